// Shared device helpers for the fieldtess B200 engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fieldtess_cuda.h"

#define FT_TPB 128              // threads (= vertex columns) per CTA tile
#define FT_WARPS (FT_TPB / 32)
#define FT_SLOT_PER_VERTEX 2    // tile slot entries per vertex column
#define FT_SLOT (FT_TPB * FT_SLOT_PER_VERTEX)
#define FT_CCH 2048             // columns per compaction chunk
#define FT_CTPB 256             // threads of the compaction kernels

namespace ft {

// Device control block at the head of the workspace.  Accumulators are
// "zero = neutral" so a plain memset initialises them; the finalize kernel
// re-zeroes the per-step ones after every step.
struct Control {
    unsigned long long maxdelta_bits;  // atomicMax over non-negative doubles
    unsigned long long bad_phi_key;    // atomicMax(~(col<<32|row)) -> min col
    unsigned long long bad_lt_key;
    unsigned long long skel_total;     // interest-skeleton nnz of the step
    unsigned long long nnz_total;      // output nnz of the step
    unsigned long long pool_next;      // overflow-pool bump pointer
    unsigned int       nan_key;        // atomicMax(INT_MAX - col) -> min col
    int                overflow;       // a tile did not fit the work buffer
    int                slow_count;     // wide columns queued for tier 2
    unsigned int       fin_count;      // finalize: CTAs done (last-block pattern)
    int                deep_count;     // tier-3 columns (slow_list + n_v)
    int                gen_count;      // tier-1.5 columns (slow_list + 2 n_v)
    int                done;           // evolve: stop flag (finalize sets it)
    int                steps_done;     // evolve: completed steps
    int                status;         // evolve: final status
    unsigned int       nonfinite;      // sticky: a kernel wrote a non-finite value
    long long          needed;         // capacity needed on overflow
    int                wide8_count;    // tier-2b columns (slow_list + 3 n_v + FT_TPB)
    int                pad2;
    long long          pad1[3];
};
static_assert(sizeof(Control) % 16 == 0, "Control must stay 16B aligned");

#define FT_FIN_MAX 1024   // finalize CTAs at most (partials in the workspace)

struct Workspace {
    Control*      ctl;
    double*       tile_bm;      // [num_tiles] per-tile base mass (fast path)
    double*       vbm;          // [n_v] base mass of wide columns (tier 2)
    unsigned int* slow_mask;    // [num_tiles * FT_WARPS] wide columns of each tile
    int*          slow_list;    // tier-2 queue [0, n_v), tier-3 at +n_v, tier-1.5 lists at +2 n_v (128 per
                                //   tile), tier-2b queue at +3 n_v + FT_TPB
    long long*    chunk_off;    // [num_chunks + 2] compaction chunk offsets
    double*       fin_part;     // [FT_FIN_MAX] finalize partial sums (base mass)
    double*       fin_maxd;     // [FT_FIN_MAX] finalize partial maxima
    long long*    fin_cnt;      // [FT_FIN_MAX] finalize partial nnz
    long long*    fin_skel;     // [FT_FIN_MAX] finalize partial skeleton nnz
    double*       tile_maxd;    // [num_tiles] per-tile max |delta| (fast path)
    int2*         tile_cs;      // [num_tiles] per-tile (nnz, skeleton nnz) (fast path)
    int*          tile_gen;     // [num_tiles] tier-1.5 columns of the tile (list at slow_list + 2 n_v + 128 t)
    int           num_tiles;
    int           num_chunks;
};

__host__ __device__ inline int num_tiles_for(int n_v) { return (n_v + FT_TPB - 1) / FT_TPB; }
__host__ __device__ inline int num_chunks_for(int n_v) { return (n_v + FT_CCH - 1) / FT_CCH; }

inline size_t workspace_bytes(int n_v) {
    size_t t = (size_t)num_tiles_for(n_v), c = (size_t)num_chunks_for(n_v);
    const size_t v = (size_t)n_v;
    return sizeof(Control) + t * sizeof(double) + v * sizeof(double) + t * FT_WARPS * sizeof(unsigned int) +
           (4 * v + FT_TPB) * sizeof(int) + t * sizeof(int) + (c + 2) * sizeof(long long) + 4 * FT_FIN_MAX * sizeof(double) +
           t * (sizeof(double) + sizeof(int2)) + 1024;
}

static_assert(FT_WARPS == 4, "slow_mask is read as one uint4 per tile");

inline char* align16(char* p) { return (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15); }

inline Workspace carve_workspace(void* base, int n_v) {
    Workspace w;
    char* p = (char*)base;
    w.ctl = (Control*)p;
    p += sizeof(Control);
    w.num_tiles = num_tiles_for(n_v);
    w.num_chunks = num_chunks_for(n_v);
    w.tile_bm = (double*)p;
    p += (size_t)w.num_tiles * sizeof(double);
    w.vbm = (double*)p;
    p += (size_t)n_v * sizeof(double);
    w.chunk_off = (long long*)p;
    p += ((size_t)w.num_chunks + 2) * sizeof(long long);
    w.fin_part = (double*)p;
    p += FT_FIN_MAX * sizeof(double);
    w.fin_maxd = (double*)p;
    p += FT_FIN_MAX * sizeof(double);
    w.fin_cnt = (long long*)p;
    p += FT_FIN_MAX * sizeof(long long);
    w.fin_skel = (long long*)p;
    p += FT_FIN_MAX * sizeof(long long);
    w.tile_maxd = (double*)p;
    p += (size_t)w.num_tiles * sizeof(double);
    w.tile_cs = (int2*)p;
    p += (size_t)w.num_tiles * sizeof(int2);
    w.tile_gen = (int*)p;
    p += (size_t)w.num_tiles * sizeof(int);
    p = align16(p);
    w.slow_mask = (unsigned int*)p;
    p += (size_t)w.num_tiles * FT_WARPS * sizeof(unsigned int);
    w.slow_list = (int*)p;
    p += (4 * (size_t)n_v + FT_TPB) * sizeof(int);
    return w;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive scan of one int per thread over a block of NT threads; returns
// the exclusive prefix and writes the block total.  s_scan holds NT/32 ints.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* s_scan, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    int pre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) {
        const int c = s_scan[k];
        if (k < warp) pre += c;
        tot += c;
    }
    __syncthreads();
    *total = tot;
    return pre + incl - v;
}

}  // namespace ft
