// Shared device helpers for the fieldtess B200 engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fieldtess_cuda.h"

#define FT_TPB 128              // threads (= vertex columns) per CTA tile
#define FT_WARPS (FT_TPB / 32)
#define FT_CCH 2048             // columns per compaction chunk
#define FT_GEN_TILES 3          // tiles per tier-1.5 warp (~63 flagged columns: two full chunks)
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
    unsigned long long pool_next;      // pool bump pointer of the step's output
    unsigned int       nan_key;        // atomicMax(INT_MAX - col) -> min col
    int                overflow;       // the output pool is too small
    int                slow_count;     // queue A: tier-1 columns for tier 2
    unsigned int       fin_count;      // finalize: CTAs done (last-block pattern)
    int                deep_count;     // tier-3 columns of queue A
    int                gen_count;      // queue B: tier-1.5 columns deferred to tier 2
    int                done;           // evolve: stop flag (finalize sets it)
    int                steps_done;     // evolve: completed steps
    int                status;         // evolve: final status
    unsigned int       nonfinite;      // sticky: a kernel wrote a non-finite value
    long long          needed;         // capacity needed on overflow
    int                wide8_count;    // tier-2b columns of queue A
    int                wide8b_count;   // tier-2b columns of queue B
    long long          conv_next;      // pool bump pointer of ft_tiled_from_csc
    int                deepb_count;    // tier-3 columns of queue B
    int                pad3;
    long long          pad1;
};
static_assert(sizeof(Control) % 16 == 0, "Control must stay 16B aligned");

#define FT_FIN_MAX 4096   // finalize CTAs at most (partials in the workspace)

// Statistics are kept per 32-column segment (one warp of tier 1) and per
// 128-column tile (one warp of tier 1.5), so no kernel needs a CTA barrier
// or a same-address atomic per warp; the finalize reduces them in a fixed
// order.
struct Workspace {
    Control*      ctl;
    double*       seg_bm;       // [4 num_tiles] tier-1 base mass per segment
    double*       seg_maxd;     // [4 num_tiles] tier-1 max |delta| per segment
    int2*         seg_cs;       // [4 num_tiles] tier-1 (nnz, skeleton nnz) per segment
    unsigned int* gen_mask;     // [4 num_tiles] tier-1.5 columns of each segment
    unsigned int* slow_mask;    // [4 num_tiles] tier-2 columns of each segment
    double*       gen_bm;       // [num_tiles] tier-1.5 base mass per tile group (FT_GEN_TILES tiles)
    double*       gen_maxd;     // [num_tiles]
    int2*         gen_cs;       // [num_tiles]
    double*       vbm;          // [n_v] base mass of tier-2/3 columns
    int*          slow_list;    // [3 n_v] tier-2 / 2b / 3 lists of queues A (growing up from
                                //   0, n_v, 2 n_v) and B (growing down from n_v - 1, ...)
    long long*    chunk_off;    // [num_chunks + 2] compaction chunk offsets
    double*       fin_part;     // [FT_FIN_MAX] finalize partial sums (base mass)
    double*       fin_maxd;     // [FT_FIN_MAX] finalize partial maxima
    long long*    fin_cnt;      // [FT_FIN_MAX] finalize partial nnz
    long long*    fin_skel;     // [FT_FIN_MAX] finalize partial skeleton nnz
    int           num_tiles;
    int           num_chunks;
    size_t        par_off;      // bytes between the parity-0 and parity-1 segment slots
};

__host__ __device__ inline int num_tiles_for(int n_v) { return (n_v + FT_TPB - 1) / FT_TPB; }
__host__ __device__ inline int num_chunks_for(int n_v) { return (n_v + FT_CCH - 1) / FT_CCH; }

// the per-segment slots written by tier 1 exist twice (step parity), so
// that ft_evolve can finalize step k while tier 1 of step k + 1 runs
inline size_t workspace_bytes(int n_v) {
    const size_t t = (size_t)num_tiles_for(n_v), c = (size_t)num_chunks_for(n_v), v = (size_t)n_v;
    return sizeof(Control) + 2 * 4 * t * (8 + 8 + 8 + 4 + 4) + t * (8 + 8 + 8) + v * 8 + 3 * v * 4 +
           (c + 2) * 8 + 4 * FT_FIN_MAX * 8 + 24 * 16;
}

static_assert(FT_WARPS == 4, "segment masks are read as one uint4 per tile");

inline char* align16(char* p) { return (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15); }

inline Workspace carve_workspace(void* base, int n_v) {
    Workspace w;
    char* p = (char*)base;
    w.ctl = (Control*)p;
    p += sizeof(Control);
    w.num_tiles = num_tiles_for(n_v);
    w.num_chunks = num_chunks_for(n_v);
    const size_t ns = 4 * (size_t)w.num_tiles, nt = (size_t)w.num_tiles;
    // parity 0 copies; parity 1 at par_off bytes further (ws_parity)
    char* seg0 = p;
    w.seg_bm = (double*)p;       p = align16(p + ns * 8);
    w.seg_maxd = (double*)p;     p = align16(p + ns * 8);
    w.seg_cs = (int2*)p;         p = align16(p + ns * 8);
    w.gen_mask = (unsigned int*)p; p = align16(p + ns * 4);
    w.slow_mask = (unsigned int*)p; p = align16(p + ns * 4);
    w.par_off = (size_t)(p - seg0);
    p += w.par_off;
    w.gen_bm = (double*)p;       p = align16(p + nt * 8);
    w.gen_maxd = (double*)p;     p = align16(p + nt * 8);
    w.gen_cs = (int2*)p;         p = align16(p + nt * 8);
    w.vbm = (double*)p;          p = align16(p + (size_t)n_v * 8);
    w.slow_list = (int*)p;       p = align16(p + 3 * (size_t)n_v * 4);
    w.chunk_off = (long long*)p; p = align16(p + ((size_t)w.num_chunks + 2) * 8);
    w.fin_part = (double*)p;     p += FT_FIN_MAX * 8;
    w.fin_maxd = (double*)p;     p += FT_FIN_MAX * 8;
    w.fin_cnt = (long long*)p;   p += FT_FIN_MAX * 8;
    w.fin_skel = (long long*)p;  p += FT_FIN_MAX * 8;
    return w;
}

// the workspace view of step parity `par` (its segment slots)
inline Workspace ws_parity(Workspace w, int par) {
    if (par & 1) {
        w.seg_bm = (double*)((char*)w.seg_bm + w.par_off);
        w.seg_maxd = (double*)((char*)w.seg_maxd + w.par_off);
        w.seg_cs = (int2*)((char*)w.seg_cs + w.par_off);
        w.gen_mask = (unsigned int*)((char*)w.gen_mask + w.par_off);
        w.slow_mask = (unsigned int*)((char*)w.slow_mask + w.par_off);
    }
    return w;
}

// ---------------------------------------------------------------------------
// hybrid field layout (ft_tiled, include/fieldtess_cuda.h)

constexpr int kPair = FT_SIG_PAIR;

__host__ __device__ __forceinline__ int sig_count(int s) {
    return s >= 0 ? ((s & kPair) ? 2 : 1) : (s == FT_SIG_EMPTY ? 0 : -s);
}

// read-only view of a hybrid buffer
struct HybIn {
    const int* __restrict__ sig;
    const int* __restrict__ aux;
    const void* __restrict__ v0;
    const void* __restrict__ v1;
    const int* __restrict__ pidx;
    const void* __restrict__ pval;
};

struct HybOut {
    int* __restrict__ sig;
    int* __restrict__ aux;
    void* __restrict__ v0;
    void* __restrict__ v1;
    int* __restrict__ pidx;
    void* __restrict__ pval;
};

inline HybIn hyb_in(const ft_tiled* t) { return HybIn{t->sig, t->aux, t->v0, t->v1, t->pool_idx, t->pool_val}; }
inline HybOut hyb_out(ft_tiled* t) { return HybOut{t->sig, t->aux, t->v0, t->v1, t->pool_idx, t->pool_val}; }

// entry k of column u whose signature is s and aux word a
template <typename T>
__device__ __forceinline__ int hyb_row(const HybIn& h, int s, int a, int k) {
    if (s >= 0) return k == 0 ? (s & ~kPair) : a;
    return __ldg(&h.pidx[a + k]);
}
template <typename T>
__device__ __forceinline__ double hyb_val(const HybIn& h, int u, int s, int a, int k) {
    if (s >= 0) return (double)__ldg(((const T*)(k == 0 ? h.v0 : h.v1)) + u);
    return (double)__ldg(((const T*)h.pval) + a + k);
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
