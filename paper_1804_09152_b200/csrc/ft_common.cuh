// Shared device helpers for the fieldtess B200 engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fieldtess_cuda.h"

#define FT_TPB 256              // threads per CTA of the per-vertex kernels
#define FT_WARPS (FT_TPB / 32)

namespace ft {

// Device control block at the head of the workspace.  Accumulators are
// "zero = neutral" so a plain memset initialises them, and the finalize
// kernel re-zeroes them after every step.
struct Control {
    unsigned long long ticket;         // monotonic CTA ticket -> tile id + epoch
    unsigned long long maxdelta_bits;  // atomicMax over non-negative doubles
    unsigned long long bad_phi_key;    // atomicMax(~(col<<32|row)) -> min col
    unsigned long long bad_lt_key;
    unsigned long long skel_total;     // interest-skeleton nnz of the step
    long long          nnz_total;      // output nnz (written by the last tile)
    unsigned int       nan_key;        // atomicMax(INT_MAX - col) -> min col
    int                overflow;       // a tile did not fit the output capacity
    int                done;           // evolve: stop flag (finalize sets it)
    int                steps_done;     // evolve: completed steps
    int                status;         // evolve: final status
    int                pad0;
    long long          needed;         // evolve: capacity needed on overflow
    long long          pad1[6];
};
static_assert(sizeof(Control) % 16 == 0, "Control must stay 16B aligned");

struct Workspace {
    Control*            ctl;
    unsigned long long* tile_status;   // [num_tiles] look-back words
    double*             tile_bm;       // [num_tiles] per-tile base mass
    int                 num_tiles;
};

__host__ __device__ inline int num_tiles_for(int n_v) {
    return (n_v + FT_TPB - 1) / FT_TPB;
}

inline size_t workspace_bytes(int n_v) {
    size_t t = (size_t)num_tiles_for(n_v);
    return sizeof(Control) + t * sizeof(unsigned long long) + t * sizeof(double) + 256;
}

inline Workspace carve_workspace(void* base, int n_v) {
    Workspace w;
    char* p = (char*)base;
    w.ctl = (Control*)p;
    p += sizeof(Control);
    w.num_tiles = num_tiles_for(n_v);
    w.tile_status = (unsigned long long*)p;
    p += (size_t)w.num_tiles * sizeof(unsigned long long);
    w.tile_bm = (double*)p;
    return w;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace ft
