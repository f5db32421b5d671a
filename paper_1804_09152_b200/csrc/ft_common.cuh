// Shared device helpers for the fieldtess B200 engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fieldtess_cuda.h"

#define FT_TPB 128              // threads of the generic per-column kernels
#define FT_WARPS (FT_TPB / 32)
#define FT_CCH 2048             // columns per compaction chunk
#define FT_CTPB 256             // threads of the compaction kernels

namespace ft {

// Device control block at the head of the workspace.  The per-step
// accumulators are "zero = neutral": a plain memset initialises them and the
// finalize kernel re-zeroes them after every step.  All statistics are
// order-independent (integers, a max, a fixed-point base mass), so every
// kernel folds its columns in with CTA-level atomics and the result is
// deterministic.
struct Control {
    // -- per-step accumulators (zeroed by finalize) --
    unsigned long long maxdelta_bits;  // atomicMax over non-negative doubles
    unsigned long long bad_phi_key;    // atomicMax(~(col<<32|row)) -> min col
    unsigned long long bad_lt_key;
    long long          acc_nnz;        // full step: output nnz; active step: its change
    long long          acc_skel;       // the same for the interest-skeleton nnz
    long long          acc_bm[4];      // base mass (fixed point, see fx_split) or its change
    unsigned int       nan_key;        // atomicMax(INT_MAX - col) -> min col
    int                overflow;       // the output pool is too small
    int                n_act;          // active columns of the step (prep_kernel)
    int                n_wide;         // columns handed to the warp-cooperative kernel
    int                n_deep;         // wide-kernel columns beyond its staging capacity
    int                n_w2;           // columns the three-row kernel hands to the warp kernel
    // -- persistent state --
    unsigned long long pool_next[2];   // pool bump pointer of hybrid buffer 0 / 1
    long long          tot_nnz;        // running totals of the current field
    long long          tot_skel;
    long long          tot_bm[4];
    int                full;           // the next step recomputes every column
    int                seq;            // step sequence number (mark stamps)
    int                done;           // evolve: stop flag (finalize sets it)
    int                steps_done;     // evolve: completed steps
    int                status;         // evolve: final status
    unsigned int       nonfinite;      // sticky: a kernel wrote a non-finite value
    long long          needed;         // capacity needed on overflow
    long long          conv_next;      // pool bump pointer of ft_tiled_from_csc
    double             tol;            // evolve: the stop test (field.py:316-317),
    double             base_threshold; //   set per call by evolve_reset_kernel, so
    int                max_steps;      //   the captured graph does not depend on them
    int                n_w3;           // per step: columns the four-row kernel hands to the warp kernel
};
static_assert(sizeof(Control) % 16 == 0, "Control must stay 16B aligned");

// Workspace: the control block, then per-column arrays.
//   act[n]    active list of the step (local column indices)
//   wide[n]   columns the band kernel hands to the three-row kernel
//   w2[n]     columns the three-row kernel hands to the four-row kernel
//             (the four-row kernel's leftovers reuse wide[], read by then)
//   skc[n]    interest-skeleton size of each column when it was last computed
//   stamp[n]  mark: column is active in the step whose sequence number (mod
//             256) equals the stamp (indexed by buffer column)
//   chunk_off compaction chunk offsets (first, see carve_workspace)
struct Workspace {
    Control*       ctl;
    int*           act;
    int*           wide;
    int*           w2;
    int*           skc;
    unsigned char* stamp;
    long long*     chunk_off;
    int            n;
    int            num_chunks;
};

__host__ __device__ inline int num_chunks_for(int n_v) { return (n_v + FT_CCH - 1) / FT_CCH; }

inline size_t workspace_bytes(int n_v) {
    const size_t c = (size_t)num_chunks_for(n_v), v = (size_t)n_v;
    return sizeof(Control) + 4 * (v * 4 + 16) + (v + 80) + (c + 2) * 8 + 64;
}

inline char* align16(char* p) { return (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15); }

inline Workspace carve_workspace(void* base, int n_v) {
    Workspace w;
    char* p = (char*)base;
    w.ctl = (Control*)p;
    p += sizeof(Control);
    w.n = n_v;
    w.num_chunks = num_chunks_for(n_v);
    // chunk_off first: a compaction of a column range (fewer chunks) carves
    // the same workspace with a smaller n and must not touch the arrays
    // after it (the active-set state)
    w.chunk_off = (long long*)p; p = align16(p + ((size_t)w.num_chunks + 2) * 8);
    w.act = (int*)p;             p = align16(p + (size_t)n_v * 4);
    w.wide = (int*)p;            p = align16(p + (size_t)n_v * 4);
    w.w2 = (int*)p;              p = align16(p + (size_t)n_v * 4);
    w.skc = (int*)p;             p = align16(p + (size_t)n_v * 4);
    w.stamp = (unsigned char*)p;   // + 64 bytes of padding: prep reads 64-byte groups
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

// ---------------------------------------------------------------------------
// fixed-point base mass.  A column's base mass x (a normalised value, finite
// and >= 0) is split exactly into an integer part and three 32-bit fraction
// limbs (truncated below 2^-96); limb sums are exact integers, so the total
// is independent of the summation order and can be updated by per-column
// differences.  The reference sums the per-column base masses with numpy's
// pairwise sum (field.py:270); the fixed-point total, rounded to double, is
// within a few ulp of it.

__host__ __device__ __forceinline__ void fx_split(double x, long long (&l)[4]) {
    if (!(x > 0.0) || !(x < 9.0e15)) {   // 0, NaN, Inf: contributes nothing
        l[0] = l[1] = l[2] = l[3] = 0;
        return;
    }
    double y = floor(x);
    l[0] = (long long)y;
    double f = x - y;                      // exact
#pragma unroll
    for (int k = 1; k < 4; ++k) {
        f = f * 4294967296.0;              // exact (power of two)
        y = floor(f);
        l[k] = (long long)y;
        f = f - y;                         // exact
    }
}

// limbs (possibly unnormalised, signed) -> double
__host__ __device__ __forceinline__ double fx_value(const long long (&t)[4]) {
    long long a[4] = {t[0], t[1], t[2], t[3]};
    // carry-normalise limbs 3..1 into [0, 2^32)
#pragma unroll
    for (int k = 3; k > 0; --k) {
        const long long c = a[k] >> 32;    // arithmetic shift: floor division
        a[k] -= c * 4294967296LL;
        a[k - 1] += c;
    }
    const double s = 1.0 / 4294967296.0;
    return (((double)a[3] * s + (double)a[2]) * s + (double)a[1]) * s + (double)a[0];
}

}  // namespace ft
