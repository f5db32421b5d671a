// The reference's public sparse algebra on the device (sm_100a):
// spgemm, build_skeleton, expand_to_skeleton, normalize_columns
// (reference pkg/src/fieldtess/sparse.py:279-420, _kernels.py:14-176).
//
// These are the general-purpose building blocks the reference exports; the
// Euler step does not use them (it fuses the same arithmetic, ft_step.cu).
// Every floating-point reduction keeps the reference's order, so results are
// bitwise those of the numba kernels.
//
// spgemm is expand-sort-compress, parallel over the entries of B (any
// shape of B, a single column included): ft_spgemm_expand writes every
// product A(r, u) * B(u, j) with the key j * n_rows + r in the reference's
// generation order (u ascending over B(:, j), then r over A(:, u)); the host
// sorts the keys with a STABLE sort, so the products of one (r, j) stay in
// generation order, and ft_segment_sums adds each run sequentially -- the
// reference's dense-accumulator order (_kernels.py:26-62).

#include <climits>
#include <cstdio>

#include "ft_common.cuh"

namespace ft {

// one thread per entry p of B (column j, row u): counts[p] = nnz(A(:, u))
__global__ void spgemm_count_kernel(const int* __restrict__ a_ptr, const int* __restrict__ b_idx, long long nnz_b,
                                    long long* __restrict__ counts) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nnz_b) return;
    const int u = b_idx[p];
    counts[p] = a_ptr[u + 1] - a_ptr[u];
}

// entry p of B (column j) writes the products A(r, u) B(u, j), r over A(:, u),
// at off[p]..: with off the exclusive scan of the counts in B's entry order
// the products of column j follow u ascending, then r -- the reference's
// generation order -- whatever the shape of B (a single column included)
__global__ void spgemm_expand_kernel(const int* __restrict__ a_ptr, const int* __restrict__ a_idx,
                                     const double* __restrict__ a_val, const int* __restrict__ b_ptr,
                                     const int* __restrict__ b_idx, const double* __restrict__ b_val, int n_cols,
                                     long long nnz_b, long long n_rows, const long long* __restrict__ off,
                                     long long* __restrict__ keys, double* __restrict__ vals) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nnz_b) return;
    // the column of entry p: the last j with b_ptr[j] <= p
    int lo = 0, hi = n_cols;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b_ptr[mid] <= p) lo = mid; else hi = mid;
    }
    const int u = b_idx[p];
    const double bv = b_val[p];
    long long w = off[p];
    const long long kb = (long long)lo * n_rows;
    for (int q = a_ptr[u]; q < a_ptr[u + 1]; ++q) {
        keys[w] = kb + a_idx[q];
        vals[w] = a_val[q] * bv;
        ++w;
    }
}

// sequential sum of each run [start[s], start[s + 1]) (the last ends at n)
__global__ void segment_sum_kernel(const double* __restrict__ vals, long long n, const long long* __restrict__ start,
                                   long long n_seg, double* __restrict__ sums) {
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    const long long e = s + 1 < n_seg ? start[s + 1] : n;
    long long q = start[s];
    double acc = vals[q];          // the first product assigned (_kernels.py:45)
    for (++q; q < e; ++q) acc += vals[q];
    sums[s] = acc;
}

// interest skeleton (skeleton_count / skeleton_fill, _kernels.py:96-150):
// rows < phi > 0 > or < phi absent or == 0 and lt > 0 >, a sorted merge
// per column.  rows == nullptr: count pass into counts[j].
__global__ void skeleton_kernel(const int* __restrict__ p_ptr, const int* __restrict__ p_idx,
                                const double* __restrict__ p_val, const int* __restrict__ l_ptr,
                                const int* __restrict__ l_idx, const double* __restrict__ l_val, int n_cols,
                                int* __restrict__ counts, const int* __restrict__ s_ptr, int* __restrict__ rows) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_cols) return;
    int a = p_ptr[j], ae = p_ptr[j + 1], b = l_ptr[j], be = l_ptr[j + 1];
    int c = 0;
    const int w0 = rows ? s_ptr[j] : 0;
    while (a < ae || b < be) {
        int r = -1;
        if (b >= be || (a < ae && p_idx[a] < l_idx[b])) {
            if (p_val[a] > 0.0) r = p_idx[a];
            ++a;
        } else if (a >= ae || l_idx[b] < p_idx[a]) {
            if (l_val[b] > 0.0) r = l_idx[b];
            ++b;
        } else {
            if (p_val[a] > 0.0 || (p_val[a] == 0.0 && l_val[b] > 0.0)) r = p_idx[a];
            ++a;
            ++b;
        }
        if (r >= 0) {
            if (rows) rows[w0 + c] = r;
            ++c;
        }
    }
    if (!rows) counts[j] = c;
}

// a's values on the skeleton pattern, explicit zeros elsewhere; bad[j] =
// the last row of a nonzero of a outside the pattern, else -1
// (expand_kernel, _kernels.py:153-176)
__global__ void expand_kernel(const int* __restrict__ a_ptr, const int* __restrict__ a_idx,
                              const double* __restrict__ a_val, const int* __restrict__ s_ptr,
                              const int* __restrict__ s_idx, int n_cols, double* __restrict__ out,
                              int* __restrict__ bad) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_cols) return;
    int a = a_ptr[j];
    const int ae = a_ptr[j + 1];
    int b = -1;
    for (int p = s_ptr[j]; p < s_ptr[j + 1]; ++p) {
        const int r = s_idx[p];
        for (; a < ae && a_idx[a] < r; ++a)
            if (a_val[a] != 0.0) b = a_idx[a];
        if (a < ae && a_idx[a] == r) out[p] = a_val[a++];
        else out[p] = 0.0;
    }
    for (; a < ae; ++a)
        if (a_val[a] != 0.0) b = a_idx[a];
    bad[j] = b;
}

// v * (1 / s) per column with s the sequential column sum (np.add.at order)
// when s > 0; zero-sum columns unchanged (normalize_columns, sparse.py:399-420)
__global__ void normalize_kernel(const int* __restrict__ ptr, const double* __restrict__ val, int n_cols,
                                 double* __restrict__ out, double* __restrict__ sums) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_cols) return;
    double s = 0.0;
    for (int q = ptr[j]; q < ptr[j + 1]; ++q) s += val[q];
    const double scale = s > 0.0 ? 1.0 / s : 1.0;
    for (int q = ptr[j]; q < ptr[j + 1]; ++q) out[q] = val[q] * scale;
    sums[j] = s;
}

}  // namespace ft

static int grid_of(long long n, int tpb) { return (int)((n + tpb - 1) / tpb); }

static int launch_ok() { return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA; }

extern "C" int ft_spgemm_count(const ft_csc* a, const ft_csc* b, int64_t nnz_b, int64_t* counts, void* stream) {
    if (!a || !b || !counts || nnz_b < 0 || nnz_b > b->capacity) return FT_ERR_ARG;
    if (a->n_cols != b->n_rows) return FT_ERR_SHAPE;
    if (nnz_b > 0)
        ft::spgemm_count_kernel<<<grid_of(nnz_b, 256), 256, 0, (cudaStream_t)stream>>>(
            a->col_ptr, b->row_idx, nnz_b, (long long*)counts);
    return launch_ok();
}

extern "C" int ft_spgemm_expand(const ft_csc* a, const ft_csc* b, int64_t nnz_b, const int64_t* offsets,
                                int64_t* keys, double* vals, void* stream) {
    if (!a || !b || !offsets || !keys || !vals || nnz_b < 0 || nnz_b > b->capacity) return FT_ERR_ARG;
    if (a->n_cols != b->n_rows) return FT_ERR_SHAPE;
    const long long nr = a->n_rows > 0 ? a->n_rows : 1;
    if (nnz_b > 0 && b->n_cols > 0)
        ft::spgemm_expand_kernel<<<grid_of(nnz_b, 256), 256, 0, (cudaStream_t)stream>>>(
            a->col_ptr, a->row_idx, (const double*)a->values, b->col_ptr, b->row_idx, (const double*)b->values,
            b->n_cols, nnz_b, nr, (const long long*)offsets, (long long*)keys, vals);
    return launch_ok();
}

extern "C" int ft_segment_sums(const double* vals, int64_t n, const int64_t* starts, int64_t n_seg, double* sums,
                               void* stream) {
    if (!vals || !starts || !sums || n < 0 || n_seg < 0) return FT_ERR_ARG;
    if (n_seg > 0)
        ft::segment_sum_kernel<<<grid_of(n_seg, 256), 256, 0, (cudaStream_t)stream>>>(
            vals, n, (const long long*)starts, n_seg, sums);
    return launch_ok();
}

extern "C" int ft_skeleton(const ft_csc* phi, const ft_csc* lt, int32_t* counts, const int32_t* skel_ptr,
                           int32_t* skel_rows, void* stream) {
    if (!phi || !lt || (!counts && !skel_rows)) return FT_ERR_ARG;
    if (phi->n_rows != lt->n_rows || phi->n_cols != lt->n_cols) return FT_ERR_SHAPE;
    if (skel_rows && !skel_ptr) return FT_ERR_ARG;
    if (phi->n_cols > 0)
        ft::skeleton_kernel<<<grid_of(phi->n_cols, 256), 256, 0, (cudaStream_t)stream>>>(
            phi->col_ptr, phi->row_idx, (const double*)phi->values, lt->col_ptr, lt->row_idx,
            (const double*)lt->values, phi->n_cols, counts, skel_ptr, skel_rows);
    return launch_ok();
}

extern "C" int ft_expand(const ft_csc* a, const int32_t* skel_ptr, const int32_t* skel_rows, double* out_vals,
                         int32_t* bad_row, void* stream) {
    if (!a || !skel_ptr || !out_vals || !bad_row) return FT_ERR_ARG;
    if (a->n_cols > 0)
        ft::expand_kernel<<<grid_of(a->n_cols, 256), 256, 0, (cudaStream_t)stream>>>(
            a->col_ptr, a->row_idx, (const double*)a->values, skel_ptr, skel_rows, a->n_cols, out_vals, bad_row);
    return launch_ok();
}

extern "C" int ft_normalize_columns(const ft_csc* a, double* out_vals, double* sums, void* stream) {
    if (!a || !out_vals || !sums) return FT_ERR_ARG;
    if (a->n_cols > 0)
        ft::normalize_kernel<<<grid_of(a->n_cols, 256), 256, 0, (cudaStream_t)stream>>>(
            a->col_ptr, (const double*)a->values, a->n_cols, out_vals, sums);
    return launch_ok();
}
