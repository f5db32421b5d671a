// Per-vertex argmax labels (sm_100a).
//
// Replaces field.sharp_labels (reference pkg/src/fieldtess/field.py:324-356):
// the winner of a column is its largest cell value, ties to the lowest cell
// id (the reference's lexsort by (col, -val, row)); the base row overrides
// with UNCLAIMED = -1 only when strictly greater than the winning value
// (0.0 when the column has no cell entry).  One thread per column; the
// column is already sorted by row, so a strict '>' scan keeps the lowest
// row among equal maxima.

#include "ft_common.cuh"

namespace ft {

template <typename T>
__global__ void __launch_bounds__(FT_TPB) labels_kernel(int n_v, const int* __restrict__ ptr,
                                                        const int* __restrict__ idx,
                                                        const T* __restrict__ val,
                                                        long long* __restrict__ labels) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_v) return;
    const int c0 = __ldg(&ptr[j]);
    const int c1 = __ldg(&ptr[j + 1]);
    double base = 0.0, bv = 0.0;
    long long lab = -1;
    bool have = false;
    for (int c = c0; c < c1; ++c) {
        const int r = __ldg(&idx[c]);
        const double v = (double)__ldg(&val[c]);
        if (r == 0) {
            base = v;
        } else if (!have || v > bv) {
            have = true;
            bv = v;
            lab = r - 1;
        }
    }
    const double best = have ? bv : 0.0;
    if (base > best) lab = -1;
    labels[j] = lab;
}

}  // namespace ft

extern "C" int ft_labels(const ft_csc* phi, int32_t dtype, int64_t* labels, void* stream) {
    if (!phi || !labels) return FT_ERR_ARG;
    if (dtype != FT_F64 && dtype != FT_F32) return FT_ERR_ARG;
    const int n = phi->n_cols;
    if (n == 0) return FT_OK;
    const int grid = (n + FT_TPB - 1) / FT_TPB;
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == FT_F64)
        ft::labels_kernel<double><<<grid, FT_TPB, 0, s>>>(n, phi->col_ptr, phi->row_idx,
                                                          (const double*)phi->values, (long long*)labels);
    else
        ft::labels_kernel<float><<<grid, FT_TPB, 0, s>>>(n, phi->col_ptr, phi->row_idx,
                                                         (const float*)phi->values, (long long*)labels);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}
