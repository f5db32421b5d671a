// Dual-mesh adjacency products (sm_100a).
//
// Replaces the sparse boolean products and the isoline-crossing tests of the
// reference's dual extraction (pkg/src/fieldtess/dual.py):
//   threshold_rows        PHIbar = [phi >= thr, rows >= 1]         (:60-71)
//   vertex_adjacency      A_v = bool(PHIbar PHIbar^T), zero diag   (:85-91)
//   triangle_adjacency    B = PHIbar M, A_t = bool(B B^T), zero diag (:94-99)
//   confirm_candidates    per candidate pair, "the two threshold isolines
//                         cross inside some shared face"           (:160-215)
//                         and the junction triples of every face   (:223-231)
// Pairs and triples are integer keys collected into device hash sets (open
// addressing, atomicCAS) -- the "integer compaction" -- and handed to the
// host, which runs the order-dependent manifold guard and build_dual.
//
// The crossing test is exact: _isoline_segment / _orient / segments_intersect
// restated with the same IEEE operations (compiled with -fmad=false).

#include <climits>
#include <cmath>
#include <cstdio>

#include "ft_common.cuh"

namespace ft {

constexpr unsigned long long kEmpty = ~0ULL;
constexpr int kMaxFaceCells = 32;

struct DualParams {
    int n_v, n_f, n_rows;
    const int* ptr;
    const int* idx;
    const double* val;
    const int* faces;
    const double* area;
    double thr;
    unsigned long long* set_v;   // A_v pairs
    unsigned long long* set_t;   // A_t pairs
    unsigned long long* set_x;   // pairs with a crossing in a shared face
    unsigned long long* set_3;   // junction triples
    unsigned long long mask_v, mask_t, mask_x, mask_3;
    int* overflow;
};

__device__ __forceinline__ unsigned long long mix(unsigned long long k) {
    k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL; k ^= k >> 33;
    return k;
}

__device__ __forceinline__ void set_insert(unsigned long long* t, unsigned long long mask,
                                           unsigned long long key, int* overflow) {
    unsigned long long h = mix(key) & mask;
    for (unsigned long long probe = 0; probe <= mask; ++probe) {
        const unsigned long long old = atomicCAS(&t[h], kEmpty, key);
        if (old == kEmpty || old == key) return;
        h = (h + 1) & mask;
    }
    atomicOr(overflow, 1);
}

// PHI(r, v) or 0.0 (SparseMat.get)
__device__ __forceinline__ double phi_get(const DualParams& p, int r, int v) {
    int a = p.ptr[v], b = p.ptr[v + 1];
    while (a < b) {                  // rows are sorted: binary search
        const int m = (a + b) >> 1;
        const int x = p.idx[m];
        if (x == r) return p.val[m];
        if (x < r) a = m + 1; else b = m;
    }
    return 0.0;
}

// _isoline_segment (dual.py:107-123): false when no transversal segment
__device__ __forceinline__ bool isoline(const double* values, double thr, double* seg) {
    const double E[3][2] = {{0.0, 0.0}, {1.0, 0.0}, {0.0, 1.0}};
    const int ea[3] = {0, 1, 2}, eb[3] = {1, 2, 0};
    double rel[3];
    for (int k = 0; k < 3; ++k) rel[k] = values[k] - thr;
    int n = 0;
    for (int q = 0; q < 3; ++q) {
        const int a = ea[q], b = eb[q];
        if (rel[a] * rel[b] < 0.0) {
            const double s = rel[a] / (rel[a] - rel[b]);
            if (!isfinite(s)) return false;
            if (n < 2) {
                seg[2 * n] = E[a][0] + s * (E[b][0] - E[a][0]);
                seg[2 * n + 1] = E[a][1] + s * (E[b][1] - E[a][1]);
            }
            ++n;
        }
    }
    return n == 2;
}

__device__ __forceinline__ int orient(const double* a, const double* b, const double* c) {
    const double d = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
    return d > 0.0 ? 1 : (d < 0.0 ? -1 : 0);
}

__device__ __forceinline__ bool on_segment(const double* a, const double* b, const double* c) {
    return fmin(a[0], b[0]) <= c[0] && c[0] <= fmax(a[0], b[0]) &&
           fmin(a[1], b[1]) <= c[1] && c[1] <= fmax(a[1], b[1]);
}

// segments_intersect (dual.py:141-157), touching counts
__device__ __forceinline__ bool seg_intersect(const double* p, const double* q) {
    const int o1 = orient(p, p + 2, q), o2 = orient(p, p + 2, q + 2);
    const int o3 = orient(q, q + 2, p), o4 = orient(q, q + 2, p + 2);
    if (o1 != o2 && o3 != o4) return true;
    if (o1 == 0 && on_segment(p, p + 2, q)) return true;
    if (o2 == 0 && on_segment(p, p + 2, q + 2)) return true;
    if (o3 == 0 && on_segment(q, q + 2, p)) return true;
    if (o4 == 0 && on_segment(q, q + 2, p + 2)) return true;
    return false;
}

// thresholded cells (rows >= 1, phi >= thr) of vertex v, ascending, into c[]
__device__ __forceinline__ int vertex_cells(const DualParams& p, int v, int* c, int cap) {
    int n = 0;
    for (int q = p.ptr[v]; q < p.ptr[v + 1]; ++q) {
        const int r = p.idx[q];
        if (r >= 1 && p.val[q] >= p.thr) {
            if (n < cap) c[n] = r - 1;
            ++n;
        }
    }
    return n;
}

__global__ void dual_vertex_kernel(const DualParams p) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= p.n_v) return;
    int c[kMaxFaceCells];
    const int n = vertex_cells(p, v, c, kMaxFaceCells);
    if (n > kMaxFaceCells) { atomicOr(p.overflow, 2); return; }
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            set_insert(p.set_v, p.mask_v, (unsigned long long)c[a] * p.n_rows + c[b], p.overflow);
}

__global__ void dual_face_kernel(const DualParams p) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= p.n_f) return;
    const int fv[3] = {p.faces[3 * f], p.faces[3 * f + 1], p.faces[3 * f + 2]};
    // cells present in the face (union of its vertices' thresholded cells)
    int c[kMaxFaceCells];
    int n = 0;
    for (int k = 0; k < 3; ++k) {
        int vc[kMaxFaceCells];
        const int m = vertex_cells(p, fv[k], vc, kMaxFaceCells);
        if (m > kMaxFaceCells) { atomicOr(p.overflow, 2); return; }
        for (int i = 0; i < m; ++i) {
            int x = vc[i], pos = n;
            bool dup = false;
            for (int t = 0; t < n; ++t) dup |= (c[t] == x);
            if (dup) continue;
            if (n == kMaxFaceCells) { atomicOr(p.overflow, 2); return; }
            while (pos > 0 && c[pos - 1] > x) { c[pos] = c[pos - 1]; --pos; }
            c[pos] = x;
            ++n;
        }
    }
    if (n < 2) return;
    const bool live = p.area[f] > 0.0;
    for (int a = 0; a < n; ++a) {
        for (int b = a + 1; b < n; ++b) {
            const unsigned long long key = (unsigned long long)c[a] * p.n_rows + c[b];
            set_insert(p.set_t, p.mask_t, key, p.overflow);
            if (!live) {                 // degenerate face: the host replays the warning
                atomicOr(p.overflow, 4);
                continue;
            }
            double vi[3], vj[3];
            bool fin = true;
            for (int k = 0; k < 3; ++k) {
                vi[k] = phi_get(p, c[a] + 1, fv[k]);
                vj[k] = phi_get(p, c[b] + 1, fv[k]);
                fin &= isfinite(vi[k]) && isfinite(vj[k]);
            }
            if (!fin) {                  // non-finite interpolation: likewise
                atomicOr(p.overflow, 4);
                continue;
            }
            double si[4], sj[4];
            if (!isoline(vi, p.thr, si) || !isoline(vj, p.thr, sj)) continue;
            if (seg_intersect(si, sj)) set_insert(p.set_x, p.mask_x, key, p.overflow);
        }
    }
    if (n < 3) return;
    const unsigned long long nr = (unsigned long long)p.n_rows;
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            for (int d = b + 1; d < n; ++d)
                set_insert(p.set_3, p.mask_3, ((unsigned long long)c[a] * nr + c[b]) * nr + c[d], p.overflow);
}

// Triangles of the dual: the 3-cliques i < j < k of a symmetric adjacency
// in CSR (rows sorted, no diagonal).  One thread per undirected edge
// (i, j), i < j: a sorted merge of the rows of i and j lists the common
// neighbours k > j.  Count pass (tris == nullptr) into counts[e], fill
// pass at offsets[e].  Edges are numbered by their position in row i's
// list (only the entries j > i are edges).
__global__ void clique_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ idx,
                              long long* __restrict__ counts, const long long* __restrict__ offsets,
                              int* __restrict__ tris) {
    const int i = blockIdx.x;                 // one CTA per row i, threads over its entries
    if (i >= n) return;
    for (int q = ptr[i] + threadIdx.x; q < ptr[i + 1]; q += blockDim.x) {
        const int j = idx[q];
        long long c = 0, w = tris ? offsets[q] : 0;
        if (j > i) {
            int a = ptr[i], b = ptr[j];
            const int ae = ptr[i + 1], be = ptr[j + 1];
            while (a < ae && b < be) {
                const int x = idx[a], y = idx[b];
                if (x < y) { ++a; continue; }
                if (y < x) { ++b; continue; }
                if (x > j) {
                    if (tris) { tris[3 * w] = i; tris[3 * w + 1] = j; tris[3 * w + 2] = x; ++w; }
                    ++c;
                }
                ++a;
                ++b;
            }
        }
        if (!tris) counts[q] = c;
    }
}

}  // namespace ft

extern "C" int ft_clique_triangles(int32_t n, const int32_t* ptr, const int32_t* idx, int64_t* counts,
                                   const int64_t* offsets, int32_t* tris, void* stream) {
    if (n < 0 || !ptr || !idx || (!counts && !tris) || (tris && !offsets)) return FT_ERR_ARG;
    if (n > 0)
        ft::clique_kernel<<<n, 128, 0, (cudaStream_t)stream>>>(n, ptr, idx, (long long*)counts,
                                                              (const long long*)offsets, tris);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}

extern "C" int ft_dual_products(const ft_csc* phi, int32_t n_faces, const int32_t* faces,
                                const double* face_area, double threshold, uint64_t* set_v,
                                uint64_t* set_t, uint64_t* set_x, uint64_t* set_3, int64_t set_capacity,
                                int32_t* overflow, void* stream) {
    if (!phi || !faces || !face_area || !set_v || !set_t || !set_x || !set_3 || !overflow) return FT_ERR_ARG;
    if (set_capacity < 2 || (set_capacity & (set_capacity - 1))) return FT_ERR_ARG;
    if (!(threshold > 0.0 && threshold < 0.5)) return FT_ERR_SHAPE;
    cudaStream_t s = (cudaStream_t)stream;
    ft::DualParams p;
    p.n_v = phi->n_cols; p.n_f = n_faces; p.n_rows = phi->n_rows - 1;   // cells
    p.ptr = phi->col_ptr; p.idx = phi->row_idx; p.val = (const double*)phi->values;
    p.faces = faces; p.area = face_area; p.thr = threshold;
    p.set_v = (unsigned long long*)set_v; p.set_t = (unsigned long long*)set_t;
    p.set_x = (unsigned long long*)set_x; p.set_3 = (unsigned long long*)set_3;
    p.mask_v = p.mask_t = p.mask_x = p.mask_3 = (unsigned long long)set_capacity - 1;
    p.overflow = overflow;
    const size_t bytes = (size_t)set_capacity * sizeof(unsigned long long);
    cudaMemsetAsync(set_v, 0xff, bytes, s);
    cudaMemsetAsync(set_t, 0xff, bytes, s);
    cudaMemsetAsync(set_x, 0xff, bytes, s);
    cudaMemsetAsync(set_3, 0xff, bytes, s);
    cudaMemsetAsync(overflow, 0, sizeof(int32_t), s);
    if (p.n_v > 0) ft::dual_vertex_kernel<<<(p.n_v + 255) / 256, 256, 0, s>>>(p);
    if (p.n_f > 0) ft::dual_face_kernel<<<(p.n_f + 255) / 256, 256, 0, s>>>(p);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}
