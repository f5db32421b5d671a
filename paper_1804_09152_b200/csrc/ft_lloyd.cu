// Lloyd-step kernels (sm_100a): faces per cell, approximate centroids,
// back-projection.  Replaces the per-cell Python loop of lloyd._reseed
// (reference pkg/src/fieldtess/lloyd.py:155-172) and its helpers
// faces_by_cell / cell_triangles / approx_centroid / backproject
// (lloyd.py:21-112).
//
// EXACTNESS.  The reference's centroid and ray arithmetic is numpy; every
// reduction is restated with the rounding sequence numpy uses (measured on
// numpy 2.3 and pinned by tests against the reference):
//   areas.sum()                 1-D pairwise summation (8 accumulators,
//                               blocks of 128, recursive halving)
//   (a[:,None]*x).sum(axis=0)   sequential over rows
//   np.linalg.norm(v) (3-vector) sqrt(fma(z,z, fma(y,y, x*x)))   (BLAS ddot)
//   np.linalg.norm(x, axis=1)   sqrt((x0*x0 + x1*x1) + x2*x2)
//   einsum("ij,ij->i") / ("ij,j->i")  (a0*b0 + a2*b2) + a1*b1
//   np.cross                    a1*b2 - a2*b1 (two roundings) ...
//   np.linalg.solve (torus basis, LAPACK dgesv)
//                               x2 = b2*(1/a22); x1 = fma(-x2, a12, b1)*(1/a11)
// The library is compiled with -fmad=false; FMAs appear only where numpy's
// BLAS uses them (explicit fma()).

#include <climits>
#include <cmath>
#include <cstdio>

#include "ft_common.cuh"

namespace ft {

struct Geo {
    const double* pos;       // [n_v][3]
    const int* faces;        // [n_f][3]
    const double* area;      // [n_f]
    const double* bary;      // [n_f][3]
    const double* fnorm;     // [n_f][3]
    int n_v, n_f;
    int periodic;
    double pv[2][3];         // period vectors
    double a11, a12, a22, r11, r22;   // basis = pv[:, :2].T (a21 == 0 required)
};

// -- numpy-exact small vector helpers -----------------------------------------

__device__ __forceinline__ double dot3_einsum(const double* a, const double* b) {
    return (a[0] * b[0] + a[2] * b[2]) + a[1] * b[1];
}

__device__ __forceinline__ double norm3_blas(const double* v) {
    return sqrt(fma(v[2], v[2], fma(v[1], v[1], v[0] * v[0])));
}

__device__ __forceinline__ double norm3_axis(const double* v) {
    return sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
}

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
    const double t0 = a[1] * b[2], u0 = a[2] * b[1];
    const double t1 = a[2] * b[0], u1 = a[0] * b[2];
    const double t2 = a[0] * b[1], u2 = a[1] * b[0];
    c[0] = t0 - u0;
    c[1] = t1 - u1;
    c[2] = t2 - u2;
}

// TriMesh.wrap_deltas for one vector (mesh.py:136-157): shortest lattice
// representative; the 9 candidate shifts in the reference's order, strict
// '<' so the first minimal candidate wins.
__device__ __forceinline__ void wrap(const Geo& g, double* d) {
    if (!g.periodic) return;
    const double x2 = d[1] * g.r22;
    const double x1 = fma(-x2, g.a12, d[0]) * g.r11;
    const double n1 = floor(x1 + 0.5), n2 = floor(x2 + 0.5);
    double best[3], bd = 0.0;
    bool have = false;
    for (int di = -1; di <= 1; ++di) {
        for (int dj = -1; dj <= 1; ++dj) {
            const double c1 = n1 + (double)di, c2 = n2 + (double)dj;
            double cand[3];
            for (int k = 0; k < 3; ++k) cand[k] = d[k] - (c1 * g.pv[0][k] + c2 * g.pv[1][k]);
            const double dd = dot3_einsum(cand, cand);
            if (!have || dd < bd) {
                bd = dd;
                best[0] = cand[0]; best[1] = cand[1]; best[2] = cand[2];
                have = true;
            }
        }
    }
    d[0] = best[0]; d[1] = best[1]; d[2] = best[2];
}

// numpy's pairwise sum of x[idx[0..n)] (numpy/_core/src/umath/loops_utils.h)
__device__ double pairwise_block(const double* x, const int* idx, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = res + x[idx[i]];
        return res;
    }
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = x[idx[k]];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int k = 0; k < 8; ++k) r[k] = r[k] + x[idx[i + k]];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + x[idx[i]];
    return res;
}

__device__ double pairwise_sum(const double* x, const int* idx, int n) {
    // explicit-stack version of the recursive split (n <= 128 -> block)
    int st_lo[40], st_n[40], st_state[40];
    double st_left[40];
    int sp = 0;
    st_lo[0] = 0; st_n[0] = n; st_state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        const int lo = st_lo[sp], m = st_n[sp];
        if (m <= 128) {
            ret = pairwise_block(x, idx + lo, m);
            --sp;
            continue;
        }
        int m2 = m / 2;
        m2 -= m2 % 8;
        if (st_state[sp] == 0) {            // descend left
            st_state[sp] = 1;
            ++sp;
            st_lo[sp] = lo; st_n[sp] = m2; st_state[sp] = 0;
        } else if (st_state[sp] == 1) {     // left done: descend right
            st_left[sp] = ret;
            st_state[sp] = 2;
            ++sp;
            st_lo[sp] = lo + m2; st_n[sp] = m - m2; st_state[sp] = 0;
        } else {                            // both done
            ret = st_left[sp] + ret;
            --sp;
        }
    }
    return ret;
}

// -- faces per cell -----------------------------------------------------------

// Distinct layer rows (>= 1) of face f whose spgemm value sum_v PHI(r, v)
// (ascending vertex, M^T binary: lloyd.py:21-28 via sparse.spgemm) is
// nonzero; calls fn(r) for each in ascending row order.
template <typename Fn>
__device__ __forceinline__ void face_rows(int f, const int* faces, const int* ptr, const int* idx,
                                          const double* val, int min_row, Fn fn) {
    int v[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
    // sort the 3 vertex ids (ascending = the accumulation order)
    if (v[0] > v[1]) { int t = v[0]; v[0] = v[1]; v[1] = t; }
    if (v[1] > v[2]) { int t = v[1]; v[1] = v[2]; v[2] = t; }
    if (v[0] > v[1]) { int t = v[0]; v[0] = v[1]; v[1] = t; }
    int a[3], e[3];
    for (int k = 0; k < 3; ++k) { a[k] = ptr[v[k]]; e[k] = ptr[v[k] + 1]; }
    for (int k = 0; k < 3; ++k)     // skip rows below min_row (the base row)
        while (a[k] < e[k] && idx[a[k]] < min_row) ++a[k];
    for (;;) {
        int r = INT_MAX;
        for (int k = 0; k < 3; ++k) if (a[k] < e[k] && idx[a[k]] < r) r = idx[a[k]];
        if (r == INT_MAX) break;
        double s = 0.0;
        bool first = true;
        for (int k = 0; k < 3; ++k) {
            if (a[k] < e[k] && idx[a[k]] == r) {
                s = first ? val[a[k]] : s + val[a[k]];
                first = false;
                ++a[k];
            }
        }
        if (s != 0.0) fn(r, s);
    }
}

__global__ void face_count_kernel(int n_f, const int* faces, const int* ptr, const int* idx,
                                  const double* val, int min_row, int* cell_cnt) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_f) return;
    face_rows(f, faces, ptr, idx, val, min_row, [&](int r, double) { atomicAdd(&cell_cnt[r], 1); });
}

__global__ void face_fill_kernel(int n_f, const int* faces, const int* ptr, const int* idx,
                                 const double* val, int min_row, const int* cell_ptr, int* cursor,
                                 int* cell_faces) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_f) return;
    face_rows(f, faces, ptr, idx, val, min_row, [&](int r, double) {
        const int q = atomicAdd(&cursor[r], 1);
        cell_faces[cell_ptr[r] + q] = f;
    });
}

// values of the product for sorted (row, face) pairs: one thread per pair
__global__ void face_value_kernel(int n_rows, const int* cell_ptr, const int* cell_faces, const int* faces,
                                  const int* ptr, const int* idx, const double* val, double* out) {
    const int r = blockIdx.y;
    for (int i = cell_ptr[r] + blockIdx.x * blockDim.x + threadIdx.x; i < cell_ptr[r + 1];
         i += gridDim.x * blockDim.x) {
        const int f = cell_faces[i];
        double sv = 0.0;
        face_rows(f, faces, ptr, idx, val, r, [&](int rr, double s) { if (rr == r) sv = s; });
        out[i] = sv;
    }
}

// exclusive scan of cnt[0..n) into ptr[0..n] (single CTA, n up to ~10^6)
__global__ void __launch_bounds__(1024) scan_kernel(int n, const int* cnt, int* ptr) {
    __shared__ long long s_part[32];
    const int tid = threadIdx.x;
    const int per = (n + 1023) / 1024;
    const int b0 = tid * per;
    long long sum = 0;
    for (int k = 0; k < per; ++k) if (b0 + k < n) sum += cnt[b0 + k];
    long long incl = sum;
    const int lane = tid & 31, warp = tid >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_part[warp] = incl;
    __syncthreads();
    long long pre = 0;
    for (int k = 0; k < warp; ++k) pre += s_part[k];
    long long run = pre + incl - sum;
    for (int k = 0; k < per; ++k) {
        if (b0 + k < n) { ptr[b0 + k] = (int)run; run += cnt[b0 + k]; }
    }
    if (tid == 1023) ptr[n] = (int)run;
}

// sort each cell's face segment ascending (bitonic in shared memory)
constexpr int kSortMax = 16384;

__global__ void __launch_bounds__(1024) segment_sort_kernel(int n_rows, const int* cell_ptr, int* cell_faces,
                                                            int* big_flag) {
    extern __shared__ int s_keys[];
    for (int r = blockIdx.x; r < n_rows; r += gridDim.x) {
        const int a = cell_ptr[r], m = cell_ptr[r + 1] - a;
        if (m <= 1) continue;
        if (m > kSortMax) { if (threadIdx.x == 0) atomicExch(big_flag, 1); continue; }
        int p2 = 1;
        while (p2 < m) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) s_keys[i] = i < m ? cell_faces[a + i] : INT_MAX;
        __syncthreads();
        for (int k = 2; k <= p2; k <<= 1) {
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                    const int ixj = i ^ jj;
                    if (ixj > i) {
                        const int x = s_keys[i], y = s_keys[ixj];
                        const bool up = (i & k) == 0;
                        if ((x > y) == up) { s_keys[i] = y; s_keys[ixj] = x; }
                    }
                }
                __syncthreads();
            }
        }
        for (int i = threadIdx.x; i < m; i += blockDim.x) cell_faces[a + i] = s_keys[i];
        __syncthreads();
    }
}

// -- centroids (lloyd.py:42-64) ------------------------------------------------

#define FT_LLOYD_OK 0
#define FT_LLOYD_VANISHED 1
#define FT_LLOYD_DEGENERATE 2
#define FT_LLOYD_NULLNORMAL 3
#define FT_LLOYD_MISS 4

__global__ void centroid_kernel(Geo g, int n_cells, const int* cell_ptr, const int* cell_faces,
                                const long long* seeds, double* point, double* normal, int* status) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const int r = c + 1;
    const int a = cell_ptr[r], m = cell_ptr[r + 1] - a;
    if (m == 0) { status[c] = FT_LLOYD_VANISHED; return; }
    const int* fl = cell_faces + a;
    const double total = pairwise_sum(g.area, fl, m);
    if (!(total > 0.0)) { status[c] = FT_LLOYD_DEGENERATE; return; }
    double ref[3] = {0.0, 0.0, 0.0};
    if (g.periodic) {
        const long long s = seeds[c];
        for (int k = 0; k < 3; ++k) ref[k] = g.pos[3 * s + k];
    }
    double ps[3] = {0.0, 0.0, 0.0}, ns[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < m; ++i) {
        const int f = fl[i];
        const double ar = g.area[f];
        double b[3] = {g.bary[3 * f], g.bary[3 * f + 1], g.bary[3 * f + 2]};
        if (g.periodic) {
            double dlt[3] = {b[0] - ref[0], b[1] - ref[1], b[2] - ref[2]};
            wrap(g, dlt);
            for (int k = 0; k < 3; ++k) b[k] = ref[k] + dlt[k];
        }
        for (int k = 0; k < 3; ++k) {
            const double x = ar * b[k];
            const double y = ar * g.fnorm[3 * f + k];
            ps[k] = (i == 0) ? x : ps[k] + x;
            ns[k] = (i == 0) ? y : ns[k] + y;
        }
    }
    double pt[3];
    for (int k = 0; k < 3; ++k) pt[k] = ps[k] / total;
    const double nrm = norm3_blas(ns);
    if (nrm <= 1e-12 * total) { status[c] = FT_LLOYD_NULLNORMAL; return; }
    for (int k = 0; k < 3; ++k) {
        point[3 * c + k] = pt[k];
        normal[3 * c + k] = ns[k] / nrm;
    }
    status[c] = FT_LLOYD_OK;
}

// -- back-projection (lloyd.py:67-112), one warp per cell ---------------------

__global__ void backproject_kernel(Geo g, int n_cells, const int* cell_ptr, const int* cell_faces,
                                   const double* point, const double* normal, int* status, int* hit_vertex,
                                   double* best_abs_t = nullptr, long long* best_face = nullptr,
                                   const int* face_ids = nullptr) {
    const int lane = threadIdx.x & 31;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= n_cells) return;
    if (status[c] != FT_LLOYD_OK) { if (lane == 0) hit_vertex[c] = -1; return; }
    const int r = c + 1;
    const int a = cell_ptr[r], m = cell_ptr[r + 1] - a;
    const double P[3] = {point[3 * c], point[3 * c + 1], point[3 * c + 2]};
    const double N[3] = {normal[3 * c], normal[3 * c + 1], normal[3 * c + 2]};
    double best_t = INFINITY;
    int best_i = INT_MAX;
    for (int i = lane; i < m; i += 32) {
        const int f = cell_faces[a + i];
        const int v0 = g.faces[3 * f], v1 = g.faces[3 * f + 1], v2 = g.faces[3 * f + 2];
        double p0[3], e1[3], e2[3];
        for (int k = 0; k < 3; ++k) {
            p0[k] = g.pos[3 * v0 + k];
            e1[k] = g.pos[3 * v1 + k] - p0[k];
            e2[k] = g.pos[3 * v2 + k] - p0[k];
        }
        if (g.periodic) {
            wrap(g, e1);
            wrap(g, e2);
            double bc[3], dd[3];
            for (int k = 0; k < 3; ++k) bc[k] = p0[k] + (e1[k] + e2[k]) / 3.0;
            for (int k = 0; k < 3; ++k) dd[k] = bc[k] - P[k];
            wrap(g, dd);
            for (int k = 0; k < 3; ++k) p0[k] = (p0[k] + (P[k] + dd[k])) - bc[k];
        }
        double h[3];
        cross3(N, e2, h);
        const double det = dot3_einsum(e1, h);
        const double scale = norm3_axis(e1) * norm3_axis(e2);
        const bool ok = fabs(det) > 1e-14 * fmax(scale, 1e-300);
        double s[3] = {P[0] - p0[0], P[1] - p0[1], P[2] - p0[2]};
        const double u = dot3_einsum(s, h) / det;
        double q[3];
        cross3(s, e1, q);
        const double v = dot3_einsum(q, N) / det;
        const double t = dot3_einsum(e2, q) / det;
        const double eps = 1e-12;
        const bool hit = ok && (u >= -eps) && (v >= -eps) && (u + v <= 1.0 + eps);
        if (hit) {
            const double at = fabs(t);
            if (at < best_t || (at == best_t && i < best_i)) { best_t = at; best_i = i; }
        }
    }
    // argmin |t| over the hits, first occurrence (np.argmin)
    for (int o = 16; o > 0; o >>= 1) {
        const double ot = __shfl_down_sync(0xffffffffu, best_t, o);
        const int oi = __shfl_down_sync(0xffffffffu, best_i, o);
        if (ot < best_t || (ot == best_t && oi < best_i)) { best_t = ot; best_i = oi; }
    }
    if (lane != 0) return;
    if (best_i == INT_MAX) {
        hit_vertex[c] = -1;
        status[c] = FT_LLOYD_MISS;
        if (best_abs_t) { best_abs_t[c] = INFINITY; best_face[c] = LLONG_MAX; }
        return;
    }
    // recompute the winning face's geometry and t (same arithmetic)
    const int f = cell_faces[a + best_i];
    if (best_abs_t) {   // the cross-rank key of a partitioned back-projection
        best_abs_t[c] = best_t;
        best_face[c] = face_ids ? face_ids[f] : f;
    }
    const int vv[3] = {g.faces[3 * f], g.faces[3 * f + 1], g.faces[3 * f + 2]};
    double p0[3], e1[3], e2[3];
    for (int k = 0; k < 3; ++k) {
        p0[k] = g.pos[3 * vv[0] + k];
        e1[k] = g.pos[3 * vv[1] + k] - p0[k];
        e2[k] = g.pos[3 * vv[2] + k] - p0[k];
    }
    if (g.periodic) {
        wrap(g, e1);
        wrap(g, e2);
        double bc[3], dd[3];
        for (int k = 0; k < 3; ++k) bc[k] = p0[k] + (e1[k] + e2[k]) / 3.0;
        for (int k = 0; k < 3; ++k) dd[k] = bc[k] - P[k];
        wrap(g, dd);
        for (int k = 0; k < 3; ++k) p0[k] = (p0[k] + (P[k] + dd[k])) - bc[k];
    }
    double h[3], s[3], q[3];
    cross3(N, e2, h);
    const double det = dot3_einsum(e1, h);
    for (int k = 0; k < 3; ++k) s[k] = P[k] - p0[k];
    cross3(s, e1, q);
    const double t = dot3_einsum(e2, q) / det;
    double hp[3], corner[3][3];
    for (int k = 0; k < 3; ++k) {
        hp[k] = P[k] + t * N[k];
        corner[0][k] = p0[k];
        corner[1][k] = p0[k] + e1[k];
        corner[2][k] = p0[k] + e2[k];
    }
    int nearest = 0;
    double bd = 0.0;
    for (int k = 0; k < 3; ++k) {
        double d[3] = {corner[k][0] - hp[0], corner[k][1] - hp[1], corner[k][2] - hp[2]};
        const double dd = norm3_axis(d);
        if (k == 0 || dd < bd) { bd = dd; nearest = k; }
    }
    hit_vertex[c] = vv[nearest];
}

// -- a partitioned field: per-rank partial sums of approx_centroid ---------
// Per cell over the rank's faces (ascending): face count, sum of areas, sum
// of area * barycenter (periodic: unwrapped around the cell's seed), sum of
// area * normal -- 8 doubles per cell, summed over the ranks by an
// all-reduce, then finished by lloyd_finish_kernel.

__global__ void lloyd_partials_kernel(Geo g, int n_cells, const int* cell_ptr, const int* cell_faces,
                                      const long long* seeds, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const int r = c + 1;
    const int a = cell_ptr[r], m = cell_ptr[r + 1] - a;
    double ref[3] = {0.0, 0.0, 0.0};
    if (g.periodic) {
        const long long sd = seeds[c];
        for (int k = 0; k < 3; ++k) ref[k] = g.pos[3 * sd + k];
    }
    double tot = 0.0, ps[3] = {0.0, 0.0, 0.0}, ns[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < m; ++i) {
        const int f = cell_faces[a + i];
        const double ar = g.area[f];
        double b[3] = {g.bary[3 * f], g.bary[3 * f + 1], g.bary[3 * f + 2]};
        if (g.periodic) {
            double dlt[3] = {b[0] - ref[0], b[1] - ref[1], b[2] - ref[2]};
            wrap(g, dlt);
            for (int k = 0; k < 3; ++k) b[k] = ref[k] + dlt[k];
        }
        tot += ar;
        for (int k = 0; k < 3; ++k) {
            ps[k] += ar * b[k];
            ns[k] += ar * g.fnorm[3 * f + k];
        }
    }
    double* o = out + 8 * (size_t)c;
    o[0] = (double)m; o[1] = tot;
    for (int k = 0; k < 3; ++k) { o[2 + k] = ps[k]; o[5 + k] = ns[k]; }
}

__global__ void lloyd_finish_kernel(int n_cells, const double* sums, double* point, double* normal, int* status) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const double* o = sums + 8 * (size_t)c;
    if (o[0] == 0.0) { status[c] = FT_LLOYD_VANISHED; return; }
    const double total = o[1];
    if (!(total > 0.0)) { status[c] = FT_LLOYD_DEGENERATE; return; }
    const double ns[3] = {o[5], o[6], o[7]};
    const double nrm = norm3_blas(ns);
    if (nrm <= 1e-12 * total) { status[c] = FT_LLOYD_NULLNORMAL; return; }
    for (int k = 0; k < 3; ++k) {
        point[3 * c + k] = o[2 + k] / total;
        normal[3 * c + k] = ns[k] / nrm;
    }
    status[c] = FT_LLOYD_OK;
}

}  // namespace ft

// ---------------------------------------------------------------------------
// C ABI

static thread_local char g_lerr[256] = "";

static int lcheck(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_lerr, sizeof(g_lerr), "%s: %s", where, cudaGetErrorString(e));
        return FT_ERR_CUDA;
    }
    return FT_OK;
}

extern "C" int ft_faces_by_cell(const ft_csc* phi, int32_t min_row, int32_t n_faces, const int32_t* faces,
                                int32_t* cell_ptr, int32_t* cell_faces, double* cell_values,
                                int32_t* scratch, int32_t* big_flag, void* stream) {
    if (!phi || !faces || !cell_ptr || !scratch || !big_flag) return FT_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int nr = phi->n_rows;
    int* cnt = scratch;              // [n_rows]
    int* cursor = scratch + nr;      // [n_rows]
    if (!cell_faces) {               // counting call: cell_ptr only
        cudaMemsetAsync(scratch, 0, sizeof(int) * 2 * (size_t)nr, s);
        cudaMemsetAsync(big_flag, 0, sizeof(int), s);
        if (n_faces > 0)
            ft::face_count_kernel<<<(n_faces + 255) / 256, 256, 0, s>>>(
                n_faces, faces, phi->col_ptr, phi->row_idx, (const double*)phi->values, min_row, cnt);
        ft::scan_kernel<<<1, 1024, 0, s>>>(nr, cnt, cell_ptr);
        return lcheck("ft_faces_by_cell(count)");
    }
    if (n_faces > 0)
        ft::face_fill_kernel<<<(n_faces + 255) / 256, 256, 0, s>>>(
            n_faces, faces, phi->col_ptr, phi->row_idx, (const double*)phi->values, min_row, cell_ptr, cursor,
            cell_faces);
    static bool attr[64] = {};          // the opt-in is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
        cudaFuncSetAttribute(ft::segment_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ft::kSortMax * (int)sizeof(int));
        attr[dev & 63] = true;
    }
    ft::segment_sort_kernel<<<nr < 1184 ? nr : 1184, 1024, ft::kSortMax * sizeof(int), s>>>(
        nr, cell_ptr, cell_faces, big_flag);
    if (cell_values) {
        dim3 grid(4, nr);
        ft::face_value_kernel<<<grid, 256, 0, s>>>(nr, cell_ptr, cell_faces, faces, phi->col_ptr, phi->row_idx,
                                                   (const double*)phi->values, cell_values);
    }
    return lcheck("ft_faces_by_cell");
}

static int fill_geo(ft::Geo& g, const double* positions, int32_t n_vertices, const int32_t* faces, int32_t n_faces,
                    const double* face_area, const double* face_bary, const double* face_normal,
                    const double* period) {
    g.pos = positions; g.faces = faces; g.area = face_area; g.bary = face_bary; g.fnorm = face_normal;
    g.n_v = n_vertices; g.n_f = n_faces;
    g.periodic = period != nullptr;
    if (period) {
        for (int k = 0; k < 3; ++k) { g.pv[0][k] = period[k]; g.pv[1][k] = period[3 + k]; }
        // basis = period[:, :2].T = [[p00, p10], [p01, p11]]
        g.a11 = period[0]; g.a12 = period[3]; g.a22 = period[4];
        if (period[1] != 0.0) return FT_ERR_ARG;     // the device solve assumes a21 == 0
        g.r11 = 1.0 / g.a11; g.r22 = 1.0 / g.a22;
    } else {
        for (int k = 0; k < 3; ++k) { g.pv[0][k] = 0.0; g.pv[1][k] = 0.0; }
        g.a11 = g.a12 = g.a22 = g.r11 = g.r22 = 0.0;
    }
    return FT_OK;
}

extern "C" int ft_lloyd_centroids(const double* positions, int32_t n_vertices, const int32_t* faces,
                                  int32_t n_faces, const double* face_area, const double* face_bary,
                                  const double* face_normal, const double* period /*[6] or NULL*/,
                                  int32_t n_cells, const int32_t* cell_ptr, const int32_t* cell_faces,
                                  const int64_t* seeds, double* point, double* normal, int32_t* status,
                                  int32_t* hit_vertex, void* stream) {
    if (!positions || !faces || !cell_ptr || !cell_faces || !point || !normal || !status || !hit_vertex)
        return FT_ERR_ARG;
    ft::Geo g;
    if (fill_geo(g, positions, n_vertices, faces, n_faces, face_area, face_bary, face_normal, period) != FT_OK)
        return FT_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_cells > 0) {
        ft::centroid_kernel<<<(n_cells + 127) / 128, 128, 0, s>>>(g, n_cells, cell_ptr, cell_faces, (const long long*)seeds,
                                                                  point, normal, status);
        ft::backproject_kernel<<<(n_cells * 32 + 255) / 256, 256, 0, s>>>(g, n_cells, cell_ptr, cell_faces,
                                                                           point, normal, status, hit_vertex);
    }
    return lcheck("ft_lloyd_centroids");
}

extern "C" int ft_lloyd_backproject(const double* positions, int32_t n_vertices, const int32_t* faces,
                                    int32_t n_faces, const double* period, int32_t n_cells,
                                    const int32_t* cell_ptr, const int32_t* cell_faces, const double* point,
                                    const double* normal, int32_t* status, int32_t* hit_vertex, void* stream) {
    if (!positions || !faces || !cell_ptr || !cell_faces || !point || !normal || !status || !hit_vertex)
        return FT_ERR_ARG;
    ft::Geo g;
    if (fill_geo(g, positions, n_vertices, faces, n_faces, nullptr, nullptr, nullptr, period) != FT_OK)
        return FT_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_cells > 0)
        ft::backproject_kernel<<<(n_cells * 32 + 255) / 256, 256, 0, s>>>(g, n_cells, cell_ptr, cell_faces,
                                                                           point, normal, status, hit_vertex);
    return lcheck("ft_lloyd_backproject");
}

extern "C" int ft_lloyd_partials(const double* positions, int32_t n_vertices, const int32_t* faces, int32_t n_faces,
                                 const double* face_area, const double* face_bary, const double* face_normal,
                                 const double* period, int32_t n_cells, const int32_t* cell_ptr,
                                 const int32_t* cell_faces, const int64_t* seeds, double* sums, void* stream) {
    if (!positions || !faces || !cell_ptr || !cell_faces || !sums) return FT_ERR_ARG;
    ft::Geo g;
    if (fill_geo(g, positions, n_vertices, faces, n_faces, face_area, face_bary, face_normal, period) != FT_OK)
        return FT_ERR_ARG;
    if (n_cells > 0)
        ft::lloyd_partials_kernel<<<(n_cells + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
            g, n_cells, cell_ptr, cell_faces, (const long long*)seeds, sums);
    return lcheck("ft_lloyd_partials");
}

extern "C" int ft_lloyd_finish(int32_t n_cells, const double* sums, double* point, double* normal, int32_t* status,
                               void* stream) {
    if (!sums || !point || !normal || !status) return FT_ERR_ARG;
    if (n_cells > 0)
        ft::lloyd_finish_kernel<<<(n_cells + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n_cells, sums, point,
                                                                                         normal, status);
    return lcheck("ft_lloyd_finish");
}

extern "C" int ft_lloyd_backproject_keys(const double* positions, int32_t n_vertices, const int32_t* faces,
                                         int32_t n_faces, const double* period, int32_t n_cells,
                                         const int32_t* cell_ptr, const int32_t* cell_faces, const int32_t* face_ids,
                                         const double* point, const double* normal, int32_t* status,
                                         int32_t* hit_vertex, double* best_abs_t, int64_t* best_face,
                                         void* stream) {
    if (!positions || !faces || !cell_ptr || !cell_faces || !point || !normal || !status || !hit_vertex ||
        !best_abs_t || !best_face)
        return FT_ERR_ARG;
    ft::Geo g;
    if (fill_geo(g, positions, n_vertices, faces, n_faces, nullptr, nullptr, nullptr, period) != FT_OK)
        return FT_ERR_ARG;
    if (n_cells > 0)
        ft::backproject_kernel<<<(n_cells * 32 + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
            g, n_cells, cell_ptr, cell_faces, point, normal, status, hit_vertex, best_abs_t,
            (long long*)best_face, face_ids);
    return lcheck("ft_lloyd_backproject_keys");
}
