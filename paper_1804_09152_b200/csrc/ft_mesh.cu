// Mesh generation, geometry and the uniform Laplacian on the device
// (sm_100a): reference mesh.py:20-162 (TriMesh derived data), :168-246
// (generators), :379-431 (build_laplacian, uniform scheme).
//
// Every output is bitwise the reference's (SHA-pinned, tests/test_mesh.py):
// the arithmetic below spells out numpy's operation order with explicit
// round-to-nearest intrinsics (no contraction), and the one place numpy
// calls BLAS -- np.linalg.norm of a single 3-vector, sqrt(ddot(m, m)) --
// replays the ddot kernel's fused chain fma(z, z, fma(y, y, x * x)).
//
// Icosphere subdivision without a hash map: the reference numbers the
// midpoint of edge (u, v) by the first time the edge is met walking the
// faces in order, edges (i,j), (j,k), (k,i) per face.  With half-edge
// h = 3 f + e and its twin t(h) (the opposite half-edge), the first
// encounter of an edge is min(h, t(h)), so the midpoint id is
// n_old + #{first encounters before it} -- an exclusive scan of the flags
// h < t(h).  Twins of the next level follow from the current ones without
// any search: each half-edge splits in two halves whose twins are the
// swapped halves of its twin, and the three inner edges of the middle
// child pair up inside the parent face.

#include <cstdint>

#include "ft_common.cuh"

namespace ft {

// ||m|| of a 3-vector as numpy's 1-D norm computes it (BLAS ddot)
__device__ __forceinline__ double norm3_dot(double x, double y, double z) {
    return sqrt(__fma_rn(z, z, __fma_rn(y, y, __dmul_rn(x, x))));
}

// np.linalg.norm(a, axis=1) of an (n, 3) array: sqrt((x*x + y*y) + z*z)
__device__ __forceinline__ double norm3_axis(double x, double y, double z) {
    return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// flag[h] = 1 where half-edge h is the first encounter of its edge
__global__ void ico_flags_kernel(long long nh, const int* __restrict__ twin, int* __restrict__ flag) {
    const long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= nh) return;
    const int t = twin[h];
    flag[h] = (t < 0 || h < t) ? 1 : 0;
}

// mid[h] = id of the midpoint of h's edge; the first encounter writes the
// new position unit(p[u] + p[v]) (mesh.py:229-235).  incl = inclusive scan
// of the flags.
__global__ void ico_midpoints_kernel(long long nh, const int* __restrict__ faces, const int* __restrict__ twin,
                                     const long long* __restrict__ incl, int n_old, double* __restrict__ pos,
                                     int* __restrict__ mid) {
    const long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= nh) return;
    const int t = twin[h];
    const long long o = (t >= 0 && t < h) ? (long long)t : h;
    const int id = n_old + (int)(incl[o] - 1);
    mid[h] = id;
    if (o != h) return;
    const long long f = h / 3;
    const int e = (int)(h - 3 * f);
    const int u = faces[3 * f + e], v = faces[3 * f + (e == 2 ? 0 : e + 1)];
    const double x = __dadd_rn(pos[3LL * u], pos[3LL * v]);
    const double y = __dadd_rn(pos[3LL * u + 1], pos[3LL * v + 1]);
    const double z = __dadd_rn(pos[3LL * u + 2], pos[3LL * v + 2]);
    const double r = norm3_dot(x, y, z);
    pos[3LL * id] = __ddiv_rn(x, r);
    pos[3LL * id + 1] = __ddiv_rn(y, r);
    pos[3LL * id + 2] = __ddiv_rn(z, r);
}

// children (i,a,c), (j,b,a), (k,c,b), (a,b,c) of face f (mesh.py:238-243)
// and their twins.  First half of parent half-edge e: child e, edge 0;
// second half: child (e+1)%3, edge 2; inner edges pair with the middle child.
__global__ void ico_children_kernel(int n_faces, const int* __restrict__ faces, const int* __restrict__ twin,
                                    const int* __restrict__ mid, int* __restrict__ faces_out,
                                    int* __restrict__ twin_out) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_faces) return;
    const long long b = 3LL * f;
    const int i = faces[b], j = faces[b + 1], k = faces[b + 2];
    const int a = mid[b], bb = mid[b + 1], c = mid[b + 2];
    const long long o = 12LL * f;
    const int fv[12] = {i, a, c, j, bb, a, k, c, bb, a, bb, c};
#pragma unroll
    for (int q = 0; q < 12; ++q) faces_out[o + q] = fv[q];
    // outer halves
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const long long first = o + 3 * e;                          // child e, edge 0
        const long long second = o + 3 * (e == 2 ? 0 : e + 1) + 2;  // child (e+1)%3, edge 2
        const int t = twin[b + e];
        if (t < 0) {
            twin_out[first] = -1;
            twin_out[second] = -1;
            continue;
        }
        const long long g = t / 3;
        const int et = (int)(t - 3 * g);
        twin_out[first] = (int)(12 * g + 3 * (et == 2 ? 0 : et + 1) + 2);   // second half of the twin
        twin_out[second] = (int)(12 * g + 3 * et);                           // first half of the twin
    }
    // inner edges: (a,c)|(c,a), (b,a)|(a,b), (c,b)|(b,c)
    twin_out[o + 1] = (int)(o + 9 + 2);
    twin_out[o + 9 + 2] = (int)(o + 1);
    twin_out[o + 3 + 1] = (int)(o + 9);
    twin_out[o + 9] = (int)(o + 3 + 1);
    twin_out[o + 6 + 1] = (int)(o + 9 + 1);
    twin_out[o + 9 + 1] = (int)(o + 6 + 1);
}

// positions /= np.linalg.norm(positions, axis=1)[:, None]  (mesh.py:245)
__global__ void renormalize_kernel(int n, double* __restrict__ pos) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const double x = pos[3LL * v], y = pos[3LL * v + 1], z = pos[3LL * v + 2];
    const double r = norm3_axis(x, y, z);
    pos[3LL * v] = __ddiv_rn(x, r);
    pos[3LL * v + 1] = __ddiv_rn(y, r);
    pos[3LL * v + 2] = __ddiv_rn(z, r);
}

// equilateral torus grid (mesh.py:168-199): vertex (i, j) -> j*nx + i at
// i*a1 + j*a2, faces (v00, v10, v01), (v10, v11, v01) per lattice cell
__global__ void torus_kernel(int nx, int ny, double s, double a2x, double a2y, double* __restrict__ pos,
                             int* __restrict__ faces) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= (long long)nx * ny) return;
    const int j = (int)(v / nx), i = (int)(v - (long long)j * nx);
    const double di = (double)i, dj = (double)j;
    pos[3 * v] = __dadd_rn(__dmul_rn(di, s), __dmul_rn(dj, a2x));
    pos[3 * v + 1] = __dadd_rn(__dmul_rn(di, 0.0), __dmul_rn(dj, a2y));
    pos[3 * v + 2] = __dadd_rn(__dmul_rn(di, 0.0), __dmul_rn(dj, 0.0));
    const int ip = i + 1 == nx ? 0 : i + 1, jp = j + 1 == ny ? 0 : j + 1;
    const int v00 = j * nx + i, v10 = j * nx + ip, v01 = jp * nx + i, v11 = jp * nx + ip;
    int* f = faces + 6 * v;
    f[0] = v00; f[1] = v10; f[2] = v01;
    f[3] = v10; f[4] = v11; f[5] = v01;
}

struct Period {
    int on;
    double p[2][3];    // period vectors
    double inv[2][2];  // inverse of the 2x2 basis [p0.xy p1.xy] (columns)
    double r2;         // squared quarter of the shortest lattice offset
};

// shortest lattice representative of d (mesh.py:136-157; see TriMesh._wrap)
__device__ void wrap_delta(const Period& P, double d[3]) {
    if (!P.on) return;
    const double f0 = P.inv[0][0] * d[0] + P.inv[0][1] * d[1];
    const double f1 = P.inv[1][0] * d[0] + P.inv[1][1] * d[1];
    const double n0 = floor(f0 + 0.5), n1 = floor(f1 + 0.5);
    const double dd = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
    if (n0 == 0.0 && n1 == 0.0 && dd < P.r2) return;
    double best[3] = {0.0, 0.0, 0.0}, best_d2 = 0.0;
    bool have = false;
    for (int a = -1; a <= 1; ++a)
        for (int b = -1; b <= 1; ++b) {
            const double m0 = n0 + a, m1 = n1 + b;
            double c[3];
#pragma unroll
            for (int q = 0; q < 3; ++q)   // m * P exact (|m| <= 2): order-free
                c[q] = __dsub_rn(d[q], __dadd_rn(__dmul_rn(m0, P.p[0][q]), __dmul_rn(m1, P.p[1][q])));
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(c[0], c[0]), __dmul_rn(c[1], c[1])),
                                        __dmul_rn(c[2], c[2]));
            if (!have || d2 < best_d2) {
                have = true;
                best_d2 = d2;
                best[0] = c[0]; best[1] = c[1]; best[2] = c[2];
            }
        }
    d[0] = best[0]; d[1] = best[1]; d[2] = best[2];
}

// face area / unit normal / barycenter and the per-face vertex-area share
// (TriMesh._geometry; mesh.py:56-84)
__global__ void face_geometry_kernel(int n_faces, const double* __restrict__ pos, const int* __restrict__ faces,
                                     Period P, double* __restrict__ area, double* __restrict__ normal,
                                     double* __restrict__ bary, double* __restrict__ third) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_faces) return;
    const int v0 = faces[3LL * f], v1 = faces[3LL * f + 1], v2 = faces[3LL * f + 2];
    double p0[3], e1[3], e2[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        p0[q] = pos[3LL * v0 + q];
        e1[q] = __dsub_rn(pos[3LL * v1 + q], p0[q]);
        e2[q] = __dsub_rn(pos[3LL * v2 + q], p0[q]);
    }
    wrap_delta(P, e1);
    wrap_delta(P, e2);
    const double c0 = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
    const double c1 = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
    const double c2 = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
    const double nrm = norm3_axis(c0, c1, c2);
    const double ar = __dmul_rn(0.5, nrm);
    area[f] = ar;
    third[f] = __ddiv_rn(ar, 3.0);
    const bool pos_n = nrm > 0.0;
    normal[3LL * f] = pos_n ? __ddiv_rn(c0, nrm) : 0.0;
    normal[3LL * f + 1] = pos_n ? __ddiv_rn(c1, nrm) : 0.0;
    normal[3LL * f + 2] = pos_n ? __ddiv_rn(c2, nrm) : 0.0;
#pragma unroll
    for (int q = 0; q < 3; ++q) bary[3LL * f + q] = __dadd_rn(p0[q], __ddiv_rn(__dadd_rn(e1[q], e2[q]), 3.0));
}

// vertex_area[v] = sum of area/3 over its face corners in (face, corner)
// order (np.bincount): corners sorted stably by vertex, ptr per vertex
__global__ void vertex_area_kernel(int n_v, const long long* __restrict__ ptr, const long long* __restrict__ corner,
                                   const double* __restrict__ third, double* __restrict__ out) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_v) return;
    double s = 0.0;
    for (long long q = ptr[v]; q < ptr[v + 1]; ++q) s = __dadd_rn(s, third[corner[q] / 3]);
    out[v] = s;
}

// uniform Laplacian (mesh.py:392-400) from the sorted one-ring: column i of
// L^T is N(i) + {i} ascending, 1/deg(i) off the diagonal and -1 on it; L
// (same pattern) holds 1/deg(row) off the diagonal.
__global__ void uniform_laplacian_kernel(int n_v, const long long* __restrict__ nptr, const int* __restrict__ nidx,
                                         int* __restrict__ ptr, int* __restrict__ idx, double* __restrict__ val_t,
                                         double* __restrict__ val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n_v) return;
    ptr[i] = (int)(nptr[i] + i);
    if (i == n_v) return;
    const long long a = nptr[i], e = nptr[i + 1];
    const double wi = __ddiv_rn(1.0, (double)(e - a));
    long long w = a + i;
    bool diag = false;
    for (long long q = a; q < e; ++q) {
        const int r = nidx[q];
        if (!diag && r > i) {
            idx[w] = i; val_t[w] = -1.0; val[w] = -1.0; ++w;
            diag = true;
        }
        idx[w] = r;
        val_t[w] = wi;
        val[w] = __ddiv_rn(1.0, (double)(nptr[r + 1] - nptr[r]));
        ++w;
    }
    if (!diag) { idx[w] = i; val_t[w] = -1.0; val[w] = -1.0; }
}

}  // namespace ft

static int grid_of(long long n, int tpb) { return (int)((n + tpb - 1) / tpb); }
static int launch_ok() { return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA; }

extern "C" int ft_ico_flags(int64_t n_half, const int32_t* twin, int32_t* flag, void* stream) {
    if (n_half < 0 || !twin || !flag) return FT_ERR_ARG;
    if (n_half) ft::ico_flags_kernel<<<grid_of(n_half, 256), 256, 0, (cudaStream_t)stream>>>(n_half, twin, flag);
    return launch_ok();
}

extern "C" int ft_ico_midpoints(int32_t n_faces, const int32_t* faces, const int32_t* twin, const int64_t* incl,
                                int32_t n_old, double* positions, int32_t* mid, void* stream) {
    if (n_faces < 0 || !faces || !twin || !incl || !positions || !mid) return FT_ERR_ARG;
    const long long nh = 3LL * n_faces;
    if (nh)
        ft::ico_midpoints_kernel<<<grid_of(nh, 256), 256, 0, (cudaStream_t)stream>>>(
            nh, faces, twin, (const long long*)incl, n_old, positions, mid);
    return launch_ok();
}

extern "C" int ft_ico_children(int32_t n_faces, const int32_t* faces, const int32_t* twin, const int32_t* mid,
                               int32_t* faces_out, int32_t* twin_out, void* stream) {
    if (n_faces < 0 || !faces || !twin || !mid || !faces_out || !twin_out) return FT_ERR_ARG;
    if ((long long)n_faces * 12 > 0x7fffffffLL) return FT_ERR_SHAPE;
    if (n_faces)
        ft::ico_children_kernel<<<grid_of(n_faces, 256), 256, 0, (cudaStream_t)stream>>>(n_faces, faces, twin, mid,
                                                                                         faces_out, twin_out);
    return launch_ok();
}

extern "C" int ft_renormalize(int32_t n, double* positions, void* stream) {
    if (n < 0 || !positions) return FT_ERR_ARG;
    if (n) ft::renormalize_kernel<<<grid_of(n, 256), 256, 0, (cudaStream_t)stream>>>(n, positions);
    return launch_ok();
}

extern "C" int ft_torus_grid(int32_t nx, int32_t ny, double spacing, double* positions, int32_t* faces,
                             void* stream) {
    if (nx < 3 || ny < 3 || !positions || !faces) return FT_ERR_ARG;
    if (2LL * nx * ny * 3 > 0x7fffffffLL) return FT_ERR_SHAPE;
    const double s = spacing;
    const double a2x = 0.5 * s;                 // a2 = (0.5 s, 0.5 sqrt(3) s, 0)
    const double a2y = (0.5 * sqrt(3.0)) * s;
    ft::torus_kernel<<<grid_of((long long)nx * ny, 256), 256, 0, (cudaStream_t)stream>>>(nx, ny, s, a2x, a2y,
                                                                                         positions, faces);
    return launch_ok();
}

extern "C" int ft_face_geometry(int32_t n_faces, const double* positions, const int32_t* faces,
                                const double* period, double quarter_r2, double* area, double* normal,
                                double* barycenter, double* third, void* stream) {
    if (n_faces < 0 || !positions || !faces || !area || !normal || !barycenter || !third) return FT_ERR_ARG;
    ft::Period P = {};
    if (period) {
        P.on = 1;
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 3; ++q) P.p[r][q] = period[3 * r + q];
        const double a = P.p[0][0], b = P.p[1][0], c = P.p[0][1], d = P.p[1][1];   // [[a b] [c d]]
        const double det = a * d - b * c;
        if (det == 0.0) return FT_ERR_ARG;
        P.inv[0][0] = d / det; P.inv[0][1] = -b / det;
        P.inv[1][0] = -c / det; P.inv[1][1] = a / det;
        P.r2 = quarter_r2;
    }
    if (n_faces)
        ft::face_geometry_kernel<<<grid_of(n_faces, 256), 256, 0, (cudaStream_t)stream>>>(
            n_faces, positions, faces, P, area, normal, barycenter, third);
    return launch_ok();
}

extern "C" int ft_vertex_area(int32_t n_v, const int64_t* ptr, const int64_t* corner, const double* third,
                              double* out, void* stream) {
    if (n_v < 0 || !ptr || !corner || !third || !out) return FT_ERR_ARG;
    if (n_v)
        ft::vertex_area_kernel<<<grid_of(n_v, 256), 256, 0, (cudaStream_t)stream>>>(
            n_v, (const long long*)ptr, (const long long*)corner, third, out);
    return launch_ok();
}

extern "C" int ft_uniform_laplacian(int32_t n_v, const int64_t* nptr, const int32_t* nidx, int32_t* ptr,
                                    int32_t* idx, double* val_t, double* val, void* stream) {
    if (n_v < 0 || !nptr || !nidx || !ptr || !idx || !val_t || !val) return FT_ERR_ARG;
    ft::uniform_laplacian_kernel<<<grid_of((long long)n_v + 1, 256), 256, 0, (cudaStream_t)stream>>>(
        n_v, (const long long*)nptr, nidx, ptr, idx, val_t, val);
    return launch_ok();
}
