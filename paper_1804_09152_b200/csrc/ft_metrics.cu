// Sampled surface distance (sm_100a): for every point, the distance to the
// closest point of a triangle soup -- the O(samples x triangles) core of the
// reference's Hausdorff metric (pkg/src/fieldtess/_kernels.py:285-366,
// analysis.py:196-229).
//
// Grid: (point blocks) x (triangle chunks).  A CTA stages one chunk of
// triangles in shared memory and every thread scans it for one point; the
// chunk minima meet in a per-point atomicMin on the bit pattern of the
// squared distance (non-negative doubles order like their bits), seeded with
// the reference's initial best (1e300), so the result does not depend on
// the chunk order.  A second pass takes the square root.  The closest-point
// test follows the reference's branch structure and operation order
// (Ericson's region tests), compiled with -fmad=false: bitwise equal.

#include <cstdint>

#include "ft_common.cuh"

namespace ft {

constexpr int kTriChunk = 256;
constexpr int kPtsPerCta = 256;

__device__ __forceinline__ double closest_sq(double px, double py, double pz, const double* t) {
    const double ax = t[0], ay = t[1], az = t[2];
    const double bx = t[3], by = t[4], bz = t[5];
    const double cx = t[6], cy = t[7], cz = t[8];
    const double abx = bx - ax, aby = by - ay, abz = bz - az;
    const double acx = cx - ax, acy = cy - ay, acz = cz - az;
    const double apx = px - ax, apy = py - ay, apz = pz - az;
    const double d1 = abx * apx + aby * apy + abz * apz;
    const double d2 = acx * apx + acy * apy + acz * apz;
    double qx, qy, qz;
    if (d1 <= 0.0 && d2 <= 0.0) {                      // vertex region A
        qx = ax; qy = ay; qz = az;
    } else {
        const double bpx = px - bx, bpy = py - by, bpz = pz - bz;
        const double d3 = abx * bpx + aby * bpy + abz * bpz;
        const double d4 = acx * bpx + acy * bpy + acz * bpz;
        if (d3 >= 0.0 && d4 <= d3) {                   // vertex region B
            qx = bx; qy = by; qz = bz;
        } else {
            const double vc = d1 * d4 - d3 * d2;
            if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) { // edge AB
                const double den = d1 - d3;
                const double v = den != 0.0 ? d1 / den : 0.0;
                qx = ax + v * abx; qy = ay + v * aby; qz = az + v * abz;
            } else {
                const double cpx = px - cx, cpy = py - cy, cpz = pz - cz;
                const double d5 = abx * cpx + aby * cpy + abz * cpz;
                const double d6 = acx * cpx + acy * cpy + acz * cpz;
                if (d6 >= 0.0 && d5 <= d6) {           // vertex region C
                    qx = cx; qy = cy; qz = cz;
                } else {
                    const double vb = d5 * d2 - d1 * d6;
                    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {   // edge AC
                        const double den = d2 - d6;
                        const double w = den != 0.0 ? d2 / den : 0.0;
                        qx = ax + w * acx; qy = ay + w * acy; qz = az + w * acz;
                    } else {
                        const double va = d3 * d6 - d5 * d4;
                        if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {   // edge BC
                            const double den = (d4 - d3) + (d5 - d6);
                            const double w = den != 0.0 ? (d4 - d3) / den : 0.0;
                            qx = bx + w * (cx - bx); qy = by + w * (cy - by); qz = bz + w * (cz - bz);
                        } else {                                                  // face interior
                            const double den = va + vb + vc;
                            const double v = den != 0.0 ? vb / den : 0.0;
                            const double w = den != 0.0 ? vc / den : 0.0;
                            qx = ax + v * abx + w * acx;
                            qy = ay + v * aby + w * acy;
                            qz = az + v * abz + w * acz;
                        }
                    }
                }
            }
        }
    }
    const double dx = px - qx, dy = py - qy, dz = pz - qz;
    return dx * dx + dy * dy + dz * dz;
}

__global__ void __launch_bounds__(kPtsPerCta) ptd_kernel(const double* __restrict__ pts, int n,
                                                         const double* __restrict__ ta,
                                                         const double* __restrict__ tb,
                                                         const double* __restrict__ tc, int m,
                                                         unsigned long long* __restrict__ best) {
    __shared__ double s_t[kTriChunk * 9];
    const int i = blockIdx.x * kPtsPerCta + threadIdx.x;
    double px = 0.0, py = 0.0, pz = 0.0;
    if (i < n) { px = pts[3 * i]; py = pts[3 * i + 1]; pz = pts[3 * i + 2]; }
    double b = 1e300;
    const int n_chunks = (m + kTriChunk - 1) / kTriChunk;
    for (int ch = blockIdx.y; ch < n_chunks; ch += gridDim.y) {
        const int t0 = ch * kTriChunk;
        const int nt = min(kTriChunk, m - t0);
        __syncthreads();
        for (int k = threadIdx.x; k < nt * 3; k += blockDim.x) {
            const int t = k / 3, c = k % 3;
            s_t[t * 9 + 0 + c] = ta[(size_t)(t0 + t) * 3 + c];
            s_t[t * 9 + 3 + c] = tb[(size_t)(t0 + t) * 3 + c];
            s_t[t * 9 + 6 + c] = tc[(size_t)(t0 + t) * 3 + c];
        }
        __syncthreads();
        if (i < n) {
            for (int t = 0; t < nt; ++t) {
                const double d = closest_sq(px, py, pz, &s_t[t * 9]);
                if (d < b) b = d;
            }
        }
    }
    if (i < n && b < 1e300) atomicMin(&best[i], (unsigned long long)__double_as_longlong(b));
}

__global__ void ptd_init(unsigned long long* best, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) best[i] = (unsigned long long)__double_as_longlong(1e300);
}

__global__ void ptd_sqrt(const unsigned long long* best, int n, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = sqrt(__longlong_as_double((long long)best[i]));
}

}  // namespace ft

extern "C" int ft_point_triangle_distances(const double* points, int32_t n_points, const double* tri_a,
                                           const double* tri_b, const double* tri_c, int32_t n_tri,
                                           uint64_t* scratch, double* out, void* stream) {
    if (n_points < 0 || n_tri < 0) return FT_ERR_SHAPE;
    if (n_points == 0) return FT_OK;
    if (!points || !scratch || !out || (n_tri > 0 && (!tri_a || !tri_b || !tri_c))) return FT_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int g1 = (n_points + 255) / 256;
    ft::ptd_init<<<g1, 256, 0, s>>>((unsigned long long*)scratch, n_points);
    if (n_tri > 0) {
        const int chunks = (n_tri + ft::kTriChunk - 1) / ft::kTriChunk;
        const dim3 grid((n_points + ft::kPtsPerCta - 1) / ft::kPtsPerCta, chunks < 65535 ? chunks : 65535);
        ft::ptd_kernel<<<grid, ft::kPtsPerCta, 0, s>>>(points, n_points, tri_a, tri_b, tri_c, n_tri,
                                                       (unsigned long long*)scratch);
    }
    ft::ptd_sqrt<<<g1, 256, 0, s>>>((const unsigned long long*)scratch, n_points, out);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}
