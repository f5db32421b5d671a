// Partitioned fields: halo exchange and the cross-rank step statistics
// (sm_100a).
//
// The reference (pkg/src/fieldtess/field.py:198-321) is single-process; the
// Euler step is column-local (column j of the new field reads the columns
// u of L^T(:, j), its one-ring), so a field split into contiguous owned
// column ranges needs, per step, only the one-ring halo of each range and
// the global statistics of field.py:270-271 (max |delta|, base mass) for the
// stop test of field.py:316-317.  These kernels move halo columns between a
// rank's hybrid buffer and a fixed-slot message (counts, rows, values) that
// the host sends with ncclSend / ncclRecv, and fold the all-gathered per-rank
// records into the global record in a fixed rank order.

#include <climits>
#include <cstdio>

#include "ft_common.cuh"

namespace ft {

struct HaloParams {
    HybIn in;            // pack: the source buffer
    HybOut out;          // unpack: the destination buffer
    const int* cols;
    int n, slots;
    int* m_cnt;          // message: counts[n]
    int* m_rows;         //          rows[n*slots]
    void* m_vals;        //          values[n*slots]
    long long region;    // unpack: first pool entry of the halo region
    ft_step_stats* record;
    int* need;
    Control* ctl;
    int force;
    // unpack: the step's input buffer and the owned readers of each halo
    // column (nullable): a changed halo column stamps its readers active
    HybIn prev;
    const int* rd_ptr;
    const int* rd_idx;
    unsigned char* stamp;
};

template <typename T>
__device__ __forceinline__ bool bits_differ(T a, T b);
template <>
__device__ __forceinline__ bool bits_differ<double>(double a, double b) {
    return __double_as_longlong(a) != __double_as_longlong(b);
}
template <>
__device__ __forceinline__ bool bits_differ<float>(float a, float b) {
    return __float_as_int(a) != __float_as_int(b);
}

template <typename T>
__global__ void __launch_bounds__(256) halo_pack_kernel(const HaloParams h) {
    if (!h.force && (*(volatile const int*)&h.ctl->done ||
                     *(volatile const int*)&h.record->status != FT_STATUS_OK))
        return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h.n) return;
    const int u = h.cols[i];
    const int s = h.in.sig[u];
    const int cnt = sig_count(s);
    const int a = cnt >= 2 ? h.in.aux[u] : 0;
    h.m_cnt[i] = cnt;
    int c = cnt;
    if (c > h.slots) {
        atomicMax(h.need, c);
        h.record->status = FT_STATUS_HALO_OVERFLOW;   // same value from every writer
        c = h.slots;
    }
    const size_t o = (size_t)i * h.slots;
    T* mv = (T*)h.m_vals;
    for (int t = 0; t < c; ++t) {
        h.m_rows[o + t] = hyb_row<T>(h.in, s, a, t);
        mv[o + t] = (T)hyb_val<T>(h.in, u, s, a, t);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) halo_unpack_kernel(const HaloParams h) {
    if (!h.force && *(volatile const int*)&h.ctl->done) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h.n) return;
    const int c = min(h.m_cnt[i], h.slots);
    const int u = h.cols[i];
    const size_t o = (size_t)i * h.slots;
    const T* mv = (const T*)h.m_vals;
    bool nf = false;
    if (c == 0) {
        h.out.sig[u] = FT_SIG_EMPTY;
    } else if (c <= 2) {
        ((T*)h.out.v0)[u] = mv[o];
        nf |= !isfinite((double)mv[o]);
        if (c == 1) {
            h.out.sig[u] = h.m_rows[o];
        } else {
            h.out.sig[u] = h.m_rows[o] | kPair;
            h.out.aux[u] = h.m_rows[o + 1];
            ((T*)h.out.v1)[u] = mv[o + 1];
            nf |= !isfinite((double)mv[o + 1]);
        }
    } else {
        const long long off = h.region + (long long)i * h.slots;
        h.out.sig[u] = -c;
        h.out.aux[u] = (int)off;
        T* v = (T*)h.out.pval;
        for (int t = 0; t < c; ++t) {
            h.out.pidx[off + t] = h.m_rows[o + t];
            v[off + t] = mv[o + t];
            nf |= !isfinite((double)mv[o + t]);
        }
    }
    // a peer's non-finite value: this rank's next step checks its inputs
    if (nf) atomicOr(&h.ctl->nonfinite, 1u);
    if (!h.rd_ptr) return;
    // the column against its previous value (the step's input buffer)
    const int ps = h.prev.sig[u];
    bool changed = sig_count(ps) != c;
    if (!changed && c > 0) {
        const int pa = c >= 2 ? h.prev.aux[u] : 0;
        for (int t = 0; t < c && !changed; ++t) {
            const int r = ps >= 0 ? (t == 0 ? (ps & ~kPair) : pa) : h.prev.pidx[pa + t];
            const T x = ps >= 0 ? ((const T*)(t == 0 ? h.prev.v0 : h.prev.v1))[u] : ((const T*)h.prev.pval)[pa + t];
            changed = r != h.m_rows[o + t] || bits_differ<T>(x, mv[o + t]);
        }
    }
    if (!changed) return;
    const unsigned char cur = (unsigned char)*(volatile const int*)&h.ctl->seq;   // the next step's stamp
    for (int q = h.rd_ptr[i]; q < h.rd_ptr[i + 1]; ++q) h.stamp[h.rd_idx[q]] = cur;
}

__device__ __forceinline__ int failure_rank(int status) {
    // the reference checks expand(PHI) / expand(Lt) before NaN (field.py:238-250)
    switch (status) {
        case FT_STATUS_PATTERN: return 4;
        case FT_STATUS_NAN: return 3;
        case FT_STATUS_OVERFLOW: return 2;
        case FT_STATUS_HALO_OVERFLOW: return 1;
        default: return 0;
    }
}

__global__ void combine_kernel(const ft_step_stats* rec, int world, int rank, int max_steps, double tol,
                               double thr, Control* ctl, ft_step_stats* trace) {
    if (*(volatile int*)&ctl->done) return;
    ft_step_stats st = rec[0];
    double bm = 0.0, mxd = 0.0;
    long long nnz = 0, nsk = 0;
    int worst = 0, wr = -1;
    for (int r = 0; r < world; ++r) {          // fixed rank order
        bm = bm + rec[r].base_mass;
        mxd = fmax(mxd, rec[r].max_delta);
        nnz += rec[r].nnz_phi;
        nsk += rec[r].nnz_skel;
        const int f = failure_rank(rec[r].status);
        // the highest-priority failure, at its lowest column (the reference
        // reports the first column of the whole field)
        const int col = rec[r].status == FT_STATUS_NAN ? rec[r].nan_col : rec[r].bad_col;
        const int wcol = wr < 0 ? INT_MAX
                                : (rec[wr].status == FT_STATUS_NAN ? rec[wr].nan_col : rec[wr].bad_col);
        if (f > worst || (f == worst && f > 0 && col >= 0 && col < wcol)) { worst = f; wr = r; }
    }
    st.max_delta = mxd;
    st.base_mass = bm;
    st.nnz_phi = nnz;
    st.nnz_skel = nsk;
    st.nan_col = -1; st.bad_col = -1; st.bad_row = -1; st.bad_is_lt = 0;
    int status = FT_STATUS_OK;
    if (wr >= 0) {
        status = rec[wr].status;
        st.nan_col = rec[wr].nan_col;
        st.bad_col = rec[wr].bad_col;
        st.bad_row = rec[wr].bad_row;
        st.bad_is_lt = rec[wr].bad_is_lt;
    }
    const int stepno = ctl->steps_done + 1;
    st.step = stepno;
    st.needed = rec[rank].needed;
    const bool converged = status == FT_STATUS_OK && st.max_delta < tol && st.base_mass < thr;
    st.status = converged ? FT_STATUS_CONVERGED : status;
    trace[ctl->steps_done] = st;
    if (status != FT_STATUS_OK) {
        ctl->done = 1;
        ctl->status = status;
        ctl->needed = st.needed;
    } else {
        ctl->steps_done = stepno;
        if (converged) { ctl->done = 1; ctl->status = FT_STATUS_CONVERGED; }
        else if (stepno >= max_steps) { ctl->done = 1; ctl->status = FT_STATUS_MAXSTEPS; }
    }
}

__global__ void control_kernel(Control* ctl, int set_steps, long long* out) {
    if (set_steps >= 0) {
        ctl->full = 1;               // (re)start: the next step recomputes every owned column
        ctl->done = 0;
        ctl->status = FT_STATUS_OK;
        ctl->needed = 0;
        ctl->steps_done = set_steps;
    }
    out[0] = ctl->steps_done;
    out[1] = ctl->status;
    out[2] = ctl->needed;
}

static bool fill_halo(HaloParams& h, ft_tiled* t, const int32_t* cols, int32_t n, int32_t slots,
                      int32_t dtype, const void* msg, void* workspace, int32_t flags) {
    if (!t || !t->sig || !t->aux || !t->v0 || !t->v1 || !cols || !msg || !workspace || n < 0 || slots < 1)
        return false;
    if (dtype != FT_F64 && dtype != FT_F32) return false;
    h.in = hyb_in(t);
    h.out = hyb_out(t);
    h.cols = cols; h.n = n; h.slots = slots;
    char* m = (char*)msg;
    h.m_cnt = (int*)m;
    h.m_rows = (int*)(m + (size_t)n * 4);
    h.m_vals = m + ((4LL * n * (1 + slots) + 7) & ~7LL);   // 8-byte aligned values block
    h.region = 0;
    h.record = nullptr; h.need = nullptr;
    h.ctl = (Control*)workspace;          // the control block leads the workspace
    h.force = flags & FT_HALO_FORCE;
    h.prev = HybIn{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    h.rd_ptr = nullptr;
    h.rd_idx = nullptr;
    h.stamp = nullptr;
    return true;
}

}  // namespace ft

extern "C" int64_t ft_halo_bytes(int32_t n_cols, int32_t slots, int32_t dtype) {
    if (n_cols < 0 || slots < 1) return -1;
    const int64_t vs = dtype == FT_F64 ? 8 : 4;
    // the values block starts 8-byte aligned
    int64_t head = 4LL * n_cols * (1 + slots);
    head = (head + 7) & ~7LL;
    return head + vs * n_cols * slots;
}

extern "C" int ft_halo_pack(const ft_tiled* src, const int32_t* cols, int32_t n, int32_t slots, int32_t dtype,
                            void* msg, ft_step_stats* record, int32_t* need, void* workspace, int32_t flags,
                            void* stream) {
    ft::HaloParams h;
    if (!record || !need || !ft::fill_halo(h, const_cast<ft_tiled*>(src), cols, n, slots, dtype, msg, workspace, flags)) return FT_ERR_ARG;
    h.record = record;
    h.need = need;
    if (n == 0) return FT_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (n + 255) / 256;
    if (dtype == FT_F64) ft::halo_pack_kernel<double><<<grid, 256, 0, s>>>(h);
    else ft::halo_pack_kernel<float><<<grid, 256, 0, s>>>(h);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}

extern "C" int ft_halo_unpack(ft_tiled* dst, const int32_t* cols, int32_t n, int32_t slots, int32_t dtype,
                              const void* msg, int64_t region, void* workspace, int32_t flags, const ft_tiled* prev,
                              const int32_t* readers_ptr, const int32_t* readers_idx, void* stream) {
    ft::HaloParams h;
    if (!ft::fill_halo(h, dst, cols, n, slots, dtype, msg, workspace, flags)) return FT_ERR_ARG;
    if (region < 0 || region + (int64_t)n * slots > dst->capacity || region + (int64_t)n * slots > INT_MAX)
        return FT_ERR_SHAPE;
    h.region = region;
    if (prev && readers_ptr && readers_idx) {
        if (prev->n_cols != dst->n_cols) return FT_ERR_SHAPE;
        h.prev = ft::hyb_in(prev);
        h.rd_ptr = readers_ptr;
        h.rd_idx = readers_idx;
        h.stamp = ft::carve_workspace(workspace, dst->n_cols).stamp;
    }
    if (n == 0) return FT_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (n + 255) / 256;
    if (dtype == FT_F64) ft::halo_unpack_kernel<double><<<grid, 256, 0, s>>>(h);
    else ft::halo_unpack_kernel<float><<<grid, 256, 0, s>>>(h);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}

extern "C" int ft_domain_combine(const ft_step_stats* records, int32_t world, int32_t rank, int32_t max_steps,
                                 double tol, double base_threshold, void* workspace, ft_step_stats* trace,
                                 void* stream) {
    if (!records || !workspace || !trace || world < 1 || rank < 0 || rank >= world || max_steps < 1)
        return FT_ERR_ARG;
    ft::combine_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(records, world, rank, max_steps, tol, base_threshold,
                                                          (ft::Control*)workspace, trace);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}

extern "C" int ft_domain_control(void* workspace, int32_t set_steps, int64_t* out, void* stream) {
    if (!workspace || !out) return FT_ERR_ARG;
    ft::control_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((ft::Control*)workspace, set_steps, (long long*)out);
    return cudaGetLastError() == cudaSuccess ? FT_OK : FT_ERR_CUDA;
}
