// Fused explicit-Euler step of the layered field (sm_100a).
//
// One launch replaces the reference pipeline of field.step
// (reference pkg/src/fieldtess/field.py:198-286):
//
//   Lt = PHI L^T            spgemm_numeric      _kernels.py:26-62
//   interest skeleton       skeleton_count/fill _kernels.py:96-150
//   PHI^, Lt^ expansion     expand_kernel       _kernels.py:153-176
//   Euler update + clamp    update_kernel       _kernels.py:179-238
//   normalise + compact     column_sums_counts, normalize_compact
//                                               _kernels.py:241-282
//
// Layout: one thread per vertex column j.  The thread walks row j of L
// (= column j of L^T, ascending neighbour index u including the diagonal)
// and merges the sorted PHI columns of those neighbours into a small sorted
// register window of at most K layer rows, accumulating Lt(r, j) for each
// row in ascending-u order, exactly the order of the reference's
// accumulator (first product assigned, then +=).  PHI(r, j) itself is
// picked up when u == j.  Columns whose union of rows exceeds K are handled
// exactly by re-gathering in ascending row windows (slow path).
//
// The per-vertex output count is only known after the update (zeros are
// dropped), so output offsets come from a single-pass block scan plus a
// decoupled look-back across tiles (tile ids from a monotonic ticket, so
// predecessors are always resident and the scan cannot deadlock).
//
// EXACT mode (double storage) replays the reference arithmetic operation by
// operation; the library is compiled with -fmad=false so no FMA contraction
// happens, and sqrt / division are IEEE correctly rounded, which makes the
// output bitwise identical to the numba reference.  FAST mode stores PHI in
// float but does all arithmetic in double in the same order.

#include <climits>
#include <cstdio>

#include "ft_common.cuh"

namespace ft {

struct StepParams {
    int n_v;
    int num_tiles;
    const int* __restrict__ lap_ptr;
    const int* __restrict__ lap_idx;
    const void* __restrict__ lap_val;
    const int* __restrict__ in_ptr;
    const int* __restrict__ in_idx;
    const void* __restrict__ in_val;
    int* __restrict__ out_ptr;
    int* __restrict__ out_idx;
    void* __restrict__ out_val;
    long long cap;
    double w, a, e, eb, mu, dt;
    Workspace ws;
    int check_done;
};

struct FinalizeParams {
    Workspace ws;
    ft_step_stats* trace;
    int fixed_slot;       // 1: write trace[0] (single step), 0: trace[steps_done]
    int evolve;           // evolve mode: convergence / done handling
    int max_steps;
    double tol;
    double base_threshold;
};

// ---------------------------------------------------------------------------
// register window of layer rows for one vertex column

template <int K>
struct Win {
    int rows[K];
    double lam[K];   // Lt(r, j) accumulator (later reused for v)
    double phi[K];   // PHI(r, j) (0.0 when not stored)
    int m;
    bool more;
};

template <int K>
__device__ __forceinline__ void win_insert(Win<K>& w, int r, double prod, bool diag, double ph) {
    bool found = false;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (i < w.m && w.rows[i] == r) {
            w.lam[i] = w.lam[i] + prod;
            if (diag) w.phi[i] = ph;
            found = true;
        }
    }
    if (found) return;
    if (w.m == K) {
        w.more = true;
        if (r > w.rows[K - 1]) return;
        w.m = K - 1;  // evict the largest row; a later window picks it up
    }
    int cr = r;
    double cl = prod;
    double cp = diag ? ph : 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (i < w.m) {
            if (w.rows[i] > cr) {
                int tr = w.rows[i]; w.rows[i] = cr; cr = tr;
                double tl = w.lam[i]; w.lam[i] = cl; cl = tl;
                double tp = w.phi[i]; w.phi[i] = cp; cp = tp;
            }
        } else if (i == w.m) {
            w.rows[i] = cr; w.lam[i] = cl; w.phi[i] = cp;
        }
    }
    w.m++;
}

template <typename T>
__device__ __forceinline__ double ldv(const void* p, long long i) {
    return (double)__ldg(((const T*)p) + i);
}

// Gather rows r > lo of the union of PHI(:, u), u in L^T(:, j), with the
// Lt accumulation, into the window (the K smallest such rows).
template <typename T, int K, bool UNIFORM>
__device__ __forceinline__ void gather(Win<K>& w, int j, int lo, const StepParams& p) {
    w.m = 0;
    w.more = false;
    const int q0 = __ldg(&p.lap_ptr[j]);
    const int q1 = __ldg(&p.lap_ptr[j + 1]);
    const double invdeg = UNIFORM ? 1.0 / (double)(q1 - q0 - 1) : 0.0;
    for (int q = q0; q < q1; ++q) {
        const int u = __ldg(&p.lap_idx[q]);
        const bool diag = (u == j);
        double l;
        if (UNIFORM) l = diag ? -1.0 : invdeg;
        else l = ldv<T>(p.lap_val, q);
        const int c0 = __ldg(&p.in_ptr[u]);
        const int c1 = __ldg(&p.in_ptr[u + 1]);
        for (int c = c0; c < c1; ++c) {
            const int r = __ldg(&p.in_idx[c]);
            if (r <= lo) continue;
            const double ph = ldv<T>(p.in_val, c);
            win_insert<K>(w, r, ph * l, diag, ph);
        }
    }
}

// Column aggregates over the skeleton rows (sequential, ascending row).
struct Agg {
    int n;
    int first_row;
    double phi0;
    double sl, sp, sr;
    int bad_phi_row, bad_lt_row;
};

__device__ __forceinline__ bool in_skeleton(double ph, double lm) {
    // (PHI stored and > 0) or ((absent or == 0) and Lt stored and > 0)
    return (ph > 0.0) || (ph == 0.0 && lm > 0.0);
}

template <int K>
__device__ __forceinline__ void pass_aggregate(const Win<K>& w, Agg& g) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (i < w.m) {
            const double ph = w.phi[i];
            const double lm = w.lam[i];
            const bool in = in_skeleton(ph, lm);
            if (ph != 0.0 && !in) g.bad_phi_row = w.rows[i];
            if (lm != 0.0 && !in) g.bad_lt_row = w.rows[i];
            if (in) {
                if (g.n == 0) { g.first_row = w.rows[i]; g.phi0 = ph; }
                g.n++;
                const double lh = (lm != 0.0) ? lm : 0.0;
                g.sl = g.sl + lh;
                g.sp = g.sp + ph;
                g.sr = g.sr + sqrt(ph);
            }
        }
    }
}

// Per-column constants of the closed-form update (_kernels.py:202-214).
struct Coef {
    bool hb;
    double rb, spc, nif, agg, inv_ni, sl, sr;
};

__device__ __forceinline__ Coef make_coef(const Agg& g, const StepParams& p) {
    Coef c;
    c.hb = (g.n > 0) && (g.first_row == 0);
    c.rb = c.hb ? sqrt(g.phi0) : 0.0;
    c.spc = c.hb ? g.sp - g.phi0 : g.sp;
    const int n_cells = c.hb ? g.n - 1 : g.n;
    c.inv_ni = 1.0 / (double)g.n;
    c.nif = (double)g.n;
    double aggw = (p.w * fmax((double)n_cells - 1.0, 0.0)) * c.spc;
    if (c.hb) aggw = aggw + p.w * c.spc;
    c.agg = ((0.5 * p.a) * (c.nif - 1.0)) * g.sl + aggw;
    c.sl = g.sl;
    c.sr = g.sr;
    return c;
}

// Euler update of one skeleton entry (_kernels.py:215-238).
__device__ __forceinline__ double update_entry(int r, double ph, double lh, const Coef& c,
                                               const StepParams& p, bool& nan) {
    const double rj = sqrt(ph);
    const double al = p.a * (c.sl - lh);
    double wj, et;
    if (r == 0) {
        wj = p.w * c.spc;
        et = ((-p.eb) * rj) * (c.sr - rj);
    } else {
        wj = p.w * (c.spc - ph);
        if (c.hb) et = rj * (p.e * ((c.sr - rj) - c.rb) + p.eb * c.rb);
        else      et = (rj * p.e) * (c.sr - rj);
    }
    const double ps = c.nif * (0.5 * al + wj) - c.agg;
    const double d = ((-p.mu) * c.inv_ni) * (ps - et);
    double v = ph + d * p.dt;
    if (v != v) { nan = true; v = ph; }
    if (v > 1.0) v = 1.0;
    else if (v <= 0.0) v = 0.0;
    return v;
}

// Per-vertex results needed before the look-back.
struct VRes {
    int cnt;          // output entries (normalised value != 0)
    int nskel;        // skeleton entries
    double bm;        // base mass of the column
    double maxd;      // max |v' - phi_old|
    double inv;       // normalisation factor (valid when s > 0)
    bool spos;        // s > 0
    bool nan;
    int bad_phi_row, bad_lt_row;
};

// --- slow path: union larger than K, processed in ascending row windows ----

template <typename T, int K, bool UNIFORM>
__device__ __noinline__ void vertex_slow(int j, const StepParams& p, VRes& res) {
    Win<K> w;
    Agg g = {0, -1, 0.0, 0.0, 0.0, 0.0, -1, -1};
    int lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        pass_aggregate<K>(w, g);
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    res.nskel = g.n;
    res.bad_phi_row = g.bad_phi_row;
    res.bad_lt_row = g.bad_lt_row;
    res.nan = false;
    res.cnt = 0; res.bm = 0.0; res.maxd = 0.0; res.inv = 0.0; res.spos = false;
    if (g.n == 0) return;
    const Coef c = make_coef(g, p);
    // pass 2: column sum of updated values
    double s = 0.0;
    lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            const double lh = (lm != 0.0) ? lm : 0.0;
            s = s + update_entry(w.rows[i], ph, lh, c, p, res.nan);
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    res.spos = s > 0.0;
    res.inv = res.spos ? 1.0 / s : 0.0;
    // pass 3: normalise, count, base mass, max delta
    lo = -1;
    bool dummy = false;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            const double lh = (lm != 0.0) ? lm : 0.0;
            const double v = update_entry(w.rows[i], ph, lh, c, p, dummy);
            const double nv = res.spos ? v * res.inv : v;
            if (nv != 0.0) {
                res.cnt++;
                if (w.rows[i] == 0) res.bm = res.bm + nv;
            }
            const double dd = fabs(nv - ph);
            if (dd > res.maxd) res.maxd = dd;
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
}

template <typename T, int K, bool UNIFORM>
__device__ __noinline__ void vertex_slow_emit(int j, const StepParams& p, long long off) {
    Win<K> w;
    Agg g = {0, -1, 0.0, 0.0, 0.0, 0.0, -1, -1};
    int lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        pass_aggregate<K>(w, g);
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    if (g.n == 0) return;
    const Coef c = make_coef(g, p);
    bool dummy = false;
    double s = 0.0;
    lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            s = s + update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p, dummy);
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    const bool spos = s > 0.0;
    const double inv = spos ? 1.0 / s : 0.0;
    T* ov = (T*)p.out_val;
    lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            const double v = update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p, dummy);
            const double nv = spos ? v * inv : v;
            if (nv != 0.0) {
                p.out_idx[off] = w.rows[i];
                ov[off] = (T)nv;
                ++off;
            }
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
}

// ---------------------------------------------------------------------------
// the fused step kernel

template <typename T, int K, bool UNIFORM>
__global__ void __launch_bounds__(FT_TPB) step_kernel(const StepParams p) {
    __shared__ int s_tile;
    __shared__ unsigned int s_epoch;
    __shared__ int s_wcnt[FT_WARPS];
    __shared__ int s_wskel[FT_WARPS];
    __shared__ double s_wbm[FT_WARPS];
    __shared__ double s_wmax[FT_WARPS];
    __shared__ int s_wflag[FT_WARPS];
    __shared__ long long s_off;

    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    if (tid == 0) {
        const unsigned long long t = atomicAdd(&p.ws.ctl->ticket, 1ULL);
        s_tile = (int)(t % (unsigned long long)p.num_tiles);
        s_epoch = (unsigned int)((t / (unsigned long long)p.num_tiles) & 0x3fffffffULL);
    }
    __syncthreads();
    const int tile = s_tile;
    const unsigned int epoch = s_epoch;
    const int j = tile * FT_TPB + tid;
    const bool active = j < p.n_v;

    Win<K> w;
    VRes res;
    res.cnt = 0; res.nskel = 0; res.bm = 0.0; res.maxd = 0.0;
    res.nan = false; res.bad_phi_row = -1; res.bad_lt_row = -1;
    res.spos = false; res.inv = 0.0;
    bool slow = false;
    unsigned int skel_mask = 0;

    if (active) {
        gather<T, K, UNIFORM>(w, j, -1, p);
        if (w.more) {
            slow = true;
            vertex_slow<T, K, UNIFORM>(j, p, res);
        } else {
            Agg g = {0, -1, 0.0, 0.0, 0.0, 0.0, -1, -1};
            pass_aggregate<K>(w, g);
            res.nskel = g.n;
            res.bad_phi_row = g.bad_phi_row;
            res.bad_lt_row = g.bad_lt_row;
            if (g.n > 0) {
                const Coef c = make_coef(g, p);
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    if (i < w.m) {
                        const double ph = w.phi[i], lm = w.lam[i];
                        if (in_skeleton(ph, lm)) {
                            skel_mask |= 1u << i;
                            const double v = update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p, res.nan);
                            w.lam[i] = v;
                            s = s + v;
                        }
                    }
                }
                res.spos = s > 0.0;
                res.inv = res.spos ? 1.0 / s : 0.0;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    if (skel_mask & (1u << i)) {
                        const double nv = res.spos ? w.lam[i] * res.inv : w.lam[i];
                        if (nv != 0.0) {
                            res.cnt++;
                            if (w.rows[i] == 0) res.bm = res.bm + nv;
                        }
                        const double dd = fabs(nv - w.phi[i]);
                        if (dd > res.maxd) res.maxd = dd;
                        w.lam[i] = nv;
                    }
                }
            }
        }
        if (res.nan) atomicMax(&p.ws.ctl->nan_key, (unsigned int)(INT_MAX - j));
        if (res.bad_phi_row >= 0)
            atomicMax(&p.ws.ctl->bad_phi_key,
                      ~(((unsigned long long)j << 32) | (unsigned int)res.bad_phi_row));
        if (res.bad_lt_row >= 0)
            atomicMax(&p.ws.ctl->bad_lt_key,
                      ~(((unsigned long long)j << 32) | (unsigned int)res.bad_lt_row));
    }

    // ---- block scan of counts, block reductions ----------------------------
    int incl = res.cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    int skel = warp_sum(res.nskel);
    double bm = warp_sum(res.bm);
    double mx = res.maxd;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 31) s_wcnt[warp] = incl;
    if (lane == 0) { s_wskel[warp] = skel; s_wbm[warp] = bm; s_wmax[warp] = mx; }
    __syncthreads();
    int wpre = 0, tile_total = 0;
#pragma unroll
    for (int k = 0; k < FT_WARPS; ++k) {
        const int c = s_wcnt[k];
        if (k < warp) wpre += c;
        tile_total += c;
    }
    const int local_off = wpre + incl - res.cnt;

    // ---- decoupled look-back (warp 0) --------------------------------------
    if (warp == 0) {
        unsigned long long* st = p.ws.tile_status;
        const unsigned long long tag = (unsigned long long)epoch << 34;
        long long excl = 0;
        if (tile == 0) {
            if (lane == 0) st_relaxed_u64(&st[0], tag | (2ULL << 32) | (unsigned int)tile_total);
        } else {
            if (lane == 0) st_relaxed_u64(&st[tile], tag | (1ULL << 32) | (unsigned int)tile_total);
            int base = tile - 1;
            while (true) {
                const int t = base - lane;
                unsigned long long s;
                unsigned int flag;
                while (true) {
                    if (t >= 0) {
                        s = ld_relaxed_u64(&st[t]);
                        flag = ((s >> 34) == (unsigned long long)epoch) ? (unsigned int)((s >> 32) & 3ULL) : 0u;
                    } else {
                        s = 0ULL;
                        flag = 2u;  // before the first tile: inclusive prefix 0
                    }
                    if (__all_sync(0xffffffffu, flag != 0u)) break;
                }
                const unsigned int pm = __ballot_sync(0xffffffffu, flag == 2u);
                const int kk = pm ? (__ffs(pm) - 1) : 31;
                unsigned int v = (lane <= kk) ? (unsigned int)(s & 0xffffffffULL) : 0u;
                excl += (long long)warp_sum(v);
                excl = __shfl_sync(0xffffffffu, excl, 0);
                if (pm) break;
                base -= 32;
            }
            if (lane == 0)
                st_relaxed_u64(&st[tile], tag | (2ULL << 32) | (unsigned int)(excl + tile_total));
        }
        if (lane == 0) {
            s_off = excl;
            double tbm = 0.0, tmx = 0.0;
            int tsk = 0;
            for (int k = 0; k < FT_WARPS; ++k) { tbm = tbm + s_wbm[k]; tmx = fmax(tmx, s_wmax[k]); tsk += s_wskel[k]; }
            p.ws.tile_bm[tile] = tbm;
            if (tmx > 0.0) atomicMax(&p.ws.ctl->maxdelta_bits, (unsigned long long)__double_as_longlong(tmx));
            atomicAdd(&p.ws.ctl->skel_total, (unsigned long long)tsk);
            const long long end = excl + tile_total;
            s_wflag[0] = (end > p.cap) ? 1 : 0;
            if (end > p.cap) atomicExch(&p.ws.ctl->overflow, 1);
            if (tile == p.num_tiles - 1) {
                p.ws.ctl->nnz_total = end;
                p.out_ptr[p.n_v] = (int)end;
            }
        }
    }
    __syncthreads();
    if (!active) return;
    const long long off = s_off + local_off;
    p.out_ptr[j] = (int)off;
    if (s_wflag[0]) return;  // output does not fit: the host grows and retries
    if (slow) {
        vertex_slow_emit<T, K, UNIFORM>(j, p, off);
    } else if (res.cnt > 0) {
        T* ov = (T*)p.out_val;
        long long o = off;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if ((skel_mask & (1u << i)) && w.lam[i] != 0.0) {
                p.out_idx[o] = w.rows[i];
                ov[o] = (T)w.lam[i];
                ++o;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// per-step finalisation: deterministic base-mass reduction, stats record,
// error / convergence flags, accumulator reset.

__global__ void __launch_bounds__(1024) finalize_kernel(const FinalizeParams f) {
    Control* ctl = f.ws.ctl;
    if (f.evolve && *(volatile int*)&ctl->done) return;
    __shared__ double s_part[32];
    const int tid = threadIdx.x;
    double acc = 0.0;
    for (int t = tid; t < f.ws.num_tiles; t += blockDim.x) acc = acc + f.ws.tile_bm[t];
    acc = warp_sum(acc);
    if ((tid & 31) == 0) s_part[tid >> 5] = acc;
    __syncthreads();
    if (tid != 0) return;
    double bm = 0.0;
    const int nw = (blockDim.x + 31) >> 5;
    for (int k = 0; k < nw; ++k) bm = bm + s_part[k];

    const int slot = f.fixed_slot ? 0 : ctl->steps_done;
    ft_step_stats st;
    st.max_delta = __longlong_as_double((long long)ctl->maxdelta_bits);
    st.base_mass = bm;
    st.nnz_phi = ctl->nnz_total;
    st.nnz_skel = (long long)ctl->skel_total;
    st.nan_col = ctl->nan_key ? (int)(INT_MAX - ctl->nan_key) : -1;
    st.bad_col = -1; st.bad_row = -1; st.bad_is_lt = 0;
    const unsigned long long kp = ctl->bad_phi_key, kl = ctl->bad_lt_key;
    if (kp) { const unsigned long long k = ~kp; st.bad_col = (int)(k >> 32); st.bad_row = (int)(k & 0xffffffffULL); }
    else if (kl) { const unsigned long long k = ~kl; st.bad_col = (int)(k >> 32); st.bad_row = (int)(k & 0xffffffffULL); st.bad_is_lt = 1; }
    int status = FT_STATUS_OK;
    if (st.bad_col >= 0) status = FT_STATUS_PATTERN;
    else if (st.nan_col >= 0) status = FT_STATUS_NAN;
    else if (ctl->overflow) status = FT_STATUS_OVERFLOW;
    const int stepno = ctl->steps_done + 1;
    st.step = stepno;
    st.reserved = 0;
    bool converged = false;
    if (status == FT_STATUS_OK && f.evolve)
        converged = (st.max_delta < f.tol) && (st.base_mass < f.base_threshold);
    st.status = converged ? FT_STATUS_CONVERGED : status;
    f.trace[slot] = st;

    // reset the per-step accumulators
    ctl->maxdelta_bits = 0ULL;
    ctl->bad_phi_key = 0ULL;
    ctl->bad_lt_key = 0ULL;
    ctl->skel_total = 0ULL;
    ctl->nan_key = 0u;
    ctl->overflow = 0;
    if (f.evolve) {
        if (status != FT_STATUS_OK) {
            ctl->done = 1;
            ctl->status = status;
            ctl->needed = st.nnz_phi;
        } else {
            ctl->steps_done = stepno;
            if (converged) { ctl->done = 1; ctl->status = FT_STATUS_CONVERGED; }
            else if (stepno >= f.max_steps) { ctl->done = 1; ctl->status = FT_STATUS_MAXSTEPS; }
        }
    }
}

__global__ void evolve_reset_kernel(Control* ctl) {
    ctl->done = 0;
    ctl->steps_done = 0;
    ctl->status = FT_STATUS_OK;
    ctl->needed = 0;
}

__global__ void evolve_report_kernel(const Control* ctl, long long* control) {
    control[0] = ctl->steps_done;
    control[1] = ctl->status;
    control[2] = ctl->needed;
    control[3] = ctl->steps_done & 1;
}

// ---------------------------------------------------------------------------
// host side

typedef void (*StepKernelFn)(const StepParams);

template <int K>
static StepKernelFn pick_kernel(int dtype, bool uniform) {
    if (dtype == FT_F64) return uniform ? step_kernel<double, K, true> : step_kernel<double, K, false>;
    return uniform ? step_kernel<float, K, true> : step_kernel<float, K, false>;
}

}  // namespace ft

// ---------------------------------------------------------------------------
// C ABI

static thread_local char g_err[512] = "";

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

static int cuda_check(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
        return FT_ERR_CUDA;
    }
    return FT_OK;
}

extern "C" int ft_abi_version(void) { return FT_ABI_VERSION; }
extern "C" const char* ft_last_error(void) { return g_err; }

extern "C" size_t ft_workspace_bytes(int32_t n_vertices) {
    return ft::workspace_bytes(n_vertices < 0 ? 0 : n_vertices);
}

extern "C" int ft_workspace_init(void* workspace, size_t bytes, void* stream) {
    if (!workspace) return set_err(FT_ERR_ARG, "null workspace");
    cudaMemsetAsync(workspace, 0, bytes, (cudaStream_t)stream);
    return cuda_check("ft_workspace_init");
}

static int validate_step_args(const ft_csc* lap_t, const ft_csc* in, const ft_csc* out, int dtype,
                              size_t ws_bytes) {
    if (!lap_t || !in || !out) return set_err(FT_ERR_ARG, "null matrix descriptor");
    if (dtype != FT_F64 && dtype != FT_F32) return set_err(FT_ERR_ARG, "bad dtype");
    if (lap_t->n_rows != lap_t->n_cols) return set_err(FT_ERR_SHAPE, "Laplacian must be square");
    if (lap_t->n_cols != in->n_cols) return set_err(FT_ERR_SHAPE, "Laplacian size does not match field");
    if (in->n_cols != out->n_cols || in->n_rows != out->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    if (ws_bytes < ft::workspace_bytes(in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    return FT_OK;
}

static ft::StepParams make_params(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* in,
                                  ft_csc* out, const ft_params* prm, void* ws) {
    ft::StepParams p;
    p.n_v = in->n_cols;
    p.num_tiles = ft::num_tiles_for(p.n_v);
    p.lap_ptr = lap_t->col_ptr;
    p.lap_idx = lap_t->row_idx;
    p.lap_val = lap_t->values;
    p.in_ptr = in->col_ptr;
    p.in_idx = in->row_idx;
    p.in_val = in->values;
    p.out_ptr = out->col_ptr;
    p.out_idx = out->row_idx;
    p.out_val = out->values;
    p.cap = out->capacity;
    p.w = prm->w; p.a = prm->a; p.e = prm->e; p.eb = prm->e_base; p.mu = prm->mu; p.dt = prm->dt;
    p.ws = ft::carve_workspace(ws, p.n_v);
    p.check_done = 0;
    (void)lap_flags;
    return p;
}

static int launch_step_kernel(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
                              ft_csc* phi_out, int32_t dtype, const ft_params* params,
                              void* workspace, size_t ws_bytes, cudaStream_t s,
                              ft::Workspace* ws_out) {
    int rc = validate_step_args(lap_t, phi_in, phi_out, dtype, ws_bytes);
    if (rc != FT_OK) return rc;
    if (!params || !workspace) return set_err(FT_ERR_ARG, "null argument");
    ft::StepParams p = make_params(lap_t, lap_flags, phi_in, phi_out, params, workspace);
    if (p.n_v == 0) return set_err(FT_ERR_SHAPE, "empty field");
    ft::StepKernelFn k = ft::pick_kernel<8>(dtype, lap_flags == FT_LAP_UNIFORM);
    k<<<p.num_tiles, FT_TPB, 0, s>>>(p);
    if (ws_out) *ws_out = p.ws;
    return cuda_check("ft_step_kernel");
}

static void launch_finalize(const ft::Workspace& ws, ft_step_stats* stats, cudaStream_t s) {
    ft::FinalizeParams f;
    f.ws = ws; f.trace = stats; f.fixed_slot = 1; f.evolve = 0;
    f.max_steps = 1; f.tol = 0.0; f.base_threshold = 0.0;
    ft::finalize_kernel<<<1, 1024, 0, s>>>(f);
}

extern "C" int ft_step_kernel(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
                              ft_csc* phi_out, int32_t dtype, const ft_params* params,
                              void* workspace, size_t ws_bytes, void* stream) {
    return launch_step_kernel(lap_t, lap_flags, phi_in, phi_out, dtype, params, workspace,
                              ws_bytes, (cudaStream_t)stream, nullptr);
}

extern "C" int ft_step_finalize(void* workspace, size_t ws_bytes, int32_t n_vertices,
                                ft_step_stats* stats, void* stream) {
    if (!workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (ws_bytes < ft::workspace_bytes(n_vertices)) return set_err(FT_ERR_ARG, "workspace too small");
    launch_finalize(ft::carve_workspace(workspace, n_vertices), stats, (cudaStream_t)stream);
    return cuda_check("ft_step_finalize");
}

extern "C" int ft_step(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
                       ft_csc* phi_out, int32_t dtype, const ft_params* params, void* workspace,
                       size_t ws_bytes, ft_step_stats* stats, void* stream) {
    if (!stats) return set_err(FT_ERR_ARG, "null stats");
    cudaStream_t s = (cudaStream_t)stream;
    ft::Workspace ws;
    int rc = launch_step_kernel(lap_t, lap_flags, phi_in, phi_out, dtype, params, workspace,
                                ws_bytes, s, &ws);
    if (rc != FT_OK) return rc;
    launch_finalize(ws, stats, s);
    return cuda_check("ft_step");
}

extern "C" int ft_evolve(const ft_csc* lap_t, int32_t lap_flags, ft_csc* phi_a, ft_csc* phi_b,
                         int32_t dtype, const ft_params* params, int32_t max_steps, double tol,
                         double base_threshold, void* workspace, size_t ws_bytes,
                         ft_step_stats* trace, int64_t* control, void* stream) {
    int rc = validate_step_args(lap_t, phi_a, phi_b, dtype, ws_bytes);
    if (rc != FT_OK) return rc;
    if (!params || !trace || !control || !workspace) return set_err(FT_ERR_ARG, "null argument");
    if (max_steps < 1) return set_err(FT_ERR_SHAPE, "max_steps must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    ft::StepParams pab = make_params(lap_t, lap_flags, phi_a, phi_b, params, workspace);
    ft::StepParams pba = make_params(lap_t, lap_flags, phi_b, phi_a, params, workspace);
    if (pab.n_v == 0) return set_err(FT_ERR_SHAPE, "empty field");
    pab.check_done = pba.check_done = 1;
    ft::StepKernelFn k = ft::pick_kernel<8>(dtype, lap_flags == FT_LAP_UNIFORM);
    ft::FinalizeParams f;
    f.ws = pab.ws; f.trace = trace; f.fixed_slot = 0; f.evolve = 1;
    f.max_steps = max_steps; f.tol = tol; f.base_threshold = base_threshold;
    ft::evolve_reset_kernel<<<1, 1, 0, s>>>(pab.ws.ctl);
    for (int i = 0; i < max_steps; ++i) {
        k<<<pab.num_tiles, FT_TPB, 0, s>>>((i & 1) ? pba : pab);
        ft::finalize_kernel<<<1, 1024, 0, s>>>(f);
    }
    ft::evolve_report_kernel<<<1, 1, 0, s>>>(pab.ws.ctl, (long long*)control);
    return cuda_check("ft_evolve");
}
