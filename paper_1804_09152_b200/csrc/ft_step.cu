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
// Work split: one CTA per tile of FT_TPB consecutive vertex columns, one
// thread per column.  The tile's L rows, the PHI column descriptors of all
// its (vertex, neighbour) pairs and the gathered PHI entries are staged in
// shared memory with flat, independent loads (high memory-level
// parallelism); each thread then merges its neighbours' sorted PHI columns
// into a sorted register window of at most K layer rows, accumulating
// Lt(r, j) in ascending-u order -- exactly the reference accumulator order
// (first product assigned, then +=).  PHI(r, j) itself arrives through the
// diagonal u == j.  Columns whose union exceeds K rows are processed exactly
// in ascending row windows straight from global memory (slow path).
//
// Output: the tile's entries go to its fixed slot of the tiled work buffer
// (FT_SLOT entries) or, when they do not fit, to a pool range taken with
// one atomic; column j is described by (start, count).  No CTA ever waits
// for another.  Canonical CSC comes from ft_compact.
//
// EXACT mode (double storage) replays the reference arithmetic operation by
// operation; the library is compiled with -fmad=false (no FMA contraction)
// and sqrt / division are IEEE correctly rounded, so the result is bitwise
// identical to the numba reference.  FAST mode stores PHI in float and does
// all arithmetic in double, in the same order.

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ft_common.cuh"

namespace ft {

// exact 1.0 / n for n = 0..32 (host IEEE division; entry 0 unused)
__constant__ double c_recip[33];

struct StepParams {
    int n_v;
    int num_tiles;
    const int* __restrict__ lap_ptr;
    const int* __restrict__ lap_idx;
    const void* __restrict__ lap_val;
    const int* __restrict__ in_ptr;     // canonical input (IN_CANON)
    const int2* __restrict__ in_desc;   // tiled input
    const int* __restrict__ in_idx;
    const void* __restrict__ in_val;
    int2* __restrict__ out_desc;
    int* __restrict__ out_idx;
    void* __restrict__ out_val;
    long long cap;
    double w, a, e, eb, mu, dt;
    Workspace ws;
    int check_done;
    int finite;          // all couplings finite: enables the single-row closed form
};

struct FinalizeParams {
    Workspace ws;
    ft_step_stats* trace;
    long long tiled_cap;
    int fixed_slot;       // 1: write trace[0] (single step), 0: trace[steps_done]
    int evolve;           // evolve mode: convergence / done handling
    int max_steps;
    double tol;
    double base_threshold;
};

template <bool IN_CANON>
__device__ __forceinline__ int2 load_desc(const StepParams& p, int u) {
    if (IN_CANON) {
        const int a = __ldg(&p.in_ptr[u]);
        const int b = __ldg(&p.in_ptr[u + 1]);
        return make_int2(a, b - a);
    }
    return __ldg(&p.in_desc[u]);
}

// ---------------------------------------------------------------------------
// register window of layer rows for one vertex column

template <int K>
struct Win {
    int rows[K];
    double lam[K];   // Lt(r, j) accumulator (later reused for v / v')
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
// Lt accumulation, into the window (the K smallest such rows).  Global
// memory version (fallback tiles and the windowed slow path).
template <typename T, int K, bool UNIFORM, bool IN_CANON>
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
        const int2 d = load_desc<IN_CANON>(p, u);
        for (int c = d.x; c < d.x + d.y; ++c) {
            const int r = __ldg(&p.in_idx[c]);
            if (r <= lo) continue;
            const double ph = ldv<T>(p.in_val, c);
            win_insert<K>(w, r, ph * l, diag, ph);
        }
    }
}

// ---------------------------------------------------------------------------
// shared-memory staging of a vertex tile
//
// The tile's L rows are one contiguous range of L^T, loaded coalesced; the
// PHI descriptors of all (vertex, neighbour) pairs are fetched with
// kLPV independent loads per thread, offsets come from a block scan, and
// the gathered PHI entries are fetched flat into shared memory.  Each
// thread then pays ~3 memory round trips instead of a dependent chain per
// neighbour.  Tiles beyond the staging capacity (very high degree or very
// dense bands) fall back to direct per-thread gathers (also exact).

constexpr int kLPV = 8;                    // staged L entries per vertex (capacity)
constexpr int kLMAX = FT_TPB * kLPV;       // staged L entries per tile
constexpr int kEMAX = kLMAX * 5 / 2;       // staged PHI entries per tile

template <typename T, bool UNIFORM>
struct Stage {
    int rp[FT_TPB + 1];    // L^T column pointers of the tile (absolute)
    int u[kLMAX];          // neighbour ids
    int2 oc[kLMAX];        // staged (offset, count) of PHI(:, u) per pair
    int er[kEMAX];         // gathered PHI rows
    T ev[kEMAX];           // gathered PHI values
    T lv[UNIFORM ? 1 : kLMAX];
    int scan[FT_WARPS];
};

// Phases A-C.  Returns true when the whole tile is staged (block-uniform).
// Thread t owns pairs e = t + k*FT_TPB: it loads their descriptors (kLPV
// independent loads), reserves their entries' space with one block scan,
// and gathers the entries itself -- the descriptors never leave registers.
template <typename T, bool UNIFORM, bool IN_CANON>
__device__ __forceinline__ bool stage_tile(Stage<T, UNIFORM>& s, int j0, int jn, const StepParams& p) {
    const int tid = threadIdx.x;
    // A: L rows of the tile
    if (tid < jn) s.rp[tid] = __ldg(&p.lap_ptr[j0 + tid]);
    if (tid == 0) s.rp[jn] = __ldg(&p.lap_ptr[j0 + jn]);
    __syncthreads();
    const int LB = s.rp[0];
    const int nL = s.rp[jn] - LB;
    if (nL > kLMAX) return false;
    int ur[kLPV];
#pragma unroll
    for (int k = 0; k < kLPV; ++k) {
        const int e = tid + k * FT_TPB;
        if (e < nL) {
            ur[k] = __ldg(&p.lap_idx[LB + e]);
            s.u[e] = ur[k];
            if (!UNIFORM) s.lv[e] = __ldg(((const T*)p.lap_val) + LB + e);
        }
    }
    // B: PHI descriptors of the owned pairs
    int2 dr[kLPV];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kLPV; ++k) {
        const int e = tid + k * FT_TPB;
        dr[k] = make_int2(0, 0);
        if (e < nL) dr[k] = load_desc<IN_CANON>(p, ur[k]);
    }
    int loc[kLPV];
#pragma unroll
    for (int k = 0; k < kLPV; ++k) { loc[k] = sum; sum += dr[k].y; }
    int nE;
    const int pre = block_excl_scan<FT_TPB>(sum, s.scan, &nE);
    if (nE > kEMAX) return false;
    // C: gather the owned pairs' entries; first entries go to registers
    // before any store so each thread keeps kLPV loads in flight
    {
        int r0[kLPV];
        T v0[kLPV];
#pragma unroll
        for (int k = 0; k < kLPV; ++k) {
            if (dr[k].y > 0) {
                r0[k] = __ldg(&p.in_idx[dr[k].x]);
                v0[k] = __ldg(((const T*)p.in_val) + dr[k].x);
            }
        }
#pragma unroll
        for (int k = 0; k < kLPV; ++k) {
            const int e = tid + k * FT_TPB;
            if (e < nL) {
                const int o = pre + loc[k];
                const int n = dr[k].y;
                s.oc[e] = make_int2(o, n);
                if (n > 0) { s.er[o] = r0[k]; s.ev[o] = v0[k]; }
                for (int t = 1; t < n; ++t) {
                    s.er[o + t] = __ldg(&p.in_idx[dr[k].x + t]);
                    s.ev[o + t] = __ldg(((const T*)p.in_val) + dr[k].x + t);
                }
            }
        }
    }
    __syncthreads();
    return true;
}

// Phase D: fill the register window of vertex (j0 + tid) from the stage.
// One pass over the vertex's gathered entries in entry order (= ascending
// u, the reference accumulation order): each entry's row is looked up among
// the rows seen so far (slot 0 first: inside a cell every entry has the
// same row) and its product added to that slot's Lt accumulator; unseen rows
// are appended.  PHI(r, j) comes from the diagonal pair, and the window is
// then sorted by row.
// Starting an accumulator at +0.0 instead of assigning the first product
// only changes the sign of an exact-zero sum; zero sums are not stored by
// the reference (Lt == 0 is dropped) and are outside the skeleton either
// way, so the result is bitwise the reference's.  Sets w.more when the
// union exceeds K rows.
template <int K>
__device__ __forceinline__ void win_sort(Win<K>& w, unsigned int active) {
    // insertion sort by row with warp-uniform trip counts (K <= 16)
#pragma unroll
    for (int a = 1; a < K; ++a) {
        if (!__any_sync(active, a < w.m)) break;
#pragma unroll
        for (int b = a; b > 0; --b) {
            const bool sw = (b < w.m) && (w.rows[b - 1] > w.rows[b]);
            if (sw) {
                const int tr = w.rows[b]; w.rows[b] = w.rows[b - 1]; w.rows[b - 1] = tr;
                const double tl = w.lam[b]; w.lam[b] = w.lam[b - 1]; w.lam[b - 1] = tl;
                const double tp = w.phi[b]; w.phi[b] = w.phi[b - 1]; w.phi[b - 1] = tp;
            }
        }
    }
}

template <typename T, int K, bool UNIFORM>
__device__ __forceinline__ void gather_staged(Win<K>& w, int j, const Stage<T, UNIFORM>& s,
                                              const double* recip) {
    const int tid = threadIdx.x;
    const int LB = s.rp[0];
    const int e0 = s.rp[tid] - LB;
    const int e1 = s.rp[tid + 1] - LB;
    const int deg = e1 - e0 - 1;
    const double invdeg = UNIFORM ? (deg <= 32 ? recip[deg] : 1.0 / (double)deg) : 0.0;
    w.more = false;
#pragma unroll
    for (int i = 0; i < K; ++i) { w.rows[i] = INT_MAX; w.lam[i] = 0.0; w.phi[i] = 0.0; }
    w.m = 0;
    int fd0 = 0, fd1 = 0;   // entries of the diagonal pair (u == j)
    for (int e = e0; e < e1; ++e) {
        const bool diag = (s.u[e] == j);
        const double l = UNIFORM ? (diag ? -1.0 : invdeg) : (double)s.lv[e];
        const int2 oc = s.oc[e];
        if (diag) { fd0 = oc.x; fd1 = oc.x + oc.y; }
        for (int f = oc.x; f < oc.x + oc.y; ++f) {
            const int r = s.er[f];
            const double prod = (double)s.ev[f] * l;
            if (r == w.rows[0]) {
                w.lam[0] = w.lam[0] + prod;
            } else if (w.m == 0) {
                w.rows[0] = r;
                w.lam[0] = 0.0 + prod;
                w.m = 1;
            } else {
                bool hit = false;
#pragma unroll
                for (int i = 1; i < K; ++i) {
                    if (w.rows[i] == r) { w.lam[i] = w.lam[i] + prod; hit = true; }
                }
                if (!hit) {
                    if (w.m == K) {
                        w.more = true;
                    } else {
#pragma unroll
                        for (int i = 1; i < K; ++i)
                            if (i == w.m) { w.rows[i] = r; w.lam[i] = 0.0 + prod; }
                        w.m++;
                    }
                }
            }
        }
    }
    if (w.more) return;
    for (int f = fd0; f < fd1; ++f) {
        const int r = s.er[f];
        const double ph = (double)s.ev[f];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (w.rows[i] == r) w.phi[i] = ph;
    }
    win_sort<K>(w, __activemask());
}

// ---------------------------------------------------------------------------
// per-column arithmetic (Appendix A of SURVEY.md; _kernels.py:179-282)

struct Agg {
    int n;
    int first_row;
    double phi0;
    double sl, sp, sr;
    int bad_phi_row, bad_lt_row;
};

__device__ __forceinline__ void agg_init(Agg& g) {
    g.n = 0; g.first_row = -1; g.phi0 = 0.0; g.sl = 0.0; g.sp = 0.0; g.sr = 0.0;
    g.bad_phi_row = -1; g.bad_lt_row = -1;
}

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

struct Coef {
    bool hb;
    double rb, spc, nif, agg, inv_ni, sl, sr;
};

__device__ __forceinline__ Coef make_coef(const Agg& g, const StepParams& p, const double* recip) {
    Coef c;
    c.hb = (g.n > 0) && (g.first_row == 0);
    c.rb = c.hb ? sqrt(g.phi0) : 0.0;
    c.spc = c.hb ? g.sp - g.phi0 : g.sp;
    const int n_cells = c.hb ? g.n - 1 : g.n;
    c.inv_ni = (recip && g.n <= 32) ? recip[g.n] : 1.0 / (double)g.n;
    c.nif = (double)g.n;
    double aggw = (p.w * fmax((double)n_cells - 1.0, 0.0)) * c.spc;
    if (c.hb) aggw = aggw + p.w * c.spc;
    c.agg = ((0.5 * p.a) * (c.nif - 1.0)) * g.sl + aggw;
    c.sl = g.sl;
    c.sr = g.sr;
    return c;
}

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

__device__ __forceinline__ double update_entry_sq(int r, double ph, double lh, double rj, const Coef& c,
                                                  const StepParams& p, bool& nan) {
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

struct VRes {
    int cnt;          // output entries (normalised value != 0)
    int nskel;        // skeleton entries
    double bm;        // base mass of the column
    double maxd;      // max |v' - phi_old|
    bool nan;
    int bad_phi_row, bad_lt_row;
};

__device__ __forceinline__ void vres_init(VRes& r) {
    r.cnt = 0; r.nskel = 0; r.bm = 0.0; r.maxd = 0.0;
    r.nan = false; r.bad_phi_row = -1; r.bad_lt_row = -1;
}

// Update + normalise one column held entirely in the window.  On return
// w.lam[i] holds v' for the slots flagged in out_mask (entries to emit).
template <int K>
__device__ __forceinline__ void process_window(Win<K>& w, const StepParams& p, VRes& res,
                                               unsigned int& out_mask, const double* recip) {
    const unsigned int active = __activemask();
    // skeleton membership and pattern checks (no arithmetic yet)
    unsigned int skel_mask = 0;
    int n = 0;
    res.bad_phi_row = -1;
    res.bad_lt_row = -1;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (!__any_sync(active, i < w.m)) break;
        if (i < w.m) {
            const double ph = w.phi[i], lm = w.lam[i];
            const bool in = in_skeleton(ph, lm);
            if (ph != 0.0 && !in) res.bad_phi_row = w.rows[i];
            if (lm != 0.0 && !in) res.bad_lt_row = w.rows[i];
            if (in) { skel_mask |= 1u << i; ++n; }
        }
    }
    res.nskel = n;
    out_mask = 0;
    if (n == 0) return;
    if (p.finite && n == 1) {
        // One skeleton row: with finite couplings every term of the update
        // cancels exactly (sl - lt = 0, sp_cells - phi = 0, sr - rj = 0,
        // n_cells - 1 <= 0, nif - 1 = 0), so d = +-0 and v = clamp(phi),
        // bit for bit what the reference's arithmetic produces.
        int slot = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (skel_mask == (1u << i)) slot = i;
        double ph1 = 0.0, lm1 = 0.0;
        int r1 = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i == slot) { ph1 = w.phi[i]; lm1 = w.lam[i]; r1 = w.rows[i]; }
        if (isfinite(ph1) && isfinite(lm1)) {
            double v = ph1;
            if (v > 1.0) v = 1.0;
            else if (v <= 0.0) v = 0.0;
            const double s = 0.0 + v;
            const bool spos = s > 0.0;
            const double nv = spos ? v * (1.0 / s) : v;
            if (nv != 0.0) {
                res.cnt = 1;
                out_mask = 1u << slot;
                if (r1 == 0) res.bm = nv;
            }
            const double dd = fabs(nv - ph1);
            if (dd > res.maxd) res.maxd = dd;
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (i == slot) w.lam[i] = nv;
            return;
        }
    }
    Agg g;
    agg_init(g);
    double sq[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        sq[i] = 0.0;
        if (skel_mask & (1u << i)) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (g.n == 0) { g.first_row = w.rows[i]; g.phi0 = ph; }
            g.n++;
            const double lh = (lm != 0.0) ? lm : 0.0;
            sq[i] = sqrt(ph);
            g.sl = g.sl + lh;
            g.sp = g.sp + ph;
            g.sr = g.sr + sq[i];
        }
    }
    const Coef c = make_coef(g, p, recip);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (skel_mask & (1u << i)) {
            const double ph = w.phi[i], lm = w.lam[i];
            const double v = update_entry_sq(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, sq[i], c, p, res.nan);
            w.lam[i] = v;
            s = s + v;
        }
    }
    const bool spos = s > 0.0;
    const double inv = spos ? 1.0 / s : 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (skel_mask & (1u << i)) {
            const double nv = spos ? w.lam[i] * inv : w.lam[i];
            if (nv != 0.0) {
                res.cnt++;
                out_mask |= 1u << i;
                if (w.rows[i] == 0) res.bm = res.bm + nv;
            }
            const double dd = fabs(nv - w.phi[i]);
            if (dd > res.maxd) res.maxd = dd;
            w.lam[i] = nv;
        }
    }
}

__device__ __forceinline__ void report_flags(const VRes& res, int j, const StepParams& p) {
    if (res.nan) atomicMax(&p.ws.ctl->nan_key, (unsigned int)(INT_MAX - j));
    if (res.bad_phi_row >= 0)
        atomicMax(&p.ws.ctl->bad_phi_key, ~(((unsigned long long)j << 32) | (unsigned int)res.bad_phi_row));
    if (res.bad_lt_row >= 0)
        atomicMax(&p.ws.ctl->bad_lt_key, ~(((unsigned long long)j << 32) | (unsigned int)res.bad_lt_row));
}

template <typename T, int K>
__device__ __forceinline__ void emit_window(const Win<K>& w, unsigned int out_mask, long long off,
                                            const StepParams& p) {
    T* ov = (T*)p.out_val;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (out_mask & (1u << i)) {
            p.out_idx[off] = w.rows[i];
            ov[off] = (T)w.lam[i];
            ++off;
        }
    }
}

// --- slow path: union larger than K, processed in ascending row windows ----

template <typename T, int K, bool UNIFORM, bool IN_CANON>
__device__ __noinline__ void vertex_slow(int j, const StepParams& p, VRes& res, long long emit_off,
                                         bool emit) {
    Win<K> w;
    Agg g;
    agg_init(g);
    int lo = -1;
    do {
        gather<T, K, UNIFORM, IN_CANON>(w, j, lo, p);
        pass_aggregate<K>(w, g);
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    res.nskel = g.n;
    res.bad_phi_row = g.bad_phi_row;
    res.bad_lt_row = g.bad_lt_row;
    res.nan = false;
    res.cnt = 0; res.bm = 0.0; res.maxd = 0.0;
    if (g.n == 0) return;
    const Coef c = make_coef(g, p, nullptr);
    double s = 0.0;
    lo = -1;
    do {
        gather<T, K, UNIFORM, IN_CANON>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            s = s + update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p, res.nan);
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    const bool spos = s > 0.0;
    const double inv = spos ? 1.0 / s : 0.0;
    bool dummy = false;
    T* ov = (T*)p.out_val;
    lo = -1;
    do {
        gather<T, K, UNIFORM, IN_CANON>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            const double v = update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p, dummy);
            const double nv = spos ? v * inv : v;
            if (nv != 0.0) {
                if (emit) {
                    p.out_idx[emit_off] = w.rows[i];
                    ov[emit_off] = (T)nv;
                    ++emit_off;
                }
                res.cnt++;
                if (w.rows[i] == 0) res.bm = res.bm + nv;
            }
            const double dd = fabs(nv - ph);
            if (dd > res.maxd) res.maxd = dd;
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
}

// ---------------------------------------------------------------------------
// the fused step kernel (fast path)
//
// Columns that do not fit the register window (union > K rows) and every
// column of a tile that could not be staged are left to fixup_kernel: they
// contribute no entries to the tile slot, their bit is set in slow_mask
// and the tile is queued once in slow_list.  Keeping the slow paths out of
// this kernel keeps its register footprint small.

// Tile epilogue shared by both kernels: block scan of the output counts,
// placement (tile slot, or a pool range), per-tile statistics.
struct TileOut {
    int local_off;
    long long base;   // -1: overflow, nothing is written
};

template <bool POOL_ONLY>
__device__ __forceinline__ TileOut tile_epilogue(int cnt, int nskel, double bmv, double maxd, int tile,
                                                 double* bm_slot, const StepParams& p, int* s_scan,
                                                 double* s_wbm, double* s_wmax, int* s_wskel,
                                                 long long* s_base) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int tile_total;
    TileOut o;
    o.local_off = block_excl_scan<FT_TPB>(cnt, s_scan, &tile_total);
    const int skel = warp_sum(nskel);
    const double bm = warp_sum(bmv);
    double mx = maxd;
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, k));
    if (lane == 0) { s_wskel[warp] = skel; s_wbm[warp] = bm; s_wmax[warp] = mx; }
    __syncthreads();
    if (tid == 0) {
        long long base = POOL_ONLY ? -1 : (long long)tile * FT_SLOT;
        if (tile_total > 0 && (POOL_ONLY || tile_total > FT_SLOT)) {
            const unsigned long long q = atomicAdd(&p.ws.ctl->pool_next, (unsigned long long)tile_total);
            base = (long long)p.num_tiles * FT_SLOT + (long long)q;
        }
        if (base + tile_total > p.cap) {
            atomicExch(&p.ws.ctl->overflow, 1);
            base = -1;
        }
        if (tile_total == 0 && POOL_ONLY) base = 0;
        *s_base = base;
        double tbm = 0.0, tmx = 0.0;
        int tsk = 0;
#pragma unroll
        for (int k = 0; k < FT_WARPS; ++k) { tbm = tbm + s_wbm[k]; tmx = fmax(tmx, s_wmax[k]); tsk += s_wskel[k]; }
        *bm_slot = tbm;
        if (POOL_ONLY) {
            // fixup path (rare): fold into the global accumulators
            if (tmx > 0.0) atomicMax(&p.ws.ctl->maxdelta_bits, (unsigned long long)__double_as_longlong(tmx));
            if (tsk) atomicAdd(&p.ws.ctl->skel_total, (unsigned long long)tsk);
            if (tile_total) atomicAdd(&p.ws.ctl->nnz_total, (unsigned long long)tile_total);
        } else {
            // fast path: per-tile slots, reduced by finalize_kernel (no
            // same-address atomics across the ~10^5 tiles of a step)
            p.ws.tile_maxd[tile] = tmx;
            p.ws.tile_cs[tile] = make_int2(tile_total, tsk);
        }
    }
    __syncthreads();
    o.base = *s_base;
    return o;
}

extern __shared__ __align__(16) unsigned char ft_dyn_smem[];

template <typename T, int K, bool UNIFORM, bool IN_CANON>
__global__ void __launch_bounds__(FT_TPB, 5) step_kernel(const StepParams p) {
    Stage<T, UNIFORM>& stg = *reinterpret_cast<Stage<T, UNIFORM>*>(ft_dyn_smem);
    __shared__ double s_wbm[FT_WARPS];
    __shared__ double s_wmax[FT_WARPS];
    __shared__ int s_wskel[FT_WARPS];
    __shared__ unsigned int s_wslow[FT_WARPS];
    __shared__ long long s_base;
    __shared__ double s_recip[33];

    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    if (threadIdx.x < 33) s_recip[threadIdx.x] = c_recip[threadIdx.x];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int tile = blockIdx.x;
    const int j0 = tile * FT_TPB;
    const int jn = min(FT_TPB, p.n_v - j0);
    const int j = j0 + tid;
    const bool active = tid < jn;

    const bool staged = stage_tile<T, UNIFORM, IN_CANON>(stg, j0, jn, p);

    Win<K> w;
    VRes res;
    vres_init(res);
    bool slow = false;
    unsigned int out_mask = 0;
    if (active) {
        if (staged) gather_staged<T, K, UNIFORM>(w, j, stg, s_recip);
        slow = !staged || w.more;
        if (!slow) {
            process_window<K>(w, p, res, out_mask, s_recip);
            report_flags(res, j, p);
        }
    }
    const unsigned int slow_bits = __ballot_sync(0xffffffffu, slow);
    if (lane == 0) s_wslow[warp] = slow_bits;
    const TileOut o = tile_epilogue<false>(res.cnt, res.nskel, res.bm, res.maxd, tile, &p.ws.tile_bm[tile], p,
                                           stg.scan, s_wbm, s_wmax, s_wskel, &s_base);
    if (tid == 0) {
        unsigned int any_slow = 0;
#pragma unroll
        for (int k = 0; k < FT_WARPS; ++k) any_slow |= s_wslow[k];
        p.ws.tile_bm_slow[2 * tile] = 0.0;
        p.ws.tile_bm_slow[2 * tile + 1] = 0.0;
        if (any_slow) {
            const int q = atomicAdd(&p.ws.ctl->slow_count, 1);
            p.ws.slow_list[q] = tile;
#pragma unroll
            for (int k = 0; k < FT_WARPS; ++k) p.ws.slow_mask[(size_t)tile * FT_WARPS + k] = s_wslow[k];
        }
    }
    if (!active || slow || o.base < 0) return;
    const long long off = o.base + o.local_off;
    p.out_desc[j] = make_int2((int)off, res.cnt);
    if (out_mask) emit_window<T, K>(w, out_mask, off, p);
}

// ---------------------------------------------------------------------------
// fixup kernel: the columns the fast path left behind.  One CTA per queued
// tile (grid-stride over slow_list): the tile is staged again and the slow
// columns use a KF-row window from shared memory; columns beyond KF rows
// and tiles that cannot be staged use the exact windowed global path.  The
// tile's base mass goes to tile_bm_slow[tile] (fixed reduction order).

// Warp-cooperative exact processing of one column from the stage, used by
// the fixup kernel for columns whose layer union is wider than the fast
// path's register window.  Lane k owns the column's k-th (vertex,
// neighbour) pair (chunks of 32).  Rows are visited in ascending order:
// each round the warp finds the next row (min over all pairs' entries),
// then the row's per-pair products are summed in pair order (= ascending
// u, the reference accumulation order) by a shuffle chain.  No per-column
// arrays, no width limit.
struct WarpCol {
    int e0, e1;       // the column's pairs in the stage
    int j;            // the column (vertex) id
    double invdeg;
};

template <typename T, bool UNIFORM>
__device__ __forceinline__ WarpCol warp_col(const Stage<T, UNIFORM>& s, int v, int j, const double* recip) {
    WarpCol c;
    const int LB = s.rp[0];
    c.e0 = s.rp[v] - LB;
    c.e1 = s.rp[v + 1] - LB;
    c.j = j;
    const int deg = c.e1 - c.e0 - 1;
    c.invdeg = deg <= 32 ? recip[deg] : 1.0 / (double)deg;
    return c;
}

// smallest row > lo among the column's entries (INT_MAX when none)
template <typename T, bool UNIFORM>
__device__ __forceinline__ int warp_next_row(const Stage<T, UNIFORM>& s, const WarpCol& c, int lo, int lane) {
    int best = INT_MAX;
    for (int e = c.e0 + lane; e < c.e1; e += 32) {
        const int2 oc = s.oc[e];
        for (int f = oc.x; f < oc.x + oc.y; ++f) {
            const int r = s.er[f];
            if (r > lo) { if (r < best) best = r; break; }   // rows ascend within a pair
        }
    }
    return __reduce_min_sync(0xffffffffu, best);
}

// (Lt(r, j), PHI(r, j)) of one row, identical on all lanes
template <typename T, bool UNIFORM>
__device__ __forceinline__ void warp_row(const Stage<T, UNIFORM>& s, const WarpCol& c, int r, int lane,
                                         double& lam, double& phi) {
    lam = 0.0;
    phi = 0.0;
    for (int base = c.e0; base < c.e1; base += 32) {
        const int e = base + lane;
        bool has = false;
        double prod = 0.0, ph = 0.0;
        bool diag = false;
        if (e < c.e1) {
            const int2 oc = s.oc[e];
            diag = (s.u[e] == c.j);
            for (int f = oc.x; f < oc.x + oc.y; ++f) {
                const int rr = s.er[f];
                if (rr == r) {
                    ph = (double)s.ev[f];
                    const double l = UNIFORM ? (diag ? -1.0 : c.invdeg) : (double)s.lv[e];
                    prod = ph * l;
                    has = true;
                    break;
                }
                if (rr > r) break;
            }
        }
        const unsigned int hb = __ballot_sync(0xffffffffu, has);
        const unsigned int db = __ballot_sync(0xffffffffu, has && diag);
        const int n = min(32, c.e1 - base);
        for (int k = 0; k < n; ++k) {          // in pair order: exact reference order
            const double pk = __shfl_sync(0xffffffffu, prod, k);
            if ((hb >> k) & 1u) lam = lam + pk;
        }
        if (db) phi = __shfl_sync(0xffffffffu, ph, __ffs(db) - 1);
    }
}

// pass = 0: aggregates; 1: column sum of v; 2: normalise + count; 3: emit
template <typename T, bool UNIFORM>
__device__ __forceinline__ void warp_column(const Stage<T, UNIFORM>& s, int v, int j, const StepParams& p,
                                            const double* recip, VRes& res, long long emit_off) {
    const int lane = threadIdx.x & 31;
    const WarpCol c = warp_col<T, UNIFORM>(s, v, j, recip);
    Agg g;
    agg_init(g);
    int lo = -1;
    for (;;) {
        const int r = warp_next_row<T, UNIFORM>(s, c, lo, lane);
        if (r == INT_MAX) break;
        double lm, ph;
        warp_row<T, UNIFORM>(s, c, r, lane, lm, ph);
        const bool in = in_skeleton(ph, lm);
        if (ph != 0.0 && !in) g.bad_phi_row = r;
        if (lm != 0.0 && !in) g.bad_lt_row = r;
        if (in) {
            if (g.n == 0) { g.first_row = r; g.phi0 = ph; }
            g.n++;
            g.sl = g.sl + ((lm != 0.0) ? lm : 0.0);
            g.sp = g.sp + ph;
            g.sr = g.sr + sqrt(ph);
        }
        lo = r;
    }
    res.nskel = g.n;
    res.bad_phi_row = g.bad_phi_row;
    res.bad_lt_row = g.bad_lt_row;
    if (g.n == 0) return;
    const Coef cf = make_coef(g, p, recip);
    double sum = 0.0;
    lo = -1;
    for (;;) {
        const int r = warp_next_row<T, UNIFORM>(s, c, lo, lane);
        if (r == INT_MAX) break;
        double lm, ph;
        warp_row<T, UNIFORM>(s, c, r, lane, lm, ph);
        if (in_skeleton(ph, lm)) sum = sum + update_entry(r, ph, (lm != 0.0) ? lm : 0.0, cf, p, res.nan);
        lo = r;
    }
    const bool spos = sum > 0.0;
    const double inv = spos ? 1.0 / sum : 0.0;
    bool dummy = false;
    T* ov = (T*)p.out_val;
    lo = -1;
    for (;;) {
        const int r = warp_next_row<T, UNIFORM>(s, c, lo, lane);
        if (r == INT_MAX) break;
        double lm, ph;
        warp_row<T, UNIFORM>(s, c, r, lane, lm, ph);
        if (in_skeleton(ph, lm)) {
            const double vv = update_entry(r, ph, (lm != 0.0) ? lm : 0.0, cf, p, dummy);
            const double nv = spos ? vv * inv : vv;
            if (nv != 0.0) {
                if (emit_off >= 0 && lane == 0) {
                    p.out_idx[emit_off] = r;
                    ov[emit_off] = (T)nv;
                }
                if (emit_off >= 0) ++emit_off;
                res.cnt++;
                if (r == 0) res.bm = res.bm + nv;
            }
            const double dd = fabs(nv - ph);
            if (dd > res.maxd) res.maxd = dd;
        }
        lo = r;
    }
}

// fixup kernel: the columns the fast path left behind.  Work unit = half a
// queued tile (64 columns), staged in shared memory (half tiles fit the
// stage even in dense bands); one warp per wide column (warp_column).
// Half tiles that still exceed the stage use the exact windowed
// global-memory path, one thread per column.
template <typename T, bool UNIFORM, bool IN_CANON>
__global__ void __launch_bounds__(FT_TPB) fixup_kernel(const StepParams p) {
    constexpr int HALF = FT_TPB / 2;
    Stage<T, UNIFORM>& stg = *reinterpret_cast<Stage<T, UNIFORM>*>(ft_dyn_smem);
    __shared__ int s_list[HALF];
    __shared__ int s_cnt[HALF];
    __shared__ int s_skel[HALF];
    __shared__ double s_bm[HALF];
    __shared__ double s_mx[HALF];
    __shared__ int s_ns;
    __shared__ int s_scan[FT_WARPS];
    __shared__ long long s_base;
    __shared__ double s_recip[33];
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    if (threadIdx.x < 33) s_recip[threadIdx.x] = c_recip[threadIdx.x];
    const int n_units = 2 * *(volatile int*)&p.ws.ctl->slow_count;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int q = blockIdx.x; q < n_units; q += gridDim.x) {
        const int tile = p.ws.slow_list[q >> 1];
        const int half = q & 1;
        const int v0 = half * HALF;
        const int j0 = tile * FT_TPB + v0;
        const int jn = max(0, min(HALF, p.n_v - j0));
        const unsigned int* msk = &p.ws.slow_mask[(size_t)tile * FT_WARPS + half * (HALF / 32)];
        const unsigned int m0 = msk[0], m1 = msk[1];
        if ((m0 | m1) == 0u || jn == 0) continue;   // block-uniform
        if (tid == 0) {
            int n = 0;
            for (int v = 0; v < HALF; ++v)
                if (((v < 32 ? m0 : m1) >> (v & 31)) & 1u) s_list[n++] = v;
            s_ns = n;
        }
        const bool staged = stage_tile<T, UNIFORM, IN_CANON>(stg, j0, jn, p);   // syncs
        const int ns = s_ns;
        // counting passes
        if (staged) {
            for (int k = warp; k < ns; k += FT_WARPS) {
                const int v = s_list[k];
                VRes res;
                vres_init(res);
                warp_column<T, UNIFORM>(stg, v, j0 + v, p, s_recip, res, -1);
                if (lane == 0) {
                    s_cnt[k] = res.cnt; s_skel[k] = res.nskel; s_bm[k] = res.bm; s_mx[k] = res.maxd;
                    report_flags(res, j0 + v, p);
                }
            }
        } else if (tid < ns) {
            const int v = s_list[tid];
            VRes res;
            vres_init(res);
            vertex_slow<T, 8, UNIFORM, IN_CANON>(j0 + v, p, res, 0, false);
            s_cnt[tid] = res.cnt; s_skel[tid] = res.nskel; s_bm[tid] = res.bm; s_mx[tid] = res.maxd;
            report_flags(res, j0 + v, p);
        }
        __syncthreads();
        int total;
        const int loc = block_excl_scan<FT_TPB>(tid < ns ? s_cnt[tid] : 0, s_scan, &total);
        if (tid == 0) {
            long long base = 0;
            if (total > 0) {
                base = (long long)p.num_tiles * FT_SLOT +
                       (long long)atomicAdd(&p.ws.ctl->pool_next, (unsigned long long)total);
                if (base + total > p.cap) { atomicExch(&p.ws.ctl->overflow, 1); base = -1; }
            }
            s_base = base;
            double bm = 0.0, mx = 0.0;
            long long sk = 0;
            for (int k = 0; k < ns; ++k) { bm = bm + s_bm[k]; mx = fmax(mx, s_mx[k]); sk += s_skel[k]; }
            p.ws.tile_bm_slow[2 * tile + half] = bm;
            if (mx > 0.0) atomicMax(&p.ws.ctl->maxdelta_bits, (unsigned long long)__double_as_longlong(mx));
            if (sk) atomicAdd(&p.ws.ctl->skel_total, (unsigned long long)sk);
            if (total) atomicAdd(&p.ws.ctl->nnz_total, (unsigned long long)total);
        }
        if (tid < ns) s_cnt[tid] = loc;    // reuse: column offset within the unit
        __syncthreads();
        const long long base = s_base;
        if (base >= 0) {
            if (staged) {
                for (int k = warp; k < ns; k += FT_WARPS) {
                    const int v = s_list[k];
                    const long long off = base + s_cnt[k];
                    VRes res;
                    vres_init(res);
                    warp_column<T, UNIFORM>(stg, v, j0 + v, p, s_recip, res, off);
                    if (lane == 0) p.out_desc[j0 + v] = make_int2((int)off, res.cnt);
                }
            } else if (tid < ns) {
                const int v = s_list[tid];
                const long long off = base + s_cnt[tid];
                VRes res;
                vres_init(res);
                vertex_slow<T, 8, UNIFORM, IN_CANON>(j0 + v, p, res, off, true);
                p.out_desc[j0 + v] = make_int2((int)off, res.cnt);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// per-step finalisation: deterministic two-level base-mass reduction (fixed
// per-CTA ranges, then the last CTA sums the partials in order), stats
// record, error / convergence flags, accumulator reset.

#define FT_FIN_CTAS 64
#define FT_FIN_TPB 256

__global__ void __launch_bounds__(FT_FIN_TPB) finalize_kernel(const FinalizeParams f) {
    Control* ctl = f.ws.ctl;
    if (f.evolve && *(volatile int*)&ctl->done) return;
    __shared__ double s_part[FT_FIN_TPB / 32];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int nt = f.ws.num_tiles;
    const int per = (nt + gridDim.x - 1) / gridDim.x;
    const int t0 = blockIdx.x * per, t1 = min(nt, t0 + per);
    double acc = 0.0, amx = 0.0;
    long long acnt = 0, askel = 0;
    for (int t = t0 + tid; t < t1; t += FT_FIN_TPB) {
        acc = acc + (f.ws.tile_bm[t] + (f.ws.tile_bm_slow[2 * t] + f.ws.tile_bm_slow[2 * t + 1]));
        amx = fmax(amx, f.ws.tile_maxd[t]);
        const int2 cs = f.ws.tile_cs[t];
        acnt += cs.x;
        askel += cs.y;
    }
    acc = warp_sum(acc);
    acnt = warp_sum(acnt);
    askel = warp_sum(askel);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amx = fmax(amx, __shfl_down_sync(0xffffffffu, amx, o));
    __shared__ double s_mx[FT_FIN_TPB / 32];
    __shared__ long long s_cnt[FT_FIN_TPB / 32], s_skel[FT_FIN_TPB / 32];
    if ((tid & 31) == 0) { s_part[tid >> 5] = acc; s_mx[tid >> 5] = amx; s_cnt[tid >> 5] = acnt; s_skel[tid >> 5] = askel; }
    __syncthreads();
    if (tid == 0) {
        double b = 0.0, m = 0.0;
        long long c = 0, k = 0;
        for (int q = 0; q < FT_FIN_TPB / 32; ++q) { b = b + s_part[q]; m = fmax(m, s_mx[q]); c += s_cnt[q]; k += s_skel[q]; }
        f.ws.fin_part[blockIdx.x] = b;
        f.ws.fin_maxd[blockIdx.x] = m;
        f.ws.fin_cnt[blockIdx.x] = c;
        f.ws.fin_skel[blockIdx.x] = k;
        __threadfence();
        s_last = (atomicAdd(&ctl->fin_count, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || tid >= 32) return;
    __threadfence();
    // the last CTA combines the per-CTA partials with one warp: lane l owns
    // partials l, l+32 (fixed order), then a fixed shuffle tree
    double pb = 0.0, pm = 0.0;
    long long pc = 0, pk = 0;
    for (int q = tid; q < (int)gridDim.x; q += 32) {
        pb = pb + *(volatile double*)&f.ws.fin_part[q];
        pm = fmax(pm, *(volatile double*)&f.ws.fin_maxd[q]);
        pc += *(volatile long long*)&f.ws.fin_cnt[q];
        pk += *(volatile long long*)&f.ws.fin_skel[q];
    }
    pb = warp_sum(pb);
    pc = warp_sum(pc);
    pk = warp_sum(pk);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pm = fmax(pm, __shfl_down_sync(0xffffffffu, pm, o));
    if (tid != 0) return;
    ctl->fin_count = 0u;
    const double bm = pb;
    const double mxd = fmax(pm, __longlong_as_double((long long)ctl->maxdelta_bits));
    const long long nnz = pc + (long long)ctl->nnz_total;
    const long long nsk = pk + (long long)ctl->skel_total;

    const int slot = f.fixed_slot ? 0 : ctl->steps_done;
    ft_step_stats st;
    st.max_delta = mxd;
    st.base_mass = bm;
    st.nnz_phi = nnz;
    st.nnz_skel = nsk;
    st.nan_col = ctl->nan_key ? (int)(INT_MAX - ctl->nan_key) : -1;
    st.bad_col = -1; st.bad_row = -1; st.bad_is_lt = 0;
    const unsigned long long kp = ctl->bad_phi_key, kl = ctl->bad_lt_key;
    if (kp) { const unsigned long long k = ~kp; st.bad_col = (int)(k >> 32); st.bad_row = (int)(k & 0xffffffffULL); }
    else if (kl) { const unsigned long long k = ~kl; st.bad_col = (int)(k >> 32); st.bad_row = (int)(k & 0xffffffffULL); st.bad_is_lt = 1; }
    int status = FT_STATUS_OK;
    // the reference checks expand(PHI), expand(Lt), then NaN (field.py:238-250)
    if (st.bad_col >= 0) status = FT_STATUS_PATTERN;
    else if (st.nan_col >= 0) status = FT_STATUS_NAN;
    else if (ctl->overflow) status = FT_STATUS_OVERFLOW;
    const int stepno = ctl->steps_done + 1;
    st.step = stepno;
    st.needed = (long long)f.ws.num_tiles * FT_SLOT + (long long)ctl->pool_next;
    if (st.needed < f.tiled_cap) st.needed = f.tiled_cap;
    bool converged = false;
    if (status == FT_STATUS_OK && f.evolve)
        converged = (st.max_delta < f.tol) && (st.base_mass < f.base_threshold);
    st.status = converged ? FT_STATUS_CONVERGED : status;
    f.trace[slot] = st;

    ctl->maxdelta_bits = 0ULL;
    ctl->bad_phi_key = 0ULL;
    ctl->bad_lt_key = 0ULL;
    ctl->skel_total = 0ULL;
    ctl->nnz_total = 0ULL;
    ctl->pool_next = 0ULL;
    ctl->nan_key = 0u;
    ctl->overflow = 0;
    ctl->slow_count = 0;
    if (f.evolve) {
        if (status != FT_STATUS_OK) {
            ctl->done = 1;
            ctl->status = status;
            ctl->needed = st.needed;
        } else {
            ctl->steps_done = stepno;
            if (converged) { ctl->done = 1; ctl->status = FT_STATUS_CONVERGED; }
            else if (stepno >= f.max_steps) { ctl->done = 1; ctl->status = FT_STATUS_MAXSTEPS; }
        }
    }
}

// ---------------------------------------------------------------------------
// compaction: tiled -> canonical CSC

struct CompactParams {
    int n_v;
    const int2* desc[2];
    const int* idx[2];
    const void* val[2];
    int sel;               // 0/1: source buffer; -1: pick by evolve parity
    int* out_ptr;
    int* out_idx;
    void* out_val;
    long long cap;
    Workspace ws;
    ft_step_stats* stats;  // single-step mode record (nullable)
    long long* control;    // evolve mode (nullable)
    int check_status;      // skip when stats->status reports a failed step
};

__device__ __forceinline__ int compact_source(const CompactParams& c) {
    if (c.check_status && c.stats && *(volatile int*)&c.stats->status != FT_STATUS_OK) return -1;
    if (c.sel >= 0) return c.sel;
    const int n = c.ws.ctl->steps_done;
    return n == 0 ? -1 : ((n & 1) ? 0 : 1);
}

constexpr int kCPT = FT_CCH / FT_CTPB;   // columns per thread (8)

__global__ void __launch_bounds__(FT_CTPB) compact_count_kernel(const CompactParams c) {
    __shared__ int s_scan[FT_CTPB / 32];
    const int src = compact_source(c);
    if (src < 0) return;
    const int2* desc = c.desc[src];
    const int j0 = blockIdx.x * FT_CCH + threadIdx.x * kCPT;
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kCPT; ++k)
        if (j0 + k < c.n_v) sum += __ldg(&desc[j0 + k]).y;
    int tot;
    block_excl_scan<FT_CTPB>(sum, s_scan, &tot);
    if (threadIdx.x == 0) c.ws.chunk_off[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) compact_scan_kernel(const CompactParams c) {
    __shared__ long long s_part[32];
    const int src = compact_source(c);
    const int nc = c.ws.num_chunks;
    const int tid = threadIdx.x;
    long long* off = c.ws.chunk_off;
    if (src < 0) {
        if (tid == 0 && c.control) { c.control[3] = 0; c.control[4] = 0; c.control[5] = 0; }
        return;
    }
    const int per = (nc + 1023) / 1024;
    const int b0 = tid * per;
    long long sum = 0;
    for (int k = 0; k < per; ++k)
        if (b0 + k < nc) sum += off[b0 + k];
    long long incl = sum;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_part[warp] = incl;
    __syncthreads();
    long long pre = 0, tot = 0;
    for (int k = 0; k < 32; ++k) {
        if (k < warp) pre += s_part[k];
        tot += s_part[k];
    }
    long long run = pre + incl - sum;
    for (int k = 0; k < per; ++k) {
        if (b0 + k < nc) {
            const long long v = off[b0 + k];
            off[b0 + k] = run;
            run += v;
        }
    }
    if (tid == 0) {
        off[nc] = tot;
        const bool fits = tot <= c.cap && tot <= (long long)INT_MAX;
        off[nc + 1] = fits ? 1 : 0;
        if (fits) c.out_ptr[c.n_v] = (int)tot;
        if (c.stats) {
            c.stats->nnz_phi = tot;
            if (!fits) { c.stats->status = FT_STATUS_OUT_OVERFLOW; c.stats->needed = tot; }
            else if (!c.check_status) c.stats->status = FT_STATUS_OK;
        }
        if (c.control) { c.control[3] = fits ? 1 : 2; c.control[4] = tot; c.control[5] = tot; }
    }
}

template <typename T>
__global__ void __launch_bounds__(FT_CTPB) compact_copy_kernel(const CompactParams c) {
    __shared__ int s_scan[FT_CTPB / 32];
    const int src = compact_source(c);
    if (src < 0) return;
    if (c.ws.chunk_off[c.ws.num_chunks + 1] == 0) return;  // does not fit
    const int2* desc = c.desc[src];
    const int* sidx = c.idx[src];
    const T* sval = (const T*)c.val[src];
    T* oval = (T*)c.out_val;
    const int j0 = blockIdx.x * FT_CCH + threadIdx.x * kCPT;
    int2 d[kCPT];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
        d[k] = (j0 + k < c.n_v) ? __ldg(&desc[j0 + k]) : make_int2(0, 0);
        sum += d[k].y;
    }
    int tot;
    const int pre = block_excl_scan<FT_CTPB>(sum, s_scan, &tot);
    long long o = c.ws.chunk_off[blockIdx.x] + pre;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
        if (j0 + k < c.n_v) {
            c.out_ptr[j0 + k] = (int)o;
            for (int t = 0; t < d[k].y; ++t) {
                c.out_idx[o + t] = __ldg(&sidx[d[k].x + t]);
                oval[o + t] = __ldg(&sval[d[k].x + t]);
            }
            o += d[k].y;
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
}

// ---------------------------------------------------------------------------
// host side

typedef void (*StepKernelFn)(const StepParams);

struct KernelPick {
    StepKernelFn fn;
    size_t smem;
};

template <typename T, bool UNIFORM>
static size_t stage_bytes() { return sizeof(Stage<T, UNIFORM>); }

static KernelPick with_smem(StepKernelFn fn, size_t bytes) {
    // opt in to > 48 KB dynamic shared memory once per kernel
    static StepKernelFn done[64];
    static int n_done = 0;
    bool seen = false;
    for (int i = 0; i < n_done; ++i) seen |= (done[i] == fn);
    if (!seen) {
        cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (n_done < 64) done[n_done++] = fn;
    }
    return KernelPick{fn, bytes};
}

static KernelPick pick_fixup(int dtype, bool uniform, bool in_canon) {
    if (dtype == FT_F64) {
        if (uniform) return with_smem(in_canon ? fixup_kernel<double, true, true> : fixup_kernel<double, true, false>, stage_bytes<double, true>());
        return with_smem(in_canon ? fixup_kernel<double, false, true> : fixup_kernel<double, false, false>, stage_bytes<double, false>());
    }
    if (uniform) return with_smem(in_canon ? fixup_kernel<float, true, true> : fixup_kernel<float, true, false>, stage_bytes<float, true>());
    return with_smem(in_canon ? fixup_kernel<float, false, true> : fixup_kernel<float, false, false>, stage_bytes<float, false>());
}

template <int K>
static KernelPick pick_kernel(int dtype, bool uniform, bool in_canon) {
    if (dtype == FT_F64) {
        if (uniform) return with_smem(in_canon ? step_kernel<double, K, true, true> : step_kernel<double, K, true, false>, stage_bytes<double, true>());
        return with_smem(in_canon ? step_kernel<double, K, false, true> : step_kernel<double, K, false, false>, stage_bytes<double, false>());
    }
    if (uniform) return with_smem(in_canon ? step_kernel<float, K, true, true> : step_kernel<float, K, true, false>, stage_bytes<float, true>());
    return with_smem(in_canon ? step_kernel<float, K, false, true> : step_kernel<float, K, false, false>, stage_bytes<float, false>());
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

extern "C" int64_t ft_tile_slot_entries(void) { return FT_SLOT; }

extern "C" int64_t ft_tiled_min_capacity(int32_t n_vertices) {
    return (int64_t)ft::num_tiles_for(n_vertices < 0 ? 0 : n_vertices) * FT_SLOT;
}

static int check_tiled(const ft_tiled* t, int n_rows, int n_cols) {
    if (!t || !t->desc || !t->row_idx || !t->values) return set_err(FT_ERR_ARG, "null tiled buffer");
    if (t->n_rows != n_rows || t->n_cols != n_cols) return set_err(FT_ERR_SHAPE, "tiled buffer has wrong shape");
    if (t->capacity < ft_tiled_min_capacity(n_cols) || t->capacity > (int64_t)INT_MAX)
        return set_err(FT_ERR_ARG, "tiled capacity out of range");
    if (((uintptr_t)t->desc) & 7) return set_err(FT_ERR_ARG, "tiled desc must be 8-byte aligned");
    return FT_OK;
}

static int g_window = 0;
static int g_fixup_grid = 2 * 148;

static int window_size() {
    if (g_window == 0) {
        double h[33];
        h[0] = 0.0;
        for (int n = 1; n <= 32; ++n) h[n] = 1.0 / (double)n;
        cudaMemcpyToSymbol(ft::c_recip, h, sizeof(h));
        const char* s = getenv("FT_WINDOW");
        g_window = (s && atoi(s) == 8) ? 8 : 4;   // default: 4-row register window
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            g_fixup_grid = 2 * sms;
    }
    return g_window;
}

// which = 1: fused kernel, 2: fixup kernel, 3: both
static int launch_step(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* in_canon,
                       const ft_tiled* in_tiled, ft_tiled* out, int32_t dtype,
                       const ft_params* prm, void* workspace, size_t ws_bytes, int check_done,
                       cudaStream_t s, int which = 3) {
    if (!lap_t || !out || !prm || !workspace) return set_err(FT_ERR_ARG, "null argument");
    if (dtype != FT_F64 && dtype != FT_F32) return set_err(FT_ERR_ARG, "bad dtype");
    const int n_rows = in_canon ? in_canon->n_rows : (in_tiled ? in_tiled->n_rows : -1);
    const int n_v = in_canon ? in_canon->n_cols : (in_tiled ? in_tiled->n_cols : -1);
    if (n_v < 0) return set_err(FT_ERR_ARG, "no input");
    if (lap_t->n_rows != lap_t->n_cols) return set_err(FT_ERR_SHAPE, "Laplacian must be square");
    if (lap_t->n_cols != n_v) return set_err(FT_ERR_SHAPE, "Laplacian size does not match field");
    if (n_v == 0) return set_err(FT_ERR_SHAPE, "empty field");
    int rc = check_tiled(out, n_rows, n_v);
    if (rc != FT_OK) return rc;
    if (ws_bytes < ft::workspace_bytes(n_v)) return set_err(FT_ERR_ARG, "workspace too small");
    ft::StepParams p;
    p.n_v = n_v;
    p.num_tiles = ft::num_tiles_for(n_v);
    p.lap_ptr = lap_t->col_ptr;
    p.lap_idx = lap_t->row_idx;
    p.lap_val = lap_t->values;
    p.in_ptr = in_canon ? in_canon->col_ptr : nullptr;
    p.in_desc = in_canon ? nullptr : (const int2*)in_tiled->desc;
    p.in_idx = in_canon ? in_canon->row_idx : in_tiled->row_idx;
    p.in_val = in_canon ? in_canon->values : in_tiled->values;
    p.out_desc = (int2*)out->desc;
    p.out_idx = out->row_idx;
    p.out_val = out->values;
    p.cap = out->capacity;
    p.w = prm->w; p.a = prm->a; p.e = prm->e; p.eb = prm->e_base; p.mu = prm->mu; p.dt = prm->dt;
    p.ws = ft::carve_workspace(workspace, n_v);
    p.check_done = check_done;
    p.finite = std::isfinite(p.w) && std::isfinite(p.a) && std::isfinite(p.e) && std::isfinite(p.eb) &&
               std::isfinite(p.mu) && std::isfinite(p.dt);
    const bool uni = lap_flags == FT_LAP_UNIFORM;
    const ft::KernelPick k = window_size() == 8 ? ft::pick_kernel<8>(dtype, uni, in_canon != nullptr)
                                                : ft::pick_kernel<4>(dtype, uni, in_canon != nullptr);
    if (which & 1) k.fn<<<p.num_tiles, FT_TPB, k.smem, s>>>(p);
    const ft::KernelPick fx = ft::pick_fixup(dtype, uni, in_canon != nullptr);
    if (which & 2) fx.fn<<<g_fixup_grid, FT_TPB, fx.smem, s>>>(p);
    return cuda_check("step kernel");
}

static void launch_finalize(const ft::Workspace& ws, ft_step_stats* trace, long long tiled_cap,
                            int evolve, int max_steps, double tol, double thr, cudaStream_t s) {
    ft::FinalizeParams f;
    f.ws = ws; f.trace = trace; f.tiled_cap = tiled_cap; f.fixed_slot = evolve ? 0 : 1;
    f.evolve = evolve; f.max_steps = max_steps; f.tol = tol; f.base_threshold = thr;
    ft::finalize_kernel<<<FT_FIN_CTAS, FT_FIN_TPB, 0, s>>>(f);
}

static int launch_compact(ft::CompactParams& c, int dtype, cudaStream_t s) {
    const int nc = c.ws.num_chunks;
    ft::compact_count_kernel<<<nc, FT_CTPB, 0, s>>>(c);
    ft::compact_scan_kernel<<<1, 1024, 0, s>>>(c);
    if (dtype == FT_F64) ft::compact_copy_kernel<double><<<nc, FT_CTPB, 0, s>>>(c);
    else ft::compact_copy_kernel<float><<<nc, FT_CTPB, 0, s>>>(c);
    return cuda_check("compact");
}

extern "C" int ft_step_kernel(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* in_canon,
                              const ft_tiled* in_tiled, ft_tiled* out, int32_t dtype,
                              const ft_params* params, void* workspace, size_t ws_bytes,
                              void* stream) {
    return launch_step(lap_t, lap_flags, in_canon, in_tiled, out, dtype, params, workspace, ws_bytes,
                       0, (cudaStream_t)stream, 1);
}

extern "C" int ft_step_fixup(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* in_canon,
                             const ft_tiled* in_tiled, ft_tiled* out, int32_t dtype,
                             const ft_params* params, void* workspace, size_t ws_bytes,
                             void* stream) {
    return launch_step(lap_t, lap_flags, in_canon, in_tiled, out, dtype, params, workspace, ws_bytes,
                       0, (cudaStream_t)stream, 2);
}

extern "C" int ft_step_finalize(void* workspace, size_t ws_bytes, int32_t n_vertices,
                                int64_t tiled_capacity, ft_step_stats* stats, void* stream) {
    if (!workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (ws_bytes < ft::workspace_bytes(n_vertices)) return set_err(FT_ERR_ARG, "workspace too small");
    launch_finalize(ft::carve_workspace(workspace, n_vertices), stats, tiled_capacity, 0, 1, 0.0, 0.0,
                    (cudaStream_t)stream);
    return cuda_check("ft_step_finalize");
}

static void fill_compact(ft::CompactParams& c, const ft_tiled* a, const ft_tiled* b, int sel,
                         ft_csc* dst, void* workspace) {
    c.n_v = dst->n_cols;
    c.desc[0] = (const int2*)a->desc; c.idx[0] = a->row_idx; c.val[0] = a->values;
    const ft_tiled* bb = b ? b : a;
    c.desc[1] = (const int2*)bb->desc; c.idx[1] = bb->row_idx; c.val[1] = bb->values;
    c.sel = sel;
    c.out_ptr = dst->col_ptr; c.out_idx = dst->row_idx; c.out_val = dst->values; c.cap = dst->capacity;
    c.ws = ft::carve_workspace(workspace, dst->n_cols);
    c.stats = nullptr;
    c.control = nullptr;
    c.check_status = 0;
}

extern "C" int ft_compact(const ft_tiled* src, ft_csc* dst, int32_t dtype, void* workspace,
                          size_t ws_bytes, ft_step_stats* stats, void* stream) {
    if (!src || !dst || !workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (src->n_cols != dst->n_cols || src->n_rows != dst->n_rows) return set_err(FT_ERR_SHAPE, "shape mismatch");
    if (ws_bytes < ft::workspace_bytes(dst->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    if (dst->n_cols == 0) return set_err(FT_ERR_SHAPE, "empty field");
    ft::CompactParams c;
    fill_compact(c, src, nullptr, 0, dst, workspace);
    c.stats = stats;
    return launch_compact(c, dtype, (cudaStream_t)stream);
}

extern "C" int ft_step(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
                       ft_tiled* scratch, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                       void* workspace, size_t ws_bytes, ft_step_stats* stats, void* stream) {
    if (!phi_in || !phi_out || !stats || !scratch) return set_err(FT_ERR_ARG, "null argument");
    if (phi_out->n_cols != phi_in->n_cols || phi_out->n_rows != phi_in->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = launch_step(lap_t, lap_flags, phi_in, nullptr, scratch, dtype, params, workspace, ws_bytes, 0, s);
    if (rc != FT_OK) return rc;
    ft::Workspace ws = ft::carve_workspace(workspace, phi_in->n_cols);
    launch_finalize(ws, stats, scratch->capacity, 0, 1, 0.0, 0.0, s);
    // the compaction always runs; the host ignores it if the step failed
    ft::CompactParams c;
    fill_compact(c, scratch, nullptr, 0, phi_out, workspace);
    c.stats = stats;
    c.check_status = 1;
    return launch_compact(c, dtype, s);
}

extern "C" int ft_evolve(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in,
                         ft_tiled* work_a, ft_tiled* work_b, ft_csc* phi_out, int32_t dtype,
                         const ft_params* params, int32_t max_steps, double tol,
                         double base_threshold, void* workspace, size_t ws_bytes,
                         ft_step_stats* trace, int64_t* control, void* stream) {
    if (!phi_in || !phi_out || !work_a || !work_b || !trace || !control)
        return set_err(FT_ERR_ARG, "null argument");
    if (max_steps < 1) return set_err(FT_ERR_SHAPE, "max_steps must be >= 1");
    if (phi_out->n_cols != phi_in->n_cols || phi_out->n_rows != phi_in->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    int rc = check_tiled(work_b, phi_in->n_rows, phi_in->n_cols);
    if (rc != FT_OK) return rc;
    if (ws_bytes < ft::workspace_bytes(phi_in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    ft::Workspace ws = ft::carve_workspace(workspace, phi_in->n_cols);
    ft::evolve_reset_kernel<<<1, 1, 0, s>>>(ws.ctl);
    for (int i = 0; i < max_steps; ++i) {
        ft_tiled* out = (i & 1) ? work_b : work_a;
        const ft_tiled* in_t = (i & 1) ? work_a : work_b;
        rc = launch_step(lap_t, lap_flags, i == 0 ? phi_in : nullptr, i == 0 ? nullptr : in_t, out, dtype,
                         params, workspace, ws_bytes, 1, s);
        if (rc != FT_OK) return rc;
        launch_finalize(ws, trace, out->capacity, 1, max_steps, tol, base_threshold, s);
    }
    ft::evolve_report_kernel<<<1, 1, 0, s>>>(ws.ctl, (long long*)control);
    ft::CompactParams c;
    fill_compact(c, work_a, work_b, -1, phi_out, workspace);
    c.control = (long long*)control;
    return launch_compact(c, dtype, s);
}
