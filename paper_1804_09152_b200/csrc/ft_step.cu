// Fused explicit-Euler step of the layered field (sm_100a).
//
// One step replaces the reference pipeline of field.step
// (reference pkg/src/fieldtess/field.py:198-286):
//
//   Lt = PHI L^T            spgemm_numeric      _kernels.py:26-62
//   interest skeleton       skeleton_count/fill _kernels.py:96-150
//   PHI^, Lt^ expansion     expand_kernel       _kernels.py:153-176
//   Euler update + clamp    update_kernel       _kernels.py:179-238
//   normalise + compact     column_sums_counts, normalize_compact
//                                               _kernels.py:241-282
//
// Between steps PHI is kept in the hybrid layout of ft_tiled: a column
// with at most two entries (~99% at C3) lives in four dense per-column
// arrays (signature, second row, two values), a wider one in a pool.  Every
// kernel reads a neighbour's entries directly (no descriptor indirection)
// and writes its own column at a fixed address (no placement scan, no
// inter-CTA wait).  Work split:
//   tier 1    tier1_kernel (persistent, one warp per 32-column segment at a
//             time, the next segments' L rows prefetched): classification
//             from the neighbours' row signatures; a single-row
//             neighbourhood (a cell interior, ~82% of the columns at C3)
//             takes the exact closed form v' = v * (1 / (0 + v)); the others
//             are flagged in the segment's bit masks (no atomics);
//   tier 1.5  gen_kernel, one warp per three tiles: columns with at most two
//             rows and at most two entries per neighbour, the update in one
//             pass (rows = min / max of the candidates, Lt accumulated in
//             ascending-u order -- exactly the reference accumulator order;
//             PHI(r, j) arrives through the diagonal u == j); a union of
//             three or more rows goes to queue B;
//   queue A   tier 1's wide columns, on a high-priority side stream while
//             tier 1.5 runs: queue_kernel, wide3_kernel (3-row window),
//             wide_kernel (8-row window), deep_kernel (no limit);
//   queue B   warp_kernel after tier 1.5: two columns per warp, 16 lanes
//             holding a column's neighbourhood entries, sums by shuffles in
//             the reference's order.
// Within each stream's chain, a kernel that directly follows another kernel
// (no event record or wait in between: queue B and its tier 3 after tier 1.5;
// tier 2a, 2b and tier 3 on the side stream) is a programmatic dependent
// launch: it starts with pdl_wait(), so its launch overlaps the
// predecessor's tail; the predecessors never trigger early, so an event
// recorded after them still means "finished" (FT_PDL=0 turns this off).
// Statistics go to per-segment / per-group slots that finalize_kernel
// reduces in a fixed order (deterministic base mass).  Canonical CSC comes
// from ft_compact.
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
#include <cstring>
#include <utility>

#include "ft_common.cuh"

namespace ft {

// exact 1.0 / n for n = 0..32 (host IEEE division; entry 0 unused)
__constant__ double c_recip[33];

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start before its
// predecessor in the stream has finished; it waits here, before touching
// anything the predecessor writes.  A no-op for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

struct StepParams {
    int n_v;             // owned columns (the whole field outside domain mode)
    int j_base;          // global index of the first owned column
    int num_tiles;
    const int* __restrict__ lap_ptr;
    const int* __restrict__ lap_idx;
    const void* __restrict__ lap_val;
    const int4* __restrict__ lap_pack;  // FT_LAP_PACKED: int16 deltas u - j, 8 per column
    HybIn in;
    HybOut out;
    long long cap;       // pool entries the step may use
    double w, a, e, eb, mu, dt;
    Workspace ws;
    int check_done;
    int finite;          // all couplings finite: enables the single-row closed form
    int force_check;     // FT_LAP_CHECK_FINITE: check input values for NaN / Inf
    const int* report_ids;  // nullable: caller ids of the owned columns (error reports)
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

// One tier-2/3 pipeline: its input queue and the tier-2b / tier-3 lists it
// feeds.  Queue A holds tier 1's wide columns and runs on a side stream
// concurrently with tier 1.5; queue B holds the columns tier 1.5 defers.
// Entry i of a list is base[dir * i] (A grows up, B down: disjoint).
struct Queues {
    int* q;  int* q_n;
    int* w8; int* w8_n;
    int* dp; int* dp_n;
    int dir;
};

// ---------------------------------------------------------------------------
// register window of layer rows for one vertex column

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

// row signature of an output column: its row if it holds one entry, -1 if
// more, -2 if none (tier 1 classifies from the neighbours' signatures)
__device__ __forceinline__ int sig_of(int cnt, int row1) { return cnt == 1 ? row1 : (cnt == 0 ? -2 : -1); }

template <int K>
__device__ __forceinline__ int window_row1(const int* rows, unsigned int out_mask) {
    int r = 0;
#pragma unroll
    for (int i = 0; i < K; ++i)
        if (out_mask & (1u << i)) r = rows[i];
    return r;
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

// process_window<2> as straight-line code for a window of one or two rows
// (tier 1.5): the same operations in the same order, so the result is
// bitwise identical; no loops, masks or warp votes.  A single skeleton row
// takes the general arithmetic too: with finite inputs every term cancels
// exactly (the closed form of tier 1), so no divergent shortcut is needed.
__device__ __forceinline__ void process_two(Win<2>& w, const StepParams& p, VRes& res, unsigned int& out_mask) {
    const bool h1 = w.m > 1;
    const double ph0 = w.phi[0], lm0 = w.lam[0];
    const double ph1 = h1 ? w.phi[1] : 0.0, lm1 = h1 ? w.lam[1] : 0.0;
    const bool in0 = in_skeleton(ph0, lm0);
    const bool in1 = h1 && in_skeleton(ph1, lm1);
    res.bad_phi_row = -1;
    res.bad_lt_row = -1;
    if (ph0 != 0.0 && !in0) res.bad_phi_row = w.rows[0];
    if (lm0 != 0.0 && !in0) res.bad_lt_row = w.rows[0];
    if (h1 && ph1 != 0.0 && !in1) res.bad_phi_row = w.rows[1];
    if (h1 && lm1 != 0.0 && !in1) res.bad_lt_row = w.rows[1];
    const int n = (int)in0 + (int)in1;
    res.nskel = n;
    out_mask = 0;
    if (n == 0) return;
    // aggregates over the skeleton rows in row order (Appendix A)
    const double sq0 = in0 ? sqrt(ph0) : 0.0;
    const double sq1 = in1 ? sqrt(ph1) : 0.0;
    const double lh0 = (lm0 != 0.0) ? lm0 : 0.0;
    const double lh1 = (lm1 != 0.0) ? lm1 : 0.0;
    Agg g;
    agg_init(g);
    if (in0) { g.first_row = w.rows[0]; g.phi0 = ph0; g.n = 1; g.sl = g.sl + lh0; g.sp = g.sp + ph0; g.sr = g.sr + sq0; }
    if (in1) {
        if (!in0) { g.first_row = w.rows[1]; g.phi0 = ph1; }
        g.n += 1;
        g.sl = g.sl + lh1; g.sp = g.sp + ph1; g.sr = g.sr + sq1;
    }
    const Coef c = make_coef(g, p, c_recip);
    double v0 = 0.0, v1 = 0.0, s = 0.0;
    if (in0) { v0 = update_entry_sq(w.rows[0], ph0, lh0, sq0, c, p, res.nan); s = s + v0; }
    if (in1) { v1 = update_entry_sq(w.rows[1], ph1, lh1, sq1, c, p, res.nan); s = s + v1; }
    const bool spos = s > 0.0;
    const double inv = spos ? 1.0 / s : 0.0;
    if (in0) {
        const double nv = spos ? v0 * inv : v0;
        if (nv != 0.0) { res.cnt++; out_mask |= 1u; if (w.rows[0] == 0) res.bm = res.bm + nv; }
        const double dd = fabs(nv - ph0);
        if (dd > res.maxd) res.maxd = dd;
        w.lam[0] = nv;
    }
    if (in1) {
        const double nv = spos ? v1 * inv : v1;
        if (nv != 0.0) { res.cnt++; out_mask |= 2u; if (w.rows[1] == 0) res.bm = res.bm + nv; }
        const double dd = fabs(nv - ph1);
        if (dd > res.maxd) res.maxd = dd;
        w.lam[1] = nv;
    }
}

__device__ __forceinline__ void report_flags(const VRes& res, int j, const StepParams& p) {
    if (!res.nan && res.bad_phi_row < 0 && res.bad_lt_row < 0) return;
    if (p.report_ids) j = __ldg(&p.report_ids[j - p.j_base]);   // the caller's vertex id
    if (res.nan) atomicMax(&p.ws.ctl->nan_key, (unsigned int)(INT_MAX - j));
    if (res.bad_phi_row >= 0)
        atomicMax(&p.ws.ctl->bad_phi_key, ~(((unsigned long long)j << 32) | (unsigned int)res.bad_phi_row));
    if (res.bad_lt_row >= 0)
        atomicMax(&p.ws.ctl->bad_lt_key, ~(((unsigned long long)j << 32) | (unsigned int)res.bad_lt_row));
}

// ---------------------------------------------------------------------------
// output: a column with at most two entries goes to the dense arrays, a
// wider one to the pool (offset from pool_place)

template <typename T>
__device__ __forceinline__ void put_dense(const StepParams& p, int j, int cnt, int r0, double x0, int r1,
                                          double x1) {
    if (cnt == 0) {
        p.out.sig[j] = FT_SIG_EMPTY;
        return;
    }
    ((T*)p.out.v0)[j] = (T)x0;
    bool nf = !isfinite(x0);
    if (cnt == 1) {
        p.out.sig[j] = r0;
    } else {
        p.out.sig[j] = r0 | kPair;
        p.out.aux[j] = r1;
        ((T*)p.out.v1)[j] = (T)x1;
        nf |= !isfinite(x1);
    }
    if (nf) atomicOr(&p.ws.ctl->nonfinite, 1u);
}

// the flagged window slots (ascending rows) as column j
template <typename T, int K>
__device__ __forceinline__ void emit_window(const Win<K>& w, unsigned int out_mask, int j, long long poff,
                                            const StepParams& p) {
    const int cnt = __popc(out_mask);
    if (cnt <= 2) {
        int r0 = 0, r1 = 0, k = 0;
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (out_mask & (1u << i)) {
                if (k == 0) { r0 = w.rows[i]; x0 = w.lam[i]; }
                else { r1 = w.rows[i]; x1 = w.lam[i]; }
                ++k;
            }
        }
        put_dense<T>(p, j, cnt, r0, x0, r1, x1);
        return;
    }
    p.out.sig[j] = -cnt;
    p.out.aux[j] = (int)poff;
    T* ov = (T*)p.out.pval;
    bool nf = false;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (out_mask & (1u << i)) {
            p.out.pidx[poff] = w.rows[i];
            ov[poff] = (T)w.lam[i];
            nf |= !isfinite(w.lam[i]);
            ++poff;
        }
    }
    if (nf) atomicOr(&p.ws.ctl->nonfinite, 1u);
}

// Gather rows r > lo of the union of PHI(:, u), u in L^T(:, j), with the
// Lt accumulation, into the window (the K smallest such rows).  L from the
// CSR (tier 3, any degree).
template <typename T, int K, bool UNIFORM>
__device__ __forceinline__ void gather(Win<K>& w, int j, int lo, const StepParams& p) {
    w.m = 0;
    w.more = false;
    const int q0 = __ldg(&p.lap_ptr[j - p.j_base]);   // L rows are local to the domain
    const int q1 = __ldg(&p.lap_ptr[j - p.j_base + 1]);
    const double invdeg = UNIFORM ? 1.0 / (double)(q1 - q0 - 1) : 0.0;
    for (int q = q0; q < q1; ++q) {
        const int u = __ldg(&p.lap_idx[q]);
        const bool diag = (u == j);
        double l;
        if (UNIFORM) l = diag ? -1.0 : invdeg;
        else l = ldv<T>(p.lap_val, q);
        const int s = __ldg(&p.in.sig[u]);
        const int cnt = sig_count(s);
        const int a = cnt >= 2 ? __ldg(&p.in.aux[u]) : 0;
        for (int c = 0; c < cnt; ++c) {
            const int r = hyb_row<T>(p.in, s, a, c);
            if (r <= lo) continue;
            const double ph = hyb_val<T>(p.in, u, s, a, c);
            win_insert<K>(w, r, ph * l, diag, ph);
        }
    }
}

// entries of a tier-3 column, emitted in ascending row order
struct Sink {
    int k, cnt;
    int r0, r1;
    double x0, x1;
    long long off;
};

template <typename T>
__device__ __forceinline__ void sink_put(Sink& s, int r, double x, const StepParams& p) {
    if (s.cnt <= 2) {
        if (s.k == 0) { s.r0 = r; s.x0 = x; }
        else { s.r1 = r; s.x1 = x; }
    } else {
        p.out.pidx[s.off + s.k] = r;
        ((T*)p.out.pval)[s.off + s.k] = (T)x;
        if (!isfinite(x)) atomicOr(&p.ws.ctl->nonfinite, 1u);
    }
    ++s.k;
}

// --- slow path: union larger than K, processed in ascending row windows ----
// emit == false: statistics only (res.cnt = output entries); emit == true:
// writes column j (the pool range at poff when res.cnt > 2)

template <typename T, int K, bool UNIFORM>
__device__ __noinline__ void vertex_slow(int j, const StepParams& p, VRes& res, long long poff, bool emit) {
    Win<K> w;
    Agg g;
    agg_init(g);
    int lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        pass_aggregate<K>(w, g);
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    const int cnt_known = res.cnt;
    res.nskel = g.n;
    res.bad_phi_row = g.bad_phi_row;
    res.bad_lt_row = g.bad_lt_row;
    res.nan = false;
    res.cnt = 0; res.bm = 0.0; res.maxd = 0.0;
    Sink sk;
    sk.k = 0; sk.cnt = cnt_known; sk.r0 = 0; sk.r1 = 0; sk.x0 = 0.0; sk.x1 = 0.0; sk.off = poff;
    if (g.n == 0) {
        if (emit) p.out.sig[j] = FT_SIG_EMPTY;
        return;
    }
    const Coef c = make_coef(g, p, nullptr);
    double s = 0.0;
    lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
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
    lo = -1;
    do {
        gather<T, K, UNIFORM>(w, j, lo, p);
        for (int i = 0; i < w.m; ++i) {
            const double ph = w.phi[i], lm = w.lam[i];
            if (!in_skeleton(ph, lm)) continue;
            const double v = update_entry(w.rows[i], ph, (lm != 0.0) ? lm : 0.0, c, p, dummy);
            const double nv = spos ? v * inv : v;
            if (nv != 0.0) {
                if (emit) sink_put<T>(sk, w.rows[i], nv, p);
                res.cnt++;
                if (w.rows[i] == 0) res.bm = res.bm + nv;
            }
            const double dd = fabs(nv - ph);
            if (dd > res.maxd) res.maxd = dd;
        }
        if (w.m > 0) lo = w.rows[w.m - 1];
    } while (w.more);
    if (emit) {
        if (res.cnt <= 2) put_dense<T>(p, j, res.cnt, sk.r0, sk.x0, sk.r1, sk.x1);
        else { p.out.sig[j] = -res.cnt; p.out.aux[j] = (int)poff; }
    }
}

// ---------------------------------------------------------------------------
// the L^T column of a vertex

constexpr int kMD = 8;
constexpr int kPackEmpty = -32768;

// The L^T column of j: u[0..n) in stored order.  PACKED reads one 16-byte
// row of int16 deltas (u - j; empty slots kPackEmpty; all-empty = not
// packable, read from the CSR); otherwise the CSR.  Returns n, or 0 when
// the column has no entry or more than kMD (-> wide).
template <bool PACKED>
__device__ __forceinline__ int load_lrow(const StepParams& p, int jl, int j, bool active, int (&u)[kMD],
                                         int& q0) {
    int n = 0;
    q0 = 0;
    bool csr = !PACKED;
    if (PACKED) {
        int4 pk = make_int4(0, 0, 0, 0);
        if (active) pk = __ldg(&p.lap_pack[jl]);
        const int w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            const int s = (k & 1) ? (w4[k >> 1] >> 16) : ((int)(w4[k >> 1] << 16) >> 16);
            const bool valid = active && s != kPackEmpty;
            u[k] = valid ? j + s : -1;
            n += valid ? 1 : 0;
        }
        csr = active && n == 0;
    }
    if (csr && active) {
        q0 = __ldg(&p.lap_ptr[jl]);
        n = __ldg(&p.lap_ptr[jl + 1]) - q0;
        if (n > kMD || n < 1) n = 0;
#pragma unroll
        for (int k = 0; k < kMD; ++k) u[k] = (k < n) ? __ldg(&p.lap_idx[q0 + k]) : -1;
    } else if (!PACKED) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) u[k] = -1;
    }
    return n;
}

// load_lrow with the packed row already loaded (PACKED), else the CSR
template <bool PACKED>
__device__ __forceinline__ int unpack_lrow(const StepParams& p, int4 pk, int jl, int j, bool active, int (&u)[kMD],
                                           int& q0) {
    int n = 0;
    q0 = 0;
    bool csr = !PACKED;
    if (PACKED) {
        const int w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            const int s = (k & 1) ? (w4[k >> 1] >> 16) : ((int)(w4[k >> 1] << 16) >> 16);
            const bool valid = active && s != kPackEmpty;
            u[k] = valid ? j + s : -1;
            n += valid ? 1 : 0;
        }
        csr = active && n == 0;
    }
    if (csr && active) {
        q0 = __ldg(&p.lap_ptr[jl]);
        n = __ldg(&p.lap_ptr[jl + 1]) - q0;
        if (n > kMD || n < 1) n = 0;
#pragma unroll
        for (int k = 0; k < kMD; ++k) u[k] = (k < n) ? __ldg(&p.lap_idx[q0 + k]) : -1;
    } else if (!PACKED) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) u[k] = -1;
    }
    return n;
}

template <typename T, bool UNIFORM>
__device__ __forceinline__ double lap_value(const StepParams& p, int k, int kd, int q0, double invdeg) {
    return UNIFORM ? ((k == kd) ? -1.0 : invdeg) : ldv<T>(p.lap_val, q0 + k);
}

__device__ __forceinline__ double recip_deg(int n) { return n - 1 <= 32 ? c_recip[n - 1] : 1.0 / (double)(n - 1); }

// ---------------------------------------------------------------------------
// tier 1: classification and the closed form.
//
// A column whose neighbourhood is one layer row (every non-empty neighbour
// holds one entry, of the column's own row; its phi > 0) is finished here
// with the exact single-row closed form.  The others are flagged in their
// segment's masks: at most two entries per neighbour -> tier 1.5, more (or
// no packable L row) -> tier 2.  The neighbours' VALUES are not read: the
// closed form needs them only through the finiteness of Lt, and values this
// library wrote are finite unless a kernel raised the sticky nonfinite flag
// (ft_tiled_from_csc raises it for non-finite input; FT_LAP_CHECK_FINITE and
// a raised flag switch the check on).  One warp = one 32-column segment:
// statistics and masks go to the segment's slots, no CTA barrier.

// one 32-column segment (one warp), the packed L row and the column's value
// already loaded (prefetched by the caller)
template <typename T, bool UNIFORM, bool PACKED>
__device__ __forceinline__ void tier1_segment(const StepParams& p, int seg, int lane, bool chk, int4 pk,
                                              double phs) {
    const int jl = seg * 32 + lane;
    const int j = p.j_base + jl;
    const bool active = jl < p.n_v;

    int q0 = 0;
    int u[kMD];
    const int n = unpack_lrow<PACKED>(p, pk, jl, j, active, u, q0);
    bool wide = active && n == 0;
    int kd = -1;
#pragma unroll
    for (int k = 0; k < kMD; ++k)
        if (u[k] == j) kd = k;
    if (active && kd < 0) wide = true;
    int sg[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) sg[k] = (k < n) ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
    int rs = FT_SIG_EMPTY;
#pragma unroll
    for (int k = 0; k < kMD; ++k)
        if (k == kd) rs = sg[k];
    bool same = true, big = false;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        same &= (sg[k] == FT_SIG_EMPTY) || (sg[k] == rs);
        big |= sg[k] <= -3;
    }
    bool cand = active && !wide && p.finite && rs >= 0 && rs < kPair && same && phs > 0.0;
    if (chk && cand) {
        // Lt(rs, j) must be finite for the closed form: read the values
        bool fin = true;
        double lam = 0.0;
        const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            if (k < n && sg[k] == rs) {
                const double v = ldv<T>(p.in.v0, u[k]);
                fin &= isfinite(v);
                lam = lam + v * lap_value<T, UNIFORM>(p, k, kd, q0, invdeg);
            }
        }
        cand = fin && isfinite(lam);
    }
    const bool fast = cand;
    const bool slow = active && !fast && (wide || big);
    const bool gen = active && !fast && !slow;

    double bm = 0.0, md = 0.0;
    int cnt = 0;
    // a cell interior at rest holds exactly 1.0, and 1.0 * (1 / (0 + 1.0))
    // == 1.0: a warp whose fast lanes all hold 1.0 skips the division
    const bool ones = __all_sync(0xffffffffu, !fast || phs == 1.0);
    if (fast) {
        double v = phs;
        if (v > 1.0) v = 1.0;
        const double s = 0.0 + v;
        const double nv = ones ? 1.0 : v * (1.0 / s);
        if (nv != 0.0) {
            cnt = 1;
            if (rs == 0) bm = nv;
        }
        md = fabs(nv - phs);
        p.out.sig[j] = cnt ? rs : FT_SIG_EMPTY;
        ((T*)p.out.v0)[j] = (T)nv;
        if (!isfinite(nv)) atomicOr(&p.ws.ctl->nonfinite, 1u);
    }
    const unsigned int fb = __ballot_sync(0xffffffffu, fast);
    const unsigned int gb = __ballot_sync(0xffffffffu, gen);
    const unsigned int wb = __ballot_sync(0xffffffffu, slow);
    cnt = __popc(__ballot_sync(0xffffffffu, cnt != 0));
    // cell interiors at rest give bm = md = 0: skip the shuffle trees then
    if (__any_sync(0xffffffffu, bm != 0.0)) bm = warp_sum(bm);      // fixed tree: deterministic
    if (__any_sync(0xffffffffu, md != 0.0)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_down_sync(0xffffffffu, md, o));
    }
    if (lane == 0) {
        p.ws.seg_bm[seg] = bm;
        p.ws.seg_maxd[seg] = md;
        p.ws.seg_cs[seg] = make_int2(cnt, __popc(fb));
        p.ws.gen_mask[seg] = gb;
        p.ws.slow_mask[seg] = wb;
    }
}

// persistent: each warp walks segments seg, seg + (warps in the grid), ...,
// loading the next segment's packed L row and value while it classifies
// the current one (two segments of loads in flight per warp)
template <typename T, bool UNIFORM, bool PACKED>
__global__ void __launch_bounds__(FT_TPB, 8) tier1_kernel(const StepParams p) {
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    const bool chk = p.force_check || *(volatile unsigned int*)&p.ws.ctl->nonfinite;
    const int lane = threadIdx.x & 31;
    const int nseg = FT_WARPS * p.num_tiles;
    const int nw = gridDim.x * FT_WARPS;
    int seg = (blockIdx.x * FT_TPB + threadIdx.x) >> 5;
    // two segments of loads in flight ahead of the one being classified
    int4 pk = make_int4(0, 0, 0, 0), pk1 = make_int4(0, 0, 0, 0);
    double phs = 0.0, ph1 = 0.0;
    {
        const int jl = seg * 32 + lane, jl1 = (seg + nw) * 32 + lane;
        if (seg < nseg && jl < p.n_v) {
            if (PACKED) pk = __ldg(&p.lap_pack[jl]);
            phs = ldv<T>(p.in.v0, p.j_base + jl);
        }
        if (seg + nw < nseg && jl1 < p.n_v) {
            if (PACKED) pk1 = __ldg(&p.lap_pack[jl1]);
            ph1 = ldv<T>(p.in.v0, p.j_base + jl1);
        }
    }
    for (; seg < nseg; seg += nw) {
        int4 pk2 = make_int4(0, 0, 0, 0);
        double ph2 = 0.0;
        const int jl2 = (seg + 2 * nw) * 32 + lane;
        if (seg + 2 * nw < nseg && jl2 < p.n_v) {
            if (PACKED) pk2 = __ldg(&p.lap_pack[jl2]);
            ph2 = ldv<T>(p.in.v0, p.j_base + jl2);
        }
        tier1_segment<T, UNIFORM, PACKED>(p, seg, lane, chk, pk, phs);
        pk = pk1; phs = ph1;
        pk1 = pk2; ph1 = ph2;
    }
}

// the r-th (0-based) set bit of m
__device__ __forceinline__ int nth_bit(unsigned int m, int r) {
    int pos = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const int c = __popc(m & ((1u << s) - 1u));
        if (r >= c) { r -= c; m >>= s; pos += s; }
    }
    return pos;
}

// warp-aggregated pool allocation (need entries per lane) + the global
// statistics of tiers 2/3 (few columns: one atomic per warp)
__device__ __forceinline__ long long pool_place(int need, const VRes& res, const StepParams& p, int lane,
                                                bool& fits) {
    int incl = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    long long base = 0;
    if (lane == 31 && wtot > 0) base = (long long)atomicAdd(&p.ws.ctl->pool_next, (unsigned long long)wtot);
    base = __shfl_sync(0xffffffffu, base, 31);
    fits = base + wtot <= p.cap;
    if (lane == 31 && !fits) atomicExch(&p.ws.ctl->overflow, 1);
    const int skel = warp_sum(res.nskel);
    const int nnz = warp_sum(res.cnt);
    double mx = res.maxd;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 0) {
        if (mx > 0.0) atomicMax(&p.ws.ctl->maxdelta_bits, (unsigned long long)__double_as_longlong(mx));
        if (skel) atomicAdd(&p.ws.ctl->skel_total, (unsigned long long)skel);
        if (nnz) atomicAdd(&p.ws.ctl->nnz_total, (unsigned long long)nnz);
    }
    return base + incl - need;
}

// ---------------------------------------------------------------------------
// lane-cooperative column (queue B: the tier-1.5 deferrals).  Sixteen
// lanes per column: lane e holds entry e of the neighbourhood (neighbours in L order, rows ascending within one), lanes
// with equal rows are grouped with __match_any_sync, and every sum is taken
// in the reference's order -- Lt(r, j) over the entries in L order
// (_kernels.py:36-50), the skeleton aggregates and the normaliser in
// ascending row order (_kernels.py:179-282) -- by shuffles, so the result is
// bitwise that of process_window / vertex_slow.  Neighbourhoods of more
// than 16 entries (or 16 L entries) go to the queue's tier-3 list.

struct WarpStats {
    double maxd;
    long long cnt, skel;
};

// Two columns per warp: lanes 0-15 and 16-31 each hold one column's
// neighbourhood (queue B: at most two entries per neighbour and at most 8
// neighbours, so at most 16 entries).  Every loop has a warp-uniform trip
// count, so the full-mask shuffles never diverge between the halves.
template <typename T, bool UNIFORM, bool PACKED>
__device__ __forceinline__ void half_column(int j, bool have, const StepParams& p, const Queues& qs, int lane,
                                            WarpStats& ws) {
    constexpr int W = 16;
    const unsigned int full = 0xffffffffu;
    const int sl = lane & (W - 1);               // lane within the half
    const int gb = lane & W;                     // 0 or 16
    auto half_bits = [&](unsigned int b) { return (b >> gb) & 0xffffu; };
    const int jl = j - p.j_base;
    int q0 = 0, n = 0, pu = -1;
    if (PACKED) {
        int4 pk = make_int4(0, 0, 0, 0);
        if (have) pk = __ldg(&p.lap_pack[jl]);
        const int w = (sl >> 1) == 0 ? pk.x : ((sl >> 1) == 1 ? pk.y : ((sl >> 1) == 2 ? pk.z : pk.w));
        const int d = (sl & 1) ? (w >> 16) : ((int)(w << 16) >> 16);
        const bool valid = have && sl < kMD && d != kPackEmpty;
        pu = valid ? j + d : -1;
        n = __popc(half_bits(__ballot_sync(full, valid)));   // valid slots lead
    }
    if (have && n == 0) {
        q0 = __ldg(&p.lap_ptr[jl]);
        n = __ldg(&p.lap_ptr[jl + 1]) - q0;
        pu = -1;
    }
    int u = -1, sgk = FT_SIG_EMPTY, axk = 0, ck = 0;
    double lk = 0.0;
    const bool lv = have && sl < n && n <= W;
    if (lv) {
        u = pu >= 0 ? pu : __ldg(&p.lap_idx[q0 + sl]);
        sgk = __ldg(&p.in.sig[u]);
        ck = sig_count(sgk);
        axk = ck >= 2 ? __ldg(&p.in.aux[u]) : 0;
    }
    const unsigned int dmask = half_bits(__ballot_sync(full, lv && u == j));
    const int kd = dmask ? __ffs(dmask) - 1 : -1;
    if (lv) {
        if (UNIFORM) lk = (sl == kd) ? -1.0 : 1.0 / (double)(n - 1);
        else lk = ldv<T>(p.lap_val, q0 + sl);
    }
    int incl = ck;                               // entry offsets within the half
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
        const int y = __shfl_up_sync(full, incl, o, W);
        if (sl >= o) incl += y;
    }
    const int E = __shfl_sync(full, incl, W - 1, W);
    const bool fb = have && (n > W || n < 1 || kd < 0 || E > W);   // to the tier-3 list
    if (fb && sl == 0) {
        const int q = atomicAdd(qs.dp_n, 1);
        qs.dp[qs.dir * q] = j;
    }
    const bool act = have && !fb;
    const int e0k = incl - ck;
    int myk = 0, t = 0;
    for (int k = 0; k < W; ++k) {
        const int a = __shfl_sync(full, e0k, k, W), c = __shfl_sync(full, ck, k, W);
        if (sl >= a && sl < a + c) { myk = k; t = sl - a; }
    }
    const int su = __shfl_sync(full, u, myk, W), ss = __shfl_sync(full, sgk, myk, W);
    const int sa = __shfl_sync(full, axk, myk, W);
    const double slk = __shfl_sync(full, lk, myk, W);
    const bool valid = act && sl < E;
    int r = -1 - lane;                           // unique key for lanes without an entry
    double v = 0.0;
    if (valid) {
        r = hyb_row<T>(p.in, ss, sa, t);
        v = hyb_val<T>(p.in, su, ss, sa, t);
    }
    const double prod = v * slk;                 // PHI(r, u) * L(j, u)
    const bool dg = valid && myk == kd;
    // group equal rows within the half: key = row and half
    const unsigned int grpw = __match_any_sync(full, valid ? ((r << 1) | (gb >> 4)) : r);
    const unsigned int grp = half_bits(grpw);
    const bool leader = valid && (__ffs(grp) - 1) == sl;
    const int gsz = __popc(grp);
    const int gmax = __reduce_max_sync(full, (unsigned int)gsz);
    double lam = 0.0;
    unsigned int rest = grp;
    for (int it = 0; it < gmax; ++it) {          // Lt(r, j) in L order
        const int src = rest ? __ffs(rest) - 1 : sl;
        rest = rest ? (rest & (rest - 1)) : 0u;
        const double pv = __shfl_sync(full, prod, src, W);
        if (it < gsz) lam = lam + pv;
    }
    const unsigned int dgm = grp & half_bits(__ballot_sync(full, dg));
    const double vd = __shfl_sync(full, v, dgm ? __ffs(dgm) - 1 : sl, W);
    const double ph = dgm ? vd : 0.0;
    int rank = 0;
    for (int s2 = 0; s2 < W; ++s2) {
        const int rr = __shfl_sync(full, r, s2, W);
        const bool ls = __shfl_sync(full, leader, s2, W);
        rank += (ls && rr < r) ? 1 : 0;
    }
    const int m = __popc(half_bits(__ballot_sync(full, leader)));
    const int mmax = __reduce_max_sync(full, (unsigned int)m);
    const bool in = leader && in_skeleton(ph, lam);
    int bad_phi = (leader && ph != 0.0 && !in) ? r : -1;
    int bad_lt = (leader && lam != 0.0 && !in) ? r : -1;
    const double lh = (lam != 0.0) ? lam : 0.0;
    const double sq = in ? sqrt(ph) : 0.0;
    Agg g;                                       // ascending row order
    agg_init(g);
    for (int q = 0; q < mmax; ++q) {
        const unsigned int hb = half_bits(__ballot_sync(full, leader && rank == q));
        const int lq = hb ? __ffs(hb) - 1 : 0;
        const bool iq = __shfl_sync(full, in, lq, W);
        const double phq = __shfl_sync(full, ph, lq, W), lhq = __shfl_sync(full, lh, lq, W);
        const double sqq = __shfl_sync(full, sq, lq, W);
        const int rq = __shfl_sync(full, r, lq, W);
        if (hb && iq) {
            if (g.n == 0) { g.first_row = rq; g.phi0 = phq; }
            g.n++;
            g.sl = g.sl + lhq;
            g.sp = g.sp + phq;
            g.sr = g.sr + sqq;
        }
    }
    bool nan = false;
    double vn = 0.0, s = 0.0;
    Coef c;
    if (g.n > 0) c = make_coef(g, p, c_recip);
    if (g.n > 0 && in) vn = update_entry_sq(r, ph, lh, sq, c, p, nan);
    for (int q = 0; q < mmax; ++q) {
        const unsigned int hb = half_bits(__ballot_sync(full, leader && rank == q));
        const int lq = hb ? __ffs(hb) - 1 : 0;
        const bool iq = __shfl_sync(full, in, lq, W);
        const double vq = __shfl_sync(full, vn, lq, W);
        if (g.n > 0 && hb && iq) s = s + vq;
    }
    const bool spos = s > 0.0;
    const double inv = spos ? 1.0 / s : 0.0;
    const double nv = spos ? vn * inv : vn;
    const bool out = in && nv != 0.0;
    const int cnt = __popc(half_bits(__ballot_sync(full, out)));
    int pos = 0;                                 // rank among the output rows
    for (int s2 = 0; s2 < W; ++s2) {
        const bool os = __shfl_sync(full, out, s2, W);
        const int rk = __shfl_sync(full, rank, s2, W);
        pos += (os && rk < rank) ? 1 : 0;
    }
    double bm = (out && r == 0) ? nv : 0.0;
    double dd = in ? fabs(nv - ph) : 0.0;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
        bm = bm + __shfl_xor_sync(full, bm, o, W);   // at most one nonzero term: exact
        dd = fmax(dd, __shfl_xor_sync(full, dd, o, W));
        bad_phi = max(bad_phi, __shfl_xor_sync(full, bad_phi, o, W));
        bad_lt = max(bad_lt, __shfl_xor_sync(full, bad_lt, o, W));
    }
    const bool anynan = half_bits(__ballot_sync(full, nan)) != 0;
    const int nskel = __popc(half_bits(__ballot_sync(full, in)));
    if (act && sl == 0) {
        VRes res;
        vres_init(res);
        res.nan = anynan; res.bad_phi_row = bad_phi; res.bad_lt_row = bad_lt;
        report_flags(res, j, p);
        p.ws.vbm[jl] = bm;
        ws.maxd = fmax(ws.maxd, dd);
        ws.cnt += cnt;
        ws.skel += nskel;
    }
    // output: dense for at most two rows, else a pool range
    long long off = 0;
    if (act && cnt > 2 && sl == 0) off = (long long)atomicAdd(&p.ws.ctl->pool_next, (unsigned long long)cnt);
    off = __shfl_sync(full, off, 0, W);
    if (!act) return;
    if (cnt <= 2) {
        if (cnt == 0) {
            if (sl == 0) p.out.sig[j] = FT_SIG_EMPTY;
        } else if (out) {
            if (pos == 0) {
                p.out.sig[j] = cnt == 2 ? (r | kPair) : r;
                ((T*)p.out.v0)[j] = (T)nv;
            } else {
                p.out.aux[j] = r;
                ((T*)p.out.v1)[j] = (T)nv;
            }
            if (!isfinite(nv)) atomicOr(&p.ws.ctl->nonfinite, 1u);
        }
        return;
    }
    if (off + cnt > p.cap) {
        if (sl == 0) atomicExch(&p.ws.ctl->overflow, 1);
        return;
    }
    if (sl == 0) { p.out.sig[j] = -cnt; p.out.aux[j] = (int)off; }
    if (out) {
        p.out.pidx[off + pos] = r;
        ((T*)p.out.pval)[off + pos] = (T)nv;
        if (!isfinite(nv)) atomicOr(&p.ws.ctl->nonfinite, 1u);
    }
}

// ---------------------------------------------------------------------------
// tier 1.5: the flagged columns with at most two entries per neighbour, one
// warp per group of FT_GEN_TILES tiles (~63 columns at C3: two nearly full
// chunks) with the columns on its lanes: the one-pass two-row update.  More
// than two rows -> queue B (and the tile's slow mask).  Statistics into the
// group's slots, base mass in lane order (fixed): no hot atomics.

template <typename T, bool UNIFORM, bool PACKED>
__global__ void __launch_bounds__(FT_TPB, 8) gen_kernel(const StepParams p) {
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    __shared__ int s_list[FT_WARPS][FT_GEN_TILES * FT_TPB];
    const int lane = threadIdx.x & 31;
    int* list = s_list[threadIdx.x >> 5];
    const int nwarps = gridDim.x * FT_WARPS;
    const int ngroups = (p.num_tiles + FT_GEN_TILES - 1) / FT_GEN_TILES;
    for (int t = (blockIdx.x * FT_TPB + threadIdx.x) >> 5; t < ngroups; t += nwarps) {
        // the flagged columns of the group's tiles, in vertex order
        int ng = 0;
#pragma unroll
        for (int tt = 0; tt < FT_GEN_TILES; ++tt) {
            const int tile = t * FT_GEN_TILES + tt;
            if (tile >= p.num_tiles) break;
            const uint4 g4 = *reinterpret_cast<const uint4*>(&p.ws.gen_mask[(size_t)FT_WARPS * tile]);
            const unsigned int gm[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if ((gm[q] >> lane) & 1u)
                    list[ng + __popc(gm[q] & ((1u << lane) - 1u))] = tile * FT_TPB + q * 32 + lane;
                ng += __popc(gm[q]);
            }
        }
        if (ng == 0) continue;
        __syncwarp();
        double tbm = 0.0, tmx = 0.0;
        int tcnt = 0, tskel = 0;
        for (int c0 = 0; c0 < ng; c0 += 32) {
            const bool mine = c0 + lane < ng;
            const int jl = mine ? list[c0 + lane] : 0;
            const int j = p.j_base + jl;
            int q0 = 0;
            int u[kMD];
            const int n = load_lrow<PACKED>(p, jl, j, mine, u, q0);
            int sg[kMD], ax[kMD];
#pragma unroll
            for (int k = 0; k < kMD; ++k) {
                const bool h = k < n;
                sg[k] = h ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
                ax[k] = h ? __ldg(&p.in.aux[u[k]]) : 0;
            }
            const double vj0 = mine ? ldv<T>(p.in.v0, j) : 0.0;
            const double vj1 = mine ? ldv<T>(p.in.v1, j) : 0.0;
            int kd = -1;
            bool big = false;
            int rlo = INT_MAX, rhi = -1;
#pragma unroll
            for (int k = 0; k < kMD; ++k) {
                kd = (u[k] == j) ? k : kd;
                big |= sg[k] <= -3;
                const bool h = sg[k] >= 0, pr = h && (sg[k] & kPair);
                const int x0 = h ? (sg[k] & ~kPair) : INT_MAX;
                rlo = min(rlo, x0);
                rhi = max(rhi, h ? x0 : -1);
                rlo = min(rlo, pr ? ax[k] : INT_MAX);
                rhi = max(rhi, pr ? ax[k] : -1);
            }
            // PHI(r, j) from the column's own entries (sg[kd], aux[kd])
            int sgj = FT_SIG_EMPTY, axj = 0;
#pragma unroll
            for (int k = 0; k < kMD; ++k) {
                sgj = (k == kd) ? sg[k] : sgj;
                axj = (k == kd) ? ax[k] : axj;
            }
            const bool hj = sgj >= 0, prj = hj && (sgj & kPair);
            const int xj = sgj & ~kPair;
            const double p0 = (hj && xj == rlo) ? vj0 : 0.0;
            const double p1 = (hj && xj == rhi) ? vj0 : ((prj && axj == rhi) ? vj1 : 0.0);
            // Lt(rlo, j), Lt(rhi, j) in L order; an entry of a neighbour
            // holding rows x0 < x1 goes to its row's sum (x1 == rlo and
            // x0 == rhi are impossible: rlo / rhi are the min / max)
            const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
            double l0 = 0.0, l1 = 0.0;
            bool more = false;
#pragma unroll
            for (int k = 0; k < kMD; ++k) {
                const bool h = sg[k] >= 0, pr = h && (sg[k] & kPair);
                const double l = (k < n) ? lap_value<T, UNIFORM>(p, k, kd, q0, invdeg) : 0.0;
                const int x0 = sg[k] & ~kPair;
                const double a0 = h ? ldv<T>(p.in.v0, u[k]) : 0.0;
                const double a1 = pr ? ldv<T>(p.in.v1, u[k]) : 0.0;
                const bool m0 = h && x0 == rlo;
                const bool m1a = h && x0 != rlo && x0 == rhi, m1b = pr && ax[k] == rhi;
                more |= (h && x0 != rlo && x0 != rhi) || (pr && ax[k] != rhi);
                l0 = m0 ? l0 + a0 * l : l0;
                const double c1 = m1a ? a0 : a1;
                l1 = (m1a || m1b) ? l1 + c1 * l : l1;
            }
            const bool defer = mine && (more || big || rlo == INT_MAX || kd < 0 || n == 0);
            Win<2> w;
            w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
            w.rows[1] = rhi; w.lam[1] = l1; w.phi[1] = p1;
            w.m = (rhi == rlo) ? 1 : 2;
            if (w.m == 1) { w.rows[1] = INT_MAX; w.lam[1] = 0.0; w.phi[1] = 0.0; }
            VRes res;
            vres_init(res);
            unsigned int out_mask = 0;
            const bool run = mine && !defer;
            if (run) {
                process_two(w, p, res, out_mask);
                report_flags(res, j, p);
                emit_window<T, 2>(w, out_mask, j, 0, p);
            }
            // three or more rows (rare): queue B, one atomic per chunk
            const unsigned int db = __ballot_sync(0xffffffffu, defer);
            if (db) {
                if (defer) atomicOr(&p.ws.slow_mask[jl >> 5], 1u << (jl & 31));
                int qb = 0;
                if (lane == 0) qb = atomicAdd(&p.ws.ctl->gen_count, __popc(db));
                qb = __shfl_sync(0xffffffffu, qb, 0);
                if (defer) p.ws.slow_list[(p.n_v - 1) - (qb + __popc(db & ((1u << lane) - 1u)))] = j;
            }
            // per-lane partials (lane l: list entries l, l + 32, ...), then
            // one fixed shuffle tree: the base mass is deterministic
            if (run) tbm = tbm + res.bm;
            tmx = fmax(tmx, res.maxd);
            tcnt += run ? res.cnt : 0;
            tskel += run ? res.nskel : 0;
        }
        tbm = warp_sum(tbm);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tmx = fmax(tmx, __shfl_down_sync(0xffffffffu, tmx, o));
        tcnt = warp_sum(tcnt);
        tskel = warp_sum(tskel);
        if (lane == 0 && ng > 0) {
            p.ws.gen_bm[t] = tbm;
            p.ws.gen_maxd[t] = tmx;
            p.ws.gen_cs[t] = make_int2(tcnt, tskel);
        }
        __syncwarp();
    }
}

// tier-1 wide columns (segment slow masks) -> queue A, one thread per
// segment, one atomic per warp
__global__ void __launch_bounds__(256) queue_kernel(const StepParams p) {
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    const int seg = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const unsigned int m = seg < FT_WARPS * p.num_tiles ? p.ws.slow_mask[seg] : 0u;
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (tot == 0) return;
    int qb = 0;
    if (lane == 31) qb = atomicAdd(&p.ws.ctl->slow_count, tot);
    qb = __shfl_sync(0xffffffffu, qb, 31) + incl - c;
    unsigned int mm = m;
    while (mm) {
        const int b = __ffs(mm) - 1;
        mm &= mm - 1;
        p.ws.slow_list[qb++] = p.j_base + seg * 32 + b;
    }
}

// ---------------------------------------------------------------------------
// tier 2a: the queued columns with at most three rows and at most three
// entries per neighbour: rows = min, max and the one other candidate; the
// three Lt sums in one (u, t) pass.  Others go on to tier 2b through
// slow_list + 2 n_v.

template <typename T, bool UNIFORM, bool PACKED>
__device__ __forceinline__ bool wide3(int j, const StepParams& p, Win<3>& w) {
    int q0 = 0;
    int u[kMD];
    const int n = load_lrow<PACKED>(p, j - p.j_base, j, true, u, q0);
    if (n == 0) return false;
    int sg[kMD], ax[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        sg[k] = (k < n) ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
        ax[k] = (k < n) ? __ldg(&p.in.aux[u[k]]) : 0;
    }
    int kd = -1;
    bool big = false;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        if (u[k] == j) kd = k;
        big |= sig_count(sg[k]) > 3;
    }
    if (kd < 0 || big) return false;
    int rr[kMD][3];
#pragma unroll
    for (int k = 0; k < kMD; ++k)
#pragma unroll
        for (int t = 0; t < 3; ++t) rr[k][t] = (t < sig_count(sg[k])) ? hyb_row<T>(p.in, sg[k], ax[k], t) : INT_MAX;
    int rlo = INT_MAX, rhi = -1;
#pragma unroll
    for (int k = 0; k < kMD; ++k)
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (rr[k][t] != INT_MAX) { rlo = min(rlo, rr[k][t]); rhi = max(rhi, rr[k][t]); }
    if (rlo == INT_MAX) return false;
    const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
    double l0 = 0.0, l1 = 0.0, l2 = 0.0, p0 = 0.0, p1 = 0.0, p2 = 0.0;
    int rmid = INT_MAX;
    bool more = false;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        const double l = (k < n) ? lap_value<T, UNIFORM>(p, k, kd, q0, invdeg) : 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int r = rr[k][t];
            if (r == INT_MAX) continue;
            const double a = hyb_val<T>(p.in, u[k], sg[k], ax[k], t);
            if (r == rlo) { l0 = l0 + a * l; if (k == kd) p0 = a; }
            else if (r == rhi) { l2 = l2 + a * l; if (k == kd) p2 = a; }
            else {
                if (rmid == INT_MAX) rmid = r;
                if (r == rmid) { l1 = l1 + a * l; if (k == kd) p1 = a; }
                else more = true;
            }
        }
    }
    if (more) return false;
    if (rlo == rhi) {
        w.m = 1;
        w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
    } else if (rmid == INT_MAX) {
        w.m = 2;
        w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
        w.rows[1] = rhi; w.lam[1] = l2; w.phi[1] = p2;
    } else {
        w.m = 3;
        w.rows[0] = rlo; w.lam[0] = l0; w.phi[0] = p0;
        w.rows[1] = rmid; w.lam[1] = l1; w.phi[1] = p1;
        w.rows[2] = rhi; w.lam[2] = l2; w.phi[2] = p2;
    }
    return true;
}

template <typename T, bool UNIFORM, bool PACKED>
__global__ void __launch_bounds__(FT_TPB, 4) wide3_kernel(const StepParams p, const Queues qs) {
    pdl_wait();
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    const int n_wide = *(volatile int*)qs.q_n;
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * FT_TPB;
    const int rounds = (n_wide + stride - 1) / stride;
    for (int rnd = 0; rnd < rounds; ++rnd) {
        const int i = rnd * stride + blockIdx.x * FT_TPB + threadIdx.x;
        const bool mine = i < n_wide;
        const int j = mine ? qs.q[qs.dir * i] : 0;
        VRes res;
        vres_init(res);
        Win<3> w;
        w.m = 0;
        unsigned int out_mask = 0;
        bool on = false;
        if (mine) {
            on = !wide3<T, UNIFORM, PACKED>(j, p, w);
            if (!on) {
                process_window<3>(w, p, res, out_mask, c_recip);
                report_flags(res, j, p);
            }
        }
        const unsigned int ob = __ballot_sync(0xffffffffu, on);
        if (ob) {
            int qb = 0;
            if (lane == 0) qb = atomicAdd(qs.w8_n, __popc(ob));
            qb = __shfl_sync(0xffffffffu, qb, 0);
            if (on) {
                qs.w8[qs.dir * (qb + __popc(ob & ((1u << lane) - 1u)))] = j;
                vres_init(res);
            }
        }
        bool fits;
        const int need = (mine && !on && res.cnt > 2) ? res.cnt : 0;
        const long long off = pool_place(need, res, p, lane, fits);
        if (mine && !on) {
            p.ws.vbm[j - p.j_base] = res.bm;
            if (need == 0 || fits) emit_window<T, 3>(w, out_mask, j, off, p);
        }
    }
}

// Gather for tier 2b: up to kMD L entries (signatures in registers), any
// number of entries per neighbour column (re-read from L1 in every row
// pass), up to K rows.  Returns false when the column exceeds kMD or K (the
// caller then uses vertex_slow).
template <typename T, int K, bool UNIFORM>
__device__ __forceinline__ bool gather_wide(int j, const StepParams& p, Win<K>& w) {
    const int q0 = __ldg(&p.lap_ptr[j - p.j_base]);
    const int n = __ldg(&p.lap_ptr[j - p.j_base + 1]) - q0;
    if (n > kMD || n < 1) return false;
    int u[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) u[k] = (k < n) ? __ldg(&p.lap_idx[q0 + k]) : -1;
    int sg[kMD], ax[kMD], cn[kMD];
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        sg[k] = (k < n) ? __ldg(&p.in.sig[u[k]]) : FT_SIG_EMPTY;
        ax[k] = (k < n) ? __ldg(&p.in.aux[u[k]]) : 0;
        cn[k] = sig_count(sg[k]);
    }
    int kd = -1;
#pragma unroll
    for (int k = 0; k < kMD; ++k) if (u[k] == j) kd = k;
    if (kd < 0) return false;
    const double invdeg = UNIFORM ? recip_deg(n) : 0.0;
    int lo = -1;
    w.m = 0;
#pragma unroll
    for (int i = 0; i <= K; ++i) {
        int rr = INT_MAX;
#pragma unroll
        for (int k = 0; k < kMD; ++k) {
            for (int t = 0; t < cn[k]; ++t) {
                const int x = hyb_row<T>(p.in, sg[k], ax[k], t);
                if (x > lo) { if (x < rr) rr = x; break; }   // rows ascend in a column
            }
        }
        if (i == K) return rr == INT_MAX;     // more than K rows?
        if (rr == INT_MAX) return true;       // all rows found (w.m of them)
        double lam = 0.0, ph = 0.0;
        if (rr != INT_MAX) {
#pragma unroll
            for (int k = 0; k < kMD; ++k) {
                const double l = (k < n) ? lap_value<T, UNIFORM>(p, k, kd, q0, invdeg) : 0.0;
                for (int t = 0; t < cn[k]; ++t) {
                    const int x = hyb_row<T>(p.in, sg[k], ax[k], t);
                    if (x == rr) {
                        const double vv = hyb_val<T>(p.in, u[k], sg[k], ax[k], t);
                        lam = lam + vv * l;
                        if (k == kd) ph = vv;
                    }
                    if (x >= rr) break;
                }
            }
            w.m = i + 1;
            lo = rr;
        }
        w.rows[i] = rr;
        w.lam[i] = lam;
        w.phi[i] = ph;
    }
    return true;
}

template <typename T, bool UNIFORM>
__global__ void __launch_bounds__(FT_TPB, 4) wide_kernel(const StepParams p, const Queues qs) {
    pdl_wait();
    constexpr int KW = 8;      // wider unions go to tier 3
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    const int n_wide = *(volatile int*)qs.w8_n;   // tier-2a leftovers
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * FT_TPB;
    const int rounds = (n_wide + stride - 1) / stride;
    for (int rnd = 0; rnd < rounds; ++rnd) {
        const int i = rnd * stride + blockIdx.x * FT_TPB + threadIdx.x;
        const bool mine = i < n_wide;
        const int j = mine ? qs.w8[qs.dir * i] : 0;
        VRes res;
        vres_init(res);
        Win<KW> w;
        unsigned int out_mask = 0;
        bool deep = false;
        if (mine) {
            deep = !gather_wide<T, KW, UNIFORM>(j, p, w);
            if (!deep) {
                process_window<KW>(w, p, res, out_mask, c_recip);
                report_flags(res, j, p);
            }
        }
        // tier 3: beyond the tier-2 window
        const unsigned int db = __ballot_sync(0xffffffffu, deep);
        if (db) {
            int qb = 0;
            if (lane == 0) qb = atomicAdd(qs.dp_n, __popc(db));
            qb = __shfl_sync(0xffffffffu, qb, 0);
            if (deep) {
                qs.dp[qs.dir * (qb + __popc(db & ((1u << lane) - 1u)))] = j;
                vres_init(res);    // only the columns handed to tier 3
            }
        }
        bool fits;
        const int need = (mine && !deep && res.cnt > 2) ? res.cnt : 0;
        const long long off = pool_place(need, res, p, lane, fits);
        if (mine && !deep) {
            p.ws.vbm[j - p.j_base] = res.bm;
            if (need == 0 || fits) emit_window<T, KW>(w, out_mask, j, off, p);
        }
    }
}


// one warp per listed column (grid-stride); the warp's statistics go to
// the global accumulators once
template <typename T, bool UNIFORM, bool PACKED>
__global__ void __launch_bounds__(FT_TPB, 4) warp_kernel(const StepParams p, const Queues qs) {
    pdl_wait();
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    const int nc = *(volatile const int*)qs.q_n;
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * FT_WARPS;
    WarpStats ws;
    ws.maxd = 0.0; ws.cnt = 0; ws.skel = 0;
    // two columns per warp and pass (uniform trip count over the warp)
    for (int i0 = 2 * ((blockIdx.x * FT_TPB + threadIdx.x) >> 5); i0 < nc; i0 += 2 * nw) {
        const int i = i0 + (lane >> 4);
        const bool have = i < nc;
        half_column<T, UNIFORM, PACKED>(have ? __ldg(&qs.q[qs.dir * i]) : p.j_base, have, p, qs, lane, ws);
    }
    // lanes 0 and 16 hold the halves' statistics
    ws.maxd = fmax(ws.maxd, __shfl_down_sync(0xffffffffu, ws.maxd, 16));
    ws.cnt += __shfl_down_sync(0xffffffffu, ws.cnt, 16);
    ws.skel += __shfl_down_sync(0xffffffffu, ws.skel, 16);
    if (lane == 0 && (ws.maxd > 0.0 || ws.cnt || ws.skel)) {
        if (ws.maxd > 0.0) atomicMax(&p.ws.ctl->maxdelta_bits, (unsigned long long)__double_as_longlong(ws.maxd));
        if (ws.skel) atomicAdd(&p.ws.ctl->skel_total, (unsigned long long)ws.skel);
        if (ws.cnt) atomicAdd(&p.ws.ctl->nnz_total, (unsigned long long)ws.cnt);
    }
}

// tier 3: exact windowed global-memory algorithm (no width limit)
template <typename T, bool UNIFORM>
__global__ void __launch_bounds__(FT_TPB) deep_kernel(const StepParams p, const Queues qs) {
    pdl_wait();
    if (p.check_done && *(volatile int*)&p.ws.ctl->done) return;
    const int n_deep = *(volatile int*)qs.dp_n;
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * FT_TPB;
    const int rounds = (n_deep + stride - 1) / stride;
    for (int rnd = 0; rnd < rounds; ++rnd) {
        const int i = rnd * stride + blockIdx.x * FT_TPB + threadIdx.x;
        const bool mine = i < n_deep;
        const int j = mine ? qs.dp[qs.dir * i] : 0;
        VRes res;
        vres_init(res);
        if (mine) {
            vertex_slow<T, 8, UNIFORM>(j, p, res, 0, false);
            report_flags(res, j, p);
        }
        bool fits;
        const int need = (mine && res.cnt > 2) ? res.cnt : 0;
        const long long off = pool_place(need, res, p, lane, fits);
        if (mine) {
            p.ws.vbm[j - p.j_base] = res.bm;
            if (need == 0 || fits) {
                VRes r2 = res;
                vertex_slow<T, 8, UNIFORM>(j, p, r2, off, true);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// per-step finalisation: deterministic two-level base-mass reduction (fixed
// per-CTA tile ranges, then the last CTA sums the partials in order), stats
// record, error / convergence flags, accumulator reset.

#define FT_FIN_TPB 128

__global__ void __launch_bounds__(FT_FIN_TPB) finalize_kernel(const FinalizeParams f) {
    Control* ctl = f.ws.ctl;
    if (f.evolve && *(volatile int*)&ctl->done) return;
    __shared__ double s_part[FT_FIN_TPB / 32];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    // one thread per 32-column segment, a fixed range of segments per CTA;
    // the segment's value: its tier-1 sum, its tier-2/3 columns in vertex
    // order, and (first segment of a tile) the tile's tier-1.5 sum
    const int ns = FT_WARPS * f.ws.num_tiles;
    const int per = ((ns + gridDim.x - 1) / gridDim.x + FT_FIN_TPB - 1) / FT_FIN_TPB * FT_FIN_TPB;
    const int s0 = blockIdx.x * per, s1 = min(ns, s0 + per);
    double acc = 0.0, amx = 0.0;
    long long acnt = 0, askel = 0;
    for (int sg = s0 + tid; sg < s1; sg += FT_FIN_TPB) {
        double tb = f.ws.seg_bm[sg];
        amx = fmax(amx, f.ws.seg_maxd[sg]);
        const int2 cs = f.ws.seg_cs[sg];
        acnt += cs.x;
        askel += cs.y;
        unsigned int m = f.ws.slow_mask[sg];
        while (m) {   // tier-2/3 columns of the segment, in vertex order
            const int b = __ffs(m) - 1;
            m &= m - 1;
            tb = tb + f.ws.vbm[(size_t)sg * 32 + b];
        }
        if (sg % (FT_WARPS * FT_GEN_TILES) == 0) {
            // first segment of a tier-1.5 tile group: the group's slots
            const int g = sg / (FT_WARPS * FT_GEN_TILES);
            unsigned int any = 0u;
#pragma unroll
            for (int k = 0; k < FT_WARPS * FT_GEN_TILES; ++k)
                if (sg + k < ns) any |= f.ws.gen_mask[sg + k];
            if (any) {
                tb = tb + f.ws.gen_bm[g];
                amx = fmax(amx, f.ws.gen_maxd[g]);
                const int2 gc = f.ws.gen_cs[g];
                acnt += gc.x;
                askel += gc.y;
            }
        }
        acc = acc + tb;
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
    if (!s_last) return;
    __threadfence();
    // the last CTA combines the per-CTA partials: thread t owns partials t,
    // t + FT_FIN_TPB, ... (fixed order), then fixed shuffle / warp trees
    double pb = 0.0, pm = 0.0;
    long long pc = 0, pk = 0;
    const int G = (int)gridDim.x;
    for (int q0 = tid; q0 < G; q0 += 4 * FT_FIN_TPB) {
        // four partials' loads in flight, added in the same order
        double b4[4], m4[4];
        long long c4[4], k4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int q = q0 + k * FT_FIN_TPB;
            const bool h = q < G;
            b4[k] = h ? __ldcg(&f.ws.fin_part[q]) : 0.0;
            m4[k] = h ? __ldcg(&f.ws.fin_maxd[q]) : 0.0;
            c4[k] = h ? __ldcg(&f.ws.fin_cnt[q]) : 0;
            k4[k] = h ? __ldcg(&f.ws.fin_skel[q]) : 0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (q0 + k * FT_FIN_TPB < G) pb = pb + b4[k];
            pm = fmax(pm, m4[k]);
            pc += c4[k];
            pk += k4[k];
        }
    }
    pb = warp_sum(pb);
    pc = warp_sum(pc);
    pk = warp_sum(pk);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pm = fmax(pm, __shfl_down_sync(0xffffffffu, pm, o));
    __syncthreads();
    if ((tid & 31) == 0) { s_part[tid >> 5] = pb; s_mx[tid >> 5] = pm; s_cnt[tid >> 5] = pc; s_skel[tid >> 5] = pk; }
    __syncthreads();
    if (tid != 0) return;
    pb = 0.0; pm = 0.0; pc = 0; pk = 0;
    for (int q = 0; q < FT_FIN_TPB / 32; ++q) { pb = pb + s_part[q]; pm = fmax(pm, s_mx[q]); pc += s_cnt[q]; pk += s_skel[q]; }
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
    st.needed = (long long)ctl->pool_next;
    if (ctl->conv_next > st.needed) st.needed = ctl->conv_next;
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
    ctl->conv_next = 0;
    ctl->nan_key = 0u;
    ctl->overflow = 0;
    ctl->slow_count = 0;
    ctl->deep_count = 0;
    ctl->gen_count = 0;
    ctl->wide8_count = 0;
    ctl->wide8b_count = 0;
    ctl->deepb_count = 0;
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
// canonical CSC -> hybrid layout

template <typename T>
__global__ void __launch_bounds__(256) convert_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                      const T* __restrict__ val, int n, HybOut o, long long cap,
                                                      Control* ctl) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool active = j < n;
    int c0 = 0, cnt = 0;
    if (active) {
        c0 = __ldg(&ptr[j]);
        cnt = __ldg(&ptr[j + 1]) - c0;
    }
    const int need = cnt > 2 ? cnt : 0;
    int incl = need;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
    }
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    long long base = 0;
    if (lane == 31 && wtot > 0) base = (long long)atomicAdd((unsigned long long*)&ctl->conv_next, (unsigned long long)wtot);
    base = __shfl_sync(0xffffffffu, base, 31);
    const bool fits = base + wtot <= cap;
    if (lane == 31 && !fits) atomicExch(&ctl->overflow, 1);
    if (!active) return;
    bool nf = false;
    if (cnt == 0) {
        o.sig[j] = FT_SIG_EMPTY;
    } else if (cnt <= 2) {
        const T x0 = val[c0];
        ((T*)o.v0)[j] = x0;
        nf |= !isfinite((double)x0);
        if (cnt == 1) {
            o.sig[j] = idx[c0];
        } else {
            const T x1 = val[c0 + 1];
            o.sig[j] = idx[c0] | kPair;
            o.aux[j] = idx[c0 + 1];
            ((T*)o.v1)[j] = x1;
            nf |= !isfinite((double)x1);
        }
    } else if (fits) {
        const long long off = base + incl - need;
        o.sig[j] = -cnt;
        o.aux[j] = (int)off;
        for (int t = 0; t < cnt; ++t) {
            o.pidx[off + t] = idx[c0 + t];
            const T x = val[c0 + t];
            ((T*)o.pval)[off + t] = x;
            nf |= !isfinite((double)x);
        }
    } else {
        o.sig[j] = FT_SIG_EMPTY;   // the step that follows reports the overflow
    }
    if (nf) atomicOr(&ctl->nonfinite, 1u);
}

__global__ void convert_report_kernel(Control* ctl, ft_step_stats* st, long long cap) {
    st->status = ctl->overflow ? FT_STATUS_OVERFLOW : FT_STATUS_OK;
    st->needed = ctl->conv_next > cap ? ctl->conv_next : cap;
    ctl->overflow = 0;
    ctl->conv_next = 0;
}

// ---------------------------------------------------------------------------
// compaction: hybrid -> canonical CSC

struct CompactParams {
    int n_v;
    HybIn src[2];
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
    const int* sig = c.src[src].sig;
    const int j0 = blockIdx.x * FT_CCH + threadIdx.x * kCPT;
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kCPT; ++k)
        if (j0 + k < c.n_v) sum += sig_count(__ldg(&sig[j0 + k]));
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
    const HybIn h = c.src[src];
    T* oval = (T*)c.out_val;
    const int j0 = blockIdx.x * FT_CCH + threadIdx.x * kCPT;
    int sg[kCPT];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
        sg[k] = (j0 + k < c.n_v) ? __ldg(&h.sig[j0 + k]) : FT_SIG_EMPTY;
        sum += sig_count(sg[k]);
    }
    int tot;
    const int pre = block_excl_scan<FT_CTPB>(sum, s_scan, &tot);
    long long o = c.ws.chunk_off[blockIdx.x] + pre;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
        if (j0 + k < c.n_v) {
            const int u = j0 + k;
            c.out_ptr[u] = (int)o;
            const int cnt = sig_count(sg[k]);
            const int a = cnt >= 2 ? __ldg(&h.aux[u]) : 0;
            for (int t = 0; t < cnt; ++t) {
                c.out_idx[o + t] = hyb_row<T>(h, sg[k], a, t);
                oval[o + t] = (T)hyb_val<T>(h, u, sg[k], a, t);
            }
            o += cnt;
        }
    }
}

__global__ void evolve_reset_kernel(Control* ctl) {
    ctl->nonfinite = 0u;    // ft_tiled_from_csc raises it again for non-finite input
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

__global__ void nonfinite_reset_kernel(Control* ctl) { ctl->nonfinite = 0u; }

// ---------------------------------------------------------------------------
// host side

typedef void (*StepKernelFn)(const StepParams);

static Queues queues(const StepParams& p, int which) {
    Queues q;
    int* L = p.ws.slow_list;
    Control* c = p.ws.ctl;
    const int n = p.n_v;
    if (which == 0) {
        q.q = L; q.w8 = L + n; q.dp = L + 2 * n; q.dir = 1;
        q.q_n = &c->slow_count; q.w8_n = &c->wide8_count; q.dp_n = &c->deep_count;
    } else {
        q.q = L + n - 1; q.w8 = L + 2 * n - 1; q.dp = L + 3 * n - 1; q.dir = -1;
        q.q_n = &c->gen_count; q.w8_n = &c->wide8b_count; q.dp_n = &c->deepb_count;
    }
    return q;
}

#define FT_PICK3(K, dtype, uni, packed)                                               \
    ((dtype) == FT_F64 ? ((uni) ? ((packed) ? K<double, true, true> : K<double, true, false>) \
                                : K<double, false, false>)                             \
                       : ((uni) ? ((packed) ? K<float, true, true> : K<float, true, false>)   \
                                : K<float, false, false>))
#define FT_PICK2(K, dtype, uni)                                                              \
    ((dtype) == FT_F64 ? ((uni) ? K<double, true> : K<double, false>) : ((uni) ? K<float, true> : K<float, false>))

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

extern "C" int64_t ft_tile_slot_entries(void) { return 0; }

extern "C" int64_t ft_tiled_min_capacity(int32_t n_vertices) {
    (void)n_vertices;
    return 0;
}

static int check_tiled(const ft_tiled* t, int n_rows, int n_cols) {
    if (!t || !t->sig || !t->aux || !t->v0 || !t->v1) return set_err(FT_ERR_ARG, "null hybrid buffer");
    if (n_rows < 1 || n_rows > FT_SIG_PAIR)
        return set_err(FT_ERR_SHAPE, "the hybrid layout holds at most 2^30 layer rows");
    if (t->capacity < 0 || t->capacity > (int64_t)INT_MAX) return set_err(FT_ERR_ARG, "pool capacity out of range");
    if (t->capacity > 0 && (!t->pool_idx || !t->pool_val)) return set_err(FT_ERR_ARG, "null pool");
    if (t->n_rows != n_rows || t->n_cols != n_cols) return set_err(FT_ERR_SHAPE, "hybrid buffer has wrong shape");
    return FT_OK;
}

// Per-device state (a process may drive several GPUs): whether c_recip is
// set on the device, grid sizes, the side stream with its fork / join events
// and the evolve-graph stream.  Indexed by the current device ordinal.
struct DevState {
    int init;
    int fixup_grid, sms;
    cudaStream_t side;
    cudaEvent_t fork, join;
    cudaStream_t gstream;
    cudaEvent_t gev[2];
    cudaEvent_t bdone, fdone, sjoin;   // evolve: queue B done, finalize done, side joined
};
static DevState g_dev[64];

static DevState& dev_state() {
    int d = 0;
    cudaGetDevice(&d);
    return g_dev[d & 63];
}

#define g_init (dev_state().init)
#define g_fixup_grid (dev_state().fixup_grid)
#define g_sms (dev_state().sms)
#define g_side (dev_state().side)
#define g_fork (dev_state().fork)
#define g_join (dev_state().join)
#define g_gstream (dev_state().gstream)
#define g_gev (dev_state().gev)

// FT_PROBE_EVENTS=1 (timing probes only): events at the stage boundaries of
// the last launch_step, read with ft_probe_timeline (debug export; first
// device only)
static cudaEvent_t g_pev[8];
static int g_pev_on = -1;

static void pev(int i, cudaStream_t st) {
    if (g_pev_on < 0) {
        const char* e = getenv("FT_PROBE_EVENTS");
        g_pev_on = e && atoi(e) ? 1 : 0;
        if (g_pev_on)
            for (auto& ev : g_pev) cudaEventCreate(&ev);
    }
    if (g_pev_on) cudaEventRecord(g_pev[i], st);
}

extern "C" int ft_probe_timeline(float* ms, int n) {
    if (g_pev_on != 1) return FT_ERR_ARG;
    cudaDeviceSynchronize();
    for (int i = 0; i < n && i < 8; ++i) ms[i] = -1.0f;
    for (int i = 1; i < n && i < 8; ++i)
        if (cudaEventElapsedTime(&ms[i], g_pev[0], g_pev[i]) != cudaSuccess) ms[i] = -1.0f;
    ms[0] = 0.0f;
    cudaGetLastError();
    return FT_OK;
}

static int side_init() {
    DevState& d = dev_state();
    if (d.side) return FT_OK;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&d.side, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.bdone, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.fdone, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.sjoin, cudaEventDisableTiming) != cudaSuccess) {
        d.side = nullptr;
        return FT_ERR_CUDA;
    }
    return FT_OK;
}

static int pdl_enabled() {
    static const int on = [] {
        const char* e = getenv("FT_PDL");
        return e ? atoi(e) : 1;
    }();
    return on;
}

// launch k on s, programmatically dependent on the stream's previous kernel
// (its launch and CTA ramp overlap the predecessor's tail; the kernel's
// pdl_wait() orders the memory accesses)
template <typename... KA, typename... AA>
static void launch_dep(void (*k)(KA...), int grid, int block, cudaStream_t s, AA&&... args) {
    if (!pdl_enabled() || g_pev_on == 1) {   // probe events sit between the kernels
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.stream = s;
        cudaLaunchKernelEx(&cfg, k, std::forward<AA>(args)...);
        return;
    }
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block); cfg.stream = s;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, std::forward<AA>(args)...);
}

static void lib_init() {
    DevState& d = dev_state();
    if (d.init) return;
    double h[33];
    h[0] = 0.0;
    for (int n = 1; n <= 32; ++n) h[n] = 1.0 / (double)n;
    cudaMemcpyToSymbol(ft::c_recip, h, sizeof(h));
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms = 148;
    d.fixup_grid = 4 * sms;
    d.sms = sms;
    d.init = 1;
}

// which = 1: tier 1, 2: tiers 1.5-3, 3: both
// dom == nullptr: the whole field; otherwise the owned column range of a
// partitioned field (lap_t then holds the owned columns of L^T only and the
// workspace is sized for the owned columns)
// parity: the step's segment-slot copy (ft_evolve alternates it); fin_wait
// (nullable): the previous step's finalize, waited for before tier 1.5
// touches the shared slots and accumulators; b_done (nullable): recorded
// after queue B (the side-stream finalize of this step waits on it)
static int launch_step(const ft_csc* lap_t, int32_t lap_flags, const ft_tiled* in, ft_tiled* out,
                       int32_t dtype, const ft_params* prm, void* workspace, size_t ws_bytes, int check_done,
                       cudaStream_t s, int which = 3, const ft_domain* dom = nullptr, int parity = 0,
                       cudaEvent_t fin_wait = nullptr, cudaEvent_t b_done = nullptr) {
    if (!lap_t || !out || !in || !prm || !workspace) return set_err(FT_ERR_ARG, "null argument");
    if (dtype != FT_F64 && dtype != FT_F32) return set_err(FT_ERR_ARG, "bad dtype");
    const int n_rows = in->n_rows, n_v = in->n_cols;
    if (n_v <= 0) return set_err(FT_ERR_SHAPE, "empty field");
    const int j_base = dom ? dom->col_begin : 0;
    const int n_own = dom ? dom->col_count : n_v;
    if (dom && (j_base < 0 || n_own < 1 || (long long)j_base + n_own > n_v))
        return set_err(FT_ERR_SHAPE, "domain outside the field");
    if (lap_t->n_rows != n_v || lap_t->n_cols != n_own)
        return set_err(FT_ERR_SHAPE, "Laplacian size does not match field");
    int rc = check_tiled(in, n_rows, n_v);
    if (rc == FT_OK) rc = check_tiled(out, n_rows, n_v);
    if (rc != FT_OK) return rc;
    const long long step_cap = dom ? dom->step_capacity : out->capacity;
    if (step_cap < 0 || step_cap > out->capacity) return set_err(FT_ERR_ARG, "domain step capacity out of range");
    if (ws_bytes < ft::workspace_bytes(n_own)) return set_err(FT_ERR_ARG, "workspace too small");
    ft::StepParams p;
    p.n_v = n_own;
    p.j_base = j_base;
    p.num_tiles = ft::num_tiles_for(n_own);
    p.lap_ptr = lap_t->col_ptr;
    p.lap_idx = lap_t->row_idx;
    p.lap_val = lap_t->values;
    p.in = ft::hyb_in(in);
    p.out = ft::hyb_out(out);
    p.cap = step_cap;
    p.w = prm->w; p.a = prm->a; p.e = prm->e; p.eb = prm->e_base; p.mu = prm->mu; p.dt = prm->dt;
    p.ws = ft::ws_parity(ft::carve_workspace(workspace, n_own), parity);
    p.check_done = check_done;
    p.finite = std::isfinite(p.w) && std::isfinite(p.a) && std::isfinite(p.e) && std::isfinite(p.eb) &&
               std::isfinite(p.mu) && std::isfinite(p.dt);
    const bool uni = (lap_flags & FT_LAP_UNIFORM) != 0;
    const bool packed = uni && (lap_flags & FT_LAP_PACKED) != 0;
    p.lap_pack = packed ? (const int4*)lap_t->values : nullptr;
    lib_init();
    p.force_check = (lap_flags & FT_LAP_CHECK_FINITE) != 0;
    p.report_ids = dom ? dom->report_ids : nullptr;
    if (which & 1) {
        pev(0, s);
        const ft::StepKernelFn k1 = FT_PICK3(ft::tier1_kernel, dtype, uni, packed);
        static int t1_ctas[2][2][2] = {};
        int& per_sm = t1_ctas[dtype == FT_F64][uni][packed];
        if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, FT_TPB, 0) != cudaSuccess)
            per_sm = 8;
        const int grid = per_sm * g_sms < p.num_tiles ? per_sm * g_sms : p.num_tiles;
        k1<<<grid, FT_TPB, 0, s>>>(p);
    }
    if (which & 2) {
        // queue A (tier 1's wide columns) on the high-priority side stream,
        // concurrently with tier 1.5
        if (side_init() != FT_OK) return cuda_check("side stream");
        const ft::Queues qa = ft::queues(p, 0), qb = ft::queues(p, 1);
        if (fin_wait) cudaStreamWaitEvent(s, fin_wait, 0);
        cudaEventRecord(g_fork, s);
        cudaStreamWaitEvent(g_side, g_fork, 0);
        ft::queue_kernel<<<(FT_WARPS * p.num_tiles + 255) / 256, 256, 0, g_side>>>(p);
        launch_dep(FT_PICK3(ft::wide3_kernel, dtype, uni, packed), g_fixup_grid, FT_TPB, g_side, p, qa);
        pev(3, g_side);
        launch_dep(FT_PICK2(ft::wide_kernel, dtype, uni), g_fixup_grid, FT_TPB, g_side, p, qa);
        launch_dep(FT_PICK2(ft::deep_kernel, dtype, uni), g_fixup_grid / 4, FT_TPB, g_side, p, qa);
        pev(4, g_side);
        cudaEventRecord(g_join, g_side);
        // tier 1.5, one warp per tile
        const int ngroups = (p.num_tiles + FT_GEN_TILES - 1) / FT_GEN_TILES;
        // (a normal launch: the fork event sits between tier 1 and tier 1.5)
        FT_PICK3(ft::gen_kernel, dtype, uni, packed)<<<(ngroups + FT_WARPS - 1) / FT_WARPS, FT_TPB, 0, s>>>(p);
        pev(5, s);
        // queue B: what tier 1.5 defers (unions of three or more rows), one
        // warp per column
        launch_dep(FT_PICK3(ft::warp_kernel, dtype, uni, packed), g_fixup_grid * 2, FT_TPB, s, p, qb);
        // (its tier-3 list is empty unless a column exceeds one warp)
        launch_dep(FT_PICK2(ft::deep_kernel, dtype, uni), g_fixup_grid / 8, FT_TPB, s, p, qb);
        pev(6, s);
        if (b_done) cudaEventRecord(b_done, s);
        cudaStreamWaitEvent(s, g_join, 0);
        pev(7, s);
    }
    return cuda_check("step kernel");
}

static void launch_finalize(const ft::Workspace& ws, ft_step_stats* trace, long long tiled_cap,
                            int evolve, int max_steps, double tol, double thr, cudaStream_t s, int parity = 0) {
    ft::FinalizeParams f;
    f.ws = ft::ws_parity(ws, parity); f.trace = trace; f.tiled_cap = tiled_cap; f.fixed_slot = evolve ? 0 : 1;
    f.evolve = evolve; f.max_steps = max_steps; f.tol = tol; f.base_threshold = thr;
    lib_init();
    // about one 32-column segment per thread
    int ctas = (FT_WARPS * ws.num_tiles + FT_FIN_TPB - 1) / FT_FIN_TPB;
    ctas = ctas < 1 ? 1 : (ctas > FT_FIN_MAX ? FT_FIN_MAX : ctas);
    ft::finalize_kernel<<<ctas, FT_FIN_TPB, 0, s>>>(f);
}

static int launch_convert(const ft_csc* src, ft_tiled* dst, int32_t dtype, const ft::Workspace& ws,
                          cudaStream_t s) {
    if (!src || !src->col_ptr || (!src->row_idx && src->capacity > 0)) return set_err(FT_ERR_ARG, "null argument");
    if (dtype != FT_F64 && dtype != FT_F32) return set_err(FT_ERR_ARG, "bad dtype");
    int rc = check_tiled(dst, src->n_rows, src->n_cols);
    if (rc != FT_OK) return rc;
    const int n = src->n_cols;
    if (n <= 0) return set_err(FT_ERR_SHAPE, "empty field");
    const int grid = (n + 255) / 256;
    if (dtype == FT_F64)
        ft::convert_kernel<double><<<grid, 256, 0, s>>>(src->col_ptr, src->row_idx, (const double*)src->values, n,
                                                       ft::hyb_out(dst), dst->capacity, ws.ctl);
    else
        ft::convert_kernel<float><<<grid, 256, 0, s>>>(src->col_ptr, src->row_idx, (const float*)src->values, n,
                                                      ft::hyb_out(dst), dst->capacity, ws.ctl);
    return cuda_check("ft_tiled_from_csc");
}

static int launch_compact(ft::CompactParams& c, int dtype, cudaStream_t s) {
    const int nc = c.ws.num_chunks;
    ft::compact_count_kernel<<<nc, FT_CTPB, 0, s>>>(c);
    ft::compact_scan_kernel<<<1, 1024, 0, s>>>(c);
    if (dtype == FT_F64) ft::compact_copy_kernel<double><<<nc, FT_CTPB, 0, s>>>(c);
    else ft::compact_copy_kernel<float><<<nc, FT_CTPB, 0, s>>>(c);
    return cuda_check("compact");
}

extern "C" int ft_tiled_from_csc(const ft_csc* src, ft_tiled* dst, int32_t dtype, void* workspace,
                                 size_t ws_bytes, ft_step_stats* stats, void* stream) {
    if (!src || !dst || !workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (ws_bytes < ft::workspace_bytes(src->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const ft::Workspace ws = ft::carve_workspace(workspace, src->n_cols);
    const int rc = launch_convert(src, dst, dtype, ws, s);
    if (rc != FT_OK) return rc;
    ft::convert_report_kernel<<<1, 1, 0, s>>>(ws.ctl, stats, dst->capacity);
    return cuda_check("ft_tiled_from_csc");
}

extern "C" int ft_step_kernel(const ft_csc* lap_t, int32_t lap_flags, const ft_tiled* in, ft_tiled* out,
                              int32_t dtype, const ft_params* params, void* workspace, size_t ws_bytes,
                              void* stream) {
    return launch_step(lap_t, lap_flags, in, out, dtype, params, workspace, ws_bytes, 0, (cudaStream_t)stream, 1);
}

extern "C" int ft_step_fixup(const ft_csc* lap_t, int32_t lap_flags, const ft_tiled* in, ft_tiled* out,
                             int32_t dtype, const ft_params* params, void* workspace, size_t ws_bytes,
                             void* stream) {
    return launch_step(lap_t, lap_flags, in, out, dtype, params, workspace, ws_bytes, 0, (cudaStream_t)stream, 2);
}

extern "C" int ft_step_finalize(void* workspace, size_t ws_bytes, int32_t n_vertices,
                                int64_t tiled_capacity, ft_step_stats* stats, void* stream) {
    if (!workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (ws_bytes < ft::workspace_bytes(n_vertices)) return set_err(FT_ERR_ARG, "workspace too small");
    launch_finalize(ft::carve_workspace(workspace, n_vertices), stats, tiled_capacity, 0, 1, 0.0, 0.0,
                    (cudaStream_t)stream);
    return cuda_check("ft_step_finalize");
}

static void fill_compact(ft::CompactParams& c, const ft_tiled* a, const ft_tiled* b, int sel, ft_csc* dst,
                         void* workspace) {
    c.n_v = dst->n_cols;
    c.src[0] = ft::hyb_in(a);
    c.src[1] = ft::hyb_in(b ? b : a);
    c.sel = sel;
    c.out_ptr = dst->col_ptr; c.out_idx = dst->row_idx; c.out_val = dst->values; c.cap = dst->capacity;
    c.ws = ft::carve_workspace(workspace, dst->n_cols);
    c.stats = nullptr;
    c.control = nullptr;
    c.check_status = 0;
}

extern "C" int ft_compact(const ft_tiled* src, ft_csc* dst, int32_t dtype, void* workspace, size_t ws_bytes,
                          ft_step_stats* stats, void* stream) {
    if (!src || !dst || !workspace || !stats) return set_err(FT_ERR_ARG, "null argument");
    if (src->n_cols != dst->n_cols || src->n_rows != dst->n_rows) return set_err(FT_ERR_SHAPE, "shape mismatch");
    if (ws_bytes < ft::workspace_bytes(dst->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    if (dst->n_cols == 0) return set_err(FT_ERR_SHAPE, "empty field");
    ft::CompactParams c;
    fill_compact(c, src, nullptr, 0, dst, workspace);
    c.stats = stats;
    return launch_compact(c, dtype, (cudaStream_t)stream);
}

extern "C" int ft_step(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in, ft_tiled* scratch_in,
                       ft_tiled* scratch_out, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                       void* workspace, size_t ws_bytes, ft_step_stats* stats, void* stream) {
    if (!phi_in || !phi_out || !stats || !scratch_in || !scratch_out) return set_err(FT_ERR_ARG, "null argument");
    if (phi_out->n_cols != phi_in->n_cols || phi_out->n_rows != phi_in->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    if (ws_bytes < ft::workspace_bytes(phi_in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    ft::Workspace ws = ft::carve_workspace(workspace, phi_in->n_cols);
    ft::nonfinite_reset_kernel<<<1, 1, 0, s>>>(ws.ctl);
    int rc = launch_convert(phi_in, scratch_in, dtype, ws, s);
    if (rc != FT_OK) return rc;
    rc = launch_step(lap_t, lap_flags, scratch_in, scratch_out, dtype, params, workspace, ws_bytes, 0, s);
    if (rc != FT_OK) return rc;
    const long long cap = scratch_out->capacity < scratch_in->capacity ? scratch_out->capacity : scratch_in->capacity;
    launch_finalize(ws, stats, cap, 0, 1, 0.0, 0.0, s);
    // the compaction always runs; the host ignores it if the step failed
    ft::CompactParams c;
    fill_compact(c, scratch_out, nullptr, 0, phi_out, workspace);
    c.stats = stats;
    c.check_status = 1;
    return launch_compact(c, dtype, s);
}

// The steady part of evolve (steps 1, 2, ...: a -> b, b -> a) repeats with
// period 2, so kGraphSteps steps are captured once into a CUDA graph and
// replayed; steps past max_steps / convergence are device-side no-ops (the
// kernels test the done flag).  Graphs are cached by their full launch
// configuration.
constexpr int kGraphSteps = 16;

struct GraphKey {
    const void* ptrs[18];
    long long caps[3];
    double prm[8];
    int ints[5];
    bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};

struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    bool used;
};

static GraphEntry g_graphs[8];
static int g_graph_next = 0;

// private non-blocking stream for capture and replay (the caller's stream may
// be the legacy default stream, which cannot be captured); ordered against the
// caller's stream with events
static int graph_stream_init() {
    DevState& d = dev_state();
    if (d.gstream) return FT_OK;
    if (cudaStreamCreateWithFlags(&d.gstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.gev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.gev[1], cudaEventDisableTiming) != cudaSuccess) {
        d.gstream = nullptr;
        return FT_ERR_CUDA;
    }
    return FT_OK;
}

static cudaGraphExec_t graph_lookup(const GraphKey& k) {
    for (auto& e : g_graphs)
        if (e.used && e.key == k) return e.exec;
    return nullptr;
}

static void graph_store(const GraphKey& k, cudaGraphExec_t exec) {
    GraphEntry& e = g_graphs[g_graph_next];
    g_graph_next = (g_graph_next + 1) % 8;
    if (e.used) cudaGraphExecDestroy(e.exec);
    e.key = k;
    e.exec = exec;
    e.used = true;
}

extern "C" int ft_evolve(const ft_csc* lap_t, int32_t lap_flags, const ft_csc* phi_in, ft_tiled* work_a,
                         ft_tiled* work_b, ft_csc* phi_out, int32_t dtype, const ft_params* params,
                         int32_t max_steps, double tol, double base_threshold, void* workspace,
                         size_t ws_bytes, ft_step_stats* trace, int64_t* control, void* stream) {
    if (!phi_in || !phi_out || !work_a || !work_b || !trace || !control)
        return set_err(FT_ERR_ARG, "null argument");
    if (max_steps < 1) return set_err(FT_ERR_SHAPE, "max_steps must be >= 1");
    if (phi_out->n_cols != phi_in->n_cols || phi_out->n_rows != phi_in->n_rows)
        return set_err(FT_ERR_SHAPE, "output buffer has wrong shape");
    if (ws_bytes < ft::workspace_bytes(phi_in->n_cols)) return set_err(FT_ERR_ARG, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    ft::Workspace ws = ft::carve_workspace(workspace, phi_in->n_cols);
    if (side_init() != FT_OK) return cuda_check("ft_evolve(side stream)");
    DevState& d = dev_state();
    // Step i runs on the main stream (tier 1, 1.5, queue B) and the side
    // stream (queue A); its finalize runs on the side stream once queue B is
    // done, overlapping tier 1 of step i + 1 (which writes the other parity's
    // segment slots); tier 1.5 of step i + 1 waits for that finalize.
    auto step = [&](int i, const ft_tiled* in_t, ft_tiled* out, long long cap, cudaStream_t ms,
                    bool wait_prev) -> int {
        const int r = launch_step(lap_t, lap_flags, in_t, out, dtype, params, workspace, ws_bytes, 1, ms, 3,
                                  nullptr, i & 1, wait_prev ? d.fdone : nullptr, d.bdone);
        if (r != FT_OK) return r;
        cudaStreamWaitEvent(d.side, d.bdone, 0);
        launch_finalize(ws, trace, cap, 1, max_steps, tol, base_threshold, d.side, i & 1);
        cudaEventRecord(d.fdone, d.side);
        return FT_OK;
    };
    ft::evolve_reset_kernel<<<1, 1, 0, s>>>(ws.ctl);
    // canonical input -> b, step 1: b -> a
    int rc = launch_convert(phi_in, work_b, dtype, ws, s);
    if (rc != FT_OK) return rc;
    const long long cap0 = work_a->capacity < work_b->capacity ? work_a->capacity : work_b->capacity;
    rc = step(0, work_b, work_a, cap0, s, false);
    if (rc != FT_OK) return rc;
    const int rest = max_steps - 1;
    if (rest < kGraphSteps) {
        for (int i = 1; i < max_steps; ++i) {
            ft_tiled* out = (i & 1) ? work_b : work_a;
            const ft_tiled* in_t = (i & 1) ? work_a : work_b;
            rc = step(i, in_t, out, out->capacity, s, true);
            if (rc != FT_OK) return rc;
        }
        cudaStreamWaitEvent(s, d.fdone, 0);     // the last finalize
    } else {
        GraphKey k;
        memset(&k, 0, sizeof(k));
        if (graph_stream_init() != FT_OK) return cuda_check("ft_evolve(graph stream)");
        cudaStream_t gs = g_gstream;
        const void* ptrs[18] = {lap_t->col_ptr, lap_t->row_idx, lap_t->values, work_a->sig, work_a->aux,
                                work_a->v0, work_a->v1, work_a->pool_idx, work_a->pool_val, work_b->sig,
                                work_b->aux, work_b->v0, work_b->v1, work_b->pool_idx, work_b->pool_val,
                                workspace, trace, nullptr};
        memcpy(k.ptrs, ptrs, sizeof(ptrs));
        k.caps[0] = work_a->capacity; k.caps[1] = work_b->capacity; k.caps[2] = (long long)ws_bytes;
        const double prm[8] = {params->w, params->a, params->e, params->e_base, params->mu, params->dt, tol,
                               base_threshold};
        memcpy(k.prm, prm, sizeof(prm));
        const int ints[5] = {lap_flags, dtype, max_steps, phi_in->n_cols, phi_in->n_rows};
        memcpy(k.ints, ints, sizeof(ints));
        // the graph's first step starts after the previous finalize (step 0's
        // here, the previous replay's last one inside the graph's end join)
        cudaEventRecord(g_gev[0], s);
        cudaStreamWaitEvent(gs, g_gev[0], 0);
        cudaStreamWaitEvent(gs, d.fdone, 0);
        cudaGraphExec_t exec = graph_lookup(k);
        if (!exec) {
            cudaGraph_t graph;
            if (cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
                return cuda_check("ft_evolve(begin capture)");
            for (int i = 1; i <= kGraphSteps; ++i) {
                ft_tiled* out = (i & 1) ? work_b : work_a;
                const ft_tiled* in_t = (i & 1) ? work_a : work_b;
                const int r2 = step(i, in_t, out, out->capacity, gs, i > 1);
                if (r2 != FT_OK) rc = r2;
            }
            cudaEventRecord(d.sjoin, d.side);   // the side stream rejoins the capture
            cudaStreamWaitEvent(gs, d.sjoin, 0);
            const cudaError_t ec = cudaStreamEndCapture(gs, &graph);
            if (ec != cudaSuccess || rc != FT_OK) return rc != FT_OK ? rc : cuda_check("ft_evolve(end capture)");
            // node priorities: queue A keeps its side stream's high priority
            if (cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority) != cudaSuccess) {
                cudaGraphDestroy(graph);
                return cuda_check("ft_evolve(instantiate)");
            }
            cudaGraphDestroy(graph);
            graph_store(k, exec);
        }
        for (int done = 0; done < rest; done += kGraphSteps) cudaGraphLaunch(exec, gs);
        cudaEventRecord(g_gev[1], gs);
        cudaStreamWaitEvent(s, g_gev[1], 0);
    }
    ft::evolve_report_kernel<<<1, 1, 0, s>>>(ws.ctl, (long long*)control);
    ft::CompactParams c;
    fill_compact(c, work_a, work_b, -1, phi_out, workspace);
    c.control = (long long*)control;
    return launch_compact(c, dtype, s);
}

// ---------------------------------------------------------------------------
// partitioned field: one step of the owned columns (the halo kernels and the
// combine live in ft_domain.cu)

extern "C" int ft_domain_step(const ft_csc* lap_rows, int32_t lap_flags, const ft_tiled* in, ft_tiled* out,
                              int32_t dtype, const ft_params* params, const ft_domain* dom, void* workspace,
                              size_t ws_bytes, ft_step_stats* record, void* stream) {
    if (!in || !dom || !record) return set_err(FT_ERR_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int rc = launch_step(lap_rows, lap_flags, in, out, dtype, params, workspace, ws_bytes, 1, s, 3, dom);
    if (rc != FT_OK) return rc;
    launch_finalize(ft::carve_workspace(workspace, dom->col_count), record, dom->step_capacity, 0, 1, 0.0, 0.0, s);
    return cuda_check("ft_domain_step");
}

// ---------------------------------------------------------------------------
// packed L^T neighbour table (FT_LAP_PACKED)

namespace ft {
__global__ void lap_pack_kernel(const int* __restrict__ ptr, const int* __restrict__ idx, int n_cols,
                                int col_base, int4* __restrict__ pack, int* n_csr) {
    const int jl = blockIdx.x * blockDim.x + threadIdx.x;
    if (jl >= n_cols) return;
    const int q0 = ptr[jl], n = ptr[jl + 1] - q0;
    const long long j = (long long)col_base + jl;
    int s[kMD];
    bool ok = n >= 1 && n <= kMD;
#pragma unroll
    for (int k = 0; k < kMD; ++k) {
        s[k] = kPackEmpty;
        if (ok && k < n) {
            const long long dl = (long long)idx[q0 + k] - j;
            if (dl < -32767 || dl > 32767) ok = false;
            else s[k] = (int)dl;
        }
    }
    if (!ok) {
#pragma unroll
        for (int k = 0; k < kMD; ++k) s[k] = kPackEmpty;
        atomicAdd(n_csr, 1);
    }
    int w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = (s[2 * q] & 0xffff) | (s[2 * q + 1] << 16);
    pack[jl] = make_int4(w[0], w[1], w[2], w[3]);
}
}  // namespace ft

extern "C" int ft_laplacian_pack(const ft_csc* lap_t, int32_t col_base, int16_t* pack, int32_t* n_csr,
                                 void* stream) {
    if (!lap_t || !pack || !n_csr) return set_err(FT_ERR_ARG, "null argument");
    if (((uintptr_t)pack) & 15) return set_err(FT_ERR_ARG, "pack must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(n_csr, 0, sizeof(int32_t), s);
    const int n = lap_t->n_cols;
    if (n > 0) ft::lap_pack_kernel<<<(n + 255) / 256, 256, 0, s>>>(lap_t->col_ptr, lap_t->row_idx, n, col_base,
                                                                   (int4*)pack, n_csr);
    return cuda_check("ft_laplacian_pack");
}
