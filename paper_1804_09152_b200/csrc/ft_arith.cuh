// Per-column arithmetic of the Euler step (Appendix A of SURVEY.md).
//
// Every function here replays the reference's operations in the reference's
// order (pkg/src/fieldtess/_kernels.py:179-282): the same parenthesisation,
// v * (1 / s) for the normaliser, the clamp order NaN -> > 1 -> <= 0.  The
// library is compiled with -fmad=false and sqrt / division are IEEE
// correctly rounded, so EXACT mode (double storage) is bitwise identical to
// the numba reference.
#pragma once
#include <climits>
#include <cmath>

#include "ft_common.cuh"

namespace ft {

// CouplingParams (field.py:34-71) as the kernels read them
struct Cp {
    double w, a, e, eb, mu, dt;
    int finite;          // all couplings finite: the single-row closed form is exact
};

// window of layer rows for one vertex column (ascending rows)
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

// interest skeleton (_kernels.py:96-150): (PHI stored and > 0) or ((absent
// or == 0) and Lt stored and > 0)
__device__ __forceinline__ bool in_skeleton(double ph, double lm) {
    return (ph > 0.0) || (ph == 0.0 && lm > 0.0);
}

// sqrt of a skeleton row's PHI (>= 0, never NaN: in_skeleton).  A row held
// only by Lt has PHI == 0, and sqrt(+-0) leaves CUDA's inline fast path for
// its out-of-range slow-path call (the warp branches and shuffles registers
// even when the result is then discarded); the argument is therefore kept
// in range (behind an empty asm, or the compiler folds the select back into
// sqrt(x) / sqrt(1)) and +-0 returned as itself (sqrt(+-0) == +-0: bitwise
// the same).
__device__ __forceinline__ double sqrt_skel(double x) {
    double a = x > 0.0 ? x : 1.0;
    asm("" : "+d"(a));     // opaque: the select is not folded through the sqrt
    const double r = sqrt(a);
    return x > 0.0 ? r : x;
}

// 1 / s for a positive column sum, 0 otherwise; the division never sees
// s == 0 (the same slow-path concern)
__device__ __forceinline__ double recip_pos(bool spos, double s) {
    double d = spos ? s : 1.0;
    asm("" : "+d"(d));
    const double q = 1.0 / d;
    return spos ? q : 0.0;
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
                g.sr = g.sr + sqrt_skel(ph);
            }
        }
    }
}

struct Coef {
    bool hb;
    double rb, spc, nif, agg, inv_ni, sl, sr;
};

// the column aggregates of update_kernel (_kernels.py:196-214)
__device__ __forceinline__ Coef make_coef(const Agg& g, const Cp& p, const double* recip) {
    Coef c;
    c.hb = (g.n > 0) && (g.first_row == 0);
    c.rb = c.hb ? sqrt_skel(g.phi0) : 0.0;
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

// one entry of update_kernel (_kernels.py:215-238); rj = sqrt(ph)
__device__ __forceinline__ double update_entry_sq(int r, double ph, double lh, double rj, const Coef& c,
                                                  const Cp& p, bool& nan) {
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

__device__ __forceinline__ double update_entry(int r, double ph, double lh, const Coef& c, const Cp& p,
                                               bool& nan) {
    return update_entry_sq(r, ph, lh, sqrt_skel(ph), c, p, nan);
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
__device__ __forceinline__ void process_window(Win<K>& w, const Cp& p, VRes& res, unsigned int& out_mask,
                                               const double* recip) {
    unsigned int skel_mask = 0;
    int n = 0;
    res.bad_phi_row = -1;
    res.bad_lt_row = -1;
#pragma unroll
    for (int i = 0; i < K; ++i) {
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
            sq[i] = sqrt_skel(ph);
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
    const double inv = recip_pos(spos, s);
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

// process_window<2> as straight-line code for a window of one or two rows:
// the same operations in the same order, so the result is bitwise identical.
// A single skeleton row takes the general arithmetic too: with finite inputs
// every term cancels exactly (the closed form), so no divergent shortcut is
// needed.  rows[1] is ignored when m == 1.
__device__ __forceinline__ void process_two(int m, int r0, int r1, double ph0, double lm0, double ph1, double lm1,
                                            const Cp& p, const double* recip, VRes& res, double& nv0,
                                            double& nv1, unsigned int& out_mask) {
    const bool h1 = m > 1;
    if (!h1) { ph1 = 0.0; lm1 = 0.0; }
    const bool in0 = in_skeleton(ph0, lm0);
    const bool in1 = h1 && in_skeleton(ph1, lm1);
    res.bad_phi_row = -1;
    res.bad_lt_row = -1;
    if (ph0 != 0.0 && !in0) res.bad_phi_row = r0;
    if (lm0 != 0.0 && !in0) res.bad_lt_row = r0;
    if (h1 && ph1 != 0.0 && !in1) res.bad_phi_row = r1;
    if (h1 && lm1 != 0.0 && !in1) res.bad_lt_row = r1;
    const int n = (int)in0 + (int)in1;
    res.nskel = n;
    out_mask = 0;
    nv0 = 0.0;
    nv1 = 0.0;
    if (n == 0) return;
    // aggregates over the skeleton rows in row order
    const double sq0 = in0 ? sqrt_skel(ph0) : 0.0;
    const double sq1 = in1 ? sqrt_skel(ph1) : 0.0;
    const double lh0 = (lm0 != 0.0) ? lm0 : 0.0;
    const double lh1 = (lm1 != 0.0) ? lm1 : 0.0;
    Agg g;
    agg_init(g);
    if (in0) { g.first_row = r0; g.phi0 = ph0; g.n = 1; g.sl = g.sl + lh0; g.sp = g.sp + ph0; g.sr = g.sr + sq0; }
    if (in1) {
        if (!in0) { g.first_row = r1; g.phi0 = ph1; }
        g.n += 1;
        g.sl = g.sl + lh1; g.sp = g.sp + ph1; g.sr = g.sr + sq1;
    }
    const Coef c = make_coef(g, p, recip);
    double v0 = 0.0, v1 = 0.0, s = 0.0;
    if (in0) { v0 = update_entry_sq(r0, ph0, lh0, sq0, c, p, res.nan); s = s + v0; }
    if (in1) { v1 = update_entry_sq(r1, ph1, lh1, sq1, c, p, res.nan); s = s + v1; }
    const bool spos = s > 0.0;
    const double inv = recip_pos(spos, s);
    if (in0) {
        const double nv = spos ? v0 * inv : v0;
        if (nv != 0.0) { res.cnt++; out_mask |= 1u; if (r0 == 0) res.bm = res.bm + nv; }
        const double dd = fabs(nv - ph0);
        if (dd > res.maxd) res.maxd = dd;
        nv0 = nv;
    }
    if (in1) {
        const double nv = spos ? v1 * inv : v1;
        if (nv != 0.0) { res.cnt++; out_mask |= 2u; if (r1 == 0) res.bm = res.bm + nv; }
        const double dd = fabs(nv - ph1);
        if (dd > res.maxd) res.maxd = dd;
        nv1 = nv;
    }
}

}  // namespace ft
