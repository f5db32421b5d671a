/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into, imported by, or
 * called from the product path (paper_1804_09152_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it, and only as the checker / CPU baseline.
 *
 * Plain-C restatement of one explicit Euler step of the layered field, in
 * float64, following the reference pipeline stage by stage for each vertex
 * column j (reference pkg/src/fieldtess/):
 *
 *   1. Lt(:,j) = sum_u PHI(:,u) * L^T(u,j): dense accumulator with stamps,
 *      first product assigned then +=, touched rows sorted, exact zeros
 *      dropped                               (_kernels.py:26-62)
 *   2. interest skeleton: sorted merge of PHI(:,j) and Lt(:,j); a row is
 *      kept if phi > 0, or phi == 0 / absent and lt > 0  (_kernels.py:96-150)
 *   3. expansion of PHI and Lt onto the skeleton; a nonzero outside the
 *      skeleton is a pattern violation        (_kernels.py:153-176)
 *   4. closed-form Euler update, NaN flag, clamp to [0, 1]
 *                                              (_kernels.py:179-238)
 *   5. column sum, v * (1/s), drop zeros, base mass, max |delta|
 *                                              (_kernels.py:241-282)
 *
 * Build with -ffp-contract=off (no FMA) so the arithmetic is the reference's
 * IEEE double sequence.  Columns are independent; an optional OpenMP
 * parallel-for over contiguous column chunks makes it usable as the
 * multi-core CPU baseline ("port").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int* stamp;      /* [n_rows], -1 = never touched */
    double* acc;     /* [n_rows] */
    int* touched;    /* [n_rows] */
    int* lt_rows;    /* [n_rows] */
    double* lt_vals; /* [n_rows] */
    int* sk_rows;    /* [n_rows] */
    double* phat;    /* [n_rows] */
    double* lhat;    /* [n_rows] */
    double* v;       /* [n_rows] */
    int* out_rows;   /* growable */
    double* out_vals;
    long long out_n, out_cap;
} scratch_t;

static int cmp_int(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

static void push_out(scratch_t* s, int r, double v) {
    if (s->out_n == s->out_cap) {
        s->out_cap = s->out_cap ? 2 * s->out_cap : 1024;
        s->out_rows = (int*)realloc(s->out_rows, s->out_cap * sizeof(int));
        s->out_vals = (double*)realloc(s->out_vals, s->out_cap * sizeof(double));
    }
    s->out_rows[s->out_n] = r;
    s->out_vals[s->out_n] = v;
    s->out_n++;
}

/* Process column j; appends its output entries to s->out_*.  Returns the
 * count, writes per-column diagnostics. */
static int column_step(int j, int n_rows, const int* lt_ptr, const int* lt_idx,
                       const double* lt_val, const int* p_ptr, const int* p_idx,
                       const double* p_val, const double* prm, scratch_t* s,
                       double* bm_out, double* delta_out, int* nan_out,
                       int* bad_phi_row, int* bad_lt_row, int* nskel_out) {
    const double w = prm[0], a = prm[1], e = prm[2], e_base = prm[3], mu = prm[4], dt = prm[5];
    (void)n_rows;
    /* 1. SpGEMM column */
    int k = 0;
    for (int p = lt_ptr[j]; p < lt_ptr[j + 1]; ++p) {
        int u = lt_idx[p];
        double bv = lt_val[p];
        for (int q = p_ptr[u]; q < p_ptr[u + 1]; ++q) {
            int r = p_idx[q];
            if (s->stamp[r] != j) {
                s->stamp[r] = j;
                s->acc[r] = p_val[q] * bv;
                s->touched[k++] = r;
            } else {
                s->acc[r] += p_val[q] * bv;
            }
        }
    }
    qsort(s->touched, (size_t)k, sizeof(int), cmp_int);
    int nl = 0;
    for (int t = 0; t < k; ++t) {
        int r = s->touched[t];
        double v = s->acc[r];
        if (v != 0.0) { s->lt_rows[nl] = r; s->lt_vals[nl] = v; nl++; }
    }
    /* 2. skeleton by sorted merge; 3. expansion of PHI and Lt */
    int a0 = p_ptr[j], ae = p_ptr[j + 1], b0 = 0, n = 0;
    *bad_phi_row = -1;
    *bad_lt_row = -1;
    while (a0 < ae || b0 < nl) {
        int take_a = 0, take_b = 0;
        if (b0 >= nl || (a0 < ae && p_idx[a0] < s->lt_rows[b0])) take_a = 1;
        else if (a0 >= ae || s->lt_rows[b0] < p_idx[a0]) take_b = 1;
        else take_a = take_b = 1;
        int r = take_a ? p_idx[a0] : s->lt_rows[b0];
        double ph = take_a ? p_val[a0] : 0.0;
        double lt = take_b ? s->lt_vals[b0] : 0.0;
        int keep;
        if (take_a && take_b) keep = (ph > 0.0) || (ph == 0.0 && lt > 0.0);
        else if (take_a) keep = ph > 0.0;
        else keep = lt > 0.0;
        if (keep) {
            s->sk_rows[n] = r; s->phat[n] = ph; s->lhat[n] = lt; n++;
        } else {
            if (take_a && ph != 0.0) *bad_phi_row = r;
            if (take_b && lt != 0.0) *bad_lt_row = r;
        }
        if (take_a) a0++;
        if (take_b) b0++;
    }
    *nskel_out = n;
    *nan_out = 0;
    *bm_out = 0.0;
    *delta_out = 0.0;
    if (n == 0) return 0;
    /* 4. update */
    double sl = 0.0, sp = 0.0, sr = 0.0;
    for (int p = 0; p < n; ++p) {
        sl += s->lhat[p];
        sp += s->phat[p];
        sr += sqrt(s->phat[p]);
    }
    int has_base = s->sk_rows[0] == 0;
    double rb = has_base ? sqrt(s->phat[0]) : 0.0;
    double sp_cells = has_base ? sp - s->phat[0] : sp;
    int n_cells = has_base ? n - 1 : n;
    double inv_ni = 1.0 / (double)n;
    double nif = (double)n;
    double mx = (double)n_cells - 1.0;
    double agg_w = w * (mx > 0.0 ? mx : 0.0) * sp_cells;
    if (has_base) agg_w += w * sp_cells;
    double agg = 0.5 * a * (nif - 1.0) * sl + agg_w;
    for (int p = 0; p < n; ++p) {
        double phi_j = s->phat[p];
        double rj = sqrt(phi_j);
        double al_j = a * (sl - s->lhat[p]);
        double w_j, eterm;
        if (s->sk_rows[p] == 0) {
            w_j = w * sp_cells;
            eterm = -e_base * rj * (sr - rj);
        } else {
            w_j = w * (sp_cells - phi_j);
            if (has_base) eterm = rj * (e * (sr - rj - rb) + e_base * rb);
            else eterm = rj * e * (sr - rj);
        }
        double pair_sum = nif * (0.5 * al_j + w_j) - agg;
        double d = -mu * inv_ni * (pair_sum - eterm);
        double v = phi_j + d * dt;
        if (v != v) { *nan_out = 1; v = phi_j; }
        if (v > 1.0) v = 1.0;
        else if (v <= 0.0) v = 0.0;
        s->v[p] = v;
    }
    /* 5. normalise + compact */
    double sum = 0.0;
    for (int p = 0; p < n; ++p) sum += s->v[p];
    double inv = sum > 0.0 ? 1.0 / sum : 0.0;
    double bm = 0.0, maxd = 0.0;
    int cnt = 0;
    for (int p = 0; p < n; ++p) {
        double nv = sum > 0.0 ? s->v[p] * inv : s->v[p];
        if (nv != 0.0) {
            push_out(s, s->sk_rows[p], nv);
            if (s->sk_rows[p] == 0) bm += nv;
            cnt++;
        }
        double dd = fabs(nv - s->phat[p]);
        if (dd > maxd) maxd = dd;
    }
    *bm_out = bm;
    *delta_out = maxd;
    return cnt;
}

/*
 * One step.  Returns 0 on success, 3 if out_cap is too small (out_ptr is
 * still filled so the caller can read the needed size from out_ptr[n_v]).
 * diag[0] = first NaN column or -1; diag[1] = first column with a PHI
 * pattern violation or -1, diag[2] its row; diag[3] = first column with an
 * Lt violation or -1, diag[4] its row; diag[5] = skeleton nnz.
 * bm_col / delta_col: per-column base mass and max |delta| (the host does
 * the final numpy sum / max exactly as field.py:270-271).
 */
int ft_oracle_step(int n_rows, int n_v, const int* lt_ptr, const int* lt_idx,
                   const double* lt_val, const int* p_ptr, const int* p_idx,
                   const double* p_val, int* out_ptr, int* out_idx, double* out_val,
                   long long out_cap, const double* prm, double* bm_col,
                   double* delta_col, long long* diag, int n_threads) {
    int nt = 1;
#ifdef _OPENMP
    nt = n_threads > 0 ? n_threads : omp_get_max_threads();
#else
    (void)n_threads;
#endif
    if (nt > n_v && n_v > 0) nt = n_v;
    if (nt < 1) nt = 1;
    int* counts = (int*)malloc(sizeof(int) * (size_t)(n_v > 0 ? n_v : 1));
    int* nanc = (int*)malloc(sizeof(int) * (size_t)(n_v > 0 ? n_v : 1));
    int* badp = (int*)malloc(sizeof(int) * (size_t)(n_v > 0 ? n_v : 1));
    int* badl = (int*)malloc(sizeof(int) * (size_t)(n_v > 0 ? n_v : 1));
    int* nsk = (int*)malloc(sizeof(int) * (size_t)(n_v > 0 ? n_v : 1));
    scratch_t* sc = (scratch_t*)calloc((size_t)nt, sizeof(scratch_t));
    long long* chunk_base = (long long*)calloc((size_t)nt + 1, sizeof(long long));
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        scratch_t* s = &sc[t];
        size_t nr = (size_t)(n_rows > 0 ? n_rows : 1);
        s->stamp = (int*)malloc(nr * sizeof(int));
        for (size_t r = 0; r < nr; ++r) s->stamp[r] = -1;
        s->acc = (double*)malloc(nr * sizeof(double));
        s->touched = (int*)malloc(nr * sizeof(int));
        s->lt_rows = (int*)malloc(nr * sizeof(int));
        s->lt_vals = (double*)malloc(nr * sizeof(double));
        s->sk_rows = (int*)malloc(nr * sizeof(int));
        s->phat = (double*)malloc(nr * sizeof(double));
        s->lhat = (double*)malloc(nr * sizeof(double));
        s->v = (double*)malloc(nr * sizeof(double));
        long long j0 = (long long)n_v * t / nt, j1 = (long long)n_v * (t + 1) / nt;
        for (long long j = j0; j < j1; ++j) {
            counts[j] = column_step((int)j, n_rows, lt_ptr, lt_idx, lt_val, p_ptr, p_idx, p_val,
                                    prm, s, &bm_col[j], &delta_col[j], &nanc[j], &badp[j],
                                    &badl[j], &nsk[j]);
        }
    }
    /* prefix sum -> out_ptr; chunk t's entries are contiguous */
    long long acc = 0;
    out_ptr[0] = 0;
    for (int j = 0; j < n_v; ++j) {
        acc += counts[j];
        out_ptr[j + 1] = (int)acc;
    }
    int rc = acc > out_cap ? 3 : 0;
    if (rc == 0) {
        for (int t = 0; t < nt; ++t) {
            long long j0 = (long long)n_v * t / nt;
            long long base = out_ptr[j0];
            memcpy(out_idx + base, sc[t].out_rows, (size_t)sc[t].out_n * sizeof(int));
            memcpy(out_val + base, sc[t].out_vals, (size_t)sc[t].out_n * sizeof(double));
        }
    }
    diag[0] = diag[1] = diag[2] = diag[3] = diag[4] = -1;
    diag[5] = 0;
    for (int j = 0; j < n_v; ++j) {
        diag[5] += nsk[j];
        if (diag[0] < 0 && nanc[j]) diag[0] = j;
        if (diag[1] < 0 && badp[j] >= 0) { diag[1] = j; diag[2] = badp[j]; }
        if (diag[3] < 0 && badl[j] >= 0) { diag[3] = j; diag[4] = badl[j]; }
    }
    for (int t = 0; t < nt; ++t) {
        free(sc[t].stamp); free(sc[t].acc); free(sc[t].touched); free(sc[t].lt_rows);
        free(sc[t].lt_vals); free(sc[t].sk_rows); free(sc[t].phat); free(sc[t].lhat);
        free(sc[t].v); free(sc[t].out_rows); free(sc[t].out_vals);
    }
    free(sc); free(chunk_base); free(counts); free(nanc); free(badp); free(badl); free(nsk);
    return rc;
}
