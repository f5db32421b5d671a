"""ORACLE (test infrastructure only) -- Python restatements of the hot path.

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/fieldtess/``).  Plain numpy / Python loops: use
for small meshes only, or go through :func:`step_c` (the C restatement).
"""

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


# ---------------------------------------------------------------------------
# plain CSC triple helpers


class Csc:
    """Minimal host CSC (int32 indices, float64 values) for the oracle."""

    def __init__(self, n_rows, n_cols, col_ptr, row_idx, values):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int32)
        nnz = int(self.col_ptr[-1]) if self.col_ptr.size else 0
        self.row_idx = np.ascontiguousarray(row_idx[:nnz], dtype=np.int32)
        self.values = np.ascontiguousarray(values[:nnz], dtype=np.float64)

    @classmethod
    def of(cls, m):
        return cls(m.n_rows, m.n_cols, m.col_ptr, m.row_idx, m.values)

    @property
    def nnz(self):
        return int(self.col_ptr[-1])

    def column(self, j):
        a, b = self.col_ptr[j], self.col_ptr[j + 1]
        return self.row_idx[a:b], self.values[a:b]

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        cols = np.repeat(np.arange(self.n_cols), np.diff(self.col_ptr))
        out[self.row_idx, cols] = self.values
        return out


# ---------------------------------------------------------------------------
# the step, literal per-column restatement (field.py:198-286)


def step_py(phi, lap_t, params):
    """One Euler step by a literal per-column loop.

    ``phi``: (n_rows, n_v) CSC, ``lap_t``: L^T in CSC (= reference
    ``lap.mat_t``), ``params``: object with w, a, e, e_base, mu, dt.
    Returns ``(Csc, stats)`` where stats has max_delta, base_mass,
    nnz_skel, nan_col, bad_phi (col,row) and bad_lt (col,row).
    """
    phi = Csc.of(phi)
    lap_t = Csc.of(lap_t)
    w, a, e, eb, mu, dt = (float(params.w), float(params.a), float(params.e),
                           float(params.e_base), float(params.mu),
                           float(params.dt))
    n_v = phi.n_cols
    out_cols = []
    bm_col = np.zeros(n_v)
    deltas = np.zeros(n_v)
    nan_col = bad_phi = bad_lt = None
    nnz_skel = 0
    for j in range(n_v):
        # Lt(:, j): _kernels.py:36-62 -- first product assigned, then +=
        acc = {}
        us, bvs = lap_t.column(j)
        for u, bv in zip(us.tolist(), bvs.tolist()):
            rows, vals = phi.column(u)
            for r, pv in zip(rows.tolist(), vals.tolist()):
                if r in acc:
                    acc[r] = acc[r] + pv * bv
                else:
                    acc[r] = pv * bv
        lt = {r: v for r, v in acc.items() if v != 0.0}
        prow, pval = phi.column(j)
        pcol = dict(zip(prow.tolist(), pval.tolist()))
        # skeleton + expansion: _kernels.py:96-176
        skel = []
        for r in sorted(set(pcol) | set(lt)):
            ph = pcol.get(r)
            lv = lt.get(r)
            if ph is not None and lv is not None:
                keep = ph > 0.0 or (ph == 0.0 and lv > 0.0)
            elif ph is not None:
                keep = ph > 0.0
            else:
                keep = lv > 0.0
            if keep:
                skel.append((r, ph if ph is not None else 0.0,
                             lv if lv is not None else 0.0))
            else:
                if ph is not None and ph != 0.0:
                    bad_phi = bad_phi if bad_phi and bad_phi[0] < j else (j, r)
                if lv is not None and lv != 0.0:
                    bad_lt = bad_lt if bad_lt and bad_lt[0] < j else (j, r)
        nnz_skel += len(skel)
        ni = len(skel)
        if ni == 0:
            out_cols.append([])
            continue
        # update: _kernels.py:195-238
        sl = sp = sr = 0.0
        for _, ph, lv in skel:
            sl += lv
            sp += ph
            sr += math.sqrt(ph)
        has_base = skel[0][0] == 0
        rb = math.sqrt(skel[0][1]) if has_base else 0.0
        sp_cells = sp - skel[0][1] if has_base else sp
        n_cells = ni - 1 if has_base else ni
        inv_ni = 1.0 / ni
        nif = float(ni)
        agg_w = w * max(n_cells - 1.0, 0.0) * sp_cells
        if has_base:
            agg_w += w * sp_cells
        agg = 0.5 * a * (nif - 1.0) * sl + agg_w
        vs = []
        for r, ph, lv in skel:
            rj = math.sqrt(ph)
            al_j = a * (sl - lv)
            if r == 0:
                w_j = w * sp_cells
                eterm = -eb * rj * (sr - rj)
            else:
                w_j = w * (sp_cells - ph)
                if has_base:
                    eterm = rj * (e * (sr - rj - rb) + eb * rb)
                else:
                    eterm = rj * e * (sr - rj)
            pair_sum = nif * (0.5 * al_j + w_j) - agg
            d = -mu * inv_ni * (pair_sum - eterm)
            v = ph + d * dt
            if v != v:
                if nan_col is None:
                    nan_col = j
                v = ph
            if v > 1.0:
                v = 1.0
            elif v <= 0.0:
                v = 0.0
            vs.append(v)
        # normalise + compact: _kernels.py:241-282
        s = 0.0
        for v in vs:
            s += v
        inv = 1.0 / s if s > 0.0 else 0.0
        col = []
        bm = maxd = 0.0
        for (r, ph, _), v in zip(skel, vs):
            nv = v * inv if s > 0.0 else v
            if nv != 0.0:
                col.append((r, nv))
                if r == 0:
                    bm += nv
            dd = abs(nv - ph)
            if dd > maxd:
                maxd = dd
        bm_col[j] = bm
        deltas[j] = maxd
        out_cols.append(col)
    counts = np.array([len(c) for c in out_cols], dtype=np.int64)
    col_ptr = np.zeros(n_v + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    rows = np.array([r for c in out_cols for r, _ in c], dtype=np.int32)
    vals = np.array([v for c in out_cols for _, v in c], dtype=np.float64)
    stats = {
        "max_delta": float(deltas.max()) if n_v else 0.0,
        "base_mass": float(bm_col.sum()),          # field.py:270 (numpy sum)
        "nnz_skel": nnz_skel,
        "nan_col": nan_col,
        "bad_phi": bad_phi,
        "bad_lt": bad_lt,
    }
    return Csc(phi.n_rows, n_v, col_ptr, rows, vals), stats


# ---------------------------------------------------------------------------
# the C restatement (ft_oracle.c) through ctypes


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libft_oracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", _HERE, "libft_oracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        lib = ctypes.CDLL(path)
        p = ctypes.c_void_p
        lib.ft_oracle_step.argtypes = [ctypes.c_int, ctypes.c_int, p, p, p, p, p, p,
                                       p, p, p, ctypes.c_longlong, p, p, p, p,
                                       ctypes.c_int]
        lib.ft_oracle_step.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def step_c(phi, lap_t, params, n_threads=1):
    """One Euler step through the C restatement.  Same return as step_py."""
    phi = Csc.of(phi)
    lap_t = Csc.of(lap_t)
    n_v = phi.n_cols
    prm = np.array([params.w, params.a, params.e, params.e_base, params.mu,
                    params.dt], dtype=np.float64)
    cap = max(16, 8 * phi.nnz + 8 * n_v)
    out_ptr = np.zeros(n_v + 1, dtype=np.int32)
    out_idx = np.empty(cap, dtype=np.int32)
    out_val = np.empty(cap, dtype=np.float64)
    bm_col = np.zeros(max(n_v, 1))
    delta_col = np.zeros(max(n_v, 1))
    diag = np.zeros(6, dtype=np.int64)
    lp, li, lv = lap_t.col_ptr, lap_t.row_idx, lap_t.values
    pp, pi, pv = phi.col_ptr, phi.row_idx, phi.values
    rc = _lib().ft_oracle_step(phi.n_rows, n_v, _ptr(lp), _ptr(li), _ptr(lv),
                               _ptr(pp), _ptr(pi), _ptr(pv), _ptr(out_ptr),
                               _ptr(out_idx), _ptr(out_val), cap, _ptr(prm),
                               _ptr(bm_col), _ptr(delta_col), _ptr(diag),
                               int(n_threads))
    if rc != 0:
        raise RuntimeError(f"oracle capacity {cap} too small")
    stats = {
        "max_delta": float(delta_col[:n_v].max()) if n_v else 0.0,
        "base_mass": float(bm_col[:n_v].sum()),
        "nnz_skel": int(diag[5]),
        "nan_col": None if diag[0] < 0 else int(diag[0]),
        "bad_phi": None if diag[1] < 0 else (int(diag[1]), int(diag[2])),
        "bad_lt": None if diag[3] < 0 else (int(diag[3]), int(diag[4])),
    }
    return Csc(phi.n_rows, n_v, out_ptr, out_idx, out_val), stats


def evolve_c(phi, lap_t, params, n_steps, n_threads=1):
    """``n_steps`` fixed steps through the C restatement; returns the field
    after each step is not kept -- only the final field and stats list."""
    cur = Csc.of(phi)
    trace = []
    for _ in range(n_steps):
        cur, st = step_c(cur, lap_t, params, n_threads=n_threads)
        if st["nan_col"] is not None or st["bad_phi"] or st["bad_lt"]:
            raise RuntimeError(f"oracle step failed: {st}")
        trace.append(st)
    return cur, trace


# ---------------------------------------------------------------------------
# labels (field.py:324-356) and seeding (field.py:137-166)


def labels_np(phi):
    """Argmax cell per column, ties -> lowest cell, base wins only if
    strictly greater (UNCLAIMED = -1).  Literal per-column loop."""
    phi = Csc.of(phi)
    out = np.full(phi.n_cols, -1, dtype=np.int64)
    for j in range(phi.n_cols):
        rows, vals = phi.column(j)
        base = 0.0
        best_val = None
        best_row = None
        for r, v in zip(rows.tolist(), vals.tolist()):
            if r == 0:
                base = v
            elif best_val is None or v > best_val:
                best_val, best_row = v, r
        best = best_val if best_val is not None else 0.0
        if best_row is not None:
            out[j] = best_row - 1
        if base > best:
            out[j] = -1
    return out


def init_field_np(neighbor_ptr, neighbor_idx, n_v, seeds):
    """Seed claims: each seed claims itself plus its one-ring, shared claims
    split 1/count, base 1.0 on unclaimed vertices (field.py:137-166)."""
    seeds = np.asarray(seeds, dtype=np.int64)
    cols = {}
    for k, s in enumerate(seeds.tolist()):
        claimed = [s] + neighbor_idx[neighbor_ptr[s]:neighbor_ptr[s + 1]].tolist()
        for v in claimed:
            cols.setdefault(v, []).append(k + 1)
    col_ptr = [0]
    rows, vals = [], []
    for v in range(n_v):
        cl = cols.get(v)
        if not cl:
            rows.append(0)
            vals.append(1.0)
        else:
            for r in sorted(cl):
                rows.append(r)
                vals.append(1.0 / len(cl))
        col_ptr.append(len(rows))
    return Csc(seeds.size + 1, n_v, np.array(col_ptr), np.array(rows),
               np.array(vals))


# ---------------------------------------------------------------------------
# Lloyd: faces per layer row (lloyd.py:21-28 via sparse.spgemm)


def faces_by_cell_np(phi, faces):
    """Pattern and values of M^T Phi^T: face f in row r when the sum over
    its vertices (ascending) of PHI(r, v) is nonzero; rows of the result are
    the layer rows (including the base row 0), faces ascending.  Literal
    per-face loop."""
    phi = Csc.of(phi)
    n_f = faces.shape[0]
    per_row = {}
    for f in range(n_f):
        acc = {}
        for v in sorted(int(x) for x in faces[f]):
            rows, vals = phi.column(v)
            for r, x in zip(rows.tolist(), vals.tolist()):
                acc[r] = acc[r] + x if r in acc else x
        for r, x in acc.items():
            if x != 0.0:
                per_row.setdefault(r, []).append((f, x))
    ptr = [0]
    idx, val = [], []
    for r in range(phi.n_rows):
        for f, x in per_row.get(r, []):
            idx.append(f)
            val.append(x)
        ptr.append(len(idx))
    return np.array(ptr, dtype=np.int32), np.array(idx, dtype=np.int32), np.array(val)


# ---------------------------------------------------------------------------
# dual: boolean products, crossing tests, junction triples (dual.py:60-233)


def dual_products_np(phi, faces, face_area, threshold):
    """Literal restatement: A_v pairs, A_t pairs, A_t pairs whose isolines
    cross in some shared positive-area face, and junction triples."""
    phi = Csc.of(phi)
    n_v = phi.n_cols
    cells_of_v = []
    for v in range(n_v):
        rows, vals = phi.column(v)
        cells_of_v.append(sorted(int(r) - 1 for r, x in zip(rows, vals) if r >= 1 and x >= threshold))
    pv, pt, px, tri = set(), set(), set(), set()
    for cl in cells_of_v:
        for a in range(len(cl)):
            for b in range(a + 1, len(cl)):
                pv.add((cl[a], cl[b]))
    emb = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])

    def seg(values):
        rel = values - threshold
        pts = []
        for a, b in ((0, 1), (1, 2), (2, 0)):
            if rel[a] * rel[b] < 0.0:
                s = rel[a] / (rel[a] - rel[b])
                if not np.isfinite(s):
                    return None
                pts.append(emb[a] + s * (emb[b] - emb[a]))
        return pts if len(pts) == 2 else None

    def orient(a, b, c):
        d = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
        return int(d > 0.0) - int(d < 0.0)

    def onseg(a, b, c):
        return min(a[0], b[0]) <= c[0] <= max(a[0], b[0]) and min(a[1], b[1]) <= c[1] <= max(a[1], b[1])

    def inter(p, q):
        o1, o2, o3, o4 = orient(p[0], p[1], q[0]), orient(p[0], p[1], q[1]), orient(q[0], q[1], p[0]), orient(q[0], q[1], p[1])
        return ((o1 != o2 and o3 != o4) or (o1 == 0 and onseg(p[0], p[1], q[0])) or (o2 == 0 and onseg(p[0], p[1], q[1]))
                or (o3 == 0 and onseg(q[0], q[1], p[0])) or (o4 == 0 and onseg(q[0], q[1], p[1])))

    def get(r, v):
        rows, vals = phi.column(v)
        k = np.searchsorted(rows, r)
        return float(vals[k]) if k < rows.size and rows[k] == r else 0.0

    for f in range(faces.shape[0]):
        cl = sorted(set(c for v in faces[f] for c in cells_of_v[int(v)]))
        for a in range(len(cl)):
            for b in range(a + 1, len(cl)):
                pt.add((cl[a], cl[b]))
                if face_area[f] > 0.0:
                    vi = np.array([get(cl[a] + 1, int(v)) for v in faces[f]])
                    vj = np.array([get(cl[b] + 1, int(v)) for v in faces[f]])
                    si, sj = seg(vi), seg(vj)
                    if si is not None and sj is not None and inter(si, sj):
                        px.add((cl[a], cl[b]))
                for c in range(b + 1, len(cl)):
                    tri.add((cl[a], cl[b], cl[c]))
    return sorted(pv), sorted(pt), sorted(px), sorted(tri)
