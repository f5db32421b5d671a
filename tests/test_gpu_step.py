"""Parity of the CUDA hot path (through the public API -> C-ABI) against the
reference's golden vectors and the C oracle.  EXACT mode must be bitwise."""

import numpy as np
import pytest

import paper_1804_09152_b200 as ft
from conftest import P, assert_csc_equal, csc_from, golden_npz
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

DEFAULT = ft.CouplingParams()


def as_sparse(c):
    return ft.SparseMat(c.n_rows, c.n_cols, c.col_ptr, c.row_idx, c.values, check=False)


class _Lap:
    """Minimal Laplacian-like object (duck-typed like the reference's)."""

    def __init__(self, lapt):
        self.mat_t = as_sparse(lapt)
        self.mat = ft.transpose(self.mat_t)
        self.scheme = "given"


@pytest.fixture(scope="module")
def cases():
    return golden_npz("step_cases.npz")


def test_step_cases_bitwise(cases):
    for name in cases["names"]:
        prm = ft.CouplingParams(*[float(x) for x in cases[f"{name}_params"]])
        inp = csc_from(cases, f"{name}_in")
        fld = ft.LayeredField(as_sparse(inp), np.arange(inp.n_rows - 1))
        out, st = ft.step(fld, _Lap(csc_from(cases, f"{name}_lapt")), prm)
        assert_csc_equal(out.phi, csc_from(cases, f"{name}_out"))
        ref = cases[f"{name}_stats"]
        assert st.max_delta == ref[0], name
        assert abs(st.base_mass - ref[1]) <= 1e-12 * max(1.0, abs(ref[1])), name
        assert st.nnz_phi == ref[2]


def test_multi_step_with_workspace(cases):
    inp = csc_from(cases, "multi_in")
    lap = _Lap(csc_from(cases, "multi_lapt"))
    cur = ft.LayeredField(as_sparse(inp), [20, 60])
    ws = ft.StepWorkspace()
    for _ in range(5):
        cur, _ = ft.step(cur, lap, DEFAULT, workspace=ws)
    assert_csc_equal(cur.phi, csc_from(cases, "multi_out"))


@pytest.mark.parametrize("traj", ["c1_traj.npz", "torus_traj.npz"])
def test_trajectory_bitwise_device_evolve(traj):
    t = golden_npz(traj)
    lap = _Lap(csc_from(t, "lapt"))
    cur = ft.LayeredField(as_sparse(csc_from(t, "s0")), t["seeds"])
    prev = 0
    all_stats = []
    for k in t["snaps"][1:]:
        cur, trace = ft.evolve(cur, lap, DEFAULT, max_steps=int(k) - prev, tol=0.0)
        assert len(trace) == int(k) - prev
        all_stats += trace
        prev = int(k)
        assert cur.step_count == prev
        assert_csc_equal(cur.phi, csc_from(t, f"s{k}"))
    tr = t["trace"]
    for k, st in enumerate(all_stats):
        assert st.max_delta == tr[k, 0] and st.nnz_phi == tr[k, 2], k
        assert abs(st.base_mass - tr[k, 1]) <= 1e-12 * max(1.0, tr[k, 1]), k
    assert np.array_equal(ft.sharp_labels(cur), t["labels_final"])


def test_trajectory_bitwise_step_loop():
    t = golden_npz("c1_traj.npz")
    lap = _Lap(csc_from(t, "lapt"))
    cur = ft.LayeredField(as_sparse(csc_from(t, "s0")), t["seeds"])
    ws = ft.StepWorkspace()
    for k in range(1, 101):
        cur, st = ft.step(cur, lap, DEFAULT, workspace=ws)
        assert st.nnz_phi == t["trace"][k - 1, 2]
        if k in t["snaps"]:
            assert_csc_equal(cur.phi, csc_from(t, f"s{k}"))


def test_generated_mesh_and_seeding_end_to_end():
    """Product generators + seeding + device evolve == C oracle, bitwise."""
    mesh = ft.gen_periodic_grid(200, 150)
    lap = ft.build_laplacian(mesh)
    rng = np.random.default_rng(3)
    seeds = rng.choice(mesh.n_vertices, size=120, replace=False)
    fld = ft.init_field(mesh, seeds)
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=40, tol=0.0)
    ref, rtrace = po.evolve_c(po.Csc.of(fld.phi), po.Csc.of(lap.mat_t), DEFAULT, 40, n_threads=4)
    assert_csc_equal(out.phi, ref)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]


@pytest.mark.parametrize("subdiv,n_seeds", [(4, 64), (3, 64), (3, 160)])
def test_high_band_density_all_tiers(subdiv, n_seeds):
    """Dense bands (many columns with > 2 entries per neighbour and > 8 rows
    in the union) route most columns through tiers 2 and 3; bitwise against
    the C oracle, through the device evolve and the step loop."""
    mesh = ft.gen_icosphere(subdiv)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(0).choice(mesh.n_vertices, n_seeds, replace=False)
    fld = ft.init_field(mesh, seeds)
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=40, tol=0.0)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, rtrace = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 40, n_threads=4)
    assert_csc_equal(out.phi, ref)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]
    cur = fld
    for _ in range(12):
        cur, _st = ft.step(cur, lap, DEFAULT)
    ref12, _ = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 12, n_threads=4)
    assert_csc_equal(cur.phi, ref12)


def test_fast_mode_single_step_tolerance():
    """FAST (fp32 storage) from identical inputs: |d| <= 1e-5|ref| + 2e-7."""
    t = golden_npz("c1_traj.npz")
    lap = _Lap(csc_from(t, "lapt"))
    for k in (10, 100):
        inp = csc_from(t, f"s{k}")
        f32 = ft.LayeredField(as_sparse(inp), t["seeds"], precision="fast")
        out, _ = ft.step(f32, lap, DEFAULT)
        # oracle fed the same fp32-rounded input
        rounded = po.Csc(inp.n_rows, inp.n_cols, inp.col_ptr, inp.row_idx,
                         inp.values.astype(np.float32).astype(np.float64))
        ref, _ = po.step_c(rounded, csc_from(t, "lapt"), DEFAULT)
        got = out.phi.to_dense()
        want = ref.to_dense()
        assert np.all(np.abs(got - want) <= 1e-5 * np.abs(want) + 2e-7)


def test_fast_mode_trajectory_labels():
    t = golden_npz("c1_traj.npz")
    lap = _Lap(csc_from(t, "lapt"))
    cur = ft.LayeredField(as_sparse(csc_from(t, "s0")), t["seeds"], precision="fast")
    cur, _ = ft.evolve(cur, lap, DEFAULT, max_steps=500, tol=0.0)
    agree = np.mean(ft.sharp_labels(cur) == t["labels_final"])
    assert agree >= 0.9999


def test_labels_golden():
    g = golden_npz("labels.npz")
    for name in g["names"]:
        c = csc_from(g, name)
        fld = ft.LayeredField(as_sparse(c), np.arange(c.n_rows - 1))
        assert np.array_equal(ft.sharp_labels(fld), g[f"{name}_labels"]), name


def test_numerical_blowup_reported():
    mesh = ft.gen_periodic_grid(9, 9)
    fld = ft.init_field(mesh, [40])
    with pytest.raises(ft.errors.NumericalBlowupError, match="numerical-blowup") as ei:
        ft.step(fld, ft.build_laplacian(mesh), ft.CouplingParams(a=float("inf")))
    ref_cols = []
    out, st = po.step_c(po.Csc.of(fld.phi), po.Csc.of(ft.build_laplacian(mesh).mat_t),
                        ft.CouplingParams(a=float("inf")))
    assert ei.value.column == st["nan_col"] and ei.value.step == 1
    del ref_cols, out


def test_pattern_violation_reported():
    mesh = ft.gen_periodic_grid(6, 6)
    dense = np.zeros((2, 36))
    dense[0] = 1.0
    dense[1, 5] = -0.25
    fld = ft.LayeredField(ft.SparseMat.from_dense(dense), [5])
    with pytest.raises(ft.errors.PatternViolationError, match="pattern-violation"):
        ft.step(fld, ft.build_laplacian(mesh), DEFAULT)


def test_overflow_regrows_and_matches(monkeypatch):
    """A deliberately tiny output buffer must be grown and the step redone."""
    from paper_1804_09152_b200 import field as fmod
    monkeypatch.setattr(fmod, "_initial_capacity", lambda d: 8)
    t = golden_npz("c1_traj.npz")
    lap = _Lap(csc_from(t, "lapt"))
    inp = as_sparse(csc_from(t, "s10"))
    fld = ft.LayeredField(inp, t["seeds"], step_count=10)
    out, st = ft.step(fld, lap, DEFAULT)
    assert st.realloc_count >= 1
    ref, _ = po.step_c(po.Csc.of(inp), csc_from(t, "lapt"), DEFAULT)
    assert_csc_equal(out.phi, ref)
    # and inside the device evolve loop
    out2, trace = ft.evolve(fld, lap, DEFAULT, max_steps=20, tol=0.0)
    ref2, _ = po.evolve_c(po.Csc.of(inp), csc_from(t, "lapt"), DEFAULT, 20)
    assert_csc_equal(out2.phi, ref2)


def test_tiled_pool_overflow_regrows(monkeypatch):
    """Tiles whose entries exceed their slot go to the pool; an empty pool
    must overflow, be grown, and the result still match bitwise."""
    from paper_1804_09152_b200 import field as fmod
    monkeypatch.setattr(fmod, "POOL_FRACTION", 0.0)
    monkeypatch.setattr(fmod, "POOL_MIN", 0)
    g = golden_npz("step_cases.npz")
    inp = csc_from(g, "wide12_in")
    lap = _Lap(csc_from(g, "wide12_lapt"))
    fld = ft.LayeredField(as_sparse(inp), np.arange(inp.n_rows - 1))
    out, st = ft.step(fld, lap, DEFAULT)
    assert st.realloc_count >= 1
    assert_csc_equal(out.phi, csc_from(g, "wide12_out"))
    out2, trace = ft.evolve(fld, lap, DEFAULT, max_steps=6, tol=0.0)
    ref2, _ = po.evolve_c(po.Csc.of(inp), csc_from(g, "wide12_lapt"), DEFAULT, 6)
    assert_csc_equal(out2.phi, ref2)


def test_pool_overflow_late_in_evolve_restarts_from_last_good(monkeypatch):
    """A pool overflow at a step >= 2 inside the device evolve loop: the
    failed step's later launches are no-ops, the host grows the buffers and
    continues from the last good field; the result equals the oracle
    bitwise (the field two steps back is never overwritten early)."""
    from paper_1804_09152_b200 import field as fmod
    monkeypatch.setattr(fmod, "POOL_FRACTION", 0.0)
    monkeypatch.setattr(fmod, "POOL_MIN", 0)
    mesh = ft.gen_icosphere(3)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(26).choice(mesh.n_vertices, 6, replace=False)
    fld = ft.init_field(mesh, seeds)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, rtrace = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 30)
    s2, _ = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 2)
    s3, _ = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 3)
    # at most two entries per column through step 2: the first pool column
    # (and so the overflow) appears at step 3
    assert np.diff(s2.col_ptr).max() <= 2 < np.diff(s3.col_ptr).max()
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=30, tol=0.0)
    assert trace[-1].realloc_count >= 1
    assert len(trace) == 30 and out.step_count == 30
    assert_csc_equal(out.phi, ref)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]
    assert [s.nnz_skel for s in trace] == [s["nnz_skel"] for s in rtrace]
    assert all(abs(s.base_mass - r["base_mass"]) <= 1e-12 * max(1.0, r["base_mass"]) for s, r in zip(trace, rtrace))


def test_active_set_matches_full_recomputation(monkeypatch):
    """Active-set stepping (the default on symmetric Laplacians) against
    every step recomputed in full (FT_LAP_SYMMETRIC off): identical fields
    and statistics over 120 steps of a 120x100 torus."""
    from paper_1804_09152_b200 import field as fmod
    mesh = ft.gen_periodic_grid(120, 100)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(9).choice(mesh.n_vertices, 60, replace=False)
    fld = ft.init_field(mesh, seeds)
    a, ta = ft.evolve(fld, lap, DEFAULT, max_steps=120, tol=0.0)
    monkeypatch.setattr(fmod, "ACTIVE_SET", False)
    b, tb = ft.evolve(fld, lap, DEFAULT, max_steps=120, tol=0.0)
    assert_csc_equal(a.phi, po.Csc.of(b.phi))
    for x, y in zip(ta, tb):
        assert (x.max_delta, x.nnz_phi, x.nnz_skel, x.base_mass) == (y.max_delta, y.nnz_phi, y.nnz_skel,
                                                                      y.base_mass)


def test_converged_input_returns_after_one_step():
    mesh = ft.gen_periodic_grid(9, 9)
    lap = ft.build_laplacian(mesh)
    dense = np.zeros((2, 81))
    dense[1] = 1.0
    fld = ft.LayeredField(ft.SparseMat.from_dense(dense), [0])
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=50)
    assert len(trace) == 1 and trace[0].converged and trace[0].max_delta == 0.0
    assert np.array_equal(out.phi.to_dense(), dense)


def test_evolve_input_stays_valid_and_on_step():
    mesh = ft.gen_periodic_grid(9, 9)
    lap = ft.build_laplacian(mesh)
    fld = ft.init_field(mesh, [40])
    before = fld.phi.to_dense()
    seen = []
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=30, on_step=lambda f, s: seen.append(f.step_count))
    assert seen == list(range(1, len(trace) + 1))
    assert np.array_equal(fld.phi.to_dense(), before)
    out2, trace2 = ft.evolve(fld, lap, DEFAULT, max_steps=30)
    assert len(trace2) == len(trace) and trace2[-1].converged == trace[-1].converged
    assert np.array_equal(out.phi.to_dense(), out2.phi.to_dense())


def test_four_symmetric_seeds_exhaust_base():
    mesh = ft.gen_periodic_grid(50, 50)
    lap = ft.build_laplacian(mesh)
    seeds = [50 * 12 + 12, 50 * 12 + 37, 50 * 37 + 12, 50 * 37 + 37]
    out, trace = ft.evolve(ft.init_field(mesh, seeds), lap, DEFAULT, max_steps=2500)
    assert trace[-1].converged and trace[-1].base_mass < 1e-9 * mesh.n_vertices


def _random_field(rng, n_v, n_rows, max_cnt, row_pool):
    """A field whose columns hold 0..max_cnt random rows out of ``row_pool``
    (sorted, values in (0, 1], columns normalised like the reference's)."""
    cols = []
    for _ in range(n_v):
        c = int(rng.integers(1 if max_cnt == 1 else 0, max_cnt + 1))
        rows = np.sort(rng.choice(row_pool, size=min(c, len(row_pool)), replace=False))
        vals = rng.random(rows.size) + 0.05
        vals = vals / vals.sum() if rows.size else vals
        cols.append((rows.astype(np.int32), vals))
    cnt = np.array([r.size for r, _ in cols])
    cp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    ri = np.concatenate([r for r, _ in cols]).astype(np.int32) if cp[-1] else np.zeros(0, np.int32)
    va = np.concatenate([v for _, v in cols]) if cp[-1] else np.zeros(0)
    return ft.SparseMat(n_rows, n_v, cp, ri, va, check=False)


def _tier_counts(phi, lap):
    """List counters of the control block after the column kernels of one
    (full) step, read before the finalize resets them: columns the band
    kernel handed to the warp-cooperative kernel, and those handed on to the
    serial windowed kernel."""
    import ctypes
    import torch
    from paper_1804_09152_b200 import _lib
    from paper_1804_09152_b200 import field as F
    lib = _lib.lib()
    d = ft.DeviceCSC.from_host(phi, torch.float64, torch.device("cuda"))
    ws = ft.StepWorkspace()
    ws.prepare(phi.n_cols, d.values.device)
    a = ft.DeviceTiled(phi.n_rows, phi.n_cols, 4 * phi.nnz + 64, torch.float64, d.values.device)
    b = ft.DeviceTiled(phi.n_rows, phi.n_cols, 4 * phi.nnz + 64, torch.float64, d.values.device)
    dl = F.device_laplacian(lap, "exact")
    lc, prm, st = dl.ft_csc("exact"), DEFAULT.ft_params(), F._stream_handle()
    wp, wn = ws.ws_args()
    s_c, a_c, b_c = d.ft_csc(), a.ft_tiled(), b.ft_tiled()
    rec = ctypes.c_void_p(ws.stats.data_ptr())
    assert lib.ft_tiled_from_csc(ctypes.byref(s_c), ctypes.byref(b_c), 0, wp, wn, rec, st) == 0
    assert lib.ft_step_run(ctypes.byref(lc), dl.launch_flags(), ctypes.byref(b_c), ctypes.byref(a_c), 0, 0,
                           ctypes.byref(prm), wp, wn, _lib.FT_PHASE_COLUMNS, rec, st) == 0
    c = ws.ws[:128].cpu().numpy()
    i32 = lambda o: int(c[o:o + 4].view(np.int32)[0])
    counts = {"wide": i32(84), "w2": i32(92), "deep": i32(88)}
    assert lib.ft_step_run(ctypes.byref(lc), dl.launch_flags(), ctypes.byref(b_c), ctypes.byref(a_c), 0, 0,
                           ctypes.byref(prm), wp, wn, _lib.FT_PHASE_FINALIZE, rec, st) == 0
    return counts


@pytest.mark.parametrize("max_cnt,n_pool,seed,tier", [
    (2, 6, 1, "wide"),      # two entries per column at most: band kernel, 3-row unions listed
    (3, 8, 2, "wide"),      # three-entry (pool) neighbours: the three-row kernel
    (4, 12, 3, "w2"),       # wider unions: the staged warp kernel
    (9, 16, 4, "w2"),
])
def test_random_fields_every_tier(max_cnt, n_pool, seed, tier):
    """Random fields on a small torus drive every kernel (band closed form and
    two-row update, the warp-cooperative 16-lane groups, the serial windowed
    kernel); one step and a 5-step evolve (active-set steps) are bitwise
    equal to the C oracle."""
    rng = np.random.default_rng(seed)
    mesh = ft.gen_periodic_grid(24, 20)
    lap = ft.build_laplacian(mesh)
    n_rows = 17
    phi = _random_field(rng, mesh.n_vertices, n_rows, max_cnt, np.arange(n_rows)[:n_pool])
    fld = ft.LayeredField(phi, np.arange(n_rows - 1))
    assert _tier_counts(phi, lap)[tier] > 0          # the case reaches the tier it names
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    out, st = ft.step(fld, lap, DEFAULT)
    ref1, rst = po.step_c(po.Csc.of(phi), lt, DEFAULT)
    assert_csc_equal(out.phi, ref1)
    assert st.max_delta == rst["max_delta"] and st.nnz_skel == rst["nnz_skel"]
    out5, trace = ft.evolve(fld, lap, DEFAULT, max_steps=5, tol=0.0)
    ref5, rtrace = po.evolve_c(po.Csc.of(phi), lt, DEFAULT, 5)
    assert_csc_equal(out5.phi, ref5)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]


def test_neighbourhood_beyond_staging_capacity():
    """A hub vertex adjacent to every other vertex: its neighbourhood holds
    more entries than the wide kernel stages in shared memory, so it runs
    the exact windowed algorithm from global memory; bitwise vs the oracle."""
    rng = np.random.default_rng(17)
    n = 200
    rows, cols = [], []
    for j in range(n):                  # L^T column j: the hub, the ring neighbours, itself
        nb = sorted({0, j, (j - 1) % n, (j + 1) % n} if j else set(range(n)))
        rows += nb
        cols += [j] * len(nb)
    deg = np.bincount(np.asarray(cols), minlength=n) - 1
    vals = np.where(np.asarray(rows) == np.asarray(cols), -1.0, 1.0 / deg[np.asarray(cols)])
    lapt = ft.SparseMat.from_triplets(n, n, rows, cols, vals)
    phi = _random_field(rng, n, 9, 3, np.arange(9))
    fld = ft.LayeredField(phi, np.arange(8))
    lap = _Lap(po.Csc.of(lapt))
    assert _tier_counts(phi, lap)["deep"] >= 1
    out, st = ft.step(fld, lap, DEFAULT)
    ref, rst = po.step_c(po.Csc.of(phi), po.Csc.of(lapt), DEFAULT)
    assert_csc_equal(out.phi, ref)
    assert st.max_delta == rst["max_delta"] and st.nnz_skel == rst["nnz_skel"]
    out3, _ = ft.evolve(fld, lap, DEFAULT, max_steps=3, tol=0.0)
    ref3, _ = po.evolve_c(po.Csc.of(phi), po.Csc.of(lapt), DEFAULT, 3)
    assert_csc_equal(out3.phi, ref3)


@pytest.mark.parametrize("max_cnt,n_pool,seed", [(2, 6, 11), (3, 8, 12), (4, 12, 13), (9, 16, 14)])
def test_random_fields_every_tier_fast(max_cnt, n_pool, seed):
    """FAST (fp32 storage) through every tier on random fields: one step from
    the fp32-rounded input within |d| <= 1e-5|ref| + 2e-7 of the oracle."""
    rng = np.random.default_rng(seed)
    mesh = ft.gen_periodic_grid(24, 20)
    lap = ft.build_laplacian(mesh)
    n_rows = 17
    phi = _random_field(rng, mesh.n_vertices, n_rows, max_cnt, np.arange(n_rows)[:n_pool])
    phi32 = ft.SparseMat(phi.n_rows, phi.n_cols, phi.col_ptr, phi.row_idx,
                         np.asarray(phi.values[:phi.nnz], dtype=np.float32).astype(np.float64), check=False)
    out, _ = ft.step(ft.LayeredField(phi32, np.arange(n_rows - 1), precision="fast"), lap, DEFAULT)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, _ = po.step_c(po.Csc.of(phi32), lt, DEFAULT)
    got, want = out.phi.to_dense(), ref.to_dense()
    assert np.all(np.abs(got - want) <= 1e-5 * np.abs(want) + 2e-7)


@pytest.mark.parametrize("max_steps", [1, 2, 3, 16, 17, 18, 33])
def test_evolve_chunk_boundaries(max_steps):
    """ft_evolve around its CUDA-graph chunking (step 1, then 16-step graph
    replays whose steps past max_steps are device no-ops) with each step's
    finalize on the side stream: field, trace length and per-step max |d|
    equal the C oracle's."""
    mesh = ft.gen_icosphere(3)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(7).choice(mesh.n_vertices, 40, replace=False)
    fld = ft.init_field(mesh, seeds)
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=max_steps, tol=0.0)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, rtrace = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, max_steps)
    assert len(trace) == max_steps and out.step_count == max_steps
    assert_csc_equal(out.phi, ref)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]
    assert [s.nnz_skel for s in trace] == [s["nnz_skel"] for s in rtrace]


def test_evolve_step_evolve_with_shared_workspace():
    """evolve -> step -> evolve with one StepWorkspace (cached graph, parity
    slots, side-stream finalize state carried between calls) equals 40 + 1 +
    25 oracle steps, bitwise."""
    mesh = ft.gen_icosphere(3)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(8).choice(mesh.n_vertices, 30, replace=False)
    fld = ft.init_field(mesh, seeds)
    ws = ft.StepWorkspace()
    a, _ = ft.evolve(fld, lap, DEFAULT, max_steps=40, tol=0.0, workspace=ws)
    b, _ = ft.step(a, lap, DEFAULT, workspace=ws)
    c, tr = ft.evolve(b, lap, DEFAULT, max_steps=25, tol=0.0, workspace=ws)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, _ = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 66)
    assert c.step_count == 66 and len(tr) == 25
    assert_csc_equal(c.phi, ref)


def test_step_reports_phase_times():
    """step() splits its device time over the reference's five StepStats
    phase slots (ft_step_phases kernel groups, field.py:220-285)."""
    mesh = ft.gen_icosphere(4)
    lap = ft.build_laplacian(mesh)
    fld = ft.init_field(mesh, ft.sample_seed_vertices(mesh, 64, 0))
    for _ in range(3):
        fld, st = ft.step(fld, lap, DEFAULT)
    phases = [st.skeleton_time, st.spgemm_time, st.expand_time, st.update_time, st.normalize_time]
    assert all(t >= 0.0 for t in phases)
    assert st.spgemm_time > 0.0 and st.normalize_time > 0.0 and st.skeleton_time > 0.0
    assert st.total_time == pytest.approx(sum(phases))


@pytest.mark.parametrize("subdiv,n_seeds", [(4, 64), (3, 160)])
def test_four_row_kernel_bitwise(monkeypatch, subdiv, n_seeds):
    """The four-row kernel (wide4) on small dense fields: forced on for any
    number of leftovers (FT_WIDE4_MIN=0; by default it runs only when the
    three-row kernel leaves >= 48K columns), bitwise against the C oracle
    through the device evolve and the step loop."""
    monkeypatch.setenv("FT_WIDE4_MIN", "0")
    mesh = ft.gen_icosphere(subdiv)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(0).choice(mesh.n_vertices, n_seeds, replace=False)
    fld = ft.init_field(mesh, seeds)
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=40, tol=0.0)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, rtrace = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 40, n_threads=4)
    assert_csc_equal(out.phi, ref)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]
    cur = fld
    for _ in range(12):
        cur, _st = ft.step(cur, lap, DEFAULT)
    ref12, _ = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 12, n_threads=4)
    assert_csc_equal(cur.phi, ref12)


@pytest.mark.parametrize("subdiv,n_seeds", [(4, 64), (5, 400)])
def test_dense_band_hint_bitwise(monkeypatch, subdiv, n_seeds):
    """FT_HINT_DENSE_BAND (the three-row kernel's dense-band variant: more
    CTAs per SM, the column's own entries re-read) changes speed only:
    forced on for every field (DENSE_BAND_EXTRA = 0), evolve and the step
    loop are bitwise the C oracle's."""
    monkeypatch.setattr(ft.field, "DENSE_BAND_EXTRA", 0)
    mesh = ft.gen_icosphere(subdiv)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(1).choice(mesh.n_vertices, n_seeds, replace=False)
    fld = ft.init_field(mesh, seeds)
    assert ft.field.device_laplacian(lap, "exact").launch_flags(fld.device_phi()) & ft._lib.FT_HINT_DENSE_BAND
    out, trace = ft.evolve(fld, lap, DEFAULT, max_steps=40, tol=0.0)
    lt = po.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, rtrace = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 40, n_threads=4)
    assert_csc_equal(out.phi, ref)
    assert [s.max_delta for s in trace] == [s["max_delta"] for s in rtrace]
    cur = fld
    for _ in range(6):
        cur, _st = ft.step(cur, lap, DEFAULT)
    ref6, _ = po.evolve_c(po.Csc.of(fld.phi), lt, DEFAULT, 6, n_threads=4)
    assert_csc_equal(cur.phi, ref6)


def test_dense_band_hint_fast_identical(monkeypatch):
    """FAST (fp32 storage) through the dense-band variant: the same bits
    with and without the hint."""
    mesh = ft.gen_icosphere(5)
    lap = ft.build_laplacian(mesh)
    seeds = np.random.default_rng(2).choice(mesh.n_vertices, 400, replace=False)
    fld = ft.init_field(mesh, seeds, precision="fast")
    plain, tp = ft.evolve(fld, lap, DEFAULT, max_steps=30, tol=0.0)
    monkeypatch.setattr(ft.field, "DENSE_BAND_EXTRA", 0)
    hinted, th = ft.evolve(fld, lap, DEFAULT, max_steps=30, tol=0.0)
    assert_csc_equal(hinted.phi, plain.phi)
    assert [s.max_delta for s in th] == [s.max_delta for s in tp]
