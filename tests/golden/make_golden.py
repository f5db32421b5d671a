"""Generate golden fixtures by running the REFERENCE package in this container.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--big]

The reference (``fieldtess``, pure Python + numba) is imported from
``oracle/_ref/py`` (pip-installed by ``make -C oracle ref``) or directly from
``/root/reference/pkg/src``.  It does not exist on the GPU box, so every
fixture the tests need is written here as a small ``.npz`` / ``.json`` and
committed.  Nothing in the product imports this script.

Fixtures
--------
step_cases.npz   single steps from the reference's own TestStepOracle inputs
                 (test_field.py:80-122): star hand case, 6 random fields
                 (rng 33), a 5-step torus 9x9 run, plus random params.
c1_traj.npz      config C1: icosphere-4, 64 seeds (sample_seed_vertices rng 0),
                 PHI snapshots at steps 0,1,2,10,100,500 and the stats trace.
torus_traj.npz   torus 64x64, 24 seeds: snapshots at 0,1,60,300.
labels.npz       sharp_labels on C1 snapshots + hand cases.
seeds.json       sample_seed_vertices outputs (rng 0) for several meshes.
meshes.json      SHA-256 digests of generator outputs (faces / positions /
                 L^T arrays) for icosphere 0..7 and a few tori.
c1_dual.json     dual-mesh products on C1 after 500 steps (API path).
seeds_collide.json  sample_seed_vertices with many collisions (small meshes,
                 seed counts near n_vertices, several rng seeds).
analysis.npz     analysis.py metrics: voronoi labels / margin masks (torus,
                 icosphere), triangle qualities of a dual mesh, area
                 histogram, directed surface distances and hausdorff.
--big: c2_traj.npz (icosphere-7, 1024 seeds, steps 0/100/1000) and
       c2_lloyd.json (5 Lloyd iterations, max_steps 1000).
c1_s10.field / c1_s10.trip  save_field / write_triplets output of the
                 reference (C1 at step 10) for snapshot compatibility.
dual_warnings.json  confirm_candidates warnings (degenerate face, NaN
                 layer value) of the reference on a modified C1.
c5_lloyd.json    (--only c5, ~10 min) C5 reduced window: 2 Lloyd iterations
                 at max_steps 100 on the 10M torus with 65,536 seeds + dual.
--only a,b: regenerate only the named groups (seeds_collide, analysis).
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
for cand in (os.path.join(REPO, "oracle", "_ref", "py"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "fieldtess")):
        sys.path.insert(0, cand)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import fieldtess as ft  # noqa: E402  (the reference)
from fieldtess.cli import sample_seed_vertices  # noqa: E402
from fieldtess.field import LayeredField, StepWorkspace, step  # noqa: E402


def csc_arrays(prefix, m):
    nnz = m.nnz
    return {f"{prefix}_shape": np.array([m.n_rows, m.n_cols], dtype=np.int64),
            f"{prefix}_ptr": m.col_ptr.astype(np.int32).copy(),
            f"{prefix}_idx": m.row_idx[:nnz].astype(np.int32).copy(),
            f"{prefix}_val": m.values[:nnz].astype(np.float64).copy()}


def params_array(p):
    return np.array([p.w, p.a, p.e, p.e_base, p.mu, p.dt], dtype=np.float64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def star_mesh():
    pos = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]], dtype=float)
    faces = [[0, 1, 2], [0, 2, 3], [0, 3, 4], [0, 4, 1]]
    return ft.TriMesh(pos, faces)


def make_step_cases():
    out = {}
    cases = []
    # star hand case (test_field.py:80-89)
    mesh = star_mesh()
    lap = ft.build_laplacian(mesh, "uniform")
    phi = np.zeros((2, 5))
    phi[1, 0] = 1.0
    phi[1, 1] = 0.4
    phi[0] = 1.0 - phi[1]
    cases.append(("star", lap, phi, ft.CouplingParams()))
    # random fields (test_field.py:91-107)
    grid9 = ft.gen_periodic_grid(9, 9)
    lap9 = ft.build_laplacian(grid9, "uniform")
    rng = np.random.default_rng(33)
    for trial in range(6):
        n_cells = int(rng.integers(1, 5))
        phi = np.zeros((n_cells + 1, 81))
        for r in range(1, n_cells + 1):
            support = rng.choice(81, size=rng.integers(3, 20), replace=False)
            phi[r, support] = rng.random(support.size)
        sums = phi.sum(axis=0)
        phi[0] = np.maximum(1.0 - sums, 0.0)
        phi /= phi.sum(axis=0, keepdims=True)
        params = ft.CouplingParams(w=0.2, a=1.0, e=float(rng.uniform(0, 0.5)),
                                   e_base=float(rng.uniform(0, 0.5)),
                                   mu=float(rng.uniform(0.05, 0.4)),
                                   dt=float(rng.uniform(1, 5)))
        cases.append((f"rand{trial}", lap9, phi, params))
    # many-cell dense-ish columns (exercise the wide-window path): 12 cells
    rng = np.random.default_rng(5)
    phi = np.zeros((13, 81))
    for r in range(1, 13):
        support = rng.choice(81, size=40, replace=False)
        phi[r, support] = rng.random(support.size)
    phi[0] = np.maximum(1.0 - phi.sum(axis=0), 0.0)
    phi /= phi.sum(axis=0, keepdims=True)
    cases.append(("wide12", lap9, phi, ft.CouplingParams()))
    # cotan Laplacian on icosphere-2 with 5 seeds, a few steps in
    ico2 = ft.gen_icosphere(2)
    lapc = ft.build_laplacian(ico2, "cotan-clamped")
    fld = ft.init_field(ico2, [0, 17, 40, 90, 130])
    for _ in range(3):
        fld, _ = step(fld, lapc, ft.CouplingParams())
    cases.append(("cotan_ico2", lapc, fld.phi.to_dense(), ft.CouplingParams()))

    names = []
    for name, lap, phi, params in cases:
        fld = LayeredField(ft.SparseMat.from_dense(phi), np.arange(phi.shape[0] - 1))
        res, stats = step(fld, lap, params)
        out.update(csc_arrays(f"{name}_in", fld.phi))
        out.update(csc_arrays(f"{name}_lapt", lap.mat_t))
        out.update(csc_arrays(f"{name}_out", res.phi))
        out[f"{name}_params"] = params_array(params)
        out[f"{name}_stats"] = np.array([stats.max_delta, stats.base_mass, stats.nnz_phi])
        names.append(name)
    # 5-step run on the 9x9 torus, seeds [20, 60] (test_field.py:109-122)
    fld = ft.init_field(grid9, [20, 60])
    out.update(csc_arrays("multi_in", fld.phi))
    out.update(csc_arrays("multi_lapt", lap9.mat_t))
    ws = StepWorkspace()
    cur = fld
    for _ in range(5):
        cur, _ = step(cur, lap9, ft.CouplingParams(), workspace=ws)
    out.update(csc_arrays("multi_out", cur.phi.copy()))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "step_cases.npz"), **out)
    print("step_cases:", names)


def trajectory(mesh, seeds, snaps, path, max_step):
    lap = ft.build_laplacian(mesh, "uniform")
    fld = ft.init_field(mesh, seeds)
    out = {"seeds": np.asarray(seeds, dtype=np.int64)}
    out.update(csc_arrays("lapt", lap.mat_t))
    out.update(csc_arrays("s0", fld.phi))
    trace = []
    ws = StepWorkspace()
    cur = fld
    t0 = time.time()
    for k in range(1, max_step + 1):
        cur, st = step(cur, lap, ft.CouplingParams(), workspace=ws)
        trace.append((st.max_delta, st.base_mass, st.nnz_phi))
        if k in snaps:
            out.update(csc_arrays(f"s{k}", cur.phi.copy()))
    out["snaps"] = np.array([0] + sorted(snaps), dtype=np.int64)
    out["trace"] = np.array(trace)
    out["labels_final"] = ft.sharp_labels(cur)
    np.savez_compressed(path, **out)
    print(os.path.basename(path), f"{time.time() - t0:.1f}s", "nnz", cur.phi.nnz)
    return cur


def make_labels_cases():
    out = {}
    cases = {
        "argmax": ({0: {4: 0.9, 8: 0.1}}, 9, 2),
        "base": ({0: {0: 1.0}}, 9, 1),
        "tie": ({0: {3: 0.5, 6: 0.5}}, 9, 1),
        "basetie": ({0: {0: 0.5, 2: 0.5}, 1: {0: 0.6, 1: 0.2, 3: 0.2}}, 4, 2),
        "zeros": ({0: {0: 0.0, 1: 0.0}, 1: {}}, 3, 2),
    }
    for name, (columns, n_rows, n_cols) in cases.items():
        dense = np.zeros((n_rows, n_cols))
        for col, entries in columns.items():
            for row, val in entries.items():
                dense[row, col] = val
        # keep explicit zeros like the reference test helpers would not:
        m = ft.SparseMat.from_triplets(
            n_rows, n_cols,
            [r for c, e in columns.items() for r in e],
            [c for c, e in columns.items() for _ in e],
            [v for c, e in columns.items() for v in e.values()])
        fld = LayeredField(m, np.arange(n_rows - 1))
        out.update(csc_arrays(name, m))
        out[f"{name}_labels"] = ft.sharp_labels(fld)
    out["names"] = np.array(list(cases))
    np.savez_compressed(os.path.join(HERE, "labels.npz"), **out)


def make_seeds_and_meshes():
    seeds = {}
    meshes = {}
    for name, mesh, count in [("ico4", ft.gen_icosphere(4), 64),
                              ("ico5", ft.gen_icosphere(5), 300),
                              ("torus64", ft.gen_periodic_grid(64, 64), 24),
                              ("torus40x30", ft.gen_periodic_grid(40, 30), 50)]:
        seeds[name] = sample_seed_vertices(mesh, count, 0).tolist()
    for s in range(0, 8):
        mesh = ft.gen_icosphere(s)
        lap = ft.build_laplacian(mesh, "uniform")
        meshes[f"ico{s}"] = {
            "n_vertices": mesh.n_vertices, "n_faces": mesh.n_faces,
            "faces": sha(mesh.faces.astype(np.int32)),
            "positions": sha(mesh.positions.astype(np.float64)),
            "lapt_ptr": sha(lap.mat_t.col_ptr.astype(np.int32)),
            "lapt_idx": sha(lap.mat_t.row_idx[:lap.mat_t.nnz].astype(np.int32)),
            "lapt_val": sha(lap.mat_t.values[:lap.mat_t.nnz].astype(np.float64)),
            "face_area": sha(mesh.face_area.astype(np.float64)),
            "vertex_area": sha(mesh.vertex_area.astype(np.float64)),
        }
    for nx, ny in [(3, 3), (9, 9), (64, 64), (40, 30), (200, 150)]:
        mesh = ft.gen_periodic_grid(nx, ny)
        lap = ft.build_laplacian(mesh, "uniform")
        meshes[f"torus{nx}x{ny}"] = {
            "n_vertices": mesh.n_vertices, "n_faces": mesh.n_faces,
            "faces": sha(mesh.faces.astype(np.int32)),
            "positions": sha(mesh.positions.astype(np.float64)),
            "lapt_ptr": sha(lap.mat_t.col_ptr.astype(np.int32)),
            "lapt_idx": sha(lap.mat_t.row_idx[:lap.mat_t.nnz].astype(np.int32)),
            "lapt_val": sha(lap.mat_t.values[:lap.mat_t.nnz].astype(np.float64)),
            "face_area": sha(mesh.face_area.astype(np.float64)),
            "vertex_area": sha(mesh.vertex_area.astype(np.float64)),
        }
    with open(os.path.join(HERE, "seeds.json"), "w") as fh:
        json.dump(seeds, fh)
    with open(os.path.join(HERE, "meshes.json"), "w") as fh:
        json.dump(meshes, fh, indent=1, sort_keys=True)
    return seeds


def make_c1_dual(fld, mesh, name="c1_dual.json"):
    from fieldtess import dual as dualmod
    a_v = dualmod.vertex_adjacency(fld, 0.25)
    a_t = dualmod.triangle_adjacency(fld, mesh, 0.25)
    cur = dualmod.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
    dm = dualmod.build_dual(cur, np.zeros((fld.n_cells, 3)))
    res = {
        "a_v": sorted(map(list, a_v.pairs())),
        "a_t": sorted(map(list, a_t.pairs())),
        "curated": sorted(map(list, cur.pairs())),
        "dropped": [[int(i), int(j), r] for i, j, r in cur.dropped],
        "triples": sorted(map(list, cur.junction_triples)),
        "triangles": sorted(map(sorted, dm.triangles.tolist())),
        "spurious": [list(map(int, t)) for t in dm.spurious_removed],
        "euler": int(dm.euler_characteristic()),
    }
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(res, fh)
    print(name, "triangles", len(res["triangles"]), "euler", res["euler"])


def make_dual_winding():
    """Exact oriented dual triangles (order and winding) of the reference's
    build_dual on the C1 / C2 golden fields: without cell normals, and with
    outward / inward cell normals (the majority-normal flip)."""
    from fieldtess import dual as dualmod
    out = {}
    for name, traj, snap, level in (("c1", "c1_traj.npz", 500, 4), ("c2", "c2_traj.npz", 1000, 7)):
        path = os.path.join(HERE, traj)
        if not os.path.exists(path):
            continue
        t = np.load(path)
        shp = t[f"s{snap}_shape"]
        phi = ft.SparseMat(int(shp[0]), int(shp[1]), t[f"s{snap}_ptr"], t[f"s{snap}_idx"], t[f"s{snap}_val"],
                           check=False)
        mesh = ft.gen_icosphere(level)
        fld = LayeredField(phi, t["seeds"], snap)
        a_v = dualmod.vertex_adjacency(fld, 0.25)
        a_t = dualmod.triangle_adjacency(fld, mesh, 0.25)
        cur = dualmod.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
        pos = mesh.positions[np.asarray(t["seeds"], dtype=np.int64)]
        nrm = pos / np.linalg.norm(pos, axis=1)[:, None]
        out[name] = {
            "plain": dualmod.build_dual(cur, np.zeros((fld.n_cells, 3))).triangles.tolist(),
            "outward": dualmod.build_dual(cur, pos, cell_normals=nrm).triangles.tolist(),
            "inward": dualmod.build_dual(cur, pos, cell_normals=-nrm).triangles.tolist(),
        }
        print("winding", name, len(out[name]["plain"]))
    with open(os.path.join(HERE, "dual_winding.json"), "w") as fh:
        json.dump(out, fh)


def make_snapshots():
    """Snapshot files written by the reference itself: save_field of the C1
    field at step 10 (with an extra header key) and write_triplets of the
    same matrix with comment lines (field.py:372-387, sparse.py:427-436)."""
    t = np.load(os.path.join(HERE, "c1_traj.npz"))
    phi = ft.SparseMat(int(t["s10_shape"][0]), int(t["s10_shape"][1]), t["s10_ptr"], t["s10_idx"],
                       t["s10_val"], check=False)
    fld = LayeredField(phi, t["seeds"], 10)
    params = ft.CouplingParams(dt=0.05, mu=2.5)
    from fieldtess.field import save_field
    from fieldtess.sparse import write_triplets
    save_field(fld, params, os.path.join(HERE, "c1_s10.field"), extra_header={"mesh": "icosphere-4"})
    write_triplets(phi, os.path.join(HERE, "c1_s10.trip"), comments=("fieldtess triplets", "step 10"))


def make_dual_warnings():
    """confirm_candidates on C1 step 500 with (a) one mesh vertex moved onto
    its neighbour (two zero-area faces) and (b) one NaN written into a
    layer: the reference's RuntimeWarnings in order (dual.py:187-199) and the
    curated result, at threshold 0.4 (A_t-only candidates exist there)."""
    import warnings as wmod
    THR = 0.4
    from fieldtess import dual as dualmod
    t = np.load(os.path.join(HERE, "c1_traj.npz"))
    shp = t["s500_shape"]
    base_vals = np.array(t["s500_val"], dtype=np.float64)
    mesh0 = ft.gen_icosphere(4)
    fld0 = LayeredField(ft.SparseMat(int(shp[0]), int(shp[1]), t["s500_ptr"], t["s500_idx"], base_vals,
                                     check=False), t["seeds"], 500)
    a_v = dualmod.vertex_adjacency(fld0, THR)
    a_t = dualmod.triangle_adjacency(fld0, mesh0, THR)
    cand = sorted(set(a_t.pairs()) - set(a_v.pairs()))
    b = ft.spgemm(dualmod.threshold_rows(fld0, THR), mesh0.incidence)
    foc = ft.transpose(b)

    def shared(i, j):
        return np.intersect1d(foc.column(i)[0], foc.column(j)[0])

    out = {}
    # (a) degenerate: collapse the first shared face of the first candidate
    i, j = cand[0]
    f = int(shared(i, j)[0])
    v_from, v_to = int(mesh0.faces[f][1]), int(mesh0.faces[f][0])
    pos = mesh0.positions.copy()
    pos[v_from] = pos[v_to]
    mesh1 = ft.TriMesh(pos, mesh0.faces.copy())
    # (b) non-finite: NaN at a stored entry of layer i+1 on a vertex of the
    # first shared face of the third candidate
    i2, j2 = cand[2]
    f2 = int(shared(i2, j2)[0])
    ptr, idx = t["s500_ptr"], t["s500_idx"]
    k_nan = -1
    for v in mesh0.faces[f2]:
        for k in range(ptr[v], ptr[v + 1]):
            if idx[k] == i2 + 1:
                k_nan = k
        if k_nan >= 0:
            break
    vals2 = base_vals.copy()
    vals2[k_nan] = np.nan
    fld2 = LayeredField(ft.SparseMat(int(shp[0]), int(shp[1]), ptr, idx, vals2, check=False), t["seeds"], 500)
    for name, fld, mesh, info in (("degenerate", fld0, mesh1, {"move": [v_from, v_to]}),
                                  ("nonfinite", fld2, mesh0, {"nan_entry": int(k_nan)})):
        av = dualmod.vertex_adjacency(fld, THR)
        at = dualmod.triangle_adjacency(fld, mesh, THR)
        with wmod.catch_warnings(record=True) as rec:
            wmod.simplefilter("always")
            cur = dualmod.confirm_candidates(fld, mesh, av, at, THR)
        info["warnings"] = [str(w.message) for w in rec if issubclass(w.category, RuntimeWarning)]
        info["curated"] = sorted(cur.pairs())
        info["dropped"] = [list(d) for d in cur.dropped]
        out[name] = info
        print("dual warnings", name, len(info["warnings"]), info["warnings"][:3])
    with open(os.path.join(HERE, "dual_warnings.json"), "w") as fh:
        json.dump(out, fh)


def make_cell_geometry(name, mesh, fld):
    """Reference approx_centroid / backproject for every cell of fld."""
    from fieldtess import lloyd as L
    prod = L.faces_by_cell(fld, mesh)
    n = fld.n_cells
    pts = np.full((n, 3), np.nan)
    nrm = np.full((n, 3), np.nan)
    status = np.zeros(n, dtype=np.int64)
    hit = np.full(n, -1, dtype=np.int64)
    for c in range(n):
        try:
            faces = L.cell_triangles(fld, mesh, c, product=prod)
            p, q = L.approx_centroid(fld, mesh, c, faces=faces)
            pts[c], nrm[c] = p, q
            h = L.backproject(p, q, fld, mesh, c, faces=faces)
            if h is None:
                status[c] = 4
            else:
                hit[c] = h
        except ft.errors.VanishedCellError:
            status[c] = 1
        except ft.errors.DegenerateCellError:
            status[c] = 2
        except ft.errors.NullNormalError:
            status[c] = 3
    out = {f"{name}_point": pts, f"{name}_normal": nrm, f"{name}_status": status, f"{name}_hit": hit}
    out.update(csc_arrays(f"{name}_fbc", prod))
    return out


def make_c2(seeds_c2):
    mesh = ft.gen_icosphere(7)
    c2 = trajectory(mesh, seeds_c2, {100, 1000}, os.path.join(HERE, "c2_traj.npz"), 1000)
    make_c1_dual(c2, mesh, "c2_dual.json")
    from fieldtess.lloyd import LloydState, lloyd_iterate
    lap = ft.build_laplacian(mesh, "uniform")
    t0 = time.time()
    state = lloyd_iterate(LloydState(seeds=np.asarray(seeds_c2)), mesh, lap,
                          ft.CouplingParams(), n_iter=5, max_steps=1000)
    hist = [{k: rec[k] for k in ("iteration", "seeds", "area_variance", "steps",
                                 "reseed_misses", "seed_collisions")}
            for rec in state.history]
    with open(os.path.join(HERE, "c2_lloyd.json"), "w") as fh:
        json.dump({"history": hist, "wall_s": time.time() - t0}, fh)
    print("c2_lloyd", f"{time.time() - t0:.1f}s")


def make_c5():
    """C5 (BASELINE configs[4]) on a reduced window: torus 3200 x 3125
    (10M vertices), 65,536 seeds (the exact replay of cli.sample_seed_vertices,
    pinned by seeds.json), lloyd_iterate n_iter=2 with max_steps=100 (C5's
    Lloyd definition: at the default max_steps=1000 a cell vanishes), then
    the dual mesh at threshold 0.25.  Digests only (the arrays are large)."""
    import hashlib
    from fieldtess.lloyd import LloydState, lloyd_iterate
    from fieldtess import dual as dualmod
    sys.path.insert(0, REPO)
    from paper_1804_09152_b200.seeding import sample_seed_vertices as replay
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    t0 = time.time()
    mesh = ft.gen_periodic_grid(3200, 3125)
    lap = ft.build_laplacian(mesh, "uniform")
    seeds = replay(mesh, 65536, 0)
    print("c5 setup", f"{time.time() - t0:.1f}s", flush=True)
    t1 = time.time()
    state = lloyd_iterate(LloydState(seeds=np.asarray(seeds)), mesh, lap, ft.CouplingParams(), n_iter=2,
                          max_steps=100)
    t_lloyd = time.time() - t1
    hist = [{"iteration": r["iteration"], "seeds_sha": dig(np.asarray(r["seeds"], dtype=np.int64)),
             "seeds_head": [int(x) for x in r["seeds"][:16]], "area_variance": r["area_variance"],
             "cell_areas_sha": dig(np.asarray(r["cell_areas"], dtype=np.float64)), "steps": r["steps"],
             "converged": r["converged"], "reseed_misses": r["reseed_misses"],
             "seed_collisions": r["seed_collisions"]} for r in state.history]
    print("c5 lloyd", f"{t_lloyd:.1f}s", flush=True)
    t2 = time.time()
    fld = state.field
    phi = fld.phi
    a_v = dualmod.vertex_adjacency(fld, 0.25)
    a_t = dualmod.triangle_adjacency(fld, mesh, 0.25)
    cur = dualmod.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
    pos = mesh.positions[np.asarray(fld.seed_vertices, dtype=np.int64)]
    try:
        dm = dualmod.build_dual(cur, pos)
        dual_error = None
    except ft.TessError as exc:          # the reference's own verdict is the golden
        dm, dual_error = None, {"type": type(exc).__name__, "message": str(exc)}
    pairs = np.asarray(sorted(cur.pairs()), dtype=np.int64)
    out = {"history": hist, "lloyd_wall_s": t_lloyd, "dual_wall_s": time.time() - t2,
           "phi_sha": {"col_ptr": dig(np.asarray(phi.col_ptr, dtype=np.int32)),
                       "row_idx": dig(np.asarray(phi.row_idx[:phi.nnz], dtype=np.int32)),
                       "values": dig(np.asarray(phi.values[:phi.nnz], dtype=np.float64))},
           "dual": {"n_pairs": int(pairs.shape[0]), "pairs_sha": dig(pairs),
                    "n_dropped": len(cur.dropped), "error": dual_error,
                    "n_triangles": None if dm is None else int(dm.triangles.shape[0]),
                    "triangles_sha": None if dm is None else dig(np.asarray(dm.triangles, dtype=np.int64)),
                    "spurious_removed": None if dm is None else len(dm.spurious_removed)}}
    with open(os.path.join(HERE, "c5_lloyd.json"), "w") as fh:
        json.dump(out, fh)
    print("c5 dual", f"{time.time() - t2:.1f}s", flush=True)


def make_seed_collisions():
    out = {}
    for name, mesh, count, seed in [("t20x15", ft.gen_periodic_grid(20, 15), 280, 3),
                                    ("ico2", ft.gen_icosphere(2), 160, 7),
                                    ("ico3", ft.gen_icosphere(3), 500, 11),
                                    ("t9x7s", ft.gen_periodic_grid(9, 7, 0.5), 60, 1)]:
        out[name] = {"count": count, "rng": seed,
                     "seeds": sample_seed_vertices(mesh, count, seed).tolist()}
    with open(os.path.join(HERE, "seeds_collide.json"), "w") as fh:
        json.dump(out, fh)


def make_analysis():
    from fieldtess import analysis as an
    from fieldtess.dual import build_dual
    out = {}
    torus = ft.gen_periodic_grid(20, 15)
    rng = np.random.default_rng(5)
    spos = torus.positions[rng.choice(torus.n_vertices, 9, replace=False)] + 0.1
    out["tor_spos"] = spos
    out["tor_labels"] = an.euclidean_voronoi_labels(torus, spos)
    out["tor_margin"] = an.margin_mask(torus, spos, "euclidean")
    ico = ft.gen_icosphere(3)
    sv = rng.choice(ico.n_vertices, 12, replace=False)
    out["ico_seeds"] = sv
    out["ico_labels"] = an.sphere_voronoi_labels(ico, sv)
    out["ico_margin"] = an.margin_mask(ico, sv, "sphere", factor=1.5)
    # dual of an icosphere-3 field with 24 seeds after 200 steps
    seeds = sample_seed_vertices(ico, 24, 2)
    fld, _ = ft.evolve(ft.init_field(ico, seeds), ft.build_laplacian(ico), ft.CouplingParams(),
                       max_steps=200)
    from fieldtess import dual as dualmod
    a_v = dualmod.vertex_adjacency(fld, 0.25)
    a_t = dualmod.triangle_adjacency(fld, ico, 0.25)
    cur = dualmod.confirm_candidates(fld, ico, a_v, a_t, 0.25)
    dual = build_dual(cur, ico.positions[seeds])
    q, ang = an.triangle_qualities(dual.positions, dual.triangles)
    out["dual_seeds"] = seeds
    out["dual_positions"] = np.asarray(dual.positions)
    out["dual_triangles"] = np.asarray(dual.triangles)
    out["dual_q"] = q
    out["dual_angles"] = ang
    rep = an.triangle_quality(dual)
    out["dual_report"] = np.array([rep.mean_quality, rep.min_quality, rep.mean_min_angle,
                                   rep.min_angle, rep.pct_below_30, rep.n_triangles,
                                   rep.n_degenerate], dtype=np.float64)
    areas = rng.random(50) * 3
    cnt, edges = an.cell_area_histogram(areas)
    out["hist_areas"], out["hist_counts"], out["hist_edges"] = areas, cnt, edges
    ico4 = ft.gen_icosphere(4)
    out["d_ab"] = an.directed_surface_distance(ico, ico4, 2000, 0)
    out["d_ba"] = an.directed_surface_distance(ico4, ico, 2000, 1)
    out["hausdorff_ico"] = np.array(an.hausdorff(ico, ico4, 2000, 0))
    t2 = ft.gen_periodic_grid(21, 16)
    out["d_tor"] = an.directed_surface_distance(torus, t2, 1500, 4)
    np.savez_compressed(os.path.join(HERE, "analysis.npz"), **out)


def main():
    if "--only" in sys.argv:
        for name in sys.argv[sys.argv.index("--only") + 1].split(","):
            {"seeds_collide": make_seed_collisions, "analysis": make_analysis,
             "winding": make_dual_winding, "snapshots": make_snapshots,
             "dual_warnings": make_dual_warnings, "c5": make_c5}[name]()
        return
    make_step_cases()
    make_labels_cases()
    seeds = make_seeds_and_meshes()
    ico4 = ft.gen_icosphere(4)
    c1 = trajectory(ico4, seeds["ico4"], {1, 2, 10, 100, 500},
                    os.path.join(HERE, "c1_traj.npz"), 500)
    make_c1_dual(c1, ico4)
    make_dual_winding()
    make_snapshots()
    make_dual_warnings()
    geo = make_cell_geometry("c1", ico4, c1)
    torus = ft.gen_periodic_grid(64, 64)
    tfld = trajectory(torus, seeds["torus64"], {1, 60, 300},
                      os.path.join(HERE, "torus_traj.npz"), 300)
    geo.update(make_cell_geometry("torus", torus, tfld))
    np.savez_compressed(os.path.join(HERE, "cell_geometry.npz"), **geo)
    make_seed_collisions()
    make_analysis()
    if "--big" in sys.argv:
        mesh = ft.gen_icosphere(7)
        seeds_c2 = sample_seed_vertices(mesh, 1024, 0)
        with open(os.path.join(HERE, "seeds_c2.json"), "w") as fh:
            json.dump(seeds_c2.tolist(), fh)
        make_c2(seeds_c2)


if __name__ == "__main__":
    main()
