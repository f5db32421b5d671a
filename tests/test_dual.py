"""Dual-mesh extraction parity: device adjacency products + host curation
against the reference's outputs on C1 (icosphere-4, 64 seeds, 500 steps)
and C2 (icosphere-7, 1024 seeds, 1000 steps) -- tests/golden/c{1,2}_dual.json."""

import os

import numpy as np
import pytest

import paper_1804_09152_b200 as ft
from conftest import GOLDEN, csc_from, golden_json, golden_npz


def _field(traj, snap):
    t = golden_npz(traj)
    c = csc_from(t, f"s{snap}")
    return ft.LayeredField(ft.SparseMat(c.n_rows, c.n_cols, c.col_ptr, c.row_idx, c.values,
                                        check=False), t["seeds"], step_count=snap)


def test_oracle_dual_products_match_reference():
    from oracle import pyoracle as po
    ref = golden_json("c1_dual.json")
    mesh, fld = ft.gen_icosphere(4), _field("c1_traj.npz", 500)
    pv, pt, px, tri = po.dual_products_np(fld.phi, mesh.faces, mesh.face_area, 0.25)
    assert [list(p) for p in pv] == ref["a_v"]
    assert [list(p) for p in pt] == ref["a_t"]
    assert [list(t) for t in tri] == ref["triples"]
    confirmed = set(map(tuple, ref["curated"])) - set(map(tuple, ref["a_v"]))
    assert confirmed <= set(px)
    for i, j, why in ref["dropped"]:
        if why == "no-intersection":
            assert (i, j) not in set(px)


def test_segments_intersect_cases():
    from paper_1804_09152_b200.dual import segments_intersect
    p = np.array([[0.0, 0.0], [1.0, 1.0]])
    assert segments_intersect(p, np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert not segments_intersect(p, np.array([[2.0, 2.0], [3.0, 3.5]]))
    assert segments_intersect(p, np.array([[1.0, 1.0], [2.0, 0.0]]))   # touching counts


def _check_case(name, traj, snap, mesh):
    ref = golden_json(name)
    fld = _field(traj, snap)
    a_v = ft.vertex_adjacency(fld, 0.25)
    a_t = ft.triangle_adjacency(fld, mesh, 0.25)
    assert sorted(map(list, a_v.pairs())) == ref["a_v"]
    assert sorted(map(list, a_t.pairs())) == ref["a_t"]
    cur = ft.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
    assert sorted(map(list, cur.pairs())) == ref["curated"]
    assert [[int(i), int(j), w] for i, j, w in cur.dropped] == ref["dropped"]
    assert sorted(map(list, cur.junction_triples)) == ref["triples"]
    dm = ft.build_dual(cur, np.zeros((fld.n_cells, 3)))
    assert sorted(map(sorted, dm.triangles.tolist())) == ref["triangles"]
    assert [list(map(int, t)) for t in dm.spurious_removed] == ref["spurious"]
    assert int(dm.euler_characteristic()) == ref["euler"]


@pytest.mark.gpu
def test_dual_c1_matches_reference():
    _check_case("c1_dual.json", "c1_traj.npz", 500, ft.gen_icosphere(4))


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c2_dual.json")), reason="no C2 dual golden")
def test_dual_c2_matches_reference():
    _check_case("c2_dual.json", "c2_traj.npz", 1000, ft.gen_icosphere(7))


@pytest.mark.gpu
def test_dual_from_partitioned_evolve_matches_reference():
    """C1 evolved on 3 loopback ranks (Morton-renumbered partition), the owned
    fields all-gathered (distributed.gathered_field), then the dual API: the
    reference's C1 dual, exactly."""
    from paper_1804_09152_b200 import distributed as D
    mesh = ft.gen_icosphere(4)
    lap = ft.build_laplacian(mesh)
    f0 = _field("c1_traj.npz", 0)
    ren = D.Renumbering.morton(mesh)
    part = D.Partition.even(mesh.n_vertices, 3)
    tr = D.LoopbackTransport()
    probs = [D.local_problem(f0.phi, lap, part, r, renumbering=ren) for r in range(3)]
    plans = D.build_plans(probs, tr)
    ranks = [D.DomainRank(p, pl, renumbering=ren) for p, pl in zip(probs, plans)]
    steps, _ = D.evolve_partitioned(ranks, tr, ft.CouplingParams(), max_steps=500, tol=0.0)
    assert steps == 500
    fld = D.gathered_field(ranks, tr, f0.seed_vertices, renumbering=ren)
    ref_fld = _field("c1_traj.npz", 500)
    assert np.array_equal(np.asarray(fld.phi.values[:fld.phi.nnz]), np.asarray(ref_fld.phi.values[:ref_fld.phi.nnz]))
    ref = golden_json("c1_dual.json")
    a_v = ft.vertex_adjacency(fld, 0.25)
    a_t = ft.triangle_adjacency(fld, mesh, 0.25)
    cur = ft.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
    assert sorted(map(list, cur.pairs())) == ref["curated"]
    dm = ft.build_dual(cur, np.zeros((fld.n_cells, 3)))
    assert sorted(map(sorted, dm.triangles.tolist())) == ref["triangles"]


@pytest.mark.gpu
@pytest.mark.parametrize("name,traj,snap,level", [("c1", "c1_traj.npz", 500, 4), ("c2", "c2_traj.npz", 1000, 7)])
def test_dual_winding_and_normal_flip_match_reference(name, traj, snap, level):
    """The exact triangle list of build_dual -- order, winding (the
    depth-first propagation) and the majority-normal flip with outward and
    inward cell normals -- equals the reference's (golden dual_winding.json,
    ref dual.py:284-391)."""
    ref = golden_json("dual_winding.json").get(name)
    if ref is None:
        pytest.skip("no winding golden")
    mesh = ft.gen_icosphere(level)
    fld = _field(traj, snap)
    cur = ft.confirm_candidates(fld, mesh, ft.vertex_adjacency(fld, 0.25), ft.triangle_adjacency(fld, mesh, 0.25),
                                0.25)
    pos = mesh.positions[np.asarray(fld.seed_vertices, dtype=np.int64)]
    nrm = pos / np.linalg.norm(pos, axis=1)[:, None]
    assert ft.build_dual(cur, np.zeros((fld.n_cells, 3))).triangles.tolist() == ref["plain"]
    assert ft.build_dual(cur, pos, cell_normals=nrm).triangles.tolist() == ref["outward"]
    assert ft.build_dual(cur, pos, cell_normals=-nrm).triangles.tolist() == ref["inward"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["degenerate", "nonfinite"])
def test_confirm_candidates_warnings_match_reference(case):
    """A zero-area face (one vertex moved onto its neighbour) or a NaN in a
    layer: the device crossing test skips it, the RuntimeWarnings are the
    reference's in order, and the curated adjacency is unchanged from the
    reference's (golden dual_warnings.json, ref dual.py:181-205)."""
    import warnings
    ref = golden_json("dual_warnings.json")[case]
    mesh = ft.gen_icosphere(4)
    fld = _field("c1_traj.npz", 500)
    if case == "degenerate":
        v_from, v_to = ref["move"]
        pos = mesh.positions.copy()
        pos[v_from] = pos[v_to]
        mesh = ft.TriMesh(pos, mesh.faces.copy())
    else:
        phi = fld.phi
        vals = np.array(phi.values[:phi.nnz], dtype=np.float64)
        vals[ref["nan_entry"]] = np.nan
        fld = ft.LayeredField(ft.SparseMat(phi.n_rows, phi.n_cols, phi.col_ptr, phi.row_idx[:phi.nnz], vals,
                                           check=False), fld.seed_vertices, step_count=500)
    a_v = ft.vertex_adjacency(fld, 0.4)
    a_t = ft.triangle_adjacency(fld, mesh, 0.4)
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        cur = ft.confirm_candidates(fld, mesh, a_v, a_t, 0.4)
    got = [str(w.message) for w in rec if issubclass(w.category, RuntimeWarning)]
    assert got == ref["warnings"] and got
    assert sorted(map(list, cur.pairs())) == ref["curated"]
    assert [list(d) for d in cur.dropped] == ref["dropped"]


@pytest.mark.gpu
def test_confirm_candidates_clean_field_does_not_warn():
    import warnings
    mesh, fld = ft.gen_icosphere(4), _field("c1_traj.npz", 500)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        ft.confirm_candidates(fld, mesh, ft.vertex_adjacency(fld, 0.4), ft.triangle_adjacency(fld, mesh, 0.4), 0.4)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_dual_adjacency_partitioned_without_gather(world):
    """The dual adjacency of a partitioned field from per-rank device products
    united over ranks (distributed.dual_adjacency_partitioned: no field
    gather): the reference's C1 A_v, A_t, curated pairs, triples and
    triangles, exactly."""
    from paper_1804_09152_b200 import distributed as D
    mesh = ft.gen_icosphere(4)
    lap = ft.build_laplacian(mesh)
    f0 = _field("c1_traj.npz", 0)
    ren = D.Renumbering.morton(mesh)
    part = D.Partition.even(mesh.n_vertices, world)
    tr = D.LoopbackTransport()
    probs = [D.local_problem(f0.phi, lap, part, r, renumbering=ren) for r in range(world)]
    ranks = [D.DomainRank(p, pl, renumbering=ren) for p, pl in zip(probs, D.build_plans(probs, tr))]
    D.evolve_partitioned(ranks, tr, ft.CouplingParams(), max_steps=500, tol=0.0)
    a_v, a_t, cur = D.dual_adjacency_partitioned(ranks, tr, mesh, 0.25, renumbering=ren)
    ref = golden_json("c1_dual.json")
    assert sorted(map(list, a_v.pairs())) == ref["a_v"]
    assert sorted(map(list, a_t.pairs())) == ref["a_t"]
    assert sorted(map(list, cur.pairs())) == ref["curated"]
    assert sorted(map(list, cur.junction_triples)) == ref["triples"]
    dm = ft.build_dual(cur, np.zeros((f0.n_cells, 3)))
    assert sorted(map(sorted, dm.triangles.tolist())) == ref["triangles"]
