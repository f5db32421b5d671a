"""The oracle is pinned to the reference's own outputs (golden vectors made
by tests/golden/make_golden.py from the reference package)."""

import numpy as np
import pytest

from conftest import P, assert_csc_equal, csc_from, golden_json, golden_npz
from oracle import pyoracle as po


@pytest.fixture(scope="module")
def cases():
    return golden_npz("step_cases.npz")


@pytest.mark.parametrize("impl", ["py", "c"])
def test_step_cases_bitwise(cases, impl):
    f = po.step_py if impl == "py" else po.step_c
    for name in cases["names"]:
        out, st = f(csc_from(cases, f"{name}_in"), csc_from(cases, f"{name}_lapt"),
                    P(cases[f"{name}_params"]))
        assert_csc_equal(out, csc_from(cases, f"{name}_out"))
        ref = cases[f"{name}_stats"]
        assert st["max_delta"] == ref[0] and st["base_mass"] == ref[1], name


def test_multi_step_torus9(cases):
    cur = csc_from(cases, "multi_in")
    lapt = csc_from(cases, "multi_lapt")
    for _ in range(5):
        cur, _ = po.step_c(cur, lapt, P([0.2, 1.0, 0.3, 0.2, 0.2, 5.0]))
    assert_csc_equal(cur, csc_from(cases, "multi_out"))


@pytest.mark.parametrize("traj", ["c1_traj.npz", "torus_traj.npz"])
def test_trajectory_bitwise(traj):
    t = golden_npz(traj)
    cur = csc_from(t, "s0")
    lapt = csc_from(t, "lapt")
    prm = P([0.2, 1.0, 0.3, 0.2, 0.2, 5.0])
    last = int(t["snaps"][-1])
    for k in range(1, last + 1):
        cur, st = po.step_c(cur, lapt, prm, n_threads=2)
        tr = t["trace"][k - 1]
        assert st["max_delta"] == tr[0] and st["base_mass"] == tr[1] and cur.nnz == tr[2], k
        if k in t["snaps"]:
            assert_csc_equal(cur, csc_from(t, f"s{k}"))
    assert np.array_equal(po.labels_np(cur), t["labels_final"])


def test_labels_cases():
    g = golden_npz("labels.npz")
    for name in g["names"]:
        assert np.array_equal(po.labels_np(csc_from(g, name)), g[f"{name}_labels"]), name


def test_init_field_oracle_matches_golden():
    from paper_1804_09152_b200 import gen_icosphere
    mesh = gen_icosphere(4)
    t = golden_npz("c1_traj.npz")
    phi = po.init_field_np(mesh.neighbor_ptr, mesh.neighbor_idx, mesh.n_vertices, t["seeds"])
    assert_csc_equal(phi, csc_from(t, "s0"))


def test_py_and_c_agree_on_random_fields():
    rng = np.random.default_rng(11)
    from paper_1804_09152_b200 import build_laplacian, gen_periodic_grid
    mesh = gen_periodic_grid(7, 6)
    lap = build_laplacian(mesh)
    for _ in range(10):
        n_cells = int(rng.integers(1, 9))
        dense = np.zeros((n_cells + 1, mesh.n_vertices))
        for r in range(1, n_cells + 1):
            sup = rng.choice(mesh.n_vertices, size=int(rng.integers(2, 20)), replace=False)
            dense[r, sup] = rng.random(sup.size)
        dense[0] = np.maximum(1.0 - dense.sum(axis=0), 0.0)
        dense /= dense.sum(axis=0, keepdims=True)
        from paper_1804_09152_b200 import SparseMat
        phi = SparseMat.from_dense(dense)
        prm = P([0.2, 1.0, rng.uniform(0, .5), rng.uniform(0, .5), rng.uniform(.05, .4), rng.uniform(1, 5)])
        a, sa = po.step_py(phi, lap.mat_t, prm)
        b, sb = po.step_c(phi, lap.mat_t, prm)
        assert_csc_equal(a, b)
        assert sa == sb
