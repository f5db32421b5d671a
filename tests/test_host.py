"""Host-side logic that runs without a GPU: the C-ABI library loads and
exports every declared symbol, seeding, sparse containers, snapshots."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import _lib
from conftest import REPO, assert_csc_equal, csc_from, golden_json, golden_npz


def declared_symbols():
    src = open(os.path.join(REPO, "include", "fieldtess_cuda.h")).read()
    return sorted(set(re.findall(r"\b(ft_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert syms, "no symbols parsed from the header"
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_header_constants_match_the_binding():
    """Every #define FT_* integer of the header equals the constant of the
    same name in _lib (flags, dtypes, status codes, phases, hints)."""
    src = open(os.path.join(REPO, "include", "fieldtess_cuda.h")).read()
    defs = dict(re.findall(r"^#define (FT_[A-Z0-9_]+)\s+(-?\d+)\b", src, flags=re.M))
    assert "FT_HINT_DENSE_BAND" in defs and "FT_LAP_SYMMETRIC" in defs
    for name, value in defs.items():
        if hasattr(_lib, name):
            assert getattr(_lib, name) == int(value), name
    missing = [n for n in defs if n.startswith(("FT_LAP_", "FT_HINT_", "FT_STATUS_", "FT_PHASE_", "FT_F"))
               and not hasattr(_lib, n)]
    assert not missing, missing


def test_abi_version_and_structs():
    lib = _lib.lib()
    assert lib.ft_abi_version() == _lib.ABI_VERSION
    assert ctypes.sizeof(_lib.FtStepStats) == 64
    assert lib.ft_workspace_bytes(1000) > 0


def test_init_field_matches_reference_seeding():
    t = golden_npz("c1_traj.npz")
    f = ft.init_field(ft.gen_icosphere(4), t["seeds"])
    assert_csc_equal(f.phi, csc_from(t, "s0"))
    t2 = golden_npz("torus_traj.npz")
    f2 = ft.init_field(ft.gen_periodic_grid(64, 64), t2["seeds"])
    assert_csc_equal(f2.phi, csc_from(t2, "s0"))


def test_init_field_errors_and_split():
    m = ft.gen_periodic_grid(9, 9)
    with pytest.raises(ft.errors.DuplicateSeedError):
        ft.init_field(m, [4, 4])
    with pytest.raises(ft.errors.ShapeError):
        ft.init_field(m, [81])
    f = ft.init_field(m, [40, 41])
    ring_a = set(m.neighbors(40).tolist()) | {40}
    ring_b = set(m.neighbors(41).tolist()) | {41}
    v = (ring_a & ring_b).pop()
    assert f.phi.get(1, v) == 0.5 and f.phi.get(2, v) == 0.5
    assert np.abs(f.column_sums() - 1).max() < 1e-12
    assert f.base_mass() == 81 - len(ring_a | ring_b)


def test_sparsemat_basics():
    a = ft.SparseMat.from_dense([[1, 0], [2, 3]])
    assert a.nnz == 3 and a.get(1, 0) == 2.0 and a.get(0, 1) == 0.0
    t = ft.transpose(a)
    assert np.array_equal(t.to_dense(), a.to_dense().T)
    with pytest.raises(ft.errors.ShapeError):
        ft.SparseMat(2, 1, [0, 2], [1, 0], [1.0, 1.0])
    m = ft.SparseMat.empty(3, 3, 10)
    ft.ensure_capacity(m, 11)
    assert m.capacity == 12 and m.realloc_count == 1


def test_snapshot_round_trip(tmp_path):
    t = golden_npz("c1_traj.npz")
    phi = ft.SparseMat(*t["s10_shape"], t["s10_ptr"], t["s10_idx"], t["s10_val"])
    fld = ft.LayeredField(phi, t["seeds"], step_count=10)
    p = tmp_path / "f.txt"
    ft.save_field(fld, ft.CouplingParams(), p)
    back, prm = ft.load_field(p)
    assert prm == ft.CouplingParams() and back.step_count == 10
    assert np.array_equal(back.phi.to_dense(), phi.to_dense())


def test_params_validation():
    with pytest.raises(ft.errors.ShapeError):
        ft.CouplingParams(w=0).validate()
    with pytest.raises(ft.errors.ShapeError):
        ft.CouplingParams(e=-1).validate()


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = ft.gen_periodic_grid(6, 6)
    f = ft.init_field(m, [0])
    with pytest.raises(ft.errors.BackendError):
        ft.step(f, ft.build_laplacian(m), ft.CouplingParams())


def _walk(tris):
    """The winding walk of dual.py:284-313 restated in Python (the checker)."""
    t = [list(map(int, r)) for r in tris]
    edges = {}
    for i, x in enumerate(t):
        for s in range(3):
            u, v = x[s], x[(s + 1) % 3]
            edges.setdefault((min(u, v), max(u, v)), []).append(i)
    seen = [False] * len(t)
    for root in range(len(t)):
        if seen[root]:
            continue
        seen[root] = True
        stack = [root]
        while stack:
            cur = stack.pop()
            x = t[cur]
            for s in range(3):
                u, v = x[s], x[(s + 1) % 3]
                for o in edges[(min(u, v), max(u, v))]:
                    if o == cur or seen[o]:
                        continue
                    y = t[o]
                    if (y[0] == u and y[1] == v) or (y[1] == u and y[2] == v) or (y[2] == u and y[0] == v):
                        t[o] = [y[0], y[2], y[1]]
                    seen[o] = True
                    stack.append(o)
    return np.asarray(t, dtype=np.int32).reshape(-1, 3)


def test_wind_triangles_matches_the_walk():
    """ft_wind_triangles (host C++, no GPU) is the reference's depth-first
    winding, triangle for triangle: a random closed surface, a Moebius strip
    (non-orientable: the result depends on the visiting order) and a
    non-manifold fan."""
    from paper_1804_09152_b200 import dual
    rng = np.random.default_rng(3)
    cases = []
    # an octahedron with random windings
    octa = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4], [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]])
    flip = rng.random(8) < 0.5
    octa[flip] = octa[flip][:, [0, 2, 1]]
    cases.append(octa)
    # Moebius strip of 8 triangles
    cases.append(np.array([[0, 1, 2], [1, 3, 2], [2, 3, 4], [3, 5, 4], [4, 5, 6], [5, 7, 6], [6, 7, 1], [7, 0, 1]]))
    # three triangles on one edge, then random soup
    cases.append(np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4], [2, 1, 5]]))
    cases.append(rng.integers(0, 40, size=(300, 3)))
    for c in cases:
        c = c[(c[:, 0] != c[:, 1]) & (c[:, 1] != c[:, 2]) & (c[:, 0] != c[:, 2])]
        assert np.array_equal(dual._wind(c), _walk(c))
