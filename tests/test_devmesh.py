"""Device mesh generation, derived data, uniform Laplacian and init_field
(§8(f)1-2, devmesh.py / ft_mesh.cu) -- bitwise the reference's outputs
(SHA-256 digests in tests/golden/meshes.json) and equal to the host
restatements array for array."""

import hashlib

import numpy as np
import pytest

import paper_1804_09152_b200 as ft
from conftest import golden_json

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _gen(name):
    if name.startswith("ico"):
        return ft.gen_icosphere(int(name[3:]))
    nx, ny = map(int, name[5:].split("x"))
    return ft.gen_periodic_grid(nx, ny)


@pytest.mark.parametrize("name", sorted(golden_json("meshes.json")))
def test_device_generator_bitwise(name):
    ref = golden_json("meshes.json")[name]
    m = _gen(name)
    assert m.device_arrays() is not None, "the device generator did not run"
    lap = ft.build_laplacian(m)
    assert lap.device is not None, "the device Laplacian did not run"
    nnz = lap.mat_t.nnz
    assert m.n_vertices == ref["n_vertices"] and m.n_faces == ref["n_faces"]
    assert sha(m.faces.astype(np.int32)) == ref["faces"]
    assert sha(m.positions) == ref["positions"]
    assert sha(m.face_area) == ref["face_area"]
    assert sha(m.vertex_area) == ref["vertex_area"]
    assert sha(lap.mat_t.col_ptr) == ref["lapt_ptr"]
    assert sha(lap.mat_t.row_idx[:nnz]) == ref["lapt_idx"]
    assert sha(lap.mat_t.values[:nnz]) == ref["lapt_val"]


def _host(monkeypatch, fn, *args):
    monkeypatch.setenv("FT_HOST_MESH", "1")
    try:
        return fn(*args)
    finally:
        monkeypatch.delenv("FT_HOST_MESH")


@pytest.mark.parametrize("kind,args", [("ico", (8,)), ("torus", (41, 37)), ("torus", (3, 3))])
def test_device_mesh_equals_host(monkeypatch, kind, args):
    gen = (lambda *a: ft.gen_icosphere(*a, max_subdiv=8)) if kind == "ico" else ft.gen_periodic_grid
    d = gen(*args)
    h = _host(monkeypatch, gen, *args)
    assert d.device_arrays() is not None and h.device_arrays() is None
    for attr in ("positions", "faces", "edges", "degree", "neighbor_ptr", "neighbor_idx", "face_area",
                 "face_normal", "face_barycenter", "vertex_area"):
        a, b = getattr(d, attr), getattr(h, attr)
        assert a.dtype == b.dtype and a.shape == b.shape, attr
        assert a.tobytes() == b.tobytes(), attr
    ld, lh = ft.build_laplacian(d), ft.build_laplacian(h)
    for which in ("mat", "mat_t"):
        x, y = getattr(ld, which), getattr(lh, which)
        assert np.array_equal(x.col_ptr, y.col_ptr)
        assert np.array_equal(x.row_idx[:x.nnz], y.row_idx[:y.nnz])
        assert x.values[:x.nnz].tobytes() == y.values[:y.nnz].tobytes()


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_device_init_field_equals_host(monkeypatch, precision):
    d = ft.gen_icosphere(6)
    h = _host(monkeypatch, ft.gen_icosphere, 6)
    seeds = ft.sample_seed_vertices(d, 300, 4)
    assert np.array_equal(seeds, ft.sample_seed_vertices(h, 300, 4))
    fd = ft.init_field(d, seeds, precision=precision)
    fh = ft.init_field(h, seeds, precision=precision)
    assert fd._dev is not None and fd._host is None
    a, b = fd.device_phi().to_host(), fh.device_phi().to_host()
    assert np.array_equal(a.col_ptr, b.col_ptr)
    assert np.array_equal(a.row_idx[:a.nnz], b.row_idx[:b.nnz])
    assert a.values[:a.nnz].tobytes() == b.values[:b.nnz].tobytes()


def test_device_mesh_evolve_matches_host_mesh(monkeypatch):
    """The engine on a device-built mesh + Laplacian (no host copy of L)
    gives the same field as on the host-built ones."""
    d = ft.gen_periodic_grid(64, 64)
    h = _host(monkeypatch, ft.gen_periodic_grid, 64, 64)
    seeds = ft.sample_seed_vertices(h, 24, 0)
    ld = ft.build_laplacian(d)
    out_d, tr_d = ft.evolve(ft.init_field(d, seeds), ld, ft.CouplingParams(), max_steps=60, tol=0.0)
    assert ld._mat_t is None, "the device Laplacian was copied to the host"
    from paper_1804_09152_b200 import field as F
    assert F.device_laplacian(ld, "exact").pack is not None, "uniform device Laplacian not packed"
    out_h, tr_h = ft.evolve(ft.init_field(h, seeds), ft.build_laplacian(h), ft.CouplingParams(), max_steps=60,
                            tol=0.0)
    a, b = out_d.phi, out_h.phi
    assert np.array_equal(a.col_ptr, b.col_ptr) and a.values[:a.nnz].tobytes() == b.values[:b.nnz].tobytes()
    assert [s.max_delta for s in tr_d] == [s.max_delta for s in tr_h]


def test_device_mesh_lloyd_geometry_reused():
    m = ft.gen_icosphere(4)
    from paper_1804_09152_b200.lloyd import device_mesh
    dm = device_mesh(m)
    assert dm.positions.data_ptr() == m.device_arrays()[0].data_ptr()


def test_locality_order_evolve_is_bitwise(monkeypatch):
    """A device-built unstructured mesh's Laplacian carries a Morton order;
    evolve runs permuted and returns the caller's numbering: the field and
    trace equal the unpermuted run bitwise, and an error (a NaN input: the
    pattern check fires first, as in the reference) reports the same
    column as without the order."""
    from paper_1804_09152_b200 import devmesh, field as F
    monkeypatch.setattr(devmesh, "LOCALITY_MIN_VERTICES", 0)
    mesh = ft.gen_icosphere(5)
    lap = ft.build_laplacian(mesh)
    assert lap.device.get("order") is not None
    seeds = ft.sample_seed_vertices(mesh, 80, 1)
    fld = ft.init_field(mesh, seeds)
    assert F.device_laplacian(lap, "exact").renum is not None
    out, tr = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=60, tol=0.0)
    monkeypatch.setattr(F, "LOCALITY_MIN_STEPS", 10 ** 9)       # the plain path
    ref, rtr = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=60, tol=0.0)
    a, b = out.phi, ref.phi
    assert np.array_equal(a.col_ptr, b.col_ptr) and np.array_equal(a.row_idx[:a.nnz], b.row_idx[:b.nnz])
    assert a.values[:a.nnz].tobytes() == b.values[:b.nnz].tobytes()
    assert [s.max_delta for s in tr] == [s.max_delta for s in rtr]
    assert [s.nnz_skel for s in tr] == [s.nnz_skel for s in rtr]
    # an error is reported in the caller's numbering
    phi = ref.phi
    vals = np.array(phi.values[:phi.nnz])
    vals[phi.nnz // 2] = np.nan
    bad = ft.LayeredField(ft.SparseMat(phi.n_rows, phi.n_cols, phi.col_ptr, phi.row_idx[:phi.nnz], vals,
                                       check=False), seeds, step_count=60)
    with pytest.raises(ft.TessError) as plain:
        ft.evolve(bad, lap, ft.CouplingParams(), max_steps=20, tol=0.0)
    monkeypatch.setattr(F, "LOCALITY_MIN_STEPS", 8)
    with pytest.raises(ft.TessError) as permuted:
        ft.evolve(bad, lap, ft.CouplingParams(), max_steps=20, tol=0.0)
    assert type(permuted.value) is type(plain.value) and str(permuted.value) == str(plain.value)
