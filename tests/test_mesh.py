"""Generators and Laplacian are order- and bit-identical to the reference
(SHA-256 digests of the reference's outputs in tests/golden/meshes.json)."""

import hashlib

import numpy as np
import pytest

import paper_1804_09152_b200 as ft
from conftest import golden_json


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _mesh(name):
    if name.startswith("ico"):
        return ft.gen_icosphere(int(name[3:]))
    nx, ny = map(int, name[5:].split("x"))
    return ft.gen_periodic_grid(nx, ny)


@pytest.mark.parametrize("name", sorted(golden_json("meshes.json")))
def test_generator_bitwise(name):
    ref = golden_json("meshes.json")[name]
    m = _mesh(name)
    lap = ft.build_laplacian(m)
    nnz = lap.mat_t.nnz
    assert m.n_vertices == ref["n_vertices"] and m.n_faces == ref["n_faces"]
    assert sha(m.faces.astype(np.int32)) == ref["faces"]
    assert sha(m.positions) == ref["positions"]
    assert sha(m.face_area) == ref["face_area"]
    assert sha(m.vertex_area) == ref["vertex_area"]
    assert sha(lap.mat_t.col_ptr) == ref["lapt_ptr"]
    assert sha(lap.mat_t.row_idx[:nnz]) == ref["lapt_idx"]
    assert sha(lap.mat_t.values[:nnz]) == ref["lapt_val"]


def test_icosphere_beyond_reference_cap():
    m = ft.gen_icosphere(8, max_subdiv=8)
    assert m.n_vertices == 10 * 4 ** 8 + 2 and m.n_faces == 20 * 4 ** 8
    assert m.euler_characteristic() == 2
    assert np.all(m.degree >= 5) and np.all(m.degree <= 6)


def test_laplacian_rows_sum_zero():
    m = ft.gen_icosphere(3)
    lap = ft.build_laplacian(m)
    d = lap.mat.to_dense()
    assert np.abs(d.sum(axis=1)).max() < 1e-12
    assert np.array_equal(lap.mat_t.to_dense(), d.T)


def test_cotan_laplacian_matches_golden_case():
    from conftest import csc_from, golden_npz
    g = golden_npz("step_cases.npz")
    ref = csc_from(g, "cotan_ico2_lapt")
    lap = ft.build_laplacian(ft.gen_icosphere(2), "cotan-clamped")
    assert np.array_equal(lap.mat_t.col_ptr, ref.col_ptr)
    assert np.array_equal(lap.mat_t.row_idx[:lap.mat_t.nnz], ref.row_idx)
    assert np.array_equal(lap.mat_t.values[:lap.mat_t.nnz], ref.values)


def test_torus_counts_and_degree():
    m = ft.gen_periodic_grid(5, 4)
    assert m.n_vertices == 20 and m.n_faces == 40 and m.euler_characteristic() == 0
    assert np.all(m.degree == 6)


def test_errors():
    with pytest.raises(ft.errors.MeshFormatError):
        ft.gen_periodic_grid(2, 5)
    with pytest.raises(ft.errors.MeshFormatError):
        ft.gen_icosphere(13)
    with pytest.raises(ft.errors.MeshFormatError):
        ft.TriMesh(np.zeros((3, 3)), [[0, 0, 1]])
