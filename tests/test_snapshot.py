"""Snapshot wire-format compatibility with files the REFERENCE wrote
(§8(f)3; ref field.py:372-404, sparse.py:427-464).  The fixtures
tests/golden/c1_s10.field / .trip come from the reference's own save_field /
write_triplets (tests/golden/make_golden.py, make_snapshots): loading them
must give the reference's matrix bitwise, and saving what was loaded must
reproduce the reference's bytes."""

import os

import numpy as np
import pytest

import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import sparse as sp
from paper_1804_09152_b200.errors import ShapeError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _c1_s10():
    t = np.load(os.path.join(GOLD, "c1_traj.npz"))
    return t, t["s10_ptr"], t["s10_idx"], t["s10_val"]


def test_reference_field_snapshot_loads_bitwise():
    t, ptr, idx, val = _c1_s10()
    fld, params = ft.load_field(os.path.join(GOLD, "c1_s10.field"))
    assert fld.step_count == 10
    assert np.array_equal(fld.seed_vertices, t["seeds"])
    assert params == ft.CouplingParams(dt=0.05, mu=2.5)
    phi = fld.phi
    assert (phi.n_rows, phi.n_cols) == tuple(int(x) for x in t["s10_shape"])
    assert np.array_equal(phi.col_ptr, ptr)
    assert np.array_equal(phi.row_idx[:phi.nnz], idx)
    assert phi.values[:phi.nnz].tobytes() == np.asarray(val, dtype=np.float64).tobytes()


def test_save_field_is_byte_identical_to_reference(tmp_path):
    src = os.path.join(GOLD, "c1_s10.field")
    fld, params = ft.load_field(src)
    out = tmp_path / "again.field"
    ft.save_field(fld, params, str(out), extra_header={"mesh": "icosphere-4"})
    with open(src, "rb") as a:
        ref = a.read()
    assert out.read_bytes() == ref


def test_triplets_round_trip_byte_identical(tmp_path):
    src = os.path.join(GOLD, "c1_s10.trip")
    m = sp.read_triplets(src)
    _, ptr, idx, val = _c1_s10()
    assert np.array_equal(m.col_ptr, ptr) and np.array_equal(m.row_idx[:m.nnz], idx)
    assert np.array_equal(m.values[:m.nnz], val)
    out = tmp_path / "again.trip"
    sp.write_triplets(m, str(out), comments=("fieldtess triplets", "step 10"))
    with open(src, "rb") as a:
        assert out.read_bytes() == a.read()


def test_snapshot_rejects_plain_triplets():
    with pytest.raises(ShapeError):
        ft.load_field(os.path.join(GOLD, "c1_s10.trip"))
