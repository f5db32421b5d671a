import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class P:
    """Plain parameter record (w, a, e, e_base, mu, dt)."""

    def __init__(self, arr):
        self.w, self.a, self.e, self.e_base, self.mu, self.dt = (float(x) for x in arr)


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def csc_from(g, prefix):
    from oracle.pyoracle import Csc
    sh = g[prefix + "_shape"]
    return Csc(sh[0], sh[1], g[prefix + "_ptr"], g[prefix + "_idx"], g[prefix + "_val"])


def assert_csc_equal(a, b, exact=True, rtol=0.0, atol=0.0):
    nnz_a = int(a.col_ptr[a.n_cols])
    nnz_b = int(b.col_ptr[b.n_cols])
    assert (a.n_rows, a.n_cols) == (b.n_rows, b.n_cols)
    assert np.array_equal(np.asarray(a.col_ptr, dtype=np.int64), np.asarray(b.col_ptr, dtype=np.int64))
    assert np.array_equal(np.asarray(a.row_idx[:nnz_a]), np.asarray(b.row_idx[:nnz_b]))
    va = np.asarray(a.values[:nnz_a], dtype=np.float64)
    vb = np.asarray(b.values[:nnz_b], dtype=np.float64)
    if exact:
        assert np.array_equal(va, vb), f"max |diff| {np.abs(va - vb).max()}"
    else:
        np.testing.assert_allclose(va, vb, rtol=rtol, atol=atol)
