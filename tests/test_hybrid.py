"""The hybrid ELL(2) + pool working layout (ft_tiled, ABI v5): the host
encoder, and on the GPU the canonical -> hybrid -> canonical round trip
through the C-ABI (ft_tiled_from_csc, ft_compact) with empty, one-, two-
and many-entry columns, non-finite values and a pool that overflows."""

import ctypes

import numpy as np
import pytest

from paper_1804_09152_b200.sparse import hybrid_columns

PAIR = 1 << 30


def random_csc(rng, n_cols, n_rows, max_cnt=9, dtype=np.float64):
    cnt = rng.integers(0, max_cnt + 1, n_cols)
    cnt[rng.random(n_cols) < 0.5] = 1          # mostly single entries, like a field
    cnt[: min(4, n_cols)] = [0, 1, 2, 3][: min(4, n_cols)]
    cnt = np.minimum(cnt, n_rows)
    col_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    rows = np.concatenate([np.sort(rng.choice(n_rows, c, replace=False)) for c in cnt]).astype(np.int32)
    vals = rng.random(rows.size).astype(dtype) + dtype(0.01)
    return col_ptr, rows, vals


def test_hybrid_columns_encoding():
    """Host encoder against a per-column restatement of the layout rules."""
    rng = np.random.default_rng(3)
    cp, ri, va = random_csc(rng, 500, 40)
    sig, aux, v0, v1, pidx, pval = hybrid_columns(cp, ri, va, pool_base=7)
    off = 7
    got_pool = 0
    for j in range(cp.size - 1):
        a, b = cp[j], cp[j + 1]
        c = b - a
        if c == 0:
            assert sig[j] == -1
        elif c == 1:
            assert sig[j] == ri[a] and v0[j] == va[a]
        elif c == 2:
            assert sig[j] == (ri[a] | PAIR) and aux[j] == ri[a + 1]
            assert v0[j] == va[a] and v1[j] == va[a + 1]
        else:
            assert sig[j] == -c and aux[j] == off
            assert np.array_equal(pidx[off - 7:off - 7 + c], ri[a:b])
            assert np.array_equal(pval[off - 7:off - 7 + c], va[a:b])
            off += c
            got_pool += c
    assert pidx.size == got_pool


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_hybrid_roundtrip_device(precision):
    import torch

    import paper_1804_09152_b200 as ft
    from paper_1804_09152_b200 import _lib
    from paper_1804_09152_b200 import field as F

    dt = np.float64 if precision == "exact" else np.float32
    rng = np.random.default_rng(11)
    n_cols, n_rows = 5000, 60
    cp, ri, va = random_csc(rng, n_cols, n_rows, dtype=dt)
    va[17] = np.inf                                     # non-finite values survive the trip
    src = ft.DeviceCSC.from_host(ft.SparseMat(n_rows, n_cols, cp, ri, va.astype(np.float64), check=False),
                                 torch.float64 if dt == np.float64 else torch.float32, torch.device("cuda"))
    lib = _lib.lib()
    ws = ft.StepWorkspace()
    ws.prepare(n_cols, torch.device("cuda"))
    wp, wn = ws.ws_args()
    stream = F._stream_handle()
    code = F._ft_dtype(precision)
    sig, aux, v0, v1, pidx, pval = hybrid_columns(cp, ri, va)
    for cap in (pidx.size, pidx.size // 2):             # exact fit, then a pool overflow
        hyb = ft.DeviceTiled(n_rows, n_cols, cap, src.values.dtype, src.values.device)
        rec = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device="cuda")
        s_c, h_c = src.ft_csc(), hyb.ft_tiled()
        assert lib.ft_tiled_from_csc(ctypes.byref(s_c), ctypes.byref(h_c), code, wp, wn,
                                     ctypes.c_void_p(rec.data_ptr()), stream) == 0
        r = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=_lib.STATS_DTYPE)[0]
        if cap < pidx.size:
            assert int(r["status"]) == _lib.FT_STATUS_OVERFLOW and int(r["needed"]) >= pidx.size
            continue
        assert int(r["status"]) == 0
        small = np.diff(cp) <= 2
        assert np.array_equal(hyb.sig.cpu().numpy()[small], sig[small])
        assert np.array_equal(hyb.v0.cpu().numpy()[np.diff(cp) >= 1][small[np.diff(cp) >= 1]],
                              v0[np.diff(cp) >= 1][small[np.diff(cp) >= 1]])
        out = ft.DeviceCSC.allocate(n_rows, n_cols, cp[-1] + 1, src.values.dtype, src.values.device)
        o_c = out.ft_csc()
        assert lib.ft_compact(ctypes.byref(h_c), ctypes.byref(o_c), code, wp, wn,
                              ctypes.c_void_p(rec.data_ptr()), stream) == 0
        r = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=_lib.STATS_DTYPE)[0]
        assert int(r["status"]) == 0 and int(r["nnz_phi"]) == cp[-1]
        assert np.array_equal(out.col_ptr.cpu().numpy(), cp)
        assert np.array_equal(out.row_idx[:cp[-1]].cpu().numpy(), ri)
        assert np.array_equal(out.values[:cp[-1]].cpu().numpy(), va)
        # the conversion raised the sticky non-finite flag (offset 180 of the control block)
        ctl = ws.ws[:224].cpu().numpy()
        assert int(ctl[180:184].view(np.uint32)[0]) == 1
