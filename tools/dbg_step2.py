import sys, ctypes
import numpy as np
import torch
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import field as F, _lib
from oracle import pyoracle as O

mesh = ft.gen_icosphere(4)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 64, replace=False)
lap = ft.build_laplacian(mesh)
lt = O.Csc.of(ft.field._with_diagonal(lap.mat_t))
cur = ft.init_field(mesh, seeds)
prm = ft.CouplingParams()
for k in range(7):
    cur, _ = ft.step(cur, lap, prm)
inp = O.Csc.of(cur.phi)
ref, st = O.step_c(inp, lt, prm)
# manual launch with big scratch, inspect control
dphi = cur.device_phi()
n_v = mesh.n_vertices
dl = F.device_laplacian(lap, "exact")
for pool in (0, 100000):
    ws = F.StepWorkspace(); ws.prepare(n_v, dphi.values.device)
    cap = int(_lib.lib().ft_tiled_min_capacity(n_v)) + max(pool, 1)
    t = ft.DeviceTiled(dphi.n_rows, n_v, cap, dphi.values.dtype, dphi.values.device)
    wp, wn = ws.ws_args()
    sh = F._stream_handle()
    rc = _lib.lib().ft_step_kernel(ctypes.byref(dl.lap_t["exact"].ft_csc()), dl.flags, ctypes.byref(dphi.ft_csc()), None,
                                   ctypes.byref(t.ft_tiled()), 0, ctypes.byref(prm.ft_params()), wp, wn, sh)
    torch.cuda.synchronize()
    ctl = ws.ws[:128].cpu().numpy().view(np.int64)
    print("pool", pool, "cap", cap, "rc", rc, "ctl words", ctl[:12])
    d = t.desc.view(-1, 2).cpu().numpy()
    print(" tile0 desc", d[:6].tolist(), "sum cnt tile0", d[:128, 1].sum(), "tile1", d[128:256, 1].sum())
    rc = _lib.lib().ft_step_fixup(ctypes.byref(dl.lap_t["exact"].ft_csc()), dl.flags, ctypes.byref(dphi.ft_csc()), None,
                                   ctypes.byref(t.ft_tiled()), 0, ctypes.byref(prm.ft_params()), wp, wn, sh)
    rc = _lib.lib().ft_step_finalize(wp, wn, n_v, t.capacity, ctypes.c_void_p(ws.stats.data_ptr()), sh)
    torch.cuda.synchronize()
    rec = np.frombuffer(ws.stats.cpu().numpy().tobytes(), dtype=_lib.STATS_DTYPE)[0]
    print(" record", rec)
