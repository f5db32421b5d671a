"""Stage timeline of one C3 step (fixed input state, repeated): tier 1 /
fork / queue A / tier 2a(A) / warp tail(A) on the side stream, tier 1.5 /
tail(B) on the main stream, join.  Sets FT_PROBE_EVENTS=1 (debug export
ft_probe_timeline)."""
import ctypes
import os
import sys

os.environ["FT_PROBE_EVENTS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401

import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import _lib, field as F

a = [int(x) for x in sys.argv[1:]]
nx, ny, nseeds, warm = (a + [3200, 3125, 4096, 80][len(a):])[:4]
mesh = ft.gen_periodic_grid(nx, ny)
lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, nseeds, replace=False)
n_v = mesh.n_vertices
lib = _lib.lib()
cur, _ = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=warm, tol=0.0)
dphi = cur.device_phi()
ws = ft.StepWorkspace()
ws.prepare(n_v, dphi.values.device)
ta = ft.DeviceTiled(dphi.n_rows, n_v, dphi.nnz, dphi.values.dtype, dphi.values.device)
tb = ft.DeviceTiled(dphi.n_rows, n_v, dphi.nnz, dphi.values.dtype, dphi.values.device)
dl = F.device_laplacian(lap, "exact")
lc = dl.ft_csc("exact")
fl = dl.launch_flags()
prm = ft.CouplingParams().ft_params()
st = F._stream_handle()
wp, wn = ws.ws_args()
src = dphi.ft_csc()
ac, bc = ta.ft_tiled(), tb.ft_tiled()
assert lib.ft_tiled_from_csc(ctypes.byref(src), ctypes.byref(bc), 0, wp, wn,
                             ctypes.c_void_p(ws.stats.data_ptr()), st) == 0
lib.ft_probe_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
rows = []
for i in range(25):
    lib.ft_step_kernel(ctypes.byref(lc), fl, ctypes.byref(bc), ctypes.byref(ac), 0, ctypes.byref(prm), wp, wn, st)
    lib.ft_step_fixup(ctypes.byref(lc), fl, ctypes.byref(bc), ctypes.byref(ac), 0, ctypes.byref(prm), wp, wn, st)
    lib.ft_step_finalize(wp, wn, n_v, ta.capacity, ctypes.c_void_p(ws.stats.data_ptr()), st)
    buf = (ctypes.c_float * 8)()
    assert lib.ft_probe_timeline(buf, 8) == 0
    if i >= 5:
        rows.append(list(buf))
r = np.median(np.array(rows), axis=0) * 1e3
names = ["start", "tier1 done/fork", "queue A", "tier2a(A)", "warp(A)", "tier1.5 (main)", "warp(B) (main)",
         "join"]
for nm, x in zip(names, r):
    print(f"{nm:18s} {x:8.1f} us")
