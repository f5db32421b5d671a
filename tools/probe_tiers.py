"""Per-tier timing and tier populations of the C3 step in steady state.

usage: python tools/probe_tiers.py [nx ny seeds warm]
Times tier 1 (ft_step_kernel), tiers 1.5-3 (ft_step_fixup) and the finalize
separately with CUDA events (on the launching stream) and reads the queue
counts of the control block before the finalize resets them.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import _lib, field as F

a = [int(x) for x in sys.argv[1:]]
nx, ny, nseeds, warm = (a + [3200, 3125, 4096, 80][len(a):])[:4]
mesh = ft.gen_periodic_grid(nx, ny)
lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, nseeds, replace=False)
n_v = mesh.n_vertices
lib = _lib.lib()
fld = ft.init_field(mesh, seeds)
cur, _ = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=warm, tol=0.0)
dphi = cur.device_phi()
ws = ft.StepWorkspace()
ws.prepare(n_v, dphi.values.device)
cap = int(lib.ft_tiled_min_capacity(n_v)) + dphi.nnz
ta = ft.DeviceTiled(dphi.n_rows, n_v, cap, dphi.values.dtype, dphi.values.device)
tb = ft.DeviceTiled(dphi.n_rows, n_v, cap, dphi.values.dtype, dphi.values.device)
dl = F.device_laplacian(lap, "exact")
lc = dl.ft_csc("exact")
fl = dl.launch_flags()
prm = ft.CouplingParams().ft_params()
st = F._stream_handle()
wp, wn = ws.ws_args()
src = dphi.ft_csc()
rows = []
tb_c = tb.ft_tiled()
assert lib.ft_tiled_from_csc(ctypes.byref(src), ctypes.byref(tb_c), 0, wp, wn, ctypes.c_void_p(ws.stats.data_ptr()),
                             st) == 0
for i in range(41):
    out = ta if i % 2 == 0 else tb
    inp = tb if i % 2 == 0 else ta
    oc, ic = out.ft_tiled(), inp.ft_tiled()
    tiled = ctypes.byref(ic)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    assert lib.ft_step_kernel(ctypes.byref(lc), fl, tiled, ctypes.byref(oc), 0, ctypes.byref(prm), wp, wn,
                              st) == 0
    ev[1].record()
    assert lib.ft_step_fixup(ctypes.byref(lc), fl, tiled, ctypes.byref(oc), 0, ctypes.byref(prm), wp, wn,
                             st) == 0
    ev[2].record()
    torch.cuda.synchronize()
    ctl = ws.ws[:128].cpu().numpy()
    slow = int(ctl[56:60].view(np.int32)[0])
    deep = int(ctl[64:68].view(np.int32)[0])
    pool = int(ctl[40:48].view(np.int64)[0])
    ev3 = torch.cuda.Event(enable_timing=True)
    ev3.record()
    assert lib.ft_step_finalize(wp, wn, n_v, out.capacity, ctypes.c_void_p(ws.stats.data_ptr()), st) == 0
    ev[3].record()
    torch.cuda.synchronize()
    if i:
        rows.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev3.elapsed_time(ev[3]), slow, deep, pool))
r = np.array(rows)
print(f"n_v {n_v}  tier1 {np.median(r[:,0])*1e3:.1f} us  tier2+3 {np.median(r[:,1])*1e3:.1f} us  "
      f"finalize {np.median(r[:,2])*1e3:.1f} us  wide cols {np.median(r[:,3]):.0f} ({100*np.median(r[:,3])/n_v:.2f}%)  "
      f"deep cols {np.median(r[:,4]):.0f}  pool entries {np.median(r[:,5]):.0f}")
