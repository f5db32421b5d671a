"""Warm times of tier 1 / the fixup launches / the finalize of the C3 step
from ONE fixed input state (the same step repeated: tb -> ta), and the tier
populations of that state.  (tools/probe_timeline.py splits the fixup.)

usage: python tools/probe_fixup.py [nx ny seeds warm]
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
assert lib.ft_tiled_from_csc(ctypes.byref(src), ctypes.byref(bc), 0, wp, wn, ctypes.c_void_p(ws.stats.data_ptr()), st) == 0
t = []
for i in range(30):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    assert lib.ft_step_kernel(ctypes.byref(lc), fl, ctypes.byref(bc), ctypes.byref(ac), 0, ctypes.byref(prm), wp, wn, st) == 0
    ev[1].record()
    assert lib.ft_step_fixup(ctypes.byref(lc), fl, ctypes.byref(bc), ctypes.byref(ac), 0, ctypes.byref(prm), wp, wn, st) == 0
    ev[2].record()
    assert lib.ft_step_finalize(wp, wn, n_v, ta.capacity, ctypes.c_void_p(ws.stats.data_ptr()), st) == 0
    ev[3].record()
    torch.cuda.synchronize()
    if i >= 5:
        t.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])])
t = np.median(np.array(t), axis=0) * 1e3
print(f"tier1 {t[0]:.1f} us  fixup {t[1]:.1f} us  finalize {t[2]:.1f} us")

# tier populations of this state: masks after tier 1, queue after tier 1.5
def al(x):
    return (x + 15) & ~15
nt = (n_v + 127) // 128
ns = 4 * nt
off = 128
off_gen = al(al(al(off + ns * 8) + ns * 8) + ns * 8)
off_slow = al(off_gen + ns * 4)
assert lib.ft_step_kernel(ctypes.byref(lc), fl, ctypes.byref(bc), ctypes.byref(ac), 0, ctypes.byref(prm), wp, wn, st) == 0
torch.cuda.synchronize()
raw = ws.ws.cpu().numpy()
gm = raw[off_gen:off_gen + ns * 4].view(np.uint32)
sm = raw[off_slow:off_slow + ns * 4].view(np.uint32)
pc = lambda a: int(np.unpackbits(a.view(np.uint8)).sum())
print(f"tier-1.5 columns {pc(gm)}  tier-1 slow columns {pc(sm)}  tiles with gen {int((gm.reshape(-1, 4).any(1)).sum())} of {nt}")
assert lib.ft_step_fixup(ctypes.byref(lc), fl, ctypes.byref(bc), ctypes.byref(ac), 0, ctypes.byref(prm), wp, wn, st) == 0
torch.cuda.synchronize()
c = ws.ws[:128].cpu().numpy()
i32 = lambda o: int(c[o:o + 4].view(np.int32)[0])
print(f"tier-2 queue A {i32(56)} B (tier-1.5 deferred) {i32(68)}  tier-2b {i32(96)}  tier-3 {i32(64)}  pool {int(c[40:48].view(np.int64)[0])}")
