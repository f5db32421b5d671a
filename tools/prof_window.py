"""Profile window: C3 (or --nx/--ny/--seeds) evolved to step S untimed, then
K steps through ft_step_run between cudaProfilerStart/Stop (for
`ncu --profile-from-start off`), with per-step list sizes printed.

    python tools/prof_window.py [--start 80] [--steps 4] [--counts]
"""
import argparse, ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import _lib, field as F

ap = argparse.ArgumentParser()
ap.add_argument("--mesh", default="torus", help="torus or icoL")
ap.add_argument("--nx", type=int, default=3200)
ap.add_argument("--ny", type=int, default=3125)
ap.add_argument("--seeds", type=int, default=4096)
ap.add_argument("--start", type=int, default=80)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--counts", action="store_true")
ap.add_argument("--precision", default="exact")
args = ap.parse_args()

mesh = (ft.gen_icosphere(int(args.mesh[3:]), max_subdiv=12) if args.mesh.startswith("ico")
        else ft.gen_periodic_grid(args.nx, args.ny))
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, args.seeds, 0)
fld = ft.init_field(mesh, seeds, precision=args.precision)
cur = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=args.start, tol=0.0)[0] if args.start else fld
src = cur.device_phi()
dev = src.values.device
n = src.n_cols
ws = ft.StepWorkspace(); ws.prepare(n, dev)
cap = max(int(src.nnz * F.POOL_FRACTION), F.POOL_MIN)
ta = ft.DeviceTiled(src.n_rows, n, cap, src.values.dtype, dev)
tb = ft.DeviceTiled(src.n_rows, n, cap, src.values.dtype, dev)
dl = F.device_laplacian(lap, args.precision)
lib = _lib.lib()
lc, prm, sh = dl.ft_csc(args.precision), ft.CouplingParams().ft_params(), F._stream_handle()
fl = dl.launch_flags(src)
dt = F._ft_dtype(args.precision)
wp, wn = ws.ws_args()
rec = torch.zeros(64, dtype=torch.uint8, device=dev)
s_c, a_c, b_c = src.ft_csc(), ta.ft_tiled(), tb.ft_tiled()
assert lib.ft_tiled_from_csc(ctypes.byref(s_c), ctypes.byref(b_c), dt, wp, wn, ctypes.c_void_p(rec.data_ptr()), sh) == 0

def run(k, phases):
    i, o = (b_c, a_c) if k % 2 == 0 else (a_c, b_c)
    assert lib.ft_step_run(ctypes.byref(lc), fl, ctypes.byref(i), ctypes.byref(o), k & 1, dt, ctypes.byref(prm),
                           wp, wn, phases, ctypes.c_void_p(rec.data_ptr()), sh) == 0

# two warm steps (the first after the conversion is a full step)
for k in range(2):
    run(k, 3)
torch.cuda.synchronize()
cudart = torch.cuda.cudart()
cudart.cudaProfilerStart()
for k in range(2, 2 + args.steps):
    run(k, 1)
    if args.counts:
        torch.cuda.synchronize()
        c = ws.ws[:224].cpu().numpy().view(np.int32)
        print(f"step {args.start + k + 1}: full {c[40]} n_act {c[20]} n_wide {c[21]} n_w2 {c[23]} n_deep {c[22]}",
              flush=True)
    run(k, 2)
torch.cuda.synchronize()
cudart.cudaProfilerStop()
r = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=_lib.STATS_DTYPE)[0]
print("last step", r, flush=True)
