"""Debug driver for the active-set engine: one step, a short evolve, with
prints after every call (run under `timeout` with python -u)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1804_09152_b200 as ft
from oracle import pyoracle as po

print("import ok", flush=True)
mesh = ft.gen_periodic_grid(12, 10)
lap = ft.build_laplacian(mesh)
fld = ft.init_field(mesh, [5, 50, 90])
print("field", fld, flush=True)
out, st = ft.step(fld, lap, ft.CouplingParams())
torch.cuda.synchronize()
print("step ok", st, flush=True)
ref, rst = po.step_c(po.Csc.of(fld.phi), po.Csc.of(lap.mat_t), ft.CouplingParams())
print("step equal", np.array_equal(out.phi.to_dense(), ref.to_dense()), flush=True)
for n in (2, 3, 20):
    o2, tr = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=n, tol=0.0)
    torch.cuda.synchronize()
    r2, _ = po.evolve_c(po.Csc.of(fld.phi), po.Csc.of(lap.mat_t), ft.CouplingParams(), n)
    print("evolve", n, len(tr), np.array_equal(o2.phi.to_dense(), r2.to_dense()), flush=True)
