"""Time ft.evolve from init_field (the e2e window) on C3."""
import sys, time
import numpy as np, torch
import paper_1804_09152_b200 as ft
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 4096, replace=False)
fld = ft.init_field(mesh, seeds)
ft.evolve(fld, lap, ft.CouplingParams(), max_steps=20, tol=0.0)
torch.cuda.synchronize()
for rep in range(2):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); out, tr = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=n, tol=0.0); e1.record()
    torch.cuda.synchronize()
    print(f"evolve {n} steps from init: {e0.elapsed_time(e1):.1f} ms -> {n / e0.elapsed_time(e1) * 1e3:.0f} steps/s  reallocs {tr[-1].realloc_count}")
