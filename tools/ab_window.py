"""A/B timing of the C3 steady window through ft_evolve, the library given
by FT_LIB: steps 81..120 from the step-80 field, best of R repeats, plus the
nnz / max_delta trace (must match across variants)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_09152_b200 as ft
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
NS = int(os.environ.get("AB_SEEDS", "4096"))
seeds = ft.sample_seed_vertices(mesh, NS, 0)
prm = ft.CouplingParams()
st80, _ = ft.evolve(ft.init_field(mesh, seeds), lap, prm, max_steps=80, tol=0.0)
best = None
for r in range(5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out, tr = ft.evolve(st80, lap, prm, max_steps=40, tol=0.0); e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    best = ms if best is None else min(best, ms)
sig = hash(tuple((t.nnz_phi, t.max_delta) for t in tr))
print(json.dumps({"lib": os.environ.get("FT_LIB", "default"), "seeds": NS,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("FT_")}, "steps_per_s": 40 / (best * 1e-3),
                  "ms_per_step": best / 40, "trace_sig": sig}))
