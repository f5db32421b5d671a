"""e2e breakdown: host field -> evolve(K) -> field.phi + sharp_labels, timed per stage."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import sparse as S

mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, 4096, 0)
fld0 = ft.init_field(mesh, seeds)
cur, _ = ft.evolve(fld0, lap, ft.CouplingParams(), max_steps=80, tol=0.0)
host = cur.phi
K = 20
mode = sys.argv[1] if len(sys.argv) > 1 else "pinned"
if mode == "pageable":
    def pc(t):
        h = torch.empty(t.shape, dtype=t.dtype)
        h.copy_(t)
        return h.numpy()
    S.pinned_copy = pc
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = ft.LayeredField(host, seeds, step_count=80)
    d = f.device_phi(); torch.cuda.synchronize(); t1 = time.perf_counter()
    out, tr = ft.evolve(f, lap, ft.CouplingParams(), max_steps=K, tol=0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    ph = out.phi; t3 = time.perf_counter()
    lb = ft.sharp_labels(out); t4 = time.perf_counter()
    print(f"{mode} it{it}: upload {1e3*(t1-t0):.1f} ms, evolve {1e3*(t2-t1):.1f} ms, phi {1e3*(t3-t2):.1f} ms, "
          f"labels {1e3*(t4-t3):.1f} ms, total {1e3*(t4-t0):.1f} ms -> {K/(t4-t0):.0f} steps/s", flush=True)
