"""Setup timings of the C4 pipeline with the device mesh path:
gen_icosphere(L) -> build_laplacian -> sample_seed_vertices -> init_field."""
import sys
import time

import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_09152_b200 as ft

level = int(sys.argv[1]) if len(sys.argv) > 1 else 11
n_seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 16384


def tick(label, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"{label:>12s} {t - t0:8.2f} s   mem {torch.cuda.max_memory_allocated() / 2**30:6.1f} GiB", flush=True)
    return t


t = time.perf_counter()
torch.zeros(1, device="cuda")
t = tick("cuda init", t)
mesh = ft.gen_icosphere(level, max_subdiv=12)
t = tick("generate", t)
lap = ft.build_laplacian(mesh)
t = tick("laplacian", t)
seeds = ft.sample_seed_vertices(mesh, n_seeds, 0)
t = tick("seeds", t)
fld = ft.init_field(mesh, seeds)
t = tick("init_field", t)
out, trace = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=20, tol=0.0)
t = tick("20 steps", t)
print("n_vertices", mesh.n_vertices, "nnz", trace[-1].nnz_phi)
