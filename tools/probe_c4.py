"""C4-scale run on ONE GPU (BASELINE configs[3] names ~100M vertices at
2/4/8 GPUs; the icosphere levels are 41.9M (s=11) and 167.8M (s=12)): the
order-identical icosphere generator, the Laplacian, the seed sampler and
steps 1..120 from init_field, timed with CUDA events.

usage: PYTHONPATH=. python tools/probe_c4.py [level] [seeds] [steps]
"""
import sys
import time

import numpy as np
import torch

import paper_1804_09152_b200 as ft

level = int(sys.argv[1]) if len(sys.argv) > 1 else 11
nseeds = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 120
t = time.time()
mesh = ft.gen_icosphere(level, max_subdiv=12)
print(f"icosphere {level}: {mesh.n_vertices} vertices, {mesh.n_faces} faces, {time.time() - t:.1f} s", flush=True)
t = time.time()
lap = ft.build_laplacian(mesh)
print(f"laplacian {time.time() - t:.1f} s", flush=True)
t = time.time()
seeds = ft.sample_seed_vertices(mesh, nseeds, 0)
print(f"seed sampler ({nseeds} seeds) {time.time() - t:.1f} s", flush=True)
fld0 = ft.init_field(mesh, seeds)
ft.evolve(fld0, lap, ft.CouplingParams(), max_steps=3, tol=0.0)       # warm-up (graphs, allocators)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
fld, tr = ft.evolve(fld0, lap, ft.CouplingParams(), max_steps=steps, tol=0.0)
e1.record()
torch.cuda.synchronize()
sec = e0.elapsed_time(e1) * 1e-3
nnz = [s.nnz_phi for s in tr]
print(f"evolve steps 1..{len(tr)}: {sec:.3f} s = {len(tr) / sec:.1f} steps/s, "
      f"{mesh.n_vertices * len(tr) / sec / 1e9:.2f} G vertex-steps/s, nnz {nnz[0]} -> {max(nnz)} -> {nnz[-1]}",
      flush=True)
lab = ft.sharp_labels(fld)
print(f"labels: {np.unique(lab[lab >= 0]).size} cells hold vertices; peak GPU memory "
      f"{torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
