"""C4 on one GPU: raw icosphere numbering vs Morton-renumbered (device
renumbering of PHI and L^T), steps 81..120 timed through ft.evolve.

usage: python tools/probe_c4_order.py [level] [seeds]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_09152_b200 as ft  # noqa: E402
from paper_1804_09152_b200 import distributed as D  # noqa: E402
from paper_1804_09152_b200.mesh import Laplacian  # noqa: E402
from paper_1804_09152_b200.sparse import DeviceCSC  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n_seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
mesh = ft.gen_icosphere(level, max_subdiv=12)
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, n_seeds, 0)
prm = ft.CouplingParams()
fld0 = ft.init_field(mesh, seeds)
st80, _ = ft.evolve(fld0, lap, prm, max_steps=80, tol=0.0)


def timed(fld, lp, k=40, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, tr = ft.evolve(fld, lp, prm, max_steps=k, tol=0.0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, out, tr


ms_raw, out_raw, tr_raw = timed(st80, lap)
print(f"raw order   : {40 / (ms_raw * 1e-3):8.1f} steps/s ({ms_raw / 40:.3f} ms/step)", flush=True)

order = D.morton_order_device(mesh.device_arrays()[0])
part = D.Partition.even(mesh.n_vertices, 1)
dphi = st80.device_phi()
inverse = torch.empty_like(order)
inverse[order] = torch.arange(order.numel(), device=order.device)
lp_ptr, src = D._gather_columns(lap.device["ptr"], order)
n = mesh.n_vertices
lap2 = Laplacian._from_device(n, lp_ptr.int(), inverse[lap.device["idx"][src].long()].int(),
                              lap.device["val_t"][src], lap.device["val"][src])
cp, fsrc = D._gather_columns(dphi.col_ptr, order)
phi2 = DeviceCSC(dphi.n_rows, n, cp.int(), dphi.row_idx[fsrc].clone(), dphi.values[fsrc].clone(), int(cp[-1]))
f2 = ft.LayeredField(phi2, seeds, step_count=80)
ms_m, out_m, tr_m = timed(f2, lap2)
print(f"Morton order: {40 / (ms_m * 1e-3):8.1f} steps/s ({ms_m / 40:.3f} ms/step)", flush=True)
same = [a.max_delta for a in tr_raw] == [b.max_delta for b in tr_m] and \
       [a.nnz_phi for a in tr_raw] == [b.nnz_phi for b in tr_m]
print("identical statistics:", same, " nnz", tr_raw[-1].nnz_phi)
