#!/usr/bin/env python
"""Where the e2e time of bench.py goes (C3): upload, evolve(K), field.phi, sharp_labels.

    python tools/e2e_breakdown.py [--steps K] [--precision exact|fast]

Each stage is bracketed by torch.cuda.synchronize(); five passes from the
step-80 field, the caller holding its latest result (as in bench.py's e2e):
pass 0 is the cold call.
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1804_09152_b200 as ft  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--precision", default="exact")
    args = ap.parse_args()
    wl = argparse.Namespace(mesh="torus", nx=bench.NX, ny=bench.NY, seeds=bench.N_SEEDS)
    mesh, lap, seeds = bench.build_workload(wl)
    host0 = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=80, tol=0.0)[0].phi
    nnz0 = host0.nnz
    pinned = [torch.empty(a.size, dtype=t, pin_memory=True)
              for a, t in ((host0.col_ptr, torch.int32), (host0.row_idx[:nnz0], torch.int32),
                           (host0.values[:nnz0], torch.float64))]   # SparseMat values are float64
    pinned[0].numpy()[:] = host0.col_ptr
    pinned[1].numpy()[:] = host0.row_idx[:nnz0]
    pinned[2].numpy()[:] = host0.values[:nnz0]
    hphi = ft.SparseMat(host0.n_rows, mesh.n_vertices, pinned[0].numpy(), pinned[1].numpy(),
                        pinned[2].numpy(), check=False)
    params = ft.CouplingParams()
    held = None
    for rep in range(5):
        t = [time.perf_counter()]
        fld = ft.LayeredField(hphi, seeds, step_count=80, precision=args.precision)
        fld.device_phi()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        fin, tr = ft.evolve(fld, lap, params, max_steps=args.steps, tol=0.0)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        phi = fin.phi
        torch.cuda.synchronize(); t.append(time.perf_counter())
        lab = ft.sharp_labels(fin)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        names = ["upload", f"evolve({args.steps})", "field.phi", "sharp_labels"]
        ms = [(b - a) * 1e3 for a, b in zip(t, t[1:])]
        print(f"pass {rep}: " + ", ".join(f"{n} {m:.2f} ms" for n, m in zip(names, ms))
              + f"; total {sum(ms):.2f} ms -> {args.steps / sum(ms) * 1e3:.0f} steps/s"
              + f"; evolve alone {args.steps / ms[1] * 1e3:.0f} steps/s; nnz {phi.nnz}, labels {lab.size}")
        held = (phi, lab)
        del fin, tr


if __name__ == "__main__":
    main()
