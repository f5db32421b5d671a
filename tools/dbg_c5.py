import numpy as np, torch
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import lloyd as L
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, 65536, 0)
print("distinct seeds", np.unique(seeds).size)
fld, tr = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=1000)
print("steps", len(tr), "converged", tr[-1].converged)
state = L.LloydState(seeds=seeds, field=fld)
old = np.asarray(seeds)
_, _, status, hit = L.cell_geometry(fld, mesh, seeds=old)
print("status counts", np.bincount(status.astype(np.int64)), "hit<0", int((hit < 0).sum()))
phi = fld.phi
rows = phi.row_idx[:phi.nnz]; cols = phi.entry_columns()
cnt = np.bincount(rows, minlength=phi.n_rows)
print("cell sizes: min", cnt[1:].min(), "median", np.median(cnt[1:]), "cells with <5 vertices", int((cnt[1:] < 5).sum()))
labels = ft.sharp_labels(fld)
lab_cnt = np.bincount(labels[labels >= 0], minlength=65536)
print("label-count min", lab_cnt.min(), "cells with 0 labelled vertices", int((lab_cnt == 0).sum()))
fail = (status != 0) | (hit < 0)
cand = np.where(fail, old, hit)
print("duplicate candidates", cand.size - np.unique(cand).size)
for c in (38541, 57716):
    mine = np.sort(cols[rows == c + 1])
    print("cell", c, "members", mine.size, "old", old[c], "cand", cand[c], "status", status[c], "hit", hit[c],
          "old in members", old[c] in set(mine.tolist()))
