"""Histogram of the C3 step-80 columns by (distinct rows in the one-ring
union, max entries of a neighbour): which columns reach tiers 2a / 2b / 3.

usage: PYTHONPATH=. python tools/wide_hist.py [nx ny seeds warm]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_09152_b200 as ft  # noqa: E402

a = [int(x) for x in sys.argv[1:]]
nx, ny, nseeds, warm = (a + [3200, 3125, 4096, 80][len(a):])[:4]
mesh = ft.gen_periodic_grid(nx, ny)
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, nseeds, 0)
cur, _ = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=warm, tol=0.0)
d = cur.device_phi()
n = d.n_cols
cp = d.col_ptr.long()
cnt = cp[1:] - cp[:-1]
ent_col = torch.repeat_interleave(torch.arange(n, device=cp.device), cnt)
rows = d.row_idx[:d.nnz].long()
mt = lap.mat_t
lp = torch.from_numpy(np.asarray(mt.col_ptr, dtype=np.int64)).cuda()
li = torch.from_numpy(np.asarray(mt.row_idx[:mt.nnz], dtype=np.int64)).cuda()
deg = lp[1:] - lp[:-1]
lcol = torch.repeat_interleave(torch.arange(n, device=cp.device), deg)   # column j of each L entry (u = li)
maxent = torch.zeros(n, dtype=torch.long, device=cp.device)
maxent.scatter_reduce_(0, lcol, cnt[li], reduce="amax")
# (j, row) pairs over the one-ring: entries of u for each L entry (j, u)
pairs = []
chunk = 4_000_000
for s in range(0, lcol.numel(), chunk):
    jj, uu = lcol[s:s + chunk], li[s:s + chunk]
    c = cnt[uu]
    jrep = torch.repeat_interleave(jj, c)
    start = torch.repeat_interleave(cp[uu], c)
    off = torch.arange(c.sum(), device=cp.device) - torch.repeat_interleave(torch.cumsum(c, 0) - c, c)
    pairs.append(jrep * 70000 + rows[start + off])
keys = torch.unique(torch.cat(pairs))
ucnt = torch.bincount(keys // 70000, minlength=n)
sel = (ucnt >= 3) | (maxent >= 3)
print(f"columns {n}: union rows >= 3 or a neighbour with >= 3 entries: {int(sel.sum())}")
for r in range(1, 10):
    for e in range(1, 7):
        k = int(((ucnt == r) & (maxent == e)).sum()) if r < 9 else int(((ucnt >= r) & (maxent == e)).sum())
        if k and (r >= 3 or e >= 3):
            print(f"  rows {r}{'+' if r == 9 else ''} max-entries {e}: {k}")
