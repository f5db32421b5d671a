"""How much of a C3 step could be skipped: the fraction of 32-column
segments whose closed one-ring neighbourhood did not change between steps
t-1 and t (their step t+1 output equals their step t output).

usage: PYTHONPATH=. python tools/quiescent.py [warm]
"""
import sys

import numpy as np
import torch

import paper_1804_09152_b200 as ft

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 80
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 4096, replace=False)
a, _ = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=warm, tol=0.0)
b, _ = ft.step(a, lap, ft.CouplingParams())
pa, pb = a.device_phi(), b.device_phi()
n = pa.n_cols


def dense_cols(d):
    # (count, first row, first value, second row, second value) per column
    cp = d.col_ptr.long()
    cnt = cp[1:] - cp[:-1]
    first = cp[:-1].clamp(max=max(d.nnz - 1, 0))
    second = (cp[:-1] + 1).clamp(max=max(d.nnz - 1, 0))
    r, v = d.row_idx[:d.nnz].long(), d.values[:d.nnz]
    return cnt, r[first], v[first], r[second], v[second]


ca, cb = dense_cols(pa), dense_cols(pb)
changed = (ca[0] != cb[0]) | (ca[1] != cb[1]) | (ca[2] != cb[2]) | \
          ((ca[0] >= 2) & ((ca[3] != cb[3]) | (ca[4] != cb[4]))) | (ca[0] > 2)
mt = lap.mat_t
lp = torch.from_numpy(np.asarray(mt.col_ptr, dtype=np.int64)).cuda()
li = torch.from_numpy(np.asarray(mt.row_idx[:mt.nnz], dtype=np.int64)).cuda()
col = torch.repeat_interleave(torch.arange(n, device="cuda"), lp[1:] - lp[:-1])
nb_changed = torch.zeros(n, dtype=torch.bool, device="cuda")
nb_changed.index_put_((col,), changed[li], accumulate=True)
segs = nb_changed[: n // 32 * 32].view(-1, 32).any(1)
print(f"step {warm}->{warm + 1}: columns changed {changed.float().mean().item():.3f}, "
      f"columns with a changed neighbourhood {nb_changed.float().mean().item():.3f}, "
      f"fully quiescent 32-column segments {1 - segs.float().mean().item():.3f}")
