"""Distribution of the tier-2 ("wide") columns of C3 at step 80: union row
count and max entries per neighbour."""
import numpy as np
import paper_1804_09152_b200 as ft
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 4096, replace=False)
cur, _ = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=80, tol=0.0)
phi = cur.phi
n = phi.n_cols
cp = np.asarray(phi.col_ptr, dtype=np.int64)
cnt = np.diff(cp)
mt = ft.field._with_diagonal(lap.mat_t)
lp = np.asarray(mt.col_ptr, dtype=np.int64)
li = np.asarray(mt.row_idx[:lp[-1]], dtype=np.int64)
lj = np.repeat(np.arange(n), np.diff(lp))
maxc = np.zeros(n, dtype=np.int64)
np.maximum.at(maxc, lj, cnt[li])
# union rows per column
reps = cnt[li]
pj = np.repeat(lj, reps)
starts = np.repeat(cp[li], reps)
off = np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps)
rows = np.asarray(phi.row_idx)[starts + off].astype(np.int64)
key = np.unique(pj * 70000 + rows)
union = np.bincount(key // 70000, minlength=n)
wide = (maxc > 2) | (union > 2)
print("columns", n, "wide", int(wide.sum()))
for u in range(1, 9):
    m = wide & (union == u)
    if m.any():
        print(f" union {u}: {int(m.sum())}  of which max entries/neighbour <=3: {int((m & (maxc <= 3)).sum())}")
print(" union > 8:", int((wide & (union > 8)).sum()))
