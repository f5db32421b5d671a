"""Column statistics of the C3 field after W steps (design input)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_09152_b200 as ft
nx, ny, ns, W = 3200, 3125, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 80
mesh = ft.gen_periodic_grid(nx, ny); lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, ns, replace=False)
cur, _ = ft.evolve(ft.init_field(mesh, seeds), lap, ft.CouplingParams(), max_steps=W, tol=0.0)
phi = cur.phi
cnt = np.diff(phi.col_ptr.astype(np.int64))
print("step", W, "nnz/v", phi.nnz / mesh.n_vertices)
print("column entry-count histogram:", {int(k): int(v) for k, v in zip(*np.unique(cnt, return_counts=True))})
lp = lap.mat_t.col_ptr.astype(np.int64); li = lap.mat_t.row_idx
nb_max = np.maximum.reduceat(cnt[li], lp[:-1])
print("max neighbour count histogram:", {int(k): int(v) for k, v in zip(*np.unique(nb_max, return_counts=True))})
# union size per vertex (rows in closed neighbourhood)
rows = phi.row_idx[:phi.nnz].astype(np.int64); cols = phi.entry_columns()
# for each vertex j, union of rows over neighbours: build (j, row) pairs
pair_v = np.repeat(np.arange(mesh.n_vertices), np.diff(lp))
nbr = li.astype(np.int64)
# expand neighbour entries
starts = phi.col_ptr[nbr].astype(np.int64); c = cnt[nbr]
tot = int(c.sum()); rep_v = np.repeat(pair_v, c)
off = np.arange(tot) - np.repeat(np.cumsum(c) - c, c)
r = rows[np.repeat(starts, c) + off]
key = np.unique(rep_v * 100000 + r)
u = np.bincount(key // 100000, minlength=mesh.n_vertices)
print("union size histogram:", {int(k): int(v) for k, v in zip(*np.unique(u, return_counts=True))})
warp_u = u[: (len(u)//32)*32].reshape(-1, 32).max(axis=1)
print("warps: max union histogram:", {int(k): int(v) for k, v in zip(*np.unique(warp_u, return_counts=True))})
warp_w = nb_max[: (len(u)//32)*32].reshape(-1, 32).max(axis=1)
print("warps: max neighbour count histogram:", {int(k): int(v) for k, v in zip(*np.unique(warp_w, return_counts=True))})
