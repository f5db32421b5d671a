"""Break the bench's e2e path (host field -> evolve -> host field + labels) into parts."""
import time
import numpy as np, torch
import paper_1804_09152_b200 as ft
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 4096, replace=False)
fld0 = ft.init_field(mesh, seeds)
h = fld0.phi
nnz = h.nnz
pinned = [torch.empty(a.size, dtype=t, pin_memory=True) for a, t in ((h.col_ptr, torch.int32), (h.row_idx[:nnz], torch.int32), (h.values[:nnz], torch.float64))]
pinned[0].numpy()[:] = h.col_ptr; pinned[1].numpy()[:] = h.row_idx[:nnz]; pinned[2].numpy()[:] = h.values[:nnz]
hphi = ft.SparseMat(h.n_rows, mesh.n_vertices, pinned[0].numpy(), pinned[1].numpy(), pinned[2].numpy(), check=False)
ft.evolve(ft.LayeredField(hphi, seeds), lap, ft.CouplingParams(), max_steps=20, tol=0.0)
torch.cuda.synchronize()
for rep in range(2):
    t = [time.perf_counter()]
    f = ft.LayeredField(hphi, seeds)
    d = f.device_phi(); torch.cuda.synchronize(); t.append(time.perf_counter())
    fin, tr = ft.evolve(f, lap, ft.CouplingParams(), max_steps=200, tol=0.0); torch.cuda.synchronize(); t.append(time.perf_counter())
    ph = fin.phi; t.append(time.perf_counter())
    lab = ft.sharp_labels(fin); torch.cuda.synchronize(); t.append(time.perf_counter())
    dt = np.diff(t) * 1e3
    print(f"upload {dt[0]:.1f} ms  evolve {dt[1]:.1f} ms  phi->host {dt[2]:.1f} ms  labels {dt[3]:.1f} ms  total {sum(dt):.1f} ms")
