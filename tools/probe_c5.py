"""C5-scale run: 10M-vertex torus, 65,536 seeds -- evolve, one Lloyd
centroid / back-projection pass, dual extraction (BASELINE configs[4]).

A full Lloyd iteration at this density stops in the reference's own
_reseed (lloyd.py:155-195) with VanishedCellError: ~14% of the cells vanish
within 1000 steps (C2's reference history shows 16% misses at iteration 1)
and, among 65,536 cells, a vanished cell's old seed is soon taken by
another cell's new seed.  This probe times each GPU stage instead."""
import sys, time
import numpy as np, torch
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import dual as DU, lloyd as L

max_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
t = time.time()
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
print(f"mesh + laplacian {time.time() - t:.1f} s", flush=True)
t = time.time()
seeds = ft.sample_seed_vertices(mesh, 65536, 0)
print(f"seed sampler (65,536 seeds) {time.time() - t:.2f} s", flush=True)
fld0 = ft.init_field(mesh, seeds)
ft.evolve(fld0, lap, ft.CouplingParams(), max_steps=5)
torch.cuda.synchronize(); t = time.time()
fld, tr = ft.evolve(fld0, lap, ft.CouplingParams(), max_steps=max_steps)
torch.cuda.synchronize()
print(f"evolve {len(tr)} steps: {time.time() - t:.2f} s ({len(tr) / (time.time() - t):.0f} steps/s), "
      f"nnz {fld.device_phi().nnz}, band vertex fraction {ft.band_vertex_fraction(fld):.3f}", flush=True)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    pts, nrm, status, hit = L.cell_geometry(fld, mesh, seeds=np.asarray(seeds))
    torch.cuda.synchronize()
    print(f"lloyd centroids + back-projection (all cells): {time.time() - t:.3f} s, "
          f"vanished {int((status == 1).sum())}, misses {int((hit < 0).sum())}", flush=True)
for rep in range(2):
    t = time.time()
    a_v = DU.vertex_adjacency(fld, 0.25)
    a_t = DU.triangle_adjacency(fld, mesh, 0.25)
    cur = DU.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
    t1 = time.time()
    try:
        dm = DU.build_dual(cur, mesh.positions[seeds])
        out = f"{len(dm.triangles)} triangles"
    except ft.errors.NonManifoldError as exc:     # the reference's own check (dual.py)
        out = f"NonManifoldError ({str(exc)[:60]}...)"
    print(f"dual: products + curation {t1 - t:.2f} s, triangulation {time.time() - t1:.2f} s, {out}",
          flush=True)
