"""Locate the first divergence between loopback ranks and the single-GPU step."""
import sys
import numpy as np
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import distributed as D

world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sub = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = ft.gen_icosphere(sub, max_subdiv=12)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 64, replace=False)
lap = ft.build_laplacian(mesh)
fld = ft.init_field(mesh, seeds)
part = D.Partition.even(mesh.n_vertices, world)
print("bounds", part.bounds, "flags", D.local_problem(fld.phi, lap, part, 0).lap_flags)
for n in [1, 2, 3, 5, 10, 30, 120]:
    single, _ = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=n, tol=0.0)
    probs = [D.local_problem(fld.phi, lap, part, r) for r in range(world)]
    plans = D.build_plans(probs, D.LoopbackTransport())
    ranks = [D.DomainRank(p, pl) for p, pl in zip(probs, plans)]
    steps, tr = D.evolve_partitioned(ranks, D.LoopbackTransport(), ft.CouplingParams(), max_steps=n, tol=0.0)
    g = D.gather_field(ranks, steps)
    s = single.phi
    from oracle import pyoracle as O
    lt = O.Csc.of(ft.field._with_diagonal(lap.mat_t))
    ref, _ = O.evolve_c(O.Csc.of(fld.phi), lt, ft.CouplingParams(), n)
    for name, x in (("gathered", g), ("single", s)):
        same = np.array_equal(np.asarray(x.col_ptr), ref.col_ptr) and np.array_equal(np.asarray(x.row_idx[:ref.nnz]), ref.row_idx) and np.array_equal(np.asarray(x.values[:ref.nnz]), ref.values)
        print("  ", name, "== oracle:", same)
    bad = []
    for j in range(mesh.n_vertices):
        a0, a1 = g.col_ptr[j], g.col_ptr[j + 1]
        b0, b1 = s.col_ptr[j], s.col_ptr[j + 1]
        if not (np.array_equal(g.row_idx[a0:a1], s.row_idx[b0:b1]) and np.array_equal(g.values[a0:a1], s.values[b0:b1])):
            bad.append(j)
    print("steps", n, steps, "bad cols", len(bad), bad[:10], "owners", np.bincount(part.owner(bad), minlength=world) if bad else None,
          "slots", [r.slots for r in ranks], "halo", [r.n_halo for r in ranks])
    if bad:
        j = bad[0]
        print(" col", j, "gathered", g.row_idx[g.col_ptr[j]:g.col_ptr[j+1]], g.values[g.col_ptr[j]:g.col_ptr[j+1]])
        print(" col", j, "single  ", s.row_idx[s.col_ptr[j]:s.col_ptr[j+1]], s.values[s.col_ptr[j]:s.col_ptr[j+1]])
        break
