import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1804_09152_b200 as ft
mesh = ft.gen_periodic_grid(3200, 3125); lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, 65536, 0)
st = ft.LloydState(seeds=seeds)
ft.lloyd_iterate(st, mesh, lap, ft.CouplingParams(), 20, max_steps=100)
fld = st.field
pr = cProfile.Profile(); pr.enable()
a_v = ft.vertex_adjacency(fld, 0.25); a_t = ft.triangle_adjacency(fld, mesh, 0.25)
cur = ft.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
pos = mesh.positions[np.asarray(fld.seed_vertices, dtype=np.int64)]
dm = ft.build_dual(cur, pos)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
