"""cProfile of two C5 Lloyd iterations (max_steps 100) after a warm one."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_09152_b200 as ft
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, 65536, 0)
st = ft.LloydState(seeds=seeds)
ft.lloyd_iterate(st, mesh, lap, ft.CouplingParams(), 1, max_steps=100)
pr = cProfile.Profile()
pr.enable()
ft.lloyd_iterate(st, mesh, lap, ft.CouplingParams(), 2, max_steps=100)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
