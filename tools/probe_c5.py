"""C5 (BASELINE configs[4]): torus 3200 x 3125 (10M vertices), 65,536 seeds
(reference sampler), Lloyd iterations with a given max_steps, then the dual
mesh.  Reports per-iteration seconds, misses / collisions / area variance,
and where a cell vanishes.

usage: python tools/probe_c5.py [max_steps] [iterations] [tol]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_09152_b200 as ft

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
IT = int(sys.argv[2]) if len(sys.argv) > 2 else 20
TOL = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
t0 = time.time()
mesh = ft.gen_periodic_grid(3200, 3125)
lap = ft.build_laplacian(mesh)
seeds = ft.sample_seed_vertices(mesh, 65536, 0)
print(f"setup {time.time() - t0:.1f} s", flush=True)
st = ft.LloydState(seeds=seeds)
t = time.time()
try:
    for it in range(IT):
        ft.lloyd_iterate(st, mesh, lap, ft.CouplingParams(), 1, max_steps=M, tol=TOL)
        torch.cuda.synchronize()
        h = st.history[-1]
        print(f"iter {h['iteration']:2d}: {time.time() - t:7.2f} s steps {h['steps']} conv {h['converged']} "
              f"misses {h['reseed_misses']} coll {h['seed_collisions']} var {h['area_variance']:.6g}", flush=True)
        t = time.time()
except Exception as exc:
    print("FAILED:", type(exc).__name__, exc, flush=True)
    sys.exit(0)
t = time.time()
fld = st.field
a_v = ft.vertex_adjacency(fld, 0.25)
a_t = ft.triangle_adjacency(fld, mesh, 0.25)
cur = ft.confirm_candidates(fld, mesh, a_v, a_t, 0.25)
pos = mesh.positions[np.asarray(fld.seed_vertices, dtype=np.int64)]
dm = ft.build_dual(cur, pos)
print(f"dual: {len(cur.pairs())} edges, {dm.triangles.shape[0]} triangles, chi {dm.euler_characteristic()}, "
      f"{time.time() - t:.2f} s", flush=True)
