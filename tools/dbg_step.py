"""Step-by-step GPU vs oracle from the GPU's own input; report the first bad column."""
import sys
import numpy as np
import paper_1804_09152_b200 as ft
from oracle import pyoracle as O

sub = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh = ft.gen_icosphere(sub, max_subdiv=12)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, 64, replace=False)
lap = ft.build_laplacian(mesh)
lt = O.Csc.of(ft.field._with_diagonal(lap.mat_t))
cur = ft.init_field(mesh, seeds)
prm = ft.CouplingParams()
for k in range(30):
    inp = O.Csc.of(cur.phi)
    ref, st = O.step_c(inp, lt, prm)
    cur, gst = ft.step(cur, lap, prm)
    g = cur.phi
    bad = [j for j in range(mesh.n_vertices)
           if not (np.array_equal(g.row_idx[g.col_ptr[j]:g.col_ptr[j+1]], ref.row_idx[ref.col_ptr[j]:ref.col_ptr[j+1]])
                   and np.array_equal(g.values[g.col_ptr[j]:g.col_ptr[j+1]], ref.values[ref.col_ptr[j]:ref.col_ptr[j+1]]))]
    print("step", k + 1, "bad", len(bad), bad[:8], "stats", gst.max_delta == st["max_delta"], gst.nnz_phi, ref.nnz)
    if bad:
        for j in bad[:3]:
            us = lt.row_idx[lt.col_ptr[j]:lt.col_ptr[j+1]]
            print(" col", j, "L entries", len(us), "neighbour counts", [int(inp.col_ptr[u+1]-inp.col_ptr[u]) for u in us])
            print("   union rows", sorted(set(np.concatenate([inp.row_idx[inp.col_ptr[u]:inp.col_ptr[u+1]] for u in us]).tolist())))
            print("   gpu", g.row_idx[g.col_ptr[j]:g.col_ptr[j+1]], g.values[g.col_ptr[j]:g.col_ptr[j+1]])
            print("   ref", ref.row_idx[ref.col_ptr[j]:ref.col_ptr[j+1]], ref.values[ref.col_ptr[j]:ref.col_ptr[j+1]])
        break
