"""Trace the control block of a loopback run that must recover from overflows."""
import numpy as np

import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import distributed as D

D.POOL_FRACTION = 0.0
D.POOL_MIN = 1
nx, ny = 40, 30
mesh = ft.gen_periodic_grid(nx, ny)
seeds = np.random.default_rng(3).choice(nx * ny, 25, replace=False)
lap = ft.build_laplacian(mesh)
fld = ft.init_field(mesh, seeds)
part = D.Partition.even(mesh.n_vertices, 2, align=40)
probs = [D.local_problem(fld.phi, lap, part, r) for r in range(2)]
plans = D.build_plans(probs, D.LoopbackTransport())
ranks = [D.DomainRank(p, pl, slots=1) for p, pl in zip(probs, plans)]
orig = D.DomainRank.read_control


def rc(self):
    c = orig(self)
    print("rank", self.rank, "control", c, "step_cap", self.step_cap, "slots", self.slots,
          "caps", [b.capacity for b in self.bufs])
    return c


D.DomainRank.read_control = rc
steps, tr = D.evolve_partitioned(ranks, D.LoopbackTransport(), ft.CouplingParams(), max_steps=12,
                                 tol=0.0, sync_every=5)
for r in ranks:
    for k in range(2):
        d = r.bufs[k].desc.view(-1, 2).cpu().numpy()
        b, e = part.range(r.rank)
        print("rank", r.rank, "buf", k, "owned cnt sum", d[b:e, 1].sum())
single, _ = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=12, tol=0.0)
print("single nnz", single.phi.nnz, "trace nnz", [t.nnz_phi for t in tr])
