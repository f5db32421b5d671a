"""Quick probe: C3-like torus, time the fused step kernel (exact + fast)."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_09152_b200 as ft
from paper_1804_09152_b200 import _lib, field as F

nx, ny = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3200, 3125)
nseeds = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
t0 = time.time()
mesh = ft.gen_periodic_grid(nx, ny); lap = ft.build_laplacian(mesh)
seeds = np.random.default_rng(0).choice(mesh.n_vertices, nseeds, replace=False)
print(f"setup {time.time()-t0:.1f}s n_v={mesh.n_vertices}", flush=True)
lib = _lib.lib()
for prec in ("exact", "fast"):
    fld = ft.init_field(mesh, seeds, precision=prec)
    cur, tr = ft.evolve(fld, lap, ft.CouplingParams(), max_steps=80, tol=0.0)
    torch.cuda.synchronize()
    ws = ft.StepWorkspace(); dphi = cur.device_phi(); ws.prepare(mesh.n_vertices, dphi.values.device)
    a = ws.tiled_buffer("a", dphi, dphi.nnz); b = ws.tiled_buffer("b", dphi, dphi.nnz)
    dl = F.device_laplacian(lap, prec); lc = dl.lap_t[prec].ft_csc(); prm = ft.CouplingParams().ft_params()
    st = F._stream_handle(); wp, wn = ws.ws_args()
    evs = []
    src_c = dphi.ft_csc()
    for i in range(41):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        out = a if i % 2 == 0 else b
        inp = b if i % 2 == 0 else a
        oc, ic = out.ft_tiled(), inp.ft_tiled()
        e0.record()
        rc = lib.ft_step_kernel(ctypes.byref(lc), dl.flags, ctypes.byref(src_c) if i == 0 else None,
                                None if i == 0 else ctypes.byref(ic), ctypes.byref(oc), F._ft_dtype(prec),
                                ctypes.byref(prm), wp, wn, st)
        e1.record()
        assert rc == 0, _lib.last_error()
        lib.ft_step_fixup(ctypes.byref(lc), dl.flags, ctypes.byref(src_c) if i == 0 else None,
                          None if i == 0 else ctypes.byref(ic), ctypes.byref(oc), F._ft_dtype(prec),
                          ctypes.byref(prm), wp, wn, st)
        if i == 40:
            torch.cuda.synchronize()
            slow_tiles = int(ws.ws[56:60].cpu().view(torch.int32).item())
        lib.ft_step_finalize(wp, wn, mesh.n_vertices, out.capacity, ctypes.c_void_p(ws.stats.data_ptr()), st)
        if i: evs.append((e0, e1))
    torch.cuda.synchronize()
    rec = F._stats_from_bytes(ws.stats.cpu().numpy().tobytes())[0]
    assert int(rec['status']) == 0, rec
    ms = np.array([x.elapsed_time(y) for x, y in evs])
    nnz = int(rec['nnz_phi']); vb = 8 if prec == "exact" else 4
    byt = (4 * (mesh.n_vertices + 1) + 4 * lap.mat_t.nnz) + 2 * (4 * (mesh.n_vertices + 1) + (4 + vb) * nnz)
    print(f"{prec}: kernel(s) median {np.median(ms):.3f} ms min {ms.min():.3f}  nnz {nnz} skel {int(rec['nnz_skel'])} "
          f"alg bytes {byt/1e9:.3f} GB -> {byt/np.median(ms)/1e6:.0f} GB/s  slow tiles {slow_tiles}/{(mesh.n_vertices+127)//128}", flush=True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); cur2, tr2 = ft.evolve(cur, lap, ft.CouplingParams(), max_steps=40, tol=0.0); e1.record(); torch.cuda.synchronize()
    print(f"{prec}: evolve 40 steps {e0.elapsed_time(e1):.2f} ms -> {40/e0.elapsed_time(e1)*1e3:.0f} steps/s", flush=True)
