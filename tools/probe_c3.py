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
    out = ft.DeviceCSC.allocate(dphi.n_rows, dphi.n_cols, 3 * dphi.nnz, dphi.values.dtype, dphi.values.device)
    dl = F.device_laplacian(lap, prec); lc = dl.lap_t[prec].ft_csc(); prm = ft.CouplingParams().ft_params()
    st = F._stream_handle()
    a, b = dphi, out
    evs = []
    for i in range(40):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        ac, bc = a.ft_csc(), b.ft_csc()
        e0.record()
        lib.ft_step_kernel(ctypes.byref(lc), dl.flags, ctypes.byref(ac), ctypes.byref(bc), F._ft_dtype(prec), ctypes.byref(prm),
                           ctypes.c_void_p(ws.ws.data_ptr()), ws.ws.numel(), st)
        e1.record()
        lib.ft_step_finalize(ctypes.c_void_p(ws.ws.data_ptr()), ws.ws.numel(), mesh.n_vertices, ctypes.c_void_p(ws.stats.data_ptr()), st)
        evs.append((e0, e1))
        rec = F._stats_from_bytes(ws.stats.cpu().numpy().tobytes())[0]
        b.nnz = int(rec['nnz_phi']); a, b = b, a
    torch.cuda.synchronize()
    ms = np.array([x.elapsed_time(y) for x, y in evs])
    nnz = a.nnz; vb = 8 if prec == "exact" else 4
    byt = (4 * (mesh.n_vertices + 1) + 4 * lap.mat_t.nnz) + 2 * (4 * (mesh.n_vertices + 1) + (4 + vb) * nnz)
    print(f"{prec}: kernel median {np.median(ms):.3f} ms min {ms.min():.3f}  nnz {nnz} skel {int(rec['nnz_skel'])} "
          f"alg bytes {byt/1e9:.3f} GB -> {byt/np.median(ms)/1e6:.0f} GB/s", flush=True)
    # device evolve loop timing
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); cur2, tr2 = ft.evolve(cur, lap, ft.CouplingParams(), max_steps=40, tol=0.0); e1.record(); torch.cuda.synchronize()
    print(f"{prec}: evolve 40 steps {e0.elapsed_time(e1):.2f} ms -> {40/e0.elapsed_time(e1)*1e3:.0f} steps/s", flush=True)
