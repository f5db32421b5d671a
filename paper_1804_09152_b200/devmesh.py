"""Mesh generation, derived data and the uniform Laplacian on the GPU
(§8(f)1; reference mesh.py:20-246, 379-431).

The host generators in :mod:`mesh` are order-identical numpy restatements
that need minutes at the benchmark sizes (icosphere-12: 168M vertices); the
same outputs come from ft_mesh.cu in seconds and stay resident for the
engine.  Everything here is bitwise the reference's (SHA-pinned against
tests/golden/meshes.json by tests/test_devmesh.py).  Sorting, unique and
scans are torch primitives on the device; the arithmetic is ours.

Host copies of the results are made on first access (``TriMesh`` /
``Laplacian`` materialise lazily), so a caller that only steps the field
never pays the device-to-host traffic for edges, one-rings or L.
"""

import ctypes
import os
import warnings

import numpy as np

from . import _lib
from .errors import BackendError

_vp = ctypes.c_void_p
LOCALITY_MIN_VERTICES = 1 << 20   # device meshes this large (not tori) get a Morton order for evolve


def _torch():
    import torch
    return torch


def enabled():
    """Device generators are used when a GPU is present (FT_HOST_MESH=1
    forces the host restatements)."""
    if os.environ.get("FT_HOST_MESH", "0") == "1":
        return False
    try:
        torch = _torch()
    except ImportError:
        return False
    return torch.cuda.is_available()


def _ptr(t):
    return _vp(t.data_ptr())


def _stream():
    return _vp(_torch().cuda.current_stream().cuda_stream)


def _call(name, *args):
    rc = getattr(_lib.lib(), name)(*args)
    if rc != 0:
        raise BackendError(f"{name} failed with code {rc}: {_lib.last_error()}")


def _device():
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device())


# -- generators --------------------------------------------------------------


def _base_twins(faces):
    """Opposite half-edge of every half-edge 3 f + e of a face list (-1 on
    a boundary); the 20-face icosahedron only."""
    at = {}
    for f, tri in enumerate(faces.tolist()):
        for e in range(3):
            at[(tri[e], tri[(e + 1) % 3])] = 3 * f + e
    tw = np.full(3 * len(faces), -1, dtype=np.int32)
    for (u, v), h in at.items():
        tw[h] = at.get((v, u), -1)
    return tw


def icosphere(subdiv, base_positions, base_faces):
    """(positions (n, 3) float64, faces (20 4^L, 3) int32) on the device;
    ``base_positions`` are the unit icosahedron vertices (host, normalised as
    the reference does)."""
    torch = _torch()
    dev = _device()
    n_final = 10 * 4 ** subdiv + 2
    pos = torch.empty((n_final, 3), dtype=torch.float64, device=dev)
    pos[:12] = torch.from_numpy(np.ascontiguousarray(base_positions, dtype=np.float64)).to(dev)
    faces = torch.from_numpy(np.ascontiguousarray(base_faces, dtype=np.int32)).to(dev)
    twin = torch.from_numpy(_base_twins(np.asarray(base_faces))).to(dev)
    n_old = 12
    s = _stream()
    for _ in range(subdiv):
        n_f = faces.shape[0]
        flag = torch.empty(3 * n_f, dtype=torch.int32, device=dev)
        _call("ft_ico_flags", 3 * n_f, _ptr(twin), _ptr(flag), s)
        incl = torch.cumsum(flag, 0, dtype=torch.int64)
        del flag
        mid = torch.empty(3 * n_f, dtype=torch.int32, device=dev)
        _call("ft_ico_midpoints", n_f, _ptr(faces), _ptr(twin), _ptr(incl), n_old, _ptr(pos), _ptr(mid), s)
        n_new = int(incl[-1].item())
        del incl
        faces2 = torch.empty((4 * n_f, 3), dtype=torch.int32, device=dev)
        twin2 = torch.empty(12 * n_f, dtype=torch.int32, device=dev)
        _call("ft_ico_children", n_f, _ptr(faces), _ptr(twin), _ptr(mid), _ptr(faces2), _ptr(twin2), s)
        faces, twin = faces2, twin2
        del mid
        n_old += n_new
    if n_old != n_final:
        raise BackendError(f"icosphere subdivision produced {n_old} vertices, expected {n_final}")
    _call("ft_renormalize", n_final, _ptr(pos), s)
    return pos, faces


def torus(nx, ny, spacing):
    torch = _torch()
    dev = _device()
    pos = torch.empty((nx * ny, 3), dtype=torch.float64, device=dev)
    faces = torch.empty((2 * nx * ny, 3), dtype=torch.int32, device=dev)
    _call("ft_torus_grid", nx, ny, float(spacing), _ptr(pos), _ptr(faces), _stream())
    return pos, faces


# -- derived data ------------------------------------------------------------


def topology(n_v, faces):
    """Sorted unique undirected edges (E, 2) int64, degree (n,) int64 and
    the sorted one-ring CSR (ptr int64, idx int32) of a device face list --
    TriMesh._topology (mesh.py:20-60) on the device.  Warns on non-manifold
    edges like the reference."""
    torch = _torch()
    n = max(int(n_v), 1)
    f = faces.long()
    key = torch.minimum(f, f.roll(-1, dims=1)) * n + torch.maximum(f, f.roll(-1, dims=1))
    del f
    keys, counts = torch.unique(key.t().reshape(-1), sorted=True, return_counts=True)
    del key
    bad = int((counts > 2).sum().item())
    del counts
    if bad:
        warnings.warn(f"{bad} non-manifold edge(s) (more than 2 incident faces); neighbors are treated "
                      "uniformly", RuntimeWarning, stacklevel=4)
    e0, e1 = keys // n, keys % n
    del keys
    edges = torch.stack([e0, e1], dim=1)
    src = torch.cat([e0, e1])
    degree = torch.bincount(src, minlength=int(n_v))
    ring = torch.sort(src * n + torch.cat([e1, e0])).values
    del src, e0, e1
    idx = (ring % n).to(torch.int32)
    del ring
    ptr = torch.zeros(int(n_v) + 1, dtype=torch.int64, device=faces.device)
    torch.cumsum(degree, 0, out=ptr[1:])
    return {"edges": edges, "degree": degree, "neighbor_ptr": ptr, "neighbor_idx": idx}


def geometry(positions, faces, period_vectors=None, quarter_r2=0.0):
    """face_area, face_normal, face_barycenter, vertex_area as device
    tensors (TriMesh._geometry, mesh.py:56-84)."""
    torch = _torch()
    dev = positions.device
    n_f, n_v = faces.shape[0], positions.shape[0]
    area = torch.empty(n_f, dtype=torch.float64, device=dev)
    third = torch.empty(n_f, dtype=torch.float64, device=dev)
    normal = torch.empty((n_f, 3), dtype=torch.float64, device=dev)
    bary = torch.empty((n_f, 3), dtype=torch.float64, device=dev)
    per = None
    if period_vectors is not None:
        per = (ctypes.c_double * 6)(*np.asarray(period_vectors, dtype=np.float64).ravel().tolist())
    s = _stream()
    _call("ft_face_geometry", n_f, _ptr(positions), _ptr(faces), per, float(quarter_r2), _ptr(area),
          _ptr(normal), _ptr(bary), _ptr(third), s)
    corner = torch.sort(faces.reshape(-1), stable=True)
    ptr = torch.zeros(n_v + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.bincount(corner.values.long(), minlength=n_v), 0, out=ptr[1:])
    vertex_area = torch.empty(n_v, dtype=torch.float64, device=dev)
    _call("ft_vertex_area", n_v, _ptr(ptr), _ptr(corner.indices), _ptr(third), _ptr(vertex_area), s)
    return {"face_area": area, "face_normal": normal, "face_barycenter": bary, "vertex_area": vertex_area}


def uniform_laplacian(n_v, neighbor_ptr, neighbor_idx):
    """(ptr, idx, values of L^T, values of L) of the uniform Laplacian
    (mesh.py:392-400) on the device; L and L^T share the pattern."""
    torch = _torch()
    dev = neighbor_ptr.device
    nnz = int(neighbor_idx.numel()) + int(n_v)
    if nnz >= 2 ** 31:
        raise BackendError("Laplacian exceeds int32 indexing")
    ptr = torch.empty(int(n_v) + 1, dtype=torch.int32, device=dev)
    idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    val_t = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    _call("ft_uniform_laplacian", int(n_v), _ptr(neighbor_ptr), _ptr(neighbor_idx), _ptr(ptr), _ptr(idx),
          _ptr(val_t), _ptr(val), _stream())
    return ptr, idx, val_t, val


# -- locality renumbering ------------------------------------------------------


def _spread3_device(x):
    x = x & 0x1FFFFF
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                        (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        x = (x | (x << shift)) & mask
    return x


def morton_order_device(positions):
    """Vertices sorted by the Morton (Z-order) code of their positions
    (distributed.morton_order on the host: same codes, same stable order):
    contiguous ranges of the order are compact surface patches."""
    torch = _torch()
    lo = positions.min(dim=0).values
    span = float((positions.max(dim=0).values - lo).max().item()) or 1.0
    q = torch.floor((positions - lo) / span * (2 ** 21 - 1)).long()
    code = _spread3_device(q[:, 0]) | (_spread3_device(q[:, 1]) << 1) | (_spread3_device(q[:, 2]) << 2)
    return torch.argsort(code, stable=True)


def gather_columns(ptr, cols):
    """(new_ptr, src) of the CSC columns ``cols`` of a matrix with column
    pointers ``ptr`` (device tensors): src = the entry positions in column
    order, entries kept in stored order."""
    torch = _torch()
    p = ptr.long()
    start = p[cols]
    cnt = p[cols + 1] - start
    new_ptr = torch.zeros(cols.numel() + 1, dtype=torch.int64, device=ptr.device)
    torch.cumsum(cnt, 0, out=new_ptr[1:])
    total = int(new_ptr[-1].item())
    src = (torch.repeat_interleave(start - new_ptr[:-1], cnt, output_size=total)
           + torch.arange(total, device=ptr.device))
    return new_ptr, src
