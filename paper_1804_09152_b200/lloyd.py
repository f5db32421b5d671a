"""Lloyd-like relaxation: centroids, back-projection, reseeding (GPU).

Same API as the reference (pkg/src/fieldtess/lloyd.py:1-229): ``LloydState``,
``lloyd_iterate``, ``faces_by_cell``, ``cell_triangles``, ``approx_centroid``,
``backproject``, ``cell_areas``.

``lloyd_iterate`` runs every stage on the device except the order-dependent
collision pass, which stays sequential on the host, as in the reference
(lloyd.py:174-194):

* the evolve loops (``field.evolve``, device-side stop test);
* faces per cell, via ``ft_faces_by_cell``: the pattern of M^T Phi^T with
  faces ascending per cell;
* all cells' centroids and normals, and the back-projected vertices, via
  ``ft_lloyd_centroids``, using numpy's exact reduction orders.

The single-cell helpers ``approx_centroid`` / ``backproject`` are host numpy
restatements of the reference functions (API convenience).
"""

import ctypes
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .errors import (BackendError, DegenerateCellError, NullNormalError,
                     ShapeError, VanishedCellError)
from .field import (StepWorkspace, _check, _device, _stream_handle, evolve,
                    init_field)
from .sparse import INDEX, SparseMat

LLOYD_OK, LLOYD_VANISHED, LLOYD_DEGENERATE, LLOYD_NULLNORMAL, LLOYD_MISS = 0, 1, 2, 3, 4


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# device copies of the mesh geometry (uploaded once per mesh object)


class _DeviceMesh:
    def __init__(self, mesh, device):
        torch = _torch()

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)

        self.positions = up(mesh.positions, np.float64)
        self.faces = up(mesh.faces, np.int32)
        self.area = up(mesh.face_area, np.float64)
        self.bary = up(mesh.face_barycenter, np.float64)
        self.normal = up(mesh.face_normal, np.float64)
        self.period = (None if mesh.period_vectors is None else
                       (ctypes.c_double * 6)(*np.asarray(mesh.period_vectors, dtype=np.float64).ravel()))
        self.n_vertices = mesh.n_vertices
        self.n_faces = mesh.n_faces


def device_mesh(mesh):
    dm = getattr(mesh, "_ft_device_mesh", None)
    if dm is None:
        dm = _DeviceMesh(mesh, _device())
        try:
            mesh._ft_device_mesh = dm
        except AttributeError:
            pass
    return dm


def _phi_f64(field):
    """The field's device CSC with float64 values (FAST fields are widened)."""
    torch = _torch()
    d = field.device_phi()
    if d.values.dtype == torch.float64:
        return d
    from .sparse import DeviceCSC
    out = DeviceCSC(d.n_rows, d.n_cols, d.col_ptr, d.row_idx, d.values[:max(d.nnz, 1)].double(), d.nnz)
    return out


def _faces_by_cell_device(field, mesh, min_row, with_values):
    """(cell_ptr, cell_faces, values|None) as device tensors."""
    torch = _torch()
    dphi = _phi_f64(field)
    dm = device_mesh(mesh)
    dev = dphi.values.device
    n_rows = dphi.n_rows
    cell_ptr = torch.zeros(n_rows + 1, dtype=torch.int32, device=dev)
    scratch = torch.zeros(2 * n_rows, dtype=torch.int32, device=dev)
    big = torch.zeros(1, dtype=torch.int32, device=dev)
    c = dphi.ft_csc()
    lib = _lib.lib()
    stream = _stream_handle()
    vp = ctypes.c_void_p
    rc = lib.ft_faces_by_cell(ctypes.byref(c), int(min_row), dm.n_faces, vp(dm.faces.data_ptr()),
                              vp(cell_ptr.data_ptr()), None, None, vp(scratch.data_ptr()),
                              vp(big.data_ptr()), stream)
    _check(rc, "ft_faces_by_cell")
    total = int(cell_ptr[n_rows].item())
    cell_faces = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    values = torch.empty(max(total, 1), dtype=torch.float64, device=dev) if with_values else None
    rc = lib.ft_faces_by_cell(ctypes.byref(c), int(min_row), dm.n_faces, vp(dm.faces.data_ptr()),
                              vp(cell_ptr.data_ptr()), vp(cell_faces.data_ptr()),
                              vp(values.data_ptr()) if values is not None else None,
                              vp(scratch.data_ptr()), vp(big.data_ptr()), stream)
    _check(rc, "ft_faces_by_cell")
    if int(big.item()):
        # rows with more than 16384 faces: sort those segments on the device
        ptr = cell_ptr.cpu().numpy()
        for r in np.flatnonzero(np.diff(ptr.astype(np.int64)) > 16384):
            a, b = int(ptr[r]), int(ptr[r + 1])
            cell_faces[a:b] = torch.sort(cell_faces[a:b]).values
        if values is not None:
            raise BackendError("faces_by_cell values for rows with > 16384 faces are not supported")
    return cell_ptr, cell_faces[:total], (values[:total] if values is not None else None)


def faces_by_cell(field, mesh):
    """Face-membership product (n_f x n_rows), one column per layer:
    column r has entry f when some vertex of f carries layer r
    (lloyd.py:21-28), value = the reference's spgemm sum."""
    cell_ptr, cell_faces, values = _faces_by_cell_device(field, mesh, 0, True)
    return SparseMat(mesh.n_faces, field.n_cells + 1, cell_ptr.cpu().numpy(),
                     cell_faces.cpu().numpy().astype(INDEX), values.cpu().numpy(), check=False)


def cell_triangles(field, mesh, cell, product=None):
    """Indices of faces with at least one vertex inside the cell (lloyd.py:31-39)."""
    row = field.cell_row(cell)
    if product is None:
        product = faces_by_cell(field, mesh)
    faces, _ = product.column(row)
    if faces.size == 0:
        raise VanishedCellError(f"vanished-cell: cell {cell} has no faces")
    return faces.astype(np.int64)


def approx_centroid(field, mesh, cell, faces=None):
    """Area-weighted barycenter average and normalised area-weighted normal
    of the cell's triangles (lloyd.py:42-64)."""
    if faces is None:
        faces = cell_triangles(field, mesh, cell)
    areas = mesh.face_area[faces]
    total = float(areas.sum())
    if total <= 0.0:
        raise DegenerateCellError(f"degenerate-cell: cell {cell} has zero area")
    barys = mesh.face_barycenter[faces]
    if mesh.periodic:
        ref = mesh.positions[field.seed_vertices[cell]]
        barys = ref + mesh.wrap_deltas(barys - ref)
    point = (areas[:, None] * barys).sum(axis=0) / total
    nsum = (areas[:, None] * mesh.face_normal[faces]).sum(axis=0)
    norm = float(np.linalg.norm(nsum))
    if norm <= 1e-12 * total:
        raise NullNormalError(f"null-normal: cell {cell} normals cancel")
    return point, nsum / norm


def backproject(point, normal, field, mesh, cell, faces=None):
    """Line point +- t*normal against the cell's triangles; the smallest |t|
    hit's nearest corner vertex, or None on a miss (lloyd.py:67-112)."""
    if faces is None:
        faces = cell_triangles(field, mesh, cell)
    point = np.asarray(point, dtype=np.float64)
    normal = np.asarray(normal, dtype=np.float64)
    tri = mesh.faces[faces]
    p0 = mesh.positions[tri[:, 0]]
    if mesh.periodic:
        e1 = mesh.wrap_deltas(mesh.positions[tri[:, 1]] - p0)
        e2 = mesh.wrap_deltas(mesh.positions[tri[:, 2]] - p0)
        bc = p0 + (e1 + e2) / 3.0
        p0 = p0 + (point + mesh.wrap_deltas(bc - point)) - bc
    else:
        e1 = mesh.positions[tri[:, 1]] - p0
        e2 = mesh.positions[tri[:, 2]] - p0
    h = np.cross(np.broadcast_to(normal, e2.shape), e2)
    det = np.einsum("ij,ij->i", e1, h)
    scale = np.linalg.norm(e1, axis=1) * np.linalg.norm(e2, axis=1)
    ok = np.abs(det) > 1e-14 * np.maximum(scale, 1e-300)
    s = point - p0
    with np.errstate(divide="ignore", invalid="ignore"):
        u = np.einsum("ij,ij->i", s, h) / det
        q = np.cross(s, e1)
        v = np.einsum("ij,j->i", q, normal) / det
        t = np.einsum("ij,ij->i", e2, q) / det
    eps = 1e-12
    hit = ok & (u >= -eps) & (v >= -eps) & (u + v <= 1.0 + eps)
    if not hit.any():
        return None
    idx = np.flatnonzero(hit)
    best = idx[np.argmin(np.abs(t[idx]))]
    hp = point + t[best] * normal
    corners = np.stack([p0[best], p0[best] + e1[best], p0[best] + e2[best]])
    return int(tri[best, int(np.argmin(np.linalg.norm(corners - hp, axis=1)))])


def cell_areas(field, mesh):
    """Field-weighted area per cell: sum of vertex_area * phi (lloyd.py:115-125)."""
    phi = field.phi
    nnz = phi.nnz
    w = phi.values[:nnz] * mesh.vertex_area[phi.entry_columns()]
    sums = np.zeros(phi.n_rows)
    np.add.at(sums, phi.row_idx[:nnz], w)
    return sums[1:]


def cell_geometry(field, mesh, seeds=None):
    """All cells at once on the device: (point[n,3], normal[n,3], status[n],
    hit_vertex[n]) -- the batched form of approx_centroid + backproject."""
    torch = _torch()
    n_cells = field.n_cells
    cell_ptr, cell_faces, _ = _faces_by_cell_device(field, mesh, 1, False)
    dm = device_mesh(mesh)
    dev = cell_ptr.device
    seeds = field.seed_vertices if seeds is None else seeds
    sd = torch.from_numpy(np.ascontiguousarray(seeds, dtype=np.int64)).to(dev)
    point = torch.zeros((max(n_cells, 1), 3), dtype=torch.float64, device=dev)
    normal = torch.zeros((max(n_cells, 1), 3), dtype=torch.float64, device=dev)
    status = torch.zeros(max(n_cells, 1), dtype=torch.int32, device=dev)
    hit = torch.full((max(n_cells, 1),), -1, dtype=torch.int32, device=dev)
    vp = ctypes.c_void_p
    rc = _lib.lib().ft_lloyd_centroids(
        vp(dm.positions.data_ptr()), dm.n_vertices, vp(dm.faces.data_ptr()), dm.n_faces,
        vp(dm.area.data_ptr()), vp(dm.bary.data_ptr()), vp(dm.normal.data_ptr()),
        ctypes.cast(dm.period, ctypes.c_void_p) if dm.period is not None else None, n_cells,
        vp(cell_ptr.data_ptr()), vp(cell_faces.data_ptr()), vp(sd.data_ptr()),
        vp(point.data_ptr()), vp(normal.data_ptr()), vp(status.data_ptr()), vp(hit.data_ptr()),
        _stream_handle())
    _check(rc, "ft_lloyd_centroids")
    return (point[:n_cells].cpu().numpy(), normal[:n_cells].cpu().numpy(),
            status[:n_cells].cpu().numpy(), hit[:n_cells].cpu().numpy())


# ---------------------------------------------------------------------------
# the iteration


@dataclass
class LloydState:
    """Relaxation state: current seeds, field, and per-iteration history."""

    seeds: np.ndarray
    field: object = None
    iteration: int = 0
    history: list = dc_field(default_factory=list)

    def history_json(self):
        return self.history


def _record(state, mesh, trace, reseed_report):
    areas = cell_areas(state.field, mesh)
    state.history.append({
        "iteration": state.iteration,
        "seeds": [int(s) for s in state.seeds],
        "seed_positions": mesh.positions[state.seeds].tolist(),
        "cell_areas": areas.tolist(),
        "area_variance": float(np.var(areas)),
        "steps": len(trace),
        "converged": bool(trace[-1].converged) if trace else True,
        **reseed_report,
    })


def _reseed(state, mesh):
    """New seed per cell (device centroids + back-projection); a miss or a
    vanished / degenerate / null-normal cell keeps its old seed; collisions
    are resolved sequentially in ascending cell order (lloyd.py:155-195)."""
    old = np.asarray(state.seeds, dtype=np.int64)
    _, _, status, hit = cell_geometry(state.field, mesh, seeds=old)
    fail = (status != LLOYD_OK) | (hit < 0)
    candidates = np.where(fail, old, hit.astype(np.int64))
    misses = int(fail.sum())
    taken = set()
    collisions = 0
    seeds = np.empty(old.size, dtype=np.int64)
    members = None
    for c in range(old.size):
        pick = int(candidates[c])
        if pick in taken:
            collisions += 1
            pick = int(old[c])
        if pick in taken:
            if members is None:
                phi = state.field.phi
                members = (phi.row_idx[:phi.nnz], phi.entry_columns())
            mine = members[1][members[0] == c + 1]
            free = [int(v) for v in np.sort(mine) if int(v) not in taken]
            if not free:
                raise VanishedCellError(f"vanished-cell: no free vertex left for cell {c}")
            pick = free[0]
        taken.add(pick)
        seeds[c] = pick
    return seeds, {"reseed_misses": misses, "seed_collisions": collisions}


def lloyd_iterate(state, mesh, lap, params, n_iter, max_steps=1000, tol=1e-4):
    """``n_iter`` relaxation iterations after the initial evolve; records
    ``n_iter + 1`` passes in ``state.history`` (lloyd.py:198-229)."""
    if n_iter < 1:
        raise ShapeError("n_iter must be >= 1")
    ws = StepWorkspace()
    if state.field is None:
        state.field = init_field(mesh, state.seeds)
    if state.field.step_count == 0:
        state.field, trace = evolve(state.field, lap, params, max_steps=max_steps, tol=tol, workspace=ws)
    else:
        trace = []
    if not state.history:
        _record(state, mesh, trace, {"reseed_misses": 0, "seed_collisions": 0})
    for _ in range(n_iter):
        seeds, report = _reseed(state, mesh)
        state.seeds = seeds
        state.iteration += 1
        state.field = init_field(mesh, seeds, precision=state.field.precision)
        state.field, trace = evolve(state.field, lap, params, max_steps=max_steps, tol=tol, workspace=ws)
        _record(state, mesh, trace, report)
    return state

