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

The single-cell helpers ``approx_centroid`` / ``backproject`` run the same
kernels on one cell; ``cell_areas`` is the device sparse product PHI a.
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

        da = mesh.device_arrays() if hasattr(mesh, "device_arrays") else None
        if da is not None and da[0].device == device:
            # built on this device (devmesh): reuse, no host round trip
            self.positions, self.faces = da
            g = mesh._device_geometry()
            self.area, self.bary, self.normal = g["face_area"], g["face_barycenter"], g["face_normal"]
        else:
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
    dm = device_mesh(mesh)
    return faces_by_cell_arrays(_phi_f64(field), dm.faces, dm.n_faces, min_row, with_values)


def faces_by_cell_arrays(dphi, faces, n_faces, min_row, with_values):
    """ft_faces_by_cell on a device CSC field (float64) and a device face
    list (int32 [n_faces][3], vertex ids = the field's columns):
    (cell_ptr, cell_faces, values|None), faces ascending per row."""
    torch = _torch()
    dev = dphi.values.device
    n_rows = dphi.n_rows
    cell_ptr = torch.zeros(n_rows + 1, dtype=torch.int32, device=dev)
    scratch = torch.zeros(2 * n_rows, dtype=torch.int32, device=dev)
    big = torch.zeros(1, dtype=torch.int32, device=dev)
    c = dphi.ft_csc()
    lib = _lib.lib()
    stream = _stream_handle()
    vp = ctypes.c_void_p
    rc = lib.ft_faces_by_cell(ctypes.byref(c), int(min_row), int(n_faces), vp(faces.data_ptr()),
                              vp(cell_ptr.data_ptr()), None, None, vp(scratch.data_ptr()),
                              vp(big.data_ptr()), stream)
    _check(rc, "ft_faces_by_cell")
    total = int(cell_ptr[n_rows].item())
    cell_faces = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    values = torch.empty(max(total, 1), dtype=torch.float64, device=dev) if with_values else None
    rc = lib.ft_faces_by_cell(ctypes.byref(c), int(min_row), int(n_faces), vp(faces.data_ptr()),
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


def _single_cell(faces, device):
    """The one-cell CSR the batched Lloyd kernels take (cell 0 = row 1)."""
    torch = _torch()
    f = np.ascontiguousarray(faces, dtype=np.int32)
    ptr = torch.tensor([0, 0, f.size], dtype=torch.int32, device=device)
    lst = torch.from_numpy(f if f.size else np.zeros(1, np.int32)).to(device)
    return ptr, lst


def _geometry_status(status, cell):
    if status == LLOYD_DEGENERATE or status == LLOYD_VANISHED:
        raise DegenerateCellError(f"degenerate-cell: cell {cell} has zero area")
    if status == LLOYD_NULLNORMAL:
        raise NullNormalError(f"null-normal: cell {cell} normals cancel")


def approx_centroid(field, mesh, cell, faces=None):
    """Area-weighted mean barycenter and normalised area-weighted normal of
    the cell's triangles (lloyd.py:42-64) -- the device centroid kernel on
    one cell (numpy's reduction orders, periodic barycenters unwrapped
    around the cell's seed)."""
    torch = _torch()
    if faces is None:
        faces = cell_triangles(field, mesh, cell)
    dm = device_mesh(mesh)
    dev = dm.positions.device
    ptr, lst = _single_cell(faces, dev)
    seed = torch.tensor([int(field.seed_vertices[cell])], dtype=torch.int64, device=dev)
    out = torch.zeros(6, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    hit = torch.zeros(1, dtype=torch.int32, device=dev)
    vp = ctypes.c_void_p
    _check(_lib.lib().ft_lloyd_centroids(
        vp(dm.positions.data_ptr()), dm.n_vertices, vp(dm.faces.data_ptr()), dm.n_faces,
        vp(dm.area.data_ptr()), vp(dm.bary.data_ptr()), vp(dm.normal.data_ptr()),
        ctypes.cast(dm.period, ctypes.c_void_p) if dm.period is not None else None, 1,
        vp(ptr.data_ptr()), vp(lst.data_ptr()), vp(seed.data_ptr()), vp(out.data_ptr()),
        vp(out.data_ptr() + 24), vp(status.data_ptr()), vp(hit.data_ptr()), _stream_handle()),
        "ft_lloyd_centroids")
    _geometry_status(int(status.item()), cell)
    o = out.cpu().numpy()
    return o[:3].copy(), o[3:].copy()


def backproject(point, normal, field, mesh, cell, faces=None):
    """Cast the line ``point + t normal`` through the cell's triangles;
    the corner vertex nearest to the hit of smallest |t|, or None on a miss
    (lloyd.py:67-112) -- the device back-projection kernel on one cell."""
    torch = _torch()
    if faces is None:
        faces = cell_triangles(field, mesh, cell)
    dm = device_mesh(mesh)
    dev = dm.positions.device
    ptr, lst = _single_cell(faces, dev)
    pn = np.concatenate([np.asarray(point, dtype=np.float64).ravel(), np.asarray(normal, dtype=np.float64).ravel()])
    pnd = torch.from_numpy(pn).to(dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    hit = torch.full((1,), -1, dtype=torch.int32, device=dev)
    vp = ctypes.c_void_p
    _check(_lib.lib().ft_lloyd_backproject(
        vp(dm.positions.data_ptr()), dm.n_vertices, vp(dm.faces.data_ptr()), dm.n_faces,
        ctypes.cast(dm.period, ctypes.c_void_p) if dm.period is not None else None, 1,
        vp(ptr.data_ptr()), vp(lst.data_ptr()), vp(pnd.data_ptr()), vp(pnd.data_ptr() + 24),
        vp(status.data_ptr()), vp(hit.data_ptr()), _stream_handle()), "ft_lloyd_backproject")
    h = int(hit.item())
    return None if h < 0 else h


def cell_areas(field, mesh):
    """Field-weighted area of every cell, sum over vertices of
    vertex_area * phi (lloyd.py:115-125): the sparse product PHI a on the
    device (the products phi * area accumulated per row in vertex order,
    the reference's np.add.at order); the base row is dropped."""
    from .sparse import spgemm
    a = SparseMat(mesh.n_vertices, 1, np.array([0, mesh.n_vertices], dtype=INDEX),
                  np.arange(mesh.n_vertices, dtype=INDEX), np.asarray(mesh.vertex_area, dtype=np.float64),
                  check=False)
    prod = spgemm(field.phi, a)
    out = np.zeros(field.phi.n_rows)
    out[prod.row_idx[:prod.nnz]] = prod.values[:prod.nnz]
    return out[1:]


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
    """Relaxation state (lloyd.py:128-138): the seeds, the current field,
    the iteration counter and one history record per evolve pass."""

    seeds: np.ndarray
    field: object = None
    iteration: int = 0
    history: list = dc_field(default_factory=list)

    def history_json(self):
        return self.history


def _history_entry(state, mesh, trace, report):
    """One history record (the reference's keys, lloyd.py:141-152)."""
    seeds = np.asarray(state.seeds, dtype=np.int64)
    areas = cell_areas(state.field, mesh)
    rec = dict(iteration=state.iteration,
               seeds=seeds.tolist(),
               seed_positions=mesh.positions[seeds].tolist(),
               cell_areas=areas.tolist(),
               area_variance=float(np.var(areas)),
               steps=len(trace),
               converged=bool(trace[-1].converged) if len(trace) else True)
    rec.update(report)
    return rec


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
    """Lloyd-like relaxation (lloyd.py:198-229): unless the state's field has
    already been stepped, evolve it first; then ``n_iter`` times reseed at
    the back-projected centroids, re-seed the field and evolve again.  Each
    evolve pass appends a history record, so a fresh state ends with
    ``n_iter + 1`` records."""
    if n_iter < 1:
        raise ShapeError("n_iter must be >= 1")
    ws = StepWorkspace()

    def converge(fld):
        return evolve(fld, lap, params, max_steps=max_steps, tol=tol, workspace=ws)

    no_reseed = {"reseed_misses": 0, "seed_collisions": 0}
    if state.field is None:
        state.field = init_field(mesh, state.seeds)
    trace = []
    if state.field.step_count == 0:
        state.field, trace = converge(state.field)
    if not state.history:
        state.history.append(_history_entry(state, mesh, trace, no_reseed))
    for _ in range(n_iter):
        state.seeds, report = _reseed(state, mesh)
        state.iteration += 1
        state.field, trace = converge(init_field(mesh, state.seeds, precision=state.field.precision))
        state.history.append(_history_entry(state, mesh, trace, report))
    return state
