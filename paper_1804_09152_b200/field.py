"""Layered-field engine on the GPU: seeding, the fused Euler step, evolve.

Public API identical to the reference (pkg/src/fieldtess/field.py:34-404):
``CouplingParams``, ``StepStats``, ``LayeredField``, ``init_field``,
``step``, ``evolve``, ``sharp_labels``, ``band_vertex_fraction``,
``save_field`` / ``load_field``, ``StepWorkspace``, ``UNCLAIMED``.

What changes underneath: the field lives in HBM as CSC (``DeviceCSC``) and
one call of the C-ABI ``ft_step`` runs the whole pipeline of the reference
step (spgemm -> skeleton -> expand -> update -> normalise/compact) as a
single fused kernel; ``evolve`` runs its loop on the device (``ft_evolve``)
with the convergence test evaluated there, reading statistics back once.

Precision: ``"exact"`` (default) stores float64 and is bitwise identical to
the reference; ``"fast"`` stores float32 and computes in float64.  Choose
per field (``init_field(..., precision=)``) or globally with
:func:`set_default_precision`.
"""

import ctypes
import json
import os
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .errors import (BackendError, DuplicateSeedError, NumericalBlowupError,
                     PatternViolationError, ShapeError)
from .sparse import INDEX, DeviceCSC, DeviceTiled, SparseMat, read_triplets_stream, warm_pinned_results

UNCLAIMED = -1
BASE_EXHAUSTION_PER_VERTEX = 1e-9       # field.py:31

_PRECISIONS = ("exact", "fast")
_default_precision = "exact"


def set_default_precision(precision):
    """Select the storage precision of new fields: "exact" | "fast"."""
    global _default_precision
    if precision not in _PRECISIONS:
        raise ShapeError(f"precision must be one of {_PRECISIONS}")
    _default_precision = precision


def get_default_precision():
    return _default_precision


def _torch():
    import torch
    return torch


def _value_dtype(precision):
    torch = _torch()
    return torch.float64 if precision == "exact" else torch.float32


def _ft_dtype(precision):
    return _lib.FT_F64 if precision == "exact" else _lib.FT_F32


def _device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise BackendError("no CUDA device: the engine has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_handle():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _check(rc, where):
    if rc != _lib.FT_OK:
        msg = _lib.last_error()
        if rc == _lib.FT_ERR_SHAPE:
            raise ShapeError(msg or where)
        raise BackendError(f"{where} failed (code {rc}): {msg}")


# ---------------------------------------------------------------------------
# parameter / statistics records


@dataclass
class CouplingParams:
    """Scalar couplings of the update rule (field.py:34-71): pair penalty
    ``w``, gradient coupling ``a``, band interaction ``e`` (``e_base`` against
    the base layer), mobility ``mu`` and the Euler time step ``dt``."""

    w: float = 0.2
    a: float = 1.0
    e: float = 0.3
    e_base: float = 0.2
    mu: float = 0.2
    dt: float = 5.0

    def validate(self):
        if min(self.w, self.a, self.mu, self.dt) <= 0:
            raise ShapeError("w, a, mu, dt must be positive")
        if self.e < 0 or self.e_base < 0:
            raise ShapeError("e, e_base must be non-negative")
        return self

    def to_dict(self):
        return asdict(self)

    @classmethod
    def from_dict(cls, d):
        return cls(**{k: float(v) for k, v in d.items()})

    def ft_params(self):
        return _lib.FtParams(float(self.w), float(self.a), float(self.e),
                             float(self.e_base), float(self.mu), float(self.dt))


@dataclass
class StepStats:
    """Per-step diagnostics (field.py:74-92).  The fused engine has no
    spgemm / skeleton / expand boundaries; :func:`step` reports the device
    time of its kernel groups in the five phase slots (ft_step_phases):
    ``skeleton_time`` layout conversion + active-column selection,
    ``spgemm_time`` the band kernel (fused gather + update + normalise of
    one/two-layer columns), ``expand_time`` the three-layer kernel,
    ``update_time`` the wider-column kernels, ``normalize_time`` statistics
    + compaction.  The device evolve loop (a CUDA graph, no host between
    steps) reports each step's mean device time in ``spgemm_time``.
    ``total_time`` is the step time either way.  ``nnz_skel`` is the
    interest-skeleton size (layer-nnz updates of the step)."""

    max_delta: float
    nnz_phi: int
    base_mass: float
    spgemm_time: float = 0.0
    skeleton_time: float = 0.0
    expand_time: float = 0.0
    update_time: float = 0.0
    normalize_time: float = 0.0
    realloc_count: int = 0
    converged: bool = False
    nnz_skel: int = 0

    @property
    def total_time(self):
        return (self.spgemm_time + self.skeleton_time + self.expand_time
                + self.update_time + self.normalize_time)


# ---------------------------------------------------------------------------
# the field


class LayeredField:
    """The sparse multi-layer field: base layer row 0, cell c in row c+1.

    ``phi`` is the host :class:`SparseMat` view (materialised lazily from the
    device copy); the device CSC is created on first use.
    """

    def __init__(self, phi, seed_vertices, step_count=0, precision=None):
        self._host = None
        self._dev = None
        if isinstance(phi, DeviceCSC):
            self._dev = phi
            torch = _torch()
            self.precision = "exact" if phi.values.dtype == torch.float64 else "fast"
        else:
            self._host = phi
            self.precision = precision or _default_precision
        if self.precision not in _PRECISIONS:
            raise ShapeError(f"precision must be one of {_PRECISIONS}")
        self.seed_vertices = np.asarray(seed_vertices, dtype=np.int64)
        self.step_count = int(step_count)

    # storage ---------------------------------------------------------------

    @property
    def phi(self):
        if self._host is None:
            self._host = self._dev.to_host()
        return self._host

    @phi.setter
    def phi(self, value):
        self._host = value
        self._dev = None

    def device_phi(self):
        """The device CSC of the field (uploaded on first use)."""
        if self._dev is None:
            self._dev = DeviceCSC.from_host(self._host, _value_dtype(self.precision), _device())
        return self._dev

    def _shape(self):
        m = self._dev if self._dev is not None else self._host
        return m.n_rows, m.n_cols

    @property
    def n_cells(self):
        return self._shape()[0] - 1

    @property
    def n_vertices(self):
        return self._shape()[1]

    def copy(self):
        out = LayeredField(self.phi.copy(), self.seed_vertices.copy(), self.step_count,
                           precision=self.precision)
        return out

    def base_mass(self):
        phi = self.phi
        nnz = phi.nnz
        return float(phi.values[:nnz][phi.row_idx[:nnz] == 0].sum())

    def column_sums(self):
        phi = self.phi
        sums = np.zeros(self.n_vertices)
        np.add.at(sums, phi.entry_columns(), phi.values[:phi.nnz])
        return sums

    def cell_row(self, cell):
        if not 0 <= cell < self.n_cells:
            raise ShapeError(f"cell {cell} out of range")
        return cell + 1

    def __repr__(self):
        nnz = self._dev.nnz if self._dev is not None else self._host.nnz
        return (f"LayeredField({self.n_cells} cells, {self.n_vertices} vertices, "
                f"nnz={nnz}, steps={self.step_count}, {self.precision})")


def init_field(mesh, seeds, precision=None):
    """Seed the field: each seed claims itself plus its one-ring; vertices
    claimed k times get 1/k per claimant; unclaimed vertices carry base 1.0
    (field.py:137-166).  Vectorised: no per-seed Python loop."""
    seeds = np.asarray(seeds, dtype=np.int64).ravel()
    if seeds.size != np.unique(seeds).size:
        raise DuplicateSeedError("duplicate-seed: seed list has repeats")
    n_v = mesh.n_vertices
    if seeds.size and (seeds.min() < 0 or seeds.max() >= n_v):
        raise ShapeError("seed vertex index out of range")
    if getattr(mesh, "_topo_dev", None) is not None:
        return _init_field_device(mesh, seeds, precision)
    nptr = np.asarray(mesh.neighbor_ptr, dtype=np.int64)
    nidx = np.asarray(mesh.neighbor_idx, dtype=np.int64)
    deg = nptr[seeds + 1] - nptr[seeds]
    # claimed vertex list per seed: the seed, then its sorted one-ring
    seg = np.cumsum(deg + 1) - (deg + 1)
    total = int((deg + 1).sum())
    cl_row = np.repeat(np.arange(1, seeds.size + 1, dtype=np.int64), deg + 1)
    pos_in = np.arange(total, dtype=np.int64) - np.repeat(seg, deg + 1)
    starts = np.repeat(nptr[seeds], deg + 1)
    is_seed = pos_in == 0
    cl_col = np.where(is_seed, np.repeat(seeds, deg + 1),
                      nidx[np.minimum(starts + pos_in - 1, max(nidx.size - 1, 0))]
                      if nidx.size else 0)
    claims = np.bincount(cl_col, minlength=n_v)
    per_col = np.where(claims == 0, 1, claims)
    col_ptr = np.zeros(n_v + 1, dtype=np.int64)
    np.cumsum(per_col, out=col_ptr[1:])
    row_idx = np.zeros(int(col_ptr[-1]), dtype=INDEX)
    vals = np.ones(int(col_ptr[-1]))
    # claims sorted by (column, row); each lands at col_ptr[col] + rank
    order = np.argsort(cl_col * np.int64(seeds.size + 1) + cl_row, kind="stable")
    sc, sr = cl_col[order], cl_row[order]
    rank = np.arange(sc.size, dtype=np.int64) - np.repeat(
        np.cumsum(claims[claims > 0]) - claims[claims > 0], claims[claims > 0])
    dst = col_ptr[sc] + rank
    row_idx[dst] = sr
    vals[dst] = 1.0 / claims[sc]
    phi = SparseMat(seeds.size + 1, n_v, col_ptr.astype(INDEX), row_idx, vals, check=False)
    return LayeredField(phi, seeds, precision=precision)


def _init_field_device(mesh, seeds, precision):
    """init_field on a device-built mesh: the same claim arithmetic on the
    device one-ring, the field created directly as a device CSC (values
    1.0 / claims in float64, then the storage precision)."""
    torch = _torch()
    topo = mesh._topo_dev
    nptr, nidx = topo["neighbor_ptr"], topo["neighbor_idx"]
    dev = nptr.device
    n_v = mesh.n_vertices
    n_s = seeds.size
    s = torch.from_numpy(seeds).to(dev)
    deg = nptr[s + 1] - nptr[s]
    cnt = deg + 1
    seg = torch.cumsum(cnt, 0) - cnt
    total = int(cnt.sum().item()) if n_s else 0
    cl_row = torch.repeat_interleave(torch.arange(1, n_s + 1, device=dev), cnt)
    pos_in = torch.arange(total, device=dev) - torch.repeat_interleave(seg, cnt)
    starts = torch.repeat_interleave(nptr[s], cnt)
    ring = nidx[torch.clamp(starts + pos_in - 1, 0, max(nidx.numel() - 1, 0))].long()
    cl_col = torch.where(pos_in == 0, torch.repeat_interleave(s, cnt), ring)
    claims = torch.bincount(cl_col, minlength=n_v)
    col_ptr = torch.zeros(n_v + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.where(claims == 0, 1, claims), 0, out=col_ptr[1:])
    nnz = int(col_ptr[-1].item())
    out = DeviceCSC.allocate(n_s + 1, n_v, max(nnz, 1), _value_dtype(precision or _default_precision), dev)
    out.col_ptr.copy_(col_ptr)
    out.row_idx.zero_()
    vals = torch.ones(max(nnz, 1), dtype=torch.float64, device=dev)
    order = torch.argsort(cl_col * (n_s + 1) + cl_row, stable=True)
    sc, sr = cl_col[order], cl_row[order]
    cc = claims[claims > 0]
    rank = torch.arange(sc.numel(), device=dev) - torch.repeat_interleave(torch.cumsum(cc, 0) - cc, cc)
    dst = col_ptr[sc] + rank
    out.row_idx[dst] = sr.to(torch.int32)
    vals[dst] = 1.0 / claims[sc].double()
    out.values.copy_(vals.to(out.values.dtype))
    out.nnz = nnz
    return LayeredField(out, seeds, precision=precision)


# ---------------------------------------------------------------------------
# device-side Laplacian and workspace


class _DeviceLap:
    def __init__(self, lap_t, flags, n_v, symmetric=False):
        self.lap_t = lap_t     # dict precision -> DeviceCSC
        self.flags = flags     # FT_LAP_* of the stored values (UNIFORM / EXPLICIT)
        self.n_v = n_v
        self.symmetric = symmetric   # pattern of L^T symmetric: active-set stepping
        self.pack = None       # packed neighbour table (uniform Laplacians)
        self.n_csr = 0         # columns the pack leaves to the CSR
        self.renum = None      # the same Laplacian in a locality order (device meshes), or None

    def launch_flags(self, phi=None):
        """FT_LAP_* for the step entry points, plus the speed hints from the
        input field ``phi`` (a DeviceCSC): FT_HINT_DENSE_BAND for a dense
        band, FT_HINT_FOUR_ROW for a young one."""
        f = self.flags | (_lib.FT_LAP_PACKED if self.pack is not None else 0)
        if self.symmetric and ACTIVE_SET:
            f |= _lib.FT_LAP_SYMMETRIC
        if phi is not None:
            extra = phi.nnz - phi.n_cols
            if extra >= DENSE_BAND_EXTRA:
                f |= _lib.FT_HINT_DENSE_BAND
            if extra < phi.n_cols // YOUNG_FIELD_DIV:
                f |= _lib.FT_HINT_FOUR_ROW
        return f

    def ft_csc(self, precision):
        """ft_csc of L^T for the step entry points: with FT_LAP_PACKED the
        (never read) uniform values slot carries the packed table."""
        c = self.lap_t[precision].ft_csc()
        if self.pack is not None:
            c.values = self.pack.data_ptr()
        return c


def pack_laplacian(lap_t, col_base=0):
    """Device int16[n_cols][8] neighbour table (ft_laplacian_pack) of a
    DeviceCSC L^T; returns (tensor, columns left to the CSR)."""
    torch = _torch()
    pack = torch.empty(max(lap_t.n_cols, 1) * 8, dtype=torch.int16, device=lap_t.col_ptr.device)
    n_csr = torch.zeros(1, dtype=torch.int32, device=lap_t.col_ptr.device)
    c = lap_t.ft_csc()
    _check(_lib.lib().ft_laplacian_pack(ctypes.byref(c), int(col_base), ctypes.c_void_p(pack.data_ptr()),
                                        ctypes.c_void_p(n_csr.data_ptr()), _stream_handle()),
           "ft_laplacian_pack")
    return pack, int(n_csr.item())


def _uniform_values_exact(mat_t):
    """True when L^T holds exactly the uniform weights: 1.0/deg(j) on the
    off-diagonal of column j and -1.0 on its diagonal (mesh.py:392-400)."""
    n = mat_t.n_cols
    cp = np.asarray(mat_t.col_ptr, dtype=np.int64)
    nnz = int(cp[-1])
    rows = np.asarray(mat_t.row_idx[:nnz], dtype=np.int64)
    vals = np.asarray(mat_t.values[:nnz], dtype=np.float64)
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    cnt = np.diff(cp)
    if np.any(cnt < 2):
        return False
    diag = rows == cols
    if np.bincount(cols[diag], minlength=n).max(initial=0) != 1 or diag.sum() != n:
        return False
    want = np.where(diag, -1.0, 1.0 / (cnt[cols] - 1).astype(np.float64))
    return bool(np.array_equal(vals, want))


def _pattern_symmetric(lap):
    """True when the pattern of L^T equals the pattern of L (lap.mat is the
    transpose of lap.mat_t, both CSC with ascending rows; mesh.py:379-431
    builds both from the symmetric edge set): column j of L^T is read by
    exactly the columns it reads, which active-set stepping relies on."""
    a, b = getattr(lap, "mat", None), lap.mat_t
    if a is None or a.n_cols != b.n_cols or a.n_rows != b.n_rows:
        return False
    pa, pb = np.asarray(a.col_ptr), np.asarray(b.col_ptr)
    if not np.array_equal(pa, pb):
        return False
    nnz = int(pb[-1])
    return bool(np.array_equal(np.asarray(a.row_idx[:nnz]), np.asarray(b.row_idx[:nnz])))


def _with_diagonal(mat_t):
    """L^T with an explicit (zero) diagonal entry wherever one is missing,
    so the fused step always meets PHI(:, j) through u == j.  A zero weight
    adds +0.0 to the accumulator, which leaves every nonzero Lt entry
    bitwise unchanged."""
    n = mat_t.n_cols
    cp = np.asarray(mat_t.col_ptr, dtype=np.int64)
    nnz = int(cp[-1])
    rows = np.asarray(mat_t.row_idx[:nnz], dtype=np.int64)
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    has = np.zeros(n, dtype=bool)
    has[cols[rows == cols]] = True
    if has.all():
        return mat_t
    miss = np.flatnonzero(~has)
    return SparseMat.from_triplets(mat_t.n_rows, n, np.concatenate([rows, miss]),
                                   np.concatenate([cols, miss]),
                                   np.concatenate([np.asarray(mat_t.values[:nnz]),
                                                   np.zeros(miss.size)]))


def _lap_size(lap):
    """Vertex count of a Laplacian without materialising a device-built one."""
    dev = getattr(lap, "device", None)
    return dev["n"] if dev is not None else lap.mat.n_rows


def device_laplacian(lap, precision):
    """Upload ``lap.mat_t`` once per Laplacian object (cached on it)."""
    dev = getattr(lap, "device", None)
    warm_pinned_results(_lap_size(lap))          # first use per size: background, once
    if dev is not None:
        key = ("device", id(dev["idx"]))
    else:
        key = (id(lap.mat_t), int(lap.mat_t.col_ptr[lap.mat_t.n_cols]))
    cache = getattr(lap, "_ft_device", None)
    if cache is None or cache[0] != key:
        if dev is not None:
            # built on the device by ft_uniform_laplacian: the uniform
            # weights, a diagonal in every column and a symmetric pattern
            # by construction; the host copy is never needed
            dl = _DeviceLap({}, _lib.FT_LAP_UNIFORM, dev["n"], symmetric=True)
            dl.host = None
            n, nnz = dev["n"], int(dev["idx"].numel())
            dl.lap_t["exact"] = DeviceCSC(n, n, dev["ptr"], dev["idx"], dev["val_t"], nnz)
            if dev.get("order") is not None:
                torch = _torch()
                from .devmesh import gather_columns
                order = dev["order"]
                inverse = torch.empty_like(order)
                inverse[order] = torch.arange(order.numel(), device=order.device)
                ptr, src = gather_columns(dev["ptr"], order)
                r = _DeviceLap({}, _lib.FT_LAP_UNIFORM, n, symmetric=True)
                r.host = None
                r.lap_t["exact"] = DeviceCSC(n, n, ptr.to(torch.int32),
                                             inverse[dev["idx"][src].long()].to(torch.int32).contiguous(),
                                             dev["val_t"][src].contiguous(), nnz)
                r.order, r.inverse = order, inverse
                dl.renum = r
        else:
            mat_t = _with_diagonal(lap.mat_t)
            flags = _lib.FT_LAP_UNIFORM if _uniform_values_exact(mat_t) else _lib.FT_LAP_EXPLICIT
            dl = _DeviceLap({}, flags, mat_t.n_cols, symmetric=_pattern_symmetric(lap))
            dl.host = mat_t
        cache = (key, dl)
        try:
            lap._ft_device = cache
        except AttributeError:
            pass
    dl = cache[1]
    for d in (dl, getattr(dl, "renum", None)):
        if d is None:
            continue
        if precision not in d.lap_t:
            if d.host is None:
                ex = d.lap_t["exact"]
                d.lap_t[precision] = DeviceCSC(ex.n_rows, ex.n_cols, ex.col_ptr, ex.row_idx,
                                               ex.values.to(_value_dtype(precision)), ex.nnz)
            else:
                d.lap_t[precision] = DeviceCSC.from_host(d.host, _value_dtype(precision), _device())
        if d.pack is None and d.flags == _lib.FT_LAP_UNIFORM and PACK_LAPLACIAN:
            d.pack, d.n_csr = pack_laplacian(d.lap_t[precision])
    return dl


POOL_FRACTION = 0.25    # pool of a hybrid buffer (columns with > 2 entries), relative to nnz
PACK_LAPLACIAN = True   # uniform Laplacians: packed neighbour table (one 16-byte load per column)
POOL_MIN = 4096
ACTIVE_SET = os.environ.get("FT_ACTIVE_SET", "1") != "0"   # active-set stepping (symmetric L^T)
# entries beyond one per column at which the step runs its dense-band
# variant of the three-row kernel (FT_HINT_DENSE_BAND; speed only): C3
# (4,096 seeds on 10M vertices) carries ~0.9M, C5 (65,536 seeds) ~3.5M
DENSE_BAND_EXTRA = int(os.environ.get("FT_DENSE_BAND_EXTRA", str(1 << 21)))
# a field with fewer extra entries than n_cols / YOUNG_FIELD_DIV is young (its
# band still forming, e.g. from init_field): the four-row kernel is launched
# for it (FT_HINT_FOUR_ROW; C3 at step 80 carries 9 %, init_field ~0 %)
YOUNG_FIELD_DIV = 16


class StepWorkspace:
    """Reusable device buffers for the step pipeline (field.py:169-189): the
    workspace (per-tile partial sums, compaction scan, control block), the
    statistics record, two hybrid work buffers and a spare canonical output.
    With a shared workspace the input field's storage is recycled as a later
    output, so only the newest field stays valid (as in the reference)."""

    def __init__(self, recycle=True):
        self.ws = None
        self.ws_n = -1
        self.stats = None
        self.spare = None
        self.tiled = {}
        self.realloc_count = 0
        self.recycle = recycle   # False: scratch only, never hand out a recycled output
        self._trace = None

    def prepare(self, n_v, device):
        torch = _torch()
        if self.ws is None or self.ws_n != n_v:
            nbytes = int(_lib.lib().ft_workspace_bytes(n_v))
            self.ws = torch.zeros(nbytes, dtype=torch.int8, device=device)
            self.ws_n = n_v
            self.tiled = {}
        if self.stats is None:
            self.stats = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=device)

    def tiled_buffer(self, key, like, nnz_hint):
        """Tiled work buffer ``key`` shaped like ``like`` (created or reused)."""
        buf = self.tiled.get(key)
        if (buf is None or buf.n_rows != like.n_rows or buf.n_cols != like.n_cols
                or buf.values.dtype != like.values.dtype):
            cap = max(int(nnz_hint * POOL_FRACTION), POOL_MIN)
            buf = DeviceTiled(like.n_rows, like.n_cols, cap, like.values.dtype, like.values.device)
            self.tiled[key] = buf
        return buf

    def trace_buffer(self, n_steps, device):
        """Device statistics records for n_steps (kept: a stable address lets
        ft_evolve reuse its captured graph across calls)."""
        torch = _torch()
        nbytes = max(n_steps, 1) * _lib.STATS_BYTES
        if self._trace is None or self._trace.numel() < nbytes or self._trace.device != device:
            self._trace = torch.zeros(max(nbytes, 256 * _lib.STATS_BYTES), dtype=torch.uint8, device=device)
        return self._trace

    def take_output(self, like, capacity):
        sp = self.spare if self.recycle else None
        self.spare = None
        if (sp is not None and sp is not like and sp.n_cols == like.n_cols
                and sp.n_rows == like.n_rows and sp.values.dtype == like.values.dtype):
            if sp.grow(capacity):
                self.realloc_count += 1
            return sp
        return DeviceCSC.allocate(like.n_rows, like.n_cols, capacity, like.values.dtype,
                                  like.values.device)

    def ws_args(self):
        return ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel()


_SCRATCH = {}


def _scratch_workspace(n_v, precision, device):
    """The per-device scratch used when the caller passes no workspace: its
    work buffers, statistics records and control block persist between
    calls (so the evolve graph is captured once per field size), but it
    never recycles an output -- every call returns independent storage, as
    the reference's workspace-less calls do (field.py:198-204)."""
    key = (str(device), int(n_v), precision)
    ws = _SCRATCH.get(key)
    if ws is None:
        if len(_SCRATCH) >= 4:
            _SCRATCH.pop(next(iter(_SCRATCH)))
        ws = _SCRATCH[key] = StepWorkspace(recycle=False)
    return ws


def _initial_capacity(dphi):
    # nnz can grow by one vertex ring per step; leave headroom so a regrow
    # (which costs a re-run of the compaction) is rare; growth is >= 1.2x
    return max(2 * dphi.nnz + dphi.n_cols // 8, 1024)


def _stats_from_bytes(buf):
    return np.frombuffer(buf, dtype=_lib.STATS_DTYPE)


def _raise_step_error(rec, field_step_count):
    status = int(rec["status"])
    if status == _lib.FT_STATUS_PATTERN:
        raise PatternViolationError(
            f"pattern-violation: nonzero at ({int(rec['bad_row'])}, {int(rec['bad_col'])}) "
            "outside the skeleton")
    if status == _lib.FT_STATUS_NAN:
        raise NumericalBlowupError(int(rec["nan_col"]), field_step_count + 1)


def _compact(tiled, out, precision, ws, stream):
    """Tiled -> canonical through ft_compact (fresh statistics record)."""
    torch = _torch()
    rec_buf = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=out.values.device)
    t_c, o_c = tiled.ft_tiled(), out.ft_csc()
    wp, wn = ws.ws_args()
    _check(_lib.lib().ft_compact(ctypes.byref(t_c), ctypes.byref(o_c), _ft_dtype(precision),
                                 wp, wn, ctypes.c_void_p(rec_buf.data_ptr()), stream),
           "ft_compact")
    return _stats_from_bytes(rec_buf.cpu().numpy().tobytes())[0]


# ---------------------------------------------------------------------------
# step / evolve


def step(field, lap, params, workspace=None):
    """One explicit Euler step; returns ``(new_field, StepStats)``
    (field.py:198-286).  Converts the input into a hybrid work buffer, runs
    the fused step kernels into a second one and compacts the result into a
    canonical CSC (ft_step)."""
    torch = _torch()
    params.validate()
    n_v = field.n_vertices
    if _lap_size(lap) != n_v:
        raise ShapeError("Laplacian size does not match field")
    dphi = field.device_phi()
    ws = workspace if workspace is not None else _scratch_workspace(n_v, field.precision, dphi.values.device)
    device = dphi.values.device
    dl = device_laplacian(lap, field.precision)
    ws.prepare(n_v, device)
    scratch_in = ws.tiled_buffer("b", dphi, dphi.nnz)
    scratch = ws.tiled_buffer("a", dphi, dphi.nnz)
    out = ws.take_output(dphi, _initial_capacity(dphi))
    reallocs = ws.realloc_count
    ws.realloc_count = 0
    lap_c = dl.ft_csc(field.precision)
    prm = params.ft_params()
    stream = _stream_handle()
    lib = _lib.lib()
    wp, wn = ws.ws_args()
    phase_ms = (ctypes.c_float * 5)()
    while True:
        in_c, si_c, sc_c, out_c = dphi.ft_csc(), scratch_in.ft_tiled(), scratch.ft_tiled(), out.ft_csc()
        rc = lib.ft_step_phases(ctypes.byref(lap_c), dl.launch_flags(dphi), ctypes.byref(in_c), ctypes.byref(si_c),
                                ctypes.byref(sc_c), ctypes.byref(out_c), _ft_dtype(field.precision),
                                ctypes.byref(prm), wp, wn, ctypes.c_void_p(ws.stats.data_ptr()), phase_ms, stream)
        _check(rc, "ft_step_phases")
        rec = _stats_from_bytes(ws.stats.cpu().numpy().tobytes())[0]
        status = int(rec["status"])
        if status == _lib.FT_STATUS_OVERFLOW:
            scratch.grow(int(rec["needed"]) + int(rec["needed"]) // 5)
            scratch_in.grow(int(rec["needed"]) + int(rec["needed"]) // 5)
            reallocs += 1
            continue
        if status == _lib.FT_STATUS_OUT_OVERFLOW:
            out.grow(int(rec["needed"]))
            reallocs += 1
            rc2 = _compact(scratch, out, field.precision, ws, stream)
            if int(rc2["status"]) != _lib.FT_STATUS_OK:
                raise BackendError("compaction failed after growing the output")
        break
    _raise_step_error(rec, field.step_count)
    out.nnz = int(rec["nnz_phi"])
    ws.spare = dphi if ws.recycle else None
    new_field = LayeredField(out, field.seed_vertices, field.step_count + 1)
    stats = StepStats(max_delta=float(rec["max_delta"]), nnz_phi=int(rec["nnz_phi"]),
                      base_mass=float(rec["base_mass"]),
                      skeleton_time=phase_ms[0] * 1e-3, spgemm_time=phase_ms[1] * 1e-3,
                      expand_time=phase_ms[2] * 1e-3, update_time=phase_ms[3] * 1e-3,
                      normalize_time=phase_ms[4] * 1e-3,
                      realloc_count=reallocs, nnz_skel=int(rec["nnz_skel"]))
    return new_field, stats


def evolve(field, lap, params, max_steps=1000, tol=1e-4, workspace=None, on_step=None):
    """Step until converged or ``max_steps`` (field.py:289-321).

    Converged: max_delta < tol and base mass < 1e-9 per vertex.  Without an
    ``on_step`` callback the whole loop runs on the device (``ft_evolve``):
    the stop test is evaluated by the GPU after every step, the field stays
    in tiled form between steps and is compacted once at the end, and the
    statistics are read back once.  The caller's input field is never
    recycled.
    """
    if max_steps < 1:
        raise ShapeError("max_steps must be >= 1")
    params.validate()
    ws = workspace if workspace is not None else _scratch_workspace(
        field.n_vertices, field.precision, field.device_phi().values.device)
    base_threshold = BASE_EXHAUSTION_PER_VERTEX * field.n_vertices
    if on_step is not None:
        return _evolve_host(field, lap, params, max_steps, tol, ws, on_step, base_threshold)
    return _evolve_device(field, lap, params, max_steps, tol, ws, base_threshold)


def _evolve_host(field, lap, params, max_steps, tol, ws, on_step, base_threshold):
    trace = []
    cur = field
    first = field.device_phi()
    for _ in range(max_steps):
        cur, st = step(cur, lap, params, workspace=ws)
        if ws.spare is first:
            ws.spare = None          # never recycle the caller's storage
        on_step(cur, st)
        st.converged = st.max_delta < tol and st.base_mass < base_threshold
        trace.append(st)
        if st.converged:
            break
    return cur, trace


LOCALITY_MIN_STEPS = 8     # evolve calls this long run in the Laplacian's locality order


def _permute_columns(d, cols):
    """A DeviceCSC with column k = column cols[k] of ``d`` (entries kept)."""
    from .devmesh import gather_columns
    ptr, src = gather_columns(d.col_ptr, cols)
    nnz = int(ptr[-1].item())
    keep = max(nnz, 1)
    return DeviceCSC(d.n_rows, d.n_cols, ptr.to(d.col_ptr.dtype), d.row_idx[src][:keep].contiguous(),
                     d.values[src][:keep].contiguous(), nnz)


def _evolve_device(field, lap, params, max_steps, tol, ws, base_threshold, locality=True):
    torch = _torch()
    n_v = field.n_vertices
    if _lap_size(lap) != n_v:
        raise ShapeError("Laplacian size does not match field")
    src = field.device_phi()
    device = src.values.device
    dl = device_laplacian(lap, field.precision)
    # a device-built unstructured mesh's Laplacian carries a Morton order:
    # long evolves run with the vertices renumbered (compact one-ring
    # gathers), the field permuted in and out; L^T keeps each column's entry
    # order, so every value is bitwise the same (DESIGN 8b)
    ren = getattr(dl, "renum", None) if locality and max_steps >= LOCALITY_MIN_STEPS else None
    if ren is not None:
        src = _permute_columns(src, ren.order)
        dl = ren
    ws.prepare(n_v, device)
    wa = ws.tiled_buffer("a", src, src.nnz)
    wb = ws.tiled_buffer("b", src, src.nnz)
    out = ws.take_output(src, _initial_capacity(src))
    trace_dev = ws.trace_buffer(max_steps, device)
    control = torch.zeros(6, dtype=torch.int64, device=device)
    lap_c = dl.ft_csc(field.precision)
    prm = params.ft_params()
    stream = _stream_handle()
    lib = _lib.lib()
    wp, wn = ws.ws_args()
    trace = []
    done = 0
    reallocs = 0
    cur = src
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    while True:
        remaining = max_steps - done
        s_c, a_c, b_c, o_c = cur.ft_csc(), wa.ft_tiled(), wb.ft_tiled(), out.ft_csc()
        ev0.record()
        rc = lib.ft_evolve(ctypes.byref(lap_c), dl.launch_flags(cur), ctypes.byref(s_c), ctypes.byref(a_c),
                           ctypes.byref(b_c), ctypes.byref(o_c), _ft_dtype(field.precision),
                           ctypes.byref(prm), remaining, float(tol), float(base_threshold),
                           wp, wn, ctypes.c_void_p(trace_dev.data_ptr()),
                           ctypes.c_void_p(control.data_ptr()), stream)
        ev1.record()
        _check(rc, "ft_evolve")
        ctl = control.cpu().numpy()
        n, status, compacted = int(ctl[0]), int(ctl[1]), int(ctl[3])
        nrec = min(n + 1, remaining)
        recs = _stats_from_bytes(trace_dev[:nrec * _lib.STATS_BYTES].cpu().numpy().tobytes())
        per_step = ev0.elapsed_time(ev1) * 1e-3 / max(n, 1)
        for k in range(n):
            r = recs[k]
            trace.append(StepStats(max_delta=float(r["max_delta"]), nnz_phi=int(r["nnz_phi"]),
                                   base_mass=float(r["base_mass"]), spgemm_time=per_step,
                                   nnz_skel=int(r["nnz_skel"]),
                                   converged=int(r["status"]) == _lib.FT_STATUS_CONVERGED))
        done += n
        if n > 0:
            last_tiled = wa if n % 2 == 1 else wb
            if compacted == 2:          # canonical output too small
                out.grow(int(ctl[4]))
                reallocs += 1
                if int(_compact(last_tiled, out, field.precision, ws, stream)["status"]) != 0:
                    raise BackendError("compaction failed after growing the output")
            out.nnz = int(ctl[4])
            if cur is not src and ws.recycle:
                ws.spare = cur
            cur = out
        if status in (_lib.FT_STATUS_NAN, _lib.FT_STATUS_PATTERN):
            if ren is not None:     # report in the caller's numbering: rerun unpermuted
                return _evolve_device(field, lap, params, max_steps, tol, ws, base_threshold, locality=False)
            _raise_step_error(recs[n], field.step_count + done)
        if status == _lib.FT_STATUS_OVERFLOW:
            need = int(recs[n]["needed"])
            wa.grow(need + need // 5)
            wb.grow(need + need // 5)
            reallocs += 1
            if n > 0:
                out = ws.take_output(cur, _initial_capacity(cur))
            continue
        break
    if trace:
        trace[-1].realloc_count = reallocs
    if ren is not None:
        back = _permute_columns(cur, ren.inverse)
        if cur is not src and ws.recycle:
            ws.spare = cur
        cur = back
    elif cur is src:                    # no step completed (cannot happen without error)
        cur = src.clone()
    return LayeredField(cur, field.seed_vertices, field.step_count + done), trace


# ---------------------------------------------------------------------------
# labels and small host utilities


def sharp_labels(field):
    """Per-vertex argmax cell id (ties -> lowest id); UNCLAIMED (-1) where
    the base strictly dominates (field.py:324-356).  GPU kernel
    ``ft_labels``; returns a host int64 array."""
    torch = _torch()
    dphi = field.device_phi()
    labels = torch.empty(max(dphi.n_cols, 1), dtype=torch.int64, device=dphi.values.device)
    c = dphi.ft_csc()
    rc = _lib.lib().ft_labels(ctypes.byref(c), _ft_dtype(field.precision),
                              ctypes.c_void_p(labels.data_ptr()), _stream_handle())
    _check(rc, "ft_labels")
    from .sparse import pinned_copy
    return pinned_copy(labels[:dphi.n_cols])


def band_vertex_fraction(field):
    """Fraction of vertices carrying two or more cell layers (field.py:359-366)."""
    phi = field.phi
    nnz = phi.nnz
    cols = phi.entry_columns()[phi.row_idx[:nnz] != 0]
    counts = np.bincount(cols, minlength=phi.n_cols)
    return float((counts >= 2).sum()) / max(phi.n_cols, 1)


def save_field(field, params, path, extra_header=None):
    """Snapshot: ``#FIELD {json}`` header, ``rows cols nnz``, then one
    ``row col repr(value)`` line per entry (field.py:372-387)."""
    header = {"seeds": [int(s) for s in field.seed_vertices],
              "step_count": field.step_count, "params": params.to_dict()}
    if extra_header:
        header.update(extra_header)
    phi = field.phi
    nnz = phi.nnz
    cols = phi.entry_columns()
    with open(path, "w") as fh:
        fh.write(f"#FIELD {json.dumps(header, sort_keys=True)}\n")
        fh.write(f"{phi.n_rows} {phi.n_cols} {nnz}\n")
        fh.writelines(f"{r} {c} {v!r}\n" for r, c, v in
                      zip(phi.row_idx[:nnz].tolist(), cols.tolist(),
                          phi.values[:nnz].tolist()))


def load_field(path):
    """Read a :func:`save_field` snapshot; returns ``(field, params)``."""
    with open(path) as fh:
        first = fh.readline()
        if not first.startswith("#FIELD "):
            raise ShapeError(f"{path}: not a field snapshot")
        header = json.loads(first[len("#FIELD "):])
        phi = read_triplets_stream(fh, first_lineno=2)
    params = CouplingParams.from_dict(header["params"])
    return LayeredField(phi, np.asarray(header["seeds"], dtype=np.int64),
                        header.get("step_count", 0)), params
