"""Sparse storage: the host CSC container and its device-resident twin.

``SparseMat`` is the host-side interchange type with the reference's
interface (pkg/src/fieldtess/sparse.py:27-178): CSC, int32 ``col_ptr`` /
``row_idx``, float64 ``values``, spare capacity, canonical (strictly
increasing rows per column).  Fields coming back from the GPU are
materialised into it lazily.

``DeviceCSC`` holds the same three arrays as CUDA tensors (values float64 in
EXACT mode, float32 in FAST mode) with explicit capacity.  It is what the
C-ABI consumes (``ft_csc`` in include/fieldtess_cuda.h).
"""

import ctypes
import math
import threading
import warnings

import numpy as np

from .errors import NegativeFieldError, PatternViolationError, ShapeError

INDEX = np.int32
GROWTH = 1.2   # capacity growth factor (sparse.py:24, :212-232)


class SparseMat:
    """Host CSC matrix: int32 indices, float64 values, explicit capacity."""

    __slots__ = ("n_rows", "n_cols", "col_ptr", "row_idx", "values",
                 "realloc_count")

    def __init__(self, n_rows, n_cols, col_ptr, row_idx, values, check=True):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=INDEX)
        self.row_idx = np.ascontiguousarray(row_idx, dtype=INDEX)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.realloc_count = 0
        if self.row_idx.size != self.values.size:
            raise ShapeError("row_idx and values must have equal length")
        if check:
            self.validate()

    # construction -----------------------------------------------------------

    @classmethod
    def empty(cls, n_rows, n_cols, capacity=0):
        return cls(n_rows, n_cols, np.zeros(n_cols + 1, dtype=INDEX),
                   np.empty(capacity, dtype=INDEX),
                   np.empty(capacity, dtype=np.float64), check=False)

    @classmethod
    def identity(cls, n):
        return cls(n, n, np.arange(n + 1, dtype=INDEX), np.arange(n, dtype=INDEX),
                   np.ones(n), check=False)

    @classmethod
    def from_triplets(cls, n_rows, n_cols, rows, cols, vals, sum_dups=True):
        """Canonical matrix from (row, col, value) triplets; duplicates are
        summed and explicit zeros kept (the reference's convention)."""
        rows = np.asarray(rows, dtype=np.int64).ravel()
        cols = np.asarray(cols, dtype=np.int64).ravel()
        vals = np.asarray(vals, dtype=np.float64).ravel()
        if not rows.size == cols.size == vals.size:
            raise ShapeError("triplet arrays must have equal length")
        if rows.size and (rows.min() < 0 or rows.max() >= n_rows
                          or cols.min() < 0 or cols.max() >= n_cols):
            raise ShapeError("triplet index out of range")
        key = cols * np.int64(max(n_rows, 1)) + rows
        order = np.argsort(key, kind="stable")
        key, rows, cols, vals = key[order], rows[order], cols[order], vals[order]
        if key.size:
            head = np.empty(key.size, dtype=bool)
            head[0] = True
            np.not_equal(key[1:], key[:-1], out=head[1:])
            if not head.all():
                if not sum_dups:
                    raise ShapeError("duplicate triplet position")
                starts = np.flatnonzero(head)
                vals = np.add.reduceat(vals, starts)
                rows, cols = rows[starts], cols[starts]
        col_ptr = np.zeros(n_cols + 1, dtype=np.int64)
        np.cumsum(np.bincount(cols, minlength=n_cols), out=col_ptr[1:])
        return cls(n_rows, n_cols, col_ptr.astype(INDEX), rows.astype(INDEX),
                   vals, check=False)

    @classmethod
    def from_dense(cls, dense):
        dense = np.asarray(dense, dtype=np.float64)
        r, c = np.nonzero(dense)
        return cls.from_triplets(dense.shape[0], dense.shape[1], r, c, dense[r, c])

    # views ------------------------------------------------------------------

    @property
    def nnz(self):
        return int(self.col_ptr[self.n_cols])

    @property
    def capacity(self):
        return self.row_idx.size

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def column(self, j):
        a, b = self.col_ptr[j], self.col_ptr[j + 1]
        return self.row_idx[a:b], self.values[a:b]

    def get(self, i, j):
        rows, vals = self.column(j)
        k = np.searchsorted(rows, i)
        return float(vals[k]) if k < rows.size and rows[k] == i else 0.0

    def entry_columns(self):
        return np.repeat(np.arange(self.n_cols, dtype=np.int64),
                         np.diff(self.col_ptr.astype(np.int64)))

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        nnz = self.nnz
        out[self.row_idx[:nnz], self.entry_columns()] = self.values[:nnz]
        return out

    def copy(self):
        nnz = self.nnz
        return SparseMat(self.n_rows, self.n_cols, self.col_ptr.copy(),
                         self.row_idx[:nnz].copy(), self.values[:nnz].copy(),
                         check=False)

    def validate(self):
        cp = self.col_ptr.astype(np.int64)
        if cp.size != self.n_cols + 1 or (cp.size and cp[0] != 0):
            raise ShapeError("bad col_ptr header")
        if np.any(np.diff(cp) < 0):
            raise ShapeError("col_ptr must be non-decreasing")
        nnz = self.nnz
        if nnz > self.capacity:
            raise ShapeError("nnz exceeds capacity")
        ri = self.row_idx[:nnz].astype(np.int64)
        if nnz and (ri.min() < 0 or ri.max() >= self.n_rows):
            raise ShapeError("row index out of range")
        if nnz > 1:
            # strictly increasing inside every column: a non-increase is only
            # allowed where a new column starts
            bad = np.flatnonzero(np.diff(ri) <= 0) + 1
            starts = np.zeros(nnz, dtype=bool)
            starts[cp[1:-1][cp[1:-1] < nnz]] = True
            bad = bad[~starts[bad]]
            if bad.size:
                j = int(np.searchsorted(cp, bad[0], side="right") - 1)
                raise ShapeError(f"rows not strictly increasing in column {j}")

    def __repr__(self):
        return f"SparseMat({self.n_rows}x{self.n_cols}, nnz={self.nnz}, capacity={self.capacity})"


def ensure_capacity(mat, needed):
    """Grow host storage to ``needed`` entries, by at least 1.2x
    (sparse.py:212-232); counts reallocations."""
    needed = int(needed)
    cap = mat.capacity
    if cap >= needed:
        return mat
    new_cap = max(needed, int(math.ceil(cap * GROWTH)))
    nnz = mat.nnz
    ri = np.empty(new_cap, dtype=INDEX)
    va = np.empty(new_cap, dtype=np.float64)
    ri[:nnz] = mat.row_idx[:nnz]
    va[:nnz] = mat.values[:nnz]
    mat.row_idx, mat.values = ri, va
    mat.realloc_count += 1
    return mat


class Skeleton:
    """A sparse pattern without values: the rows of interest per column
    (sparse.py:181-209)."""

    __slots__ = ("n_rows", "n_cols", "col_ptr", "row_idx", "realloc_count")

    def __init__(self, n_rows, n_cols, col_ptr, row_idx):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=INDEX)
        self.row_idx = np.ascontiguousarray(row_idx, dtype=INDEX)
        self.realloc_count = 0

    @property
    def nnz(self):
        return int(self.col_ptr[self.n_cols])

    @property
    def capacity(self):
        return int(self.row_idx.size)

    def column(self, j):
        return self.row_idx[self.col_ptr[j]:self.col_ptr[j + 1]]

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols), dtype=bool)
        cols = np.repeat(np.arange(self.n_cols), np.diff(self.col_ptr.astype(np.int64)))
        out[self.row_idx[:self.nnz], cols] = True
        return out


def transpose(a):
    """Exact transpose in canonical CSC (host; counting sort by row)."""
    nnz = a.nnz
    rows = a.row_idx[:nnz].astype(np.int64)
    order = np.argsort(rows, kind="stable")       # stable: keeps column order
    t_ptr = np.zeros(a.n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=a.n_rows), out=t_ptr[1:])
    return SparseMat(a.n_cols, a.n_rows, t_ptr.astype(INDEX),
                     a.entry_columns()[order].astype(INDEX),
                     a.values[:nnz][order], check=False)


# ---------------------------------------------------------------------------
# device twin


def _torch():
    import torch
    return torch


_WARMED = set()
_WARM_LOCK = threading.Lock()
WARM_PINNED_MAX_BYTES = 2 << 30     # largest result set whose pinned blocks are warmed ahead


def warm_pinned_results(n_cols, nnz_hint=None):
    """Pre-allocate (and release into torch's caching host allocator) pinned
    blocks of the sizes a field of ``n_cols`` vertices returns to the host --
    col_ptr, row_idx, values, labels -- on a background thread, so the first
    ``field.phi`` / ``sharp_labels`` of a process does not pay the page
    pinning (~0.5 ms per MB) on its critical path.  Called when a Laplacian
    is first put on the device."""
    n = int(n_cols)
    nnz = int(nnz_hint) if nnz_hint is not None else n + n // 4     # a typical band: 1.1-1.4 entries/vertex
    # three sets: a caller usually still holds its previous result (and
    # perhaps a pinned copy of its input)
    sizes = [4 * (n + 1), 4 * nnz, 8 * nnz, 8 * n]
    if sum(sizes) * 3 > WARM_PINNED_MAX_BYTES:
        return None
    with _WARM_LOCK:
        if n in _WARMED:
            return None
        _WARMED.add(n)

    def work():
        torch = _torch()
        try:
            blocks = [torch.empty(sz, dtype=torch.uint8, pin_memory=True) for sz in sizes for _ in range(3)]
            del blocks
        except RuntimeError:
            pass

    th = threading.Thread(target=work, name="ft-pinned-warm", daemon=True)
    th.start()
    return th


def pinned_copy(t):
    """Device tensor -> numpy array backed by pinned host memory."""
    torch = _torch()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


class DeviceCSC:
    """CSC arrays resident on the GPU (torch CUDA tensors).

    ``values`` dtype is float64 (EXACT) or float32 (FAST).  ``nnz`` is known
    on the host once the producing step's statistics were read back.
    """

    __slots__ = ("n_rows", "n_cols", "col_ptr", "row_idx", "values", "nnz",
                 "realloc_count")

    def __init__(self, n_rows, n_cols, col_ptr, row_idx, values, nnz):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.col_ptr = col_ptr
        self.row_idx = row_idx
        self.values = values
        self.nnz = int(nnz)
        self.realloc_count = 0

    @property
    def capacity(self):
        return int(self.row_idx.numel())

    @property
    def dtype(self):
        return self.values.dtype

    @classmethod
    def allocate(cls, n_rows, n_cols, capacity, dtype, device):
        torch = _torch()
        capacity = max(int(capacity), 1)
        return cls(n_rows, n_cols,
                   torch.zeros(n_cols + 1, dtype=torch.int32, device=device),
                   torch.empty(capacity, dtype=torch.int32, device=device),
                   torch.empty(capacity, dtype=dtype, device=device), 0)

    @classmethod
    def from_host(cls, mat, dtype, device, capacity=None):
        """Upload a host CSC (any object with the SparseMat attributes)."""
        torch = _torch()
        nnz = int(mat.col_ptr[mat.n_cols])
        cap = max(nnz, int(capacity or 0), 1)
        dev = cls.allocate(mat.n_rows, mat.n_cols, cap, dtype, device)
        dev.col_ptr.copy_(torch.from_numpy(np.ascontiguousarray(mat.col_ptr, dtype=np.int32)))
        if nnz:
            dev.row_idx[:nnz].copy_(torch.from_numpy(
                np.ascontiguousarray(mat.row_idx[:nnz], dtype=np.int32)))
            vals = torch.from_numpy(np.ascontiguousarray(mat.values[:nnz], dtype=np.float64))
            if dtype == torch.float64:
                dev.values[:nnz].copy_(vals)
            else:                       # narrow on the device, not on the host
                dev.values[:nnz].copy_(vals.to(device))
        dev.nnz = nnz
        return dev

    def to_host(self):
        """Materialise as a host :class:`SparseMat` (float64 values).  The
        arrays are numpy views of pinned host tensors (one DMA each, at link
        speed; torch's caching host allocator recycles them)."""
        nnz = self.nnz
        cp = pinned_copy(self.col_ptr)
        ri = pinned_copy(self.row_idx[:nnz])
        va = pinned_copy(self.values[:nnz] if self.values.dtype == _torch().float64
                         else self.values[:nnz].double())
        return SparseMat(self.n_rows, self.n_cols, cp, ri, va, check=False)

    def grow(self, needed):
        """Reallocate the entry storage (contents discarded) to >= needed,
        by at least 1.2x, counting the reallocation."""
        torch = _torch()
        cap = self.capacity
        if cap >= needed:
            return False
        new_cap = max(int(needed), int(math.ceil(cap * GROWTH)))
        self.row_idx = torch.empty(new_cap, dtype=torch.int32, device=self.row_idx.device)
        self.values = torch.empty(new_cap, dtype=self.values.dtype, device=self.values.device)
        self.realloc_count += 1
        return True

    def clone(self, capacity=None):
        torch = _torch()
        cap = max(self.nnz, int(capacity or 0), 1)
        out = DeviceCSC.allocate(self.n_rows, self.n_cols, cap, self.values.dtype,
                                 self.values.device)
        out.col_ptr.copy_(self.col_ptr)
        if self.nnz:
            out.row_idx[:self.nnz].copy_(self.row_idx[:self.nnz])
            out.values[:self.nnz].copy_(self.values[:self.nnz])
        out.nnz = self.nnz
        del torch
        return out

    def ft_csc(self):
        from ._lib import FtCsc
        return FtCsc(self.n_rows, self.n_cols, self.col_ptr.data_ptr(),
                     self.row_idx.data_ptr(), self.values.data_ptr(), self.capacity)

    def __repr__(self):
        return (f"DeviceCSC({self.n_rows}x{self.n_cols}, nnz={self.nnz}, "
                f"capacity={self.capacity}, {self.values.dtype})")


class DeviceTiled:
    """Working storage of a field on the GPU between Euler steps (``ft_tiled``
    in include/fieldtess_cuda.h), the hybrid layout: a column with at most
    two entries in the dense per-column arrays ``sig`` (row signature),
    ``aux`` (second row), ``v0`` / ``v1`` (values); a wider column in the
    pool (``pool_idx`` / ``pool_val``, offset in ``aux``)."""

    __slots__ = ("n_rows", "n_cols", "sig", "aux", "v0", "v1", "pool_idx", "pool_val")

    def __init__(self, n_rows, n_cols, capacity, dtype, device):
        torch = _torch()
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        n = max(self.n_cols, 1)
        self.sig = torch.full((n,), -1, dtype=torch.int32, device=device)   # all columns empty
        self.aux = torch.zeros(n, dtype=torch.int32, device=device)
        self.v0 = torch.zeros(n, dtype=dtype, device=device)
        self.v1 = torch.zeros(n, dtype=dtype, device=device)
        cap = max(int(capacity), 1)
        self.pool_idx = torch.empty(cap, dtype=torch.int32, device=device)
        self.pool_val = torch.empty(cap, dtype=dtype, device=device)

    @property
    def capacity(self):
        return int(self.pool_idx.numel())

    @property
    def values(self):
        return self.v0

    def grow(self, needed, keep=False):
        """Pool of at least ``needed`` entries (>= GROWTH x); ``keep`` copies
        the old pool (the dense arrays are never reallocated)."""
        torch = _torch()
        if self.capacity >= needed:
            return False
        new_cap = max(int(needed), int(math.ceil(self.capacity * GROWTH)))
        old_i, old_v = self.pool_idx, self.pool_val
        self.pool_idx = torch.empty(new_cap, dtype=torch.int32, device=old_i.device)
        self.pool_val = torch.empty(new_cap, dtype=old_v.dtype, device=old_v.device)
        if keep:
            self.pool_idx[:old_i.numel()].copy_(old_i)
            self.pool_val[:old_v.numel()].copy_(old_v)
        return True

    def ft_tiled(self, col_begin=0, n_cols=None):
        """The ``ft_tiled`` struct, or a view of columns [col_begin,
        col_begin + n_cols)."""
        from ._lib import FtTiled
        n = self.n_cols if n_cols is None else int(n_cols)
        vs = self.v0.element_size()
        return FtTiled(self.n_rows, n, self.sig.data_ptr() + 4 * col_begin,
                       self.aux.data_ptr() + 4 * col_begin, self.v0.data_ptr() + vs * col_begin,
                       self.v1.data_ptr() + vs * col_begin, self.pool_idx.data_ptr(),
                       self.pool_val.data_ptr(), self.capacity)


def hybrid_columns(col_ptr, row_idx, values, pool_base=0):
    """Host arrays of the hybrid layout for the CSC columns (col_ptr,
    row_idx, values): (sig, aux, v0, v1, pool_idx, pool_val); wide columns
    take consecutive pool entries from ``pool_base`` in column order."""
    col_ptr = np.asarray(col_ptr, dtype=np.int64)
    cnt = np.diff(col_ptr)
    n = cnt.size
    start = col_ptr[:-1]
    nnz = int(col_ptr[-1]) if n else 0
    first = np.minimum(start, max(nnz - 1, 0))
    second = np.minimum(start + 1, max(nnz - 1, 0))
    r0 = row_idx[first] if nnz else np.zeros(n, dtype=np.int32)
    r1 = row_idx[second] if nnz else np.zeros(n, dtype=np.int32)
    x0 = values[first] if nnz else np.zeros(n, dtype=values.dtype)
    x1 = values[second] if nnz else np.zeros(n, dtype=values.dtype)
    wide = cnt > 2
    wcnt = np.where(wide, cnt, 0)
    woff = pool_base + np.cumsum(wcnt) - wcnt
    sig = np.where(cnt == 0, -1, np.where(cnt == 1, r0, np.where(cnt == 2, r0 | (1 << 30), -cnt)))
    aux = np.where(cnt == 2, r1, np.where(wide, woff, 0))
    sel = np.repeat(wide, cnt)
    pidx = row_idx[:nnz][sel]
    pval = values[:nnz][sel]
    return (sig.astype(np.int32), aux.astype(np.int32), np.where(cnt >= 1, x0, 0).astype(values.dtype),
            np.where(cnt == 2, x1, 0).astype(values.dtype), pidx.astype(np.int32), pval)


# ---------------------------------------------------------------------------
# the reference's public sparse algebra, on the device (csrc/ft_sparse.cu;
# sparse.py:279-464).  Host SparseMat in, host SparseMat out; every
# floating-point reduction keeps the reference's order (bitwise equal).


class SpgemmScratch:
    """Reusable scratch of :func:`spgemm` (sparse.py:243-271).  The device
    product needs no dense accumulators; the object is kept for the API and
    counts the reallocations of its expansion buffers."""

    def __init__(self):
        self.realloc_count = 0
        self._keys = None
        self._vals = None

    def buffers(self, n, device):
        torch = _torch()
        if self._keys is None or self._keys.numel() < n or self._keys.device != device:
            cap = max(int(n), int(math.ceil((0 if self._keys is None else self._keys.numel()) * GROWTH)), 1)
            self._keys = torch.empty(cap, dtype=torch.int64, device=device)
            self._vals = torch.empty(cap, dtype=torch.float64, device=device)
            self.realloc_count += 1
        return self._keys[:n], self._vals[:n]


def _dev():
    from .field import _device
    return _device()


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _lib_call(name, *args):
    from . import _lib
    rc = getattr(_lib.lib(), name)(*args)
    if rc != 0:
        if rc == _lib.FT_ERR_SHAPE:
            raise ShapeError(f"{name}: shape mismatch")
        from .errors import BackendError
        raise BackendError(f"{name} failed (code {rc}): {_lib.last_error()}")


def _upload64(mat, device):
    torch = _torch()
    return DeviceCSC.from_host(mat, torch.float64, device)


def spgemm(a, b, out=None, scratch=None):
    """Sparse product ``C = A @ B`` in canonical CSC (sparse.py:279-330),
    bitwise equal to the reference: expand the products on the device in
    the reference's order, stable-sort them by (column, row), add every run
    sequentially (first term assigned), drop exact zeros."""
    torch = _torch()
    if a.n_cols != b.n_rows:
        raise ShapeError(f"shape mismatch: {a.shape} @ {b.shape}")
    n_rows, n_cols = a.n_rows, b.n_cols
    dev = _dev()
    da, db = _upload64(a, dev), _upload64(b, dev)
    ca, cb = da.ft_csc(), db.ft_csc()
    nnz_b = db.nnz
    counts = torch.zeros(max(nnz_b, 1), dtype=torch.int64, device=dev)
    _lib_call("ft_spgemm_count", ctypes.byref(ca), ctypes.byref(cb), nnz_b, ctypes.c_void_p(counts.data_ptr()),
              _stream())
    off = torch.zeros(nnz_b + 1, dtype=torch.int64, device=dev)
    if nnz_b:
        torch.cumsum(counts[:nnz_b], 0, out=off[1:])
    total = int(off[-1].item())
    col_ptr = np.zeros(n_cols + 1, dtype=INDEX)
    rows = np.zeros(0, dtype=INDEX)
    vals = np.zeros(0)
    if total:
        scratch = scratch if scratch is not None else SpgemmScratch()
        keys, pv = scratch.buffers(total, dev)
        _lib_call("ft_spgemm_expand", ctypes.byref(ca), ctypes.byref(cb), nnz_b, ctypes.c_void_p(off.data_ptr()),
                  ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(pv.data_ptr()), _stream())
        sk, perm = torch.sort(keys, stable=True)
        sv = pv[perm]
        head = torch.ones(total, dtype=torch.bool, device=dev)
        head[1:] = sk[1:] != sk[:-1]
        starts = torch.nonzero(head).flatten()
        sums = torch.empty(starts.numel(), dtype=torch.float64, device=dev)
        _lib_call("ft_segment_sums", ctypes.c_void_p(sv.data_ptr()), total, ctypes.c_void_p(starts.data_ptr()),
                  starts.numel(), ctypes.c_void_p(sums.data_ptr()), _stream())
        keep = sums != 0.0                          # the reference drops exact zeros
        key = sk[starts][keep]
        nr = max(n_rows, 1)
        cols = key // nr
        cnt = torch.bincount(cols, minlength=n_cols)
        col_ptr[1:] = torch.cumsum(cnt, 0).cpu().numpy()
        rows = (key % nr).to(torch.int32).cpu().numpy()
        vals = sums[keep].cpu().numpy()
    nnz = int(col_ptr[-1])
    if out is None:
        return SparseMat(n_rows, n_cols, col_ptr, rows, vals, check=False)
    if out.n_rows != n_rows or out.n_cols != n_cols:
        raise ShapeError("output buffer has wrong shape")
    ensure_capacity(out, nnz)
    out.col_ptr = col_ptr
    out.row_idx[:nnz] = rows
    out.values[:nnz] = vals
    return out


def build_skeleton(phi, lt, out=None):
    """Rows of interest per column: ``phi > 0`` or (``phi == 0`` and
    ``lt > 0``) (sparse.py:345-371), a sorted merge per column on the
    device (count, prefix sum, fill)."""
    torch = _torch()
    if phi.shape != lt.shape:
        raise ShapeError(f"shape mismatch: {phi.shape} vs {lt.shape}")
    n_cols = phi.n_cols
    dev = _dev()
    dp, dl = _upload64(phi, dev), _upload64(lt, dev)
    cp, cl = dp.ft_csc(), dl.ft_csc()
    counts = torch.zeros(max(n_cols, 1), dtype=torch.int32, device=dev)
    _lib_call("ft_skeleton", ctypes.byref(cp), ctypes.byref(cl), ctypes.c_void_p(counts.data_ptr()), None, None,
              _stream())
    ptr = torch.zeros(n_cols + 1, dtype=torch.int32, device=dev)
    if n_cols:
        torch.cumsum(counts[:n_cols], 0, out=ptr[1:])
    nnz = int(ptr[-1].item())
    rows = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    if nnz:
        _lib_call("ft_skeleton", ctypes.byref(cp), ctypes.byref(cl), None, ctypes.c_void_p(ptr.data_ptr()),
                  ctypes.c_void_p(rows.data_ptr()), _stream())
    col_ptr = ptr.cpu().numpy()
    row_idx = rows[:nnz].cpu().numpy()
    if out is None:
        return Skeleton(phi.n_rows, n_cols, col_ptr, row_idx)
    out.col_ptr = col_ptr
    if out.row_idx is None or out.row_idx.size < nnz:
        size = nnz if out.row_idx is None else max(nnz, int(math.ceil(out.row_idx.size * GROWTH)))
        out.row_idx = np.empty(size, dtype=INDEX)
        out.realloc_count += 1
    out.row_idx[:nnz] = row_idx
    return out


def expand_to_skeleton(a, skel, out_values=None):
    """``a`` on the skeleton pattern with explicit zeros elsewhere
    (sparse.py:374-396); a nonzero of ``a`` outside the pattern raises
    :class:`PatternViolationError` (first such column, its last offending
    row -- the reference's report)."""
    torch = _torch()
    if (a.n_rows, a.n_cols) != (skel.n_rows, skel.n_cols):
        raise ShapeError(f"shape mismatch: {a.shape} vs ({skel.n_rows}, {skel.n_cols})")
    nnz = skel.nnz
    dev = _dev()
    da = _upload64(a, dev)
    ca = da.ft_csc()
    sp = torch.from_numpy(np.ascontiguousarray(skel.col_ptr, dtype=np.int32)).to(dev)
    sr = torch.from_numpy(np.ascontiguousarray(skel.row_idx[:max(nnz, 1)] if nnz else np.zeros(1, INDEX),
                                               dtype=np.int32)).to(dev)
    vals = torch.zeros(max(nnz, 1), dtype=torch.float64, device=dev)
    bad = torch.full((max(a.n_cols, 1),), -1, dtype=torch.int32, device=dev)
    _lib_call("ft_expand", ctypes.byref(ca), ctypes.c_void_p(sp.data_ptr()), ctypes.c_void_p(sr.data_ptr()),
              ctypes.c_void_p(vals.data_ptr()), ctypes.c_void_p(bad.data_ptr()), _stream())
    badh = bad[:a.n_cols].cpu().numpy()
    offenders = np.flatnonzero(badh >= 0)
    if offenders.size:
        j = int(offenders[0])
        raise PatternViolationError(f"pattern-violation: nonzero at ({badh[j]}, {j}) outside the skeleton")
    v = vals[:nnz].cpu().numpy()
    if out_values is not None and out_values.size >= nnz:
        out_values[:nnz] = v
        v = out_values[:nnz]
    return SparseMat(skel.n_rows, skel.n_cols, skel.col_ptr, skel.row_idx[:nnz], v, check=False)


def normalize_columns(a):
    """Scale every positive-sum column to unit sum, ``v * (1 / s)`` with the
    column sum in entry order (sparse.py:399-420); negative entries raise
    :class:`NegativeFieldError`, zero-sum columns stay untouched with a
    warning, explicit zeros are kept."""
    torch = _torch()
    nnz = a.nnz
    vals = np.asarray(a.values[:nnz], dtype=np.float64)
    if nnz and vals.min() < 0:
        raise NegativeFieldError("negative-field: negative entry in input")
    dev = _dev()
    da = _upload64(a, dev)
    ca = da.ft_csc()
    out = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    sums = torch.empty(max(a.n_cols, 1), dtype=torch.float64, device=dev)
    _lib_call("ft_normalize_columns", ctypes.byref(ca), ctypes.c_void_p(out.data_ptr()),
              ctypes.c_void_p(sums.data_ptr()), _stream())
    s = sums[:a.n_cols].cpu().numpy()
    zero = np.flatnonzero((s == 0) & (np.diff(a.col_ptr.astype(np.int64)) > 0))
    if zero.size:
        warnings.warn(f"normalize_columns: {zero.size} zero-sum column(s) left untouched (first: {zero[0]})",
                      RuntimeWarning, stacklevel=2)
    return SparseMat(a.n_rows, a.n_cols, a.col_ptr.copy(), a.row_idx[:nnz].copy(), out[:nnz].cpu().numpy(),
                     check=False)


# ---------------------------------------------------------------------------
# text triplet interchange (sparse.py:427-464): "rows cols nnz" header, one
# "row col value" line per entry, '#' comment lines


def write_triplets(mat, path, comments=()):
    """Write ``mat`` as text triplets (values with ``repr``: round-trips)."""
    nnz = mat.nnz
    cols = mat.entry_columns()
    lines = [f"# {c}\n" for c in comments]
    lines.append(f"{mat.n_rows} {mat.n_cols} {nnz}\n")
    lines += [f"{r} {c} {v!r}\n" for r, c, v in
              zip(mat.row_idx[:nnz].tolist(), cols.tolist(), np.asarray(mat.values[:nnz], dtype=float).tolist())]
    with open(path, "w") as fh:
        fh.writelines(lines)


def read_triplets_stream(fh, first_lineno=1):
    """Parse triplet lines from an open text stream (``first_lineno``: the
    file line number of the stream's first line, for error messages)."""
    header = None
    rows, cols, vals = [], [], []
    for lineno, raw in enumerate(fh, first_lineno):
        parts = raw.split()
        if not parts or parts[0].startswith("#"):
            continue
        if len(parts) != 3:
            raise ShapeError(f"line {lineno}: bad triplet {'header' if header is None else 'entry'}")
        if header is None:
            header = tuple(int(x) for x in parts)
        else:
            rows.append(int(parts[0]))
            cols.append(int(parts[1]))
            vals.append(float(parts[2]))
    if header is None:
        raise ShapeError("empty triplet file")
    n_rows, n_cols, nnz = header
    if len(rows) != nnz:
        raise ShapeError(f"header says {nnz} entries, found {len(rows)}")
    return SparseMat.from_triplets(n_rows, n_cols, rows, cols, vals)


def read_triplets(path):
    """Read :func:`write_triplets` output."""
    with open(path) as fh:
        return read_triplets_stream(fh)
