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

import math

import numpy as np

from .errors import ShapeError

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
            dev.values[:nnz].copy_(vals.to(dtype))
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
    """Tiled working storage of a field on the GPU (``ft_tiled`` in
    include/fieldtess_cuda.h): per-column (start, count) descriptors, entries
    in per-tile slots plus an overflow pool.  Used between Euler steps."""

    __slots__ = ("n_rows", "n_cols", "desc", "row_idx", "values", "sig")

    def __init__(self, n_rows, n_cols, capacity, dtype, device):
        torch = _torch()
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.desc = torch.zeros(2 * max(n_cols, 1), dtype=torch.int32, device=device)
        self.row_idx = torch.empty(int(capacity), dtype=torch.int32, device=device)
        self.values = torch.empty(int(capacity), dtype=dtype, device=device)
        # row signature per column (row of a single entry, -1 more, -2 none)
        self.sig = torch.full((max(n_cols, 1),), -2, dtype=torch.int32, device=device)

    @property
    def capacity(self):
        return int(self.row_idx.numel())

    def grow(self, needed):
        torch = _torch()
        if self.capacity >= needed:
            return False
        new_cap = max(int(needed), int(math.ceil(self.capacity * GROWTH)))
        self.row_idx = torch.empty(new_cap, dtype=torch.int32, device=self.row_idx.device)
        self.values = torch.empty(new_cap, dtype=self.values.dtype, device=self.values.device)
        return True

    def ft_tiled(self):
        from ._lib import FtTiled
        return FtTiled(self.n_rows, self.n_cols, self.desc.data_ptr(), self.row_idx.data_ptr(),
                       self.values.data_ptr(), self.capacity, self.sig.data_ptr())
