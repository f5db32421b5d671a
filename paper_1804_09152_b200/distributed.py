"""Partitioned fields: one rank per GPU, vertex row-partition + halo exchange.

The reference evolves one field in one process (pkg/src/fieldtess/field.py:
289-321).  Column j of a new field reads only the columns u of L^T(:, j)
(its one-ring, _kernels.py:14-74), so a field whose vertices are split into
contiguous owned ranges steps independently per range given the one-ring
halo of the range.  Per Euler step every rank runs

    ft_domain_step      its owned columns (the single-GPU kernels, unchanged)
    ft_halo_pack        the owned columns each peer reads -> one message/peer
    all-gather          the per-rank statistics records (NCCL)
    ft_domain_combine   global max |delta|, base mass, stop test (fixed order)
    send / recv         the halo messages (NCCL over NVLink)
    ft_halo_unpack      the peers' messages -> the halo columns

with no host synchronisation: the stop test runs on every GPU from the
same gathered records, so the ranks stop at the same step, and the host only
reads the control block every ``sync_every`` steps.  The owned columns are
bitwise identical to the single-GPU :func:`field.evolve`; the global base
mass is summed in rank order (rounding may differ from the one-GPU
reduction tree at the 1e-16 relative level).

Two transports share one driver: :class:`TorchTransport` (torch.distributed;
NCCL for CUDA tensors, gloo for CPU tensors) for one rank per process, and
:class:`LoopbackTransport` for several ranks of one process on one device
(sequential, no rank waits for another inside a kernel), used by the tests.
"""

import ctypes

import numpy as np

from . import _lib
from . import field as F
from .devmesh import gather_columns as _gather_columns, morton_order_device  # noqa: F401 (public API)
from .errors import BackendError, ShapeError
from .field import (BASE_EXHAUSTION_PER_VERTEX, POOL_FRACTION, POOL_MIN, StepStats, _check,
                    _ft_dtype, _raise_step_error, _stats_from_bytes, _stream_handle,
                    _value_dtype)
from .sparse import INDEX, GROWTH, DeviceCSC, DeviceTiled, SparseMat, hybrid_columns

DEFAULT_SLOTS = 7      # halo message entries per column (grows on demand)


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# partition and halo plan (host)


class Partition:
    """Contiguous owned vertex ranges: rank r owns [bounds[r], bounds[r+1])."""

    def __init__(self, bounds):
        b = np.asarray(bounds, dtype=np.int64)
        if b.ndim != 1 or b.size < 2 or b[0] != 0 or np.any(np.diff(b) < 1):
            raise ShapeError("partition bounds must start at 0 and increase strictly")
        self.bounds = b

    @classmethod
    def even(cls, n_vertices, world, align=1):
        """Near-equal ranges, boundaries rounded to multiples of ``align``
        (e.g. a grid row, so the halo is whole rows)."""
        if world < 1 or n_vertices < world:
            raise ShapeError("need 1 <= world <= n_vertices")
        units = -(-n_vertices // align)
        cuts = [min(n_vertices, (units * r // world) * align) for r in range(world + 1)]
        cuts[-1] = n_vertices
        return cls(cuts)

    @property
    def world(self):
        return self.bounds.size - 1

    @property
    def n_vertices(self):
        return int(self.bounds[-1])

    def range(self, rank):
        return int(self.bounds[rank]), int(self.bounds[rank + 1])

    def owner(self, cols):
        return np.searchsorted(self.bounds, np.asarray(cols), side="right") - 1


class HaloPlan:
    """Which columns a rank receives from / sends to each peer.

    ``recv[q]``: sorted global columns owned by q that this rank's owned L^T
    columns read; ``send[q]``: this rank's owned columns q reads."""

    def __init__(self, rank, partition, recv, send):
        self.rank = rank
        self.partition = partition
        self.recv = {int(q): np.asarray(v, dtype=np.int32) for q, v in recv.items() if len(v)}
        self.send = {int(q): np.asarray(v, dtype=np.int32) for q, v in send.items() if len(v)}

    @staticmethod
    def needed(rank, partition, lap_idx):
        """recv lists from the owned L^T columns' row indices."""
        b, e = partition.range(rank)
        need = np.unique(np.asarray(lap_idx, dtype=np.int64))
        halo = need[(need < b) | (need >= e)]
        own = partition.owner(halo)
        return {int(q): halo[own == q] for q in np.unique(own)}

    @property
    def halo_cols(self):
        return int(sum(v.size for v in self.recv.values()))

    @property
    def peers(self):
        return sorted(set(self.recv) | set(self.send))


def build_plans(problems, transport):
    """Halo plans of the local ranks (a host collective over all ranks)."""
    recvs = [HaloPlan.needed(p.rank, p.partition, p.lap_idx) for p in problems]
    sends = transport.exchange_lists(recvs)
    return [HaloPlan(p.rank, p.partition, r, s) for p, r, s in zip(problems, recvs, sends)]


class LocalProblem:
    """What one rank holds: the owned columns of L^T (CSC with global row
    indices, n_rows = n_vertices) and the initial field on its owned + halo
    columns (``cols`` sorted, CSC-like ``col_ptr`` / ``row_idx`` /
    ``values`` over them)."""

    def __init__(self, rank, partition, n_rows, lap_ptr, lap_idx, lap_val, lap_flags, cols,
                 col_ptr, row_idx, values, symmetric=False):
        self.rank = rank
        self.symmetric = bool(symmetric)   # L^T pattern symmetric: active-set stepping
        self.partition = partition
        self.n_rows = int(n_rows)
        self.lap_ptr = np.ascontiguousarray(lap_ptr, dtype=INDEX)
        self.lap_idx = np.ascontiguousarray(lap_idx, dtype=INDEX)
        self.lap_val = np.ascontiguousarray(lap_val, dtype=np.float64)
        self.lap_flags = int(lap_flags)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.row_idx = np.ascontiguousarray(row_idx, dtype=INDEX)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        b, e = partition.range(rank)
        if self.lap_ptr.size != e - b + 1:
            raise ShapeError("L^T columns do not match the owned range")


def _slice_problem(field_phi, mat_t, flags, partition, rank, symmetric=False):
    b, e = partition.range(rank)
    cp = np.asarray(mat_t.col_ptr, dtype=np.int64)
    q0, q1 = int(cp[b]), int(cp[e])
    lap_ptr = cp[b:e + 1] - q0
    lap_idx = np.asarray(mat_t.row_idx[q0:q1])
    lap_val = np.asarray(mat_t.values[q0:q1], dtype=np.float64)
    need = np.unique(lap_idx.astype(np.int64))
    cols = np.union1d(np.arange(b, e, dtype=np.int64), need)
    fcp = np.asarray(field_phi.col_ptr, dtype=np.int64)
    cnt = fcp[cols + 1] - fcp[cols]
    col_ptr = np.zeros(cols.size + 1, dtype=np.int64)
    np.cumsum(cnt, out=col_ptr[1:])
    src = np.repeat(fcp[cols], cnt) + (np.arange(int(col_ptr[-1])) - np.repeat(col_ptr[:-1], cnt))
    return LocalProblem(rank, partition, field_phi.n_rows, lap_ptr, lap_idx, lap_val, flags, cols,
                        col_ptr, np.asarray(field_phi.row_idx)[src],
                        np.asarray(field_phi.values, dtype=np.float64)[src], symmetric=symmetric)


def _laplacian_t(lap):
    from .field import _uniform_values_exact, _with_diagonal
    mat_t = _with_diagonal(lap.mat_t)
    flags = _lib.FT_LAP_UNIFORM if _uniform_values_exact(mat_t) else _lib.FT_LAP_EXPLICIT
    return mat_t, flags


def local_problem(field_phi, lap, partition, rank, renumbering=None):
    """Slice a host field (SparseMat) and a Laplacian for one rank; with a
    :class:`Renumbering` the partition is over the renumbered vertices."""
    sym = F._pattern_symmetric(lap)        # a renumbering keeps the pattern symmetric
    if renumbering is not None:
        return _slice_problem(renumbering.field(field_phi), renumbering.laplacian_t(lap),
                              renumbering.lap_flags, partition, rank, symmetric=sym)
    mat_t, flags = _laplacian_t(lap)
    return _slice_problem(field_phi, mat_t, flags, partition, rank, symmetric=sym)


# -- locality renumbering -------------------------------------------------------


def _spread3(x):
    """Spread the low 21 bits of x to every third bit (Morton code)."""
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                        (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        x = (x | (x << np.uint64(shift))) & np.uint64(mask)
    return x


def morton_order(positions):
    """Vertices sorted by the Morton (Z-order) code of their positions:
    contiguous ranges of the order are compact patches of the surface."""
    p = np.asarray(positions, dtype=np.float64)
    lo = p.min(axis=0)
    span = float((p.max(axis=0) - lo).max()) or 1.0
    q = np.floor((p - lo) / span * (2 ** 21 - 1)).astype(np.uint64)
    code = _spread3(q[:, 0]) | (_spread3(q[:, 1]) << np.uint64(1)) | (_spread3(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable")


class Renumbering:
    """A vertex renumbering for partitioning: new vertex k is old vertex
    ``order[k]``.  Every L^T column keeps its entries in the ORIGINAL order
    (the kernels accumulate in stored order, so the step stays bitwise the
    reference's); only the indices change.  Layer rows (cells) do not."""

    def __init__(self, order):
        self.order = np.asarray(order, dtype=np.int64)
        self.inverse = np.empty_like(self.order)
        self.inverse[self.order] = np.arange(self.order.size)
        self.lap_flags = None
        self._lap = None

    @classmethod
    def morton(cls, mesh):
        return cls(morton_order(mesh.positions))

    def _columns(self, m, rows_map=None):
        cp = np.asarray(m.col_ptr, dtype=np.int64)
        cnt = cp[1:] - cp[:-1]
        new_cnt = cnt[self.order]
        new_cp = np.zeros(cnt.size + 1, dtype=np.int64)
        np.cumsum(new_cnt, out=new_cp[1:])
        src = np.repeat(cp[self.order], new_cnt) + (np.arange(int(new_cp[-1])) -
                                                    np.repeat(new_cp[:-1], new_cnt))
        rows = np.asarray(m.row_idx)[src]
        if rows_map is not None:
            rows = rows_map[rows]
        return SparseMat(m.n_rows, m.n_cols, new_cp, rows, np.asarray(m.values, dtype=np.float64)[src],
                         check=False)

    def field(self, phi):
        """PHI with its vertex columns renumbered."""
        return self._columns(phi)

    def laplacian_t(self, lap):
        """L^T renumbered: column k = old column order[k], row indices mapped,
        entries kept in the original order (cached per Laplacian)."""
        if self._lap is None or self._lap[0] is not lap:
            mat_t, flags = _laplacian_t(lap)
            self.lap_flags = flags
            self._lap = (lap, self._columns(mat_t, self.inverse))
        return self._lap[1]

    def restore(self, phi_new):
        """A renumbered field back in the caller's vertex numbering."""
        back = Renumbering(self.inverse)
        return back._columns(phi_new)

    def old_vertex(self, k):
        return int(self.order[k]) if k >= 0 else k


def local_problem_device(phi, lap, order, partition, rank):
    """:func:`local_problem` with a :class:`Renumbering` ``order`` computed
    on the device: ``phi`` a DeviceCSC field, ``lap`` a device-built uniform
    Laplacian (``lap.device``), ``order`` a device permutation (new vertex k
    = old vertex order[k], e.g. :func:`morton_order_device`).  Only this
    rank's owned + halo columns are gathered; the result is the same
    LocalProblem the host path builds (tests/test_distributed.py)."""
    torch = _torch()
    dev = lap.device
    if dev is None:
        raise ShapeError("local_problem_device needs a device-built Laplacian")
    b, e = partition.range(rank)
    inverse = torch.empty_like(order)
    inverse[order] = torch.arange(order.numel(), device=order.device)
    lap_ptr, src = _gather_columns(dev["ptr"], order[b:e])
    lap_idx = inverse[dev["idx"][src].long()]
    lap_val = dev["val_t"][src]
    need = torch.unique(lap_idx)
    cols = torch.unique(torch.cat([torch.arange(b, e, device=order.device), need]))
    col_ptr, fsrc = _gather_columns(phi.col_ptr, order[cols])
    host = lambda t: t.cpu().numpy()
    return LocalProblem(rank, partition, phi.n_rows, host(lap_ptr), host(lap_idx), host(lap_val),
                        _lib.FT_LAP_UNIFORM, host(cols), host(col_ptr), host(phi.row_idx[fsrc]),
                        host(phi.values[fsrc].double()), symmetric=True)


# torus stencil of gen_periodic_grid (vertex (i, j) -> j*nx + i; faces
# (v00, v10, v01), (v10, v11, v01)): the one-ring of (i, j)
_GRID_RING = ((1, 0), (-1, 0), (0, 1), (0, -1), (1, -1), (-1, 1))


def _grid_ring(v, nx, ny):
    i, j = v % nx, v // nx
    return np.stack([((j + dj) % ny) * nx + (i + di) % nx for di, dj in _GRID_RING], axis=1)


def periodic_grid_problem(nx, ny, seeds, partition, rank):
    """The rank-local problem of ``init_field(gen_periodic_grid(nx, ny),
    seeds)`` with the uniform Laplacian, built from the lattice stencil
    without the global mesh (weak-scaling runs whose global mesh does not
    fit one host process).  Identical to :func:`local_problem` on the
    globally built objects (tests/test_distributed.py)."""
    b, e = partition.range(rank)
    n_v = nx * ny
    if partition.n_vertices != n_v:
        raise ShapeError("partition does not cover the grid")
    own = np.arange(b, e, dtype=np.int64)
    ring = _grid_ring(own, nx, ny)
    lt = np.sort(np.concatenate([own[:, None], ring], axis=1), axis=1)
    deg = 6
    lap_idx = lt.reshape(-1)
    lap_val = np.where(lt == own[:, None], -1.0, 1.0 / deg).reshape(-1)
    lap_ptr = np.arange(0, 7 * own.size + 1, 7, dtype=np.int64)
    need = np.unique(lap_idx)
    cols = np.union1d(own, need)
    # seeds claim themselves and their one-ring (field.py:137-166): rows =
    # seed position + 1, 1/k for a vertex claimed k times
    seeds = np.asarray(seeds, dtype=np.int64).ravel()
    if seeds.size != np.unique(seeds).size:
        from .errors import DuplicateSeedError
        raise DuplicateSeedError("duplicate-seed: seed list has repeats")
    cl_col = np.concatenate([seeds[:, None], _grid_ring(seeds, nx, ny)], axis=1).reshape(-1)
    cl_row = np.repeat(np.arange(1, seeds.size + 1, dtype=np.int64), 7)
    pos = np.searchsorted(cols, cl_col)
    keep = (pos < cols.size) & (cols[np.minimum(pos, cols.size - 1)] == cl_col)
    cl_col, cl_row, pos = cl_col[keep], cl_row[keep], pos[keep]
    claims = np.bincount(pos, minlength=cols.size)
    per = np.where(claims == 0, 1, claims)
    col_ptr = np.zeros(cols.size + 1, dtype=np.int64)
    np.cumsum(per, out=col_ptr[1:])
    row_idx = np.zeros(int(col_ptr[-1]), dtype=INDEX)
    vals = np.ones(int(col_ptr[-1]))
    order = np.lexsort((cl_row, pos))
    sp, sr = pos[order], cl_row[order]
    first = np.searchsorted(sp, sp, side="left")
    dst = col_ptr[sp] + (np.arange(sp.size) - first)
    row_idx[dst] = sr
    vals[dst] = 1.0 / claims[sp]
    return LocalProblem(rank, partition, seeds.size + 1, lap_ptr, lap_idx, lap_val,
                        _lib.FT_LAP_UNIFORM, cols, col_ptr, row_idx, vals, symmetric=True)


# ---------------------------------------------------------------------------
# transports


class TorchTransport:
    """One rank per process over torch.distributed (NCCL for CUDA tensors,
    gloo for CPU tensors).  ``ranks`` is always this process's single rank."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def exchange_lists(self, recvs):
        (recv,) = recvs
        allr = [None] * self.world
        self.dist.all_gather_object(allr, {q: v for q, v in recv.items()}, group=self.group)
        return [{q: allr[q][self.rank] for q in range(self.world)
                 if q != self.rank and self.rank in allr[q]}]

    def all_gather(self, ranks):
        (r,) = ranks
        if self.nccl:
            self.dist.all_gather_into_tensor(r.gathered, r.record, group=self.group)
        elif r.record.device.type == "cpu":
            self.dist.all_gather(list(r.gathered.chunk(self.world)), r.record, group=self.group)
        else:                       # gloo with device buffers: staged through the host
            g = r.gathered.cpu()
            self.dist.all_gather(list(g.chunk(self.world)), r.record.cpu(), group=self.group)
            r.gathered.copy_(g)

    def exchange(self, ranks):
        (r,) = ranks
        d = self.dist
        # gloo cannot send device tensors: stage the messages through the host
        host = not self.nccl and any(t.device.type != "cpu"
                                     for t in list(r.send_msg.values()) + list(r.recv_msg.values()))
        recv = {q: (t.cpu() if host else t) for q, t in r.recv_msg.items()}
        ops = []
        for q in r.plan.peers:
            if q in r.plan.send:
                m = r.send_msg[q]
                ops.append(d.P2POp(d.isend, m.cpu() if host else m, q, group=self.group))
            if q in r.plan.recv:
                ops.append(d.P2POp(d.irecv, recv[q], q, group=self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()
        if host:
            for q, t in recv.items():
                r.recv_msg[q].copy_(t)

    def all_reduce(self, tensors, op):
        """In-place all-reduce ("sum" / "min" / "max") of this rank's tensor."""
        (t,) = tensors
        ops = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX}
        if self.nccl or t.device.type == "cpu":
            self.dist.all_reduce(t, op=ops[op], group=self.group)
        else:
            h = t.cpu()
            self.dist.all_reduce(h, op=ops[op], group=self.group)
            t.copy_(h)

    def gather_objects(self, objs):
        (o,) = objs
        out = [None] * self.world
        self.dist.all_gather_object(out, o, group=self.group)
        return out

    def max_int(self, values):
        torch = _torch()
        (v,) = values
        dev = "cuda" if self.nccl else "cpu"
        t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def gather_owned(self, ranks, steps_done):
        """Every rank's owned columns, in rank order, on every rank: (column
        counts, rows, values) as host arrays per rank (all_gather of the
        padded device arrays: NCCL over NVLink)."""
        torch = _torch()
        (r,) = ranks
        f = r.owned_field(steps_done)
        dev = f.values.device if self.nccl else "cpu"
        cnt = (f.col_ptr[1:] - f.col_ptr[:-1]).to(torch.int32)
        sizes = torch.tensor([r.n_own, f.nnz], dtype=torch.int64, device=dev)
        all_sizes = [torch.zeros_like(sizes) for _ in range(self.world)]
        self.dist.all_gather(all_sizes, sizes, group=self.group)
        all_sizes = [tuple(int(x) for x in t.cpu()) for t in all_sizes]
        mo = max(a for a, _ in all_sizes)
        mn = max(max(b for _, b in all_sizes), 1)

        def pad(t, n):
            out = torch.zeros(n, dtype=t.dtype, device=dev)
            out[:t.numel()] = t.to(dev)
            return out

        parts = []
        for t, n in ((cnt, mo), (f.row_idx[:f.nnz], mn), (f.values[:f.nnz].double(), mn)):
            mine = pad(t, n)
            got = [torch.zeros_like(mine) for _ in range(self.world)]
            self.dist.all_gather(got, mine, group=self.group)
            parts.append([g.cpu().numpy() for g in got])
        return [(parts[0][q][:a], parts[1][q][:b], parts[2][q][:b]) for q, (a, b) in enumerate(all_sizes)]


class LoopbackTransport:
    """All ranks live in this process (one device): collectives are copies.
    The ranks' kernels run one after another; none waits on another."""

    def exchange_lists(self, recvs):
        sends = [dict() for _ in recvs]
        for r, recv in enumerate(recvs):
            for q, cols in recv.items():
                sends[q][r] = cols
        return sends

    def all_gather(self, ranks):
        torch = _torch()
        cat = torch.cat([r.record for r in ranks])
        for r in ranks:
            r.gathered.copy_(cat)

    def exchange(self, ranks):
        for r in ranks:
            for q in r.plan.recv:
                r.recv_msg[q].copy_(ranks[q].send_msg[r.rank])

    def max_int(self, values):
        return max(int(v) for v in values)

    def all_reduce(self, tensors, op):
        torch = _torch()
        red = {"sum": lambda a, b: a + b, "min": torch.minimum, "max": torch.maximum}[op]
        acc = tensors[0].clone()
        for t in tensors[1:]:
            acc = red(acc, t)
        for t in tensors:
            t.copy_(acc)

    def gather_objects(self, objs):
        return list(objs)

    def gather_owned(self, ranks, steps_done):
        out = []
        for r in sorted(ranks, key=lambda x: x.g_begin):
            h = r.owned_field(steps_done).to_host()
            cp = np.asarray(h.col_ptr, dtype=np.int64)
            out.append((np.diff(cp).astype(np.int32), np.asarray(h.row_idx[:cp[-1]]),
                        np.asarray(h.values[:cp[-1]], dtype=np.float64)))
        return out


# ---------------------------------------------------------------------------
# one rank's device state


class DomainRank:
    """Device state of one rank.  Its columns are LOCAL: the sorted union of
    the owned columns and the halo, numbered 0 .. n_loc-1 in global order,
    so the owned ones are the range [col_begin, col_begin + n_own) and the
    buffers scale with the rank's share of the field, not the whole field.
    Holds the owned L^T columns (local row indices), two tiled buffers over
    the local columns, the workspace, the statistics records and the halo
    messages."""

    def __init__(self, problem, plan, precision="exact", slots=DEFAULT_SLOTS, device=None,
                 renumbering=None):
        torch = _torch()
        if device is None:
            if not torch.cuda.is_available():
                raise BackendError("no CUDA device: the engine has no CPU fallback")
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.renumbering = renumbering
        self.lib = _lib.lib()
        self.rank = problem.rank
        self.partition = problem.partition
        self.world = problem.partition.world
        self.plan = plan
        self.precision = precision
        self.ftd = _ft_dtype(precision)
        self.vdtype = _value_dtype(precision)
        self.n_rows = problem.n_rows
        self.n_v = problem.partition.n_vertices
        g_begin, g_end = problem.partition.range(problem.rank)
        self.g_begin = g_begin
        self.n_own = g_end - g_begin
        self.cols = problem.cols                      # local column k = global column cols[k]
        self.n_loc = int(self.cols.size)
        local = lambda g: np.searchsorted(self.cols, np.asarray(g, dtype=np.int64)).astype(np.int32)
        self.col_begin = int(local(g_begin))
        lap_idx = local(problem.lap_idx)
        lap = SparseMat(self.n_loc, self.n_own, problem.lap_ptr, lap_idx, problem.lap_val, check=False)
        self.lap = DeviceCSC.from_host(lap, self.vdtype, device)
        self.lap_c = self.lap.ft_csc()
        self.lap_flags = problem.lap_flags
        if problem.symmetric and F.ACTIVE_SET:
            self.lap_flags |= _lib.FT_LAP_SYMMETRIC
        # NaN / pattern errors report global (caller) vertex ids
        gids = np.arange(g_begin, g_end, dtype=np.int64)
        if renumbering is not None:
            gids = renumbering.order[gids]
        self.report_ids = torch.from_numpy(gids.astype(np.int32)).to(device)
        self.pack = None
        if problem.lap_flags == _lib.FT_LAP_UNIFORM and F.PACK_LAPLACIAN:
            self.pack, _ = F.pack_laplacian(self.lap, col_base=self.col_begin)
            self.lap_c.values = self.pack.data_ptr()
            self.lap_flags |= _lib.FT_LAP_PACKED
        self.ws = torch.zeros(int(self.lib.ft_workspace_bytes(self.n_loc)), dtype=torch.int8,
                              device=device)
        self.record = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=device)
        self.gathered = torch.zeros(self.world * _lib.STATS_BYTES, dtype=torch.uint8, device=device)
        self.need = torch.zeros(1, dtype=torch.int32, device=device)
        self.ctl_out = torch.zeros(3, dtype=torch.int64, device=device)
        # control snapshots in flight (device, pinned host, event) x 2
        self.snap = [(torch.zeros(3, dtype=torch.int64, device=device),
                      torch.zeros(3, dtype=torch.int64, pin_memory=True),
                      torch.cuda.Event()) for _ in range(2)]
        self.trace = None
        self.steps_done = 0            # steps completed by previous evolve calls
        self.step_events = None        # list: (start, end) CUDA events per ft_domain_step
        # halo layout (local columns): peers ascending, columns of a peer
        # consecutive; per received column, the owned columns that read it
        own_j = np.repeat(np.arange(self.n_own, dtype=np.int64) + self.col_begin,
                          np.diff(np.asarray(problem.lap_ptr, dtype=np.int64)))
        order = np.argsort(lap_idx, kind="stable")
        rd_key, rd_val = lap_idx[order].astype(np.int64), own_j[order]
        self.recv_cols, self.send_cols, self.readers = {}, {}, {}
        for q, v in plan.recv.items():
            lv = local(v)
            lo = np.searchsorted(rd_key, lv, side="left")
            hi = np.searchsorted(rd_key, lv, side="right")
            ptr = np.concatenate([[0], np.cumsum(hi - lo)]).astype(np.int32)
            idx = (np.concatenate([rd_val[a:b] for a, b in zip(lo, hi)]) if lv.size
                   else np.zeros(0)).astype(np.int32)
            self.recv_cols[q] = torch.from_numpy(lv).to(device)
            self.readers[q] = (torch.from_numpy(ptr).to(device),
                               torch.from_numpy(idx if idx.size else np.zeros(1, np.int32)).to(device))
        for q, v in plan.send.items():
            self.send_cols[q] = torch.from_numpy(local(v)).to(device)
        self.recv_off = {}
        off = 0
        for q in sorted(plan.recv):
            self.recv_off[q] = off
            off += plan.recv[q].size
        self.n_halo = off
        own_mask = (problem.cols >= g_begin) & (problem.cols < g_end)
        own_nnz = int(np.sum(np.diff(problem.col_ptr)[own_mask]))
        self.step_cap = max(
            int(own_nnz * POOL_FRACTION), POOL_MIN)
        self.slots = int(slots)
        self.bufs = [None, None]
        self.meta = [None, None]       # (ft_tiled struct, step_capacity, slots) per buffer
        self._alloc_messages()
        self._upload(problem)
        self.reallocs = 0

    # -- buffers -------------------------------------------------------------

    def _alloc_messages(self):
        torch = _torch()
        hb = self.lib.ft_halo_bytes
        self.send_msg = {q: torch.zeros(int(hb(v.size, self.slots, self.ftd)), dtype=torch.uint8,
                                        device=self.device) for q, v in self.plan.send.items()}
        self.recv_msg = {q: torch.zeros(int(hb(v.size, self.slots, self.ftd)), dtype=torch.uint8,
                                        device=self.device) for q, v in self.plan.recv.items()}

    def _need_capacity(self):
        return self.step_cap + self.n_halo * self.slots

    def _buffer(self, k, capacity):
        """Buffer k with at least ``capacity`` entries.  A grown buffer keeps
        its contents: launches enqueued after a failed step (device no-ops)
        may grow the buffer that holds the state the host rewinds to."""
        buf = self.bufs[k]
        if buf is None or buf.capacity < capacity:
            old = buf
            if old is not None:
                self.reallocs += 1
                capacity = max(capacity, int(old.capacity * GROWTH))
            buf = DeviceTiled(self.n_rows, self.n_loc, capacity, self.vdtype, self.device)
            if old is not None:
                for name in ("sig", "aux", "v0", "v1"):
                    getattr(buf, name).copy_(getattr(old, name))
                buf.pool_idx[:old.capacity].copy_(old.pool_idx)
                buf.pool_val[:old.capacity].copy_(old.pool_val)
            self.bufs[k] = buf
        return buf

    def _upload(self, problem):
        torch = _torch()
        sig, aux, v0, v1, pidx, pval = hybrid_columns(problem.col_ptr, problem.row_idx,
                                                      problem.values.astype(np.float64))
        buf = self._buffer(0, max(self._need_capacity(), pidx.size, 1))
        dev = self.device
        buf.sig.copy_(torch.from_numpy(sig).to(dev))          # the local columns, in order
        buf.aux.copy_(torch.from_numpy(aux).to(dev))
        buf.v0.copy_(torch.from_numpy(v0).to(dev, self.vdtype))
        buf.v1.copy_(torch.from_numpy(v1).to(dev, self.vdtype))
        if pidx.size:
            buf.pool_idx[:pidx.size].copy_(torch.from_numpy(pidx).to(dev))
            buf.pool_val[:pidx.size].copy_(torch.from_numpy(pval).to(dev, self.vdtype))
        self.meta[0] = (buf.ft_tiled(), 0, self.slots)
        # values of unknown origin: the first step checks them unless finite
        self.first_check = not bool(np.all(np.isfinite(problem.values)))
        self._buffer(1, self._need_capacity())
        self.meta[1] = None

    def _as_output(self, k):
        """Buffer k about to receive a step: large enough for the current step
        capacity and halo slots (contents discarded when reallocated)."""
        buf = self._buffer(k, self._need_capacity())
        self.meta[k] = (buf.ft_tiled(), self.step_cap, self.slots)
        return self.meta[k]

    # -- the per-step launches (all asynchronous) ----------------------------

    def begin(self, total_steps):
        torch = _torch()
        if self.trace is None or self.trace.numel() < total_steps * _lib.STATS_BYTES:
            old = self.trace
            self.trace = torch.zeros(total_steps * _lib.STATS_BYTES, dtype=torch.uint8,
                                     device=self.device)
            if old is not None:
                self.trace[:old.numel()].copy_(old)
        self.set_control(self.steps_done)

    def launch_step(self, i, prm, stream):
        lib = self.lib
        in_t = self.meta[i % 2][0]
        out_t, step_cap, slots = self._as_output((i + 1) % 2)
        dom = _lib.FtDomain(self.col_begin, self.n_own, step_cap, self.report_ids.data_ptr(), (i + 1) % 2, 0)
        wp, wn = ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel()
        rec = ctypes.c_void_p(self.record.data_ptr())
        if self.step_events is not None:
            torch = _torch()
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            self.step_events.append(ev)
        flags = self.lap_flags | (_lib.FT_LAP_CHECK_FINITE if (i == 0 and self.first_check) else 0)
        _check(lib.ft_domain_step(ctypes.byref(self.lap_c), flags, ctypes.byref(in_t),
                                  ctypes.byref(out_t), self.ftd, ctypes.byref(prm),
                                  ctypes.byref(dom), wp, wn, rec, stream), "ft_domain_step")
        if self.step_events is not None:
            self.step_events[-1][1].record()
        for q, cols in self.send_cols.items():
            _check(lib.ft_halo_pack(ctypes.byref(out_t), ctypes.c_void_p(cols.data_ptr()),
                                    cols.numel(), slots, self.ftd,
                                    ctypes.c_void_p(self.send_msg[q].data_ptr()), rec,
                                    ctypes.c_void_p(self.need.data_ptr()), wp, 0, stream),
                   "ft_halo_pack")

    def launch_combine(self, max_steps, tol, base_threshold, stream):
        _check(self.lib.ft_domain_combine(ctypes.c_void_p(self.gathered.data_ptr()), self.world,
                                          self.rank, max_steps, float(tol), float(base_threshold),
                                          ctypes.c_void_p(self.ws.data_ptr()),
                                          ctypes.c_void_p(self.trace.data_ptr()), stream),
               "ft_domain_combine")

    def launch_unpack(self, i, stream, flags=0):
        out_t, step_cap, slots = self.meta[(i + 1) % 2]
        prev = self.meta[i % 2][0]            # the step's input: the halo's previous values
        track = bool(self.lap_flags & _lib.FT_LAP_SYMMETRIC)
        for q, cols in self.recv_cols.items():
            rp, ri = self.readers[q]
            _check(self.lib.ft_halo_unpack(ctypes.byref(out_t), ctypes.c_void_p(cols.data_ptr()),
                                           cols.numel(), slots, self.ftd,
                                           ctypes.c_void_p(self.recv_msg[q].data_ptr()),
                                           step_cap + self.recv_off[q] * slots,
                                           ctypes.c_void_p(self.ws.data_ptr()), flags,
                                           ctypes.byref(prev) if track else None,
                                           ctypes.c_void_p(rp.data_ptr()) if track else None,
                                           ctypes.c_void_p(ri.data_ptr()) if track else None, stream),
                   "ft_halo_unpack")

    # -- control -------------------------------------------------------------

    def set_control(self, steps_done):
        _check(self.lib.ft_domain_control(ctypes.c_void_p(self.ws.data_ptr()), int(steps_done),
                                          ctypes.c_void_p(self.ctl_out.data_ptr()),
                                          _stream_handle()), "ft_domain_control")

    def read_control(self):
        _check(self.lib.ft_domain_control(ctypes.c_void_p(self.ws.data_ptr()), -1,
                                          ctypes.c_void_p(self.ctl_out.data_ptr()),
                                          _stream_handle()), "ft_domain_control")
        c = self.ctl_out.cpu().numpy()
        return int(c[0]), int(c[1]), int(c[2])

    def snapshot(self, k):
        """Asynchronous copy of the control block into snapshot slot k."""
        dev, host, ev = self.snap[k]
        _check(self.lib.ft_domain_control(ctypes.c_void_p(self.ws.data_ptr()), -1,
                                          ctypes.c_void_p(dev.data_ptr()), _stream_handle()),
               "ft_domain_control")
        host.copy_(dev, non_blocking=True)
        ev.record()

    def snapshot_wait(self, k):
        _dev, host, ev = self.snap[k]
        ev.synchronize()
        c = host.numpy()
        return int(c[0]), int(c[1]), int(c[2])

    def read_trace(self, n):
        if n <= 0:
            return _stats_from_bytes(b"")
        return _stats_from_bytes(self.trace[:n * _lib.STATS_BYTES].cpu().numpy().tobytes())

    def grow_step_capacity(self, needed):
        if needed > self.step_cap:
            self.step_cap = max(int(needed), int(self.step_cap * GROWTH))

    def set_slots(self, need):
        if need > self.slots:
            self.slots = int(need)
            self._alloc_messages()
        self.need.zero_()

    # -- results -------------------------------------------------------------

    def owned_field(self, steps_done):
        """The owned columns after ``steps_done`` steps as a DeviceCSC
        (n_rows x n_own), compacted from the tiled buffer."""
        torch = _torch()
        buf = self.bufs[steps_done % 2]
        src = buf.ft_tiled(self.col_begin, self.n_own)
        sg = buf.sig[self.col_begin:self.col_begin + self.n_own]
        counts = torch.where(sg >= (1 << 30), 2, torch.where(sg >= 0, 1, torch.where(sg == -1, 0, -sg)))
        cap = max(1, int(counts.sum().item()))
        out = DeviceCSC.allocate(self.n_rows, self.n_own, cap, self.vdtype, self.device)
        o_c = out.ft_csc()
        rec = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=self.device)
        _check(self.lib.ft_compact(ctypes.byref(src), ctypes.byref(o_c), self.ftd,
                                   ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                   ctypes.c_void_p(rec.data_ptr()), _stream_handle()),
               "ft_compact")
        r = _stats_from_bytes(rec.cpu().numpy().tobytes())[0]
        if int(r["status"]) != _lib.FT_STATUS_OK:
            raise BackendError("compaction of the owned columns failed")
        out.nnz = int(r["nnz_phi"])
        return out


    def pack_final(self, steps_done, stream):
        """Pack the owned columns the peers read from the field after
        ``steps_done`` steps (forced: the last step's own pack ran before the
        stop flag, but its unpack was a no-op)."""
        buf_t, _cap, slots = self.meta[steps_done % 2]
        scratch = _torch().zeros(_lib.STATS_BYTES, dtype=_torch().uint8, device=self.device)
        self._scratch_rec = scratch
        for q, cols in self.send_cols.items():
            _check(self.lib.ft_halo_pack(ctypes.byref(buf_t), ctypes.c_void_p(cols.data_ptr()), cols.numel(),
                                         slots, self.ftd, ctypes.c_void_p(self.send_msg[q].data_ptr()),
                                         ctypes.c_void_p(scratch.data_ptr()), ctypes.c_void_p(self.need.data_ptr()),
                                         ctypes.c_void_p(self.ws.data_ptr()), _lib.FT_HALO_FORCE, stream),
                   "ft_halo_pack")

    def unpack_final(self, steps_done, stream):
        """The peers' owned columns -> the halo of the field after
        ``steps_done`` steps (forced, no activity stamps)."""
        buf_t, cap, slots = self.meta[steps_done % 2]
        for q, cols in self.recv_cols.items():
            _check(self.lib.ft_halo_unpack(ctypes.byref(buf_t), ctypes.c_void_p(cols.data_ptr()), cols.numel(),
                                           slots, self.ftd, ctypes.c_void_p(self.recv_msg[q].data_ptr()),
                                           cap + self.recv_off[q] * slots, ctypes.c_void_p(self.ws.data_ptr()),
                                           _lib.FT_HALO_FORCE, None, None, None, stream), "ft_halo_unpack")

    def local_field(self, steps_done):
        """All local columns (owned + halo) after ``steps_done`` steps as a
        float64 DeviceCSC (n_rows x n_loc) -- the input of the partitioned
        Lloyd step, whose faces reach one ring beyond the owned range."""
        torch = _torch()
        buf = self.bufs[steps_done % 2]
        src = buf.ft_tiled()
        sg = buf.sig
        counts = torch.where(sg >= (1 << 30), 2, torch.where(sg >= 0, 1, torch.where(sg == -1, 0, -sg)))
        cap = max(1, int(counts.sum().item()))
        out = DeviceCSC.allocate(self.n_rows, self.n_loc, cap, self.vdtype, self.device)
        o_c = out.ft_csc()
        rec = torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=self.device)
        _check(self.lib.ft_compact(ctypes.byref(src), ctypes.byref(o_c), self.ftd,
                                   ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                   ctypes.c_void_p(rec.data_ptr()), _stream_handle()), "ft_compact")
        r = _stats_from_bytes(rec.cpu().numpy().tobytes())[0]
        if int(r["status"]) != _lib.FT_STATUS_OK:
            raise BackendError("compaction of the local columns failed")
        out.nnz = int(r["nnz_phi"])
        if out.values.dtype != torch.float64:
            out.values = out.values.double()
        return out

    def lloyd_faces(self, mesh, renumbering=None):
        """The rank's faces for the partitioned Lloyd step (cached per mesh):
        those whose first vertex the rank owns, ascending.  Returns
        (faces in local column ids, faces in mesh vertex ids, global face
        ids, area, barycenter, normal) as device arrays."""
        torch = _torch()
        key = id(mesh)
        if getattr(self, "_lloyd_faces", None) is not None and self._lloyd_faces[0] == key:
            return self._lloyd_faces[1]
        f = np.asarray(mesh.faces, dtype=np.int64)
        fn = renumbering.inverse[f] if renumbering is not None else f       # partition numbering
        own = (fn[:, 0] >= self.g_begin) & (fn[:, 0] < self.g_begin + self.n_own)
        ids = np.flatnonzero(own)
        loc = np.searchsorted(self.cols, fn[ids])
        if ids.size and not np.all(self.cols[np.minimum(loc, self.cols.size - 1)] == fn[ids]):
            raise BackendError("a face reaches beyond the rank's one-ring halo")
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(self.device)
        faces = (up(loc if ids.size else np.zeros((1, 3)), np.int32), up(f[ids] if ids.size else np.zeros((1, 3)), np.int32),
                 up(ids if ids.size else np.zeros(1), np.int32), up(mesh.face_area[ids], np.float64),
                 up(mesh.face_barycenter[ids], np.float64), up(mesh.face_normal[ids], np.float64),
                 int(ids.size))
        self._lloyd_faces = (key, faces)
        return faces

    def owned_labels(self, steps_done=None, field=None):
        """Argmax cell labels of the owned vertices (ft_labels, field.py:
        324-356) as a device int64 tensor."""
        torch = _torch()
        f = field if field is not None else self.owned_field(
            self.steps_done if steps_done is None else steps_done)
        labels = torch.empty(max(self.n_own, 1), dtype=torch.int64, device=self.device)
        c = f.ft_csc()
        _check(self.lib.ft_labels(ctypes.byref(c), self.ftd, ctypes.c_void_p(labels.data_ptr()),
                                  _stream_handle()), "ft_labels")
        return labels[:self.n_own]


# ---------------------------------------------------------------------------
# the driver


def evolve_partitioned(ranks, transport, params, max_steps=1000, tol=1e-4,
                       base_threshold=None, sync_every=16):
    """Evolve a partitioned field (one :class:`DomainRank` per local rank)
    by up to ``max_steps`` more steps, stopping when converged, exactly as
    :func:`field.evolve` (field.py:289-321).  Returns ``(steps, trace)`` of
    this call; the fields stay on the devices (:meth:`DomainRank.owned_field`)
    and a later call resumes from them.

    The host enqueues ``sync_every`` steps per chunk and reads the control
    block of chunk c (an asynchronous snapshot) only after chunk c+1 is
    enqueued, so the GPUs never wait for the host.  After a failed step the
    remaining launches are device no-ops; the host grows what overflowed and
    rewinds to the failed step."""
    if max_steps < 1:
        raise ShapeError("max_steps must be >= 1")
    params.validate()
    n_v = ranks[0].n_v
    thr = BASE_EXHAUSTION_PER_VERTEX * n_v if base_threshold is None else base_threshold
    prm = params.ft_params()
    stream = _stream_handle()
    s0 = ranks[0].steps_done
    total = s0 + max_steps
    for r in ranks:
        r.begin(total)

    def enqueue(i, end, slot):
        for s in range(i, end):
            for r in ranks:
                r.launch_step(s, prm, stream)
            transport.all_gather(ranks)
            for r in ranks:
                r.launch_combine(total, tol, thr, stream)
            transport.exchange(ranks)
            for r in ranks:
                r.launch_unpack(s, stream)
        for r in ranks:
            r.snapshot(slot)

    i = s0
    inflight = []          # (snapshot slot, chunk end), oldest first
    nslot = 0
    while True:
        while i < total and len(inflight) < 2:
            end = min(i + sync_every, total)
            enqueue(i, end, nslot)
            inflight.append((nslot, end))
            nslot ^= 1
            i = end
        slot, _end = inflight.pop(0)
        ctl = [r.snapshot_wait(slot) for r in ranks]
        done, status = ctl[0][0], ctl[0][1]
        if any(c[:2] != (done, status) for c in ctl):
            raise BackendError("ranks disagree on the step count")
        if status in (_lib.FT_STATUS_CONVERGED, _lib.FT_STATUS_MAXSTEPS):
            break
        if status == _lib.FT_STATUS_OK:
            continue
        _torch().cuda.synchronize()         # let the no-op launches drain
        if status == _lib.FT_STATUS_OVERFLOW:
            for r, c in zip(ranks, ctl):
                r.grow_step_capacity(c[2] + c[2] // 5)
        elif status == _lib.FT_STATUS_HALO_OVERFLOW:
            need = transport.max_int([int(r.need.item()) for r in ranks])
            for r in ranks:
                r.set_slots(need)
        else:
            # error columns are already in the caller's numbering (report_ids)
            _raise_step_error(ranks[0].read_trace(done + 1)[done], done)
            raise BackendError(f"partitioned step failed with status {status}")
        for r in ranks:                     # rewind: redo the failed step
            r.set_control(done)
        i = done
        inflight = []
    _torch().cuda.synchronize()
    steps = ranks[0].read_control()[0]
    recs = ranks[0].read_trace(steps)[s0:]
    for r in ranks:
        r.steps_done = steps
    trace = [StepStats(max_delta=float(x["max_delta"]), nnz_phi=int(x["nnz_phi"]),
                       base_mass=float(x["base_mass"]), nnz_skel=int(x["nnz_skel"]),
                       converged=int(x["status"]) == _lib.FT_STATUS_CONVERGED) for x in recs]
    if trace:
        trace[-1].realloc_count = sum(r.reallocs for r in ranks)
    return steps - s0, trace


def gather_field(ranks, steps_done=None, n_rows=None, renumbering=None):
    """Host SparseMat of the whole field from local ranks covering every
    owned range (loopback runs; a multi-process run gathers per rank)."""
    parts = sorted(ranks, key=lambda r: r.g_begin)
    ptrs, idx, vals = [np.zeros(1, dtype=np.int64)], [], []
    base = 0
    for r in parts:
        h = r.owned_field(r.steps_done if steps_done is None else steps_done).to_host()
        cp = np.asarray(h.col_ptr, dtype=np.int64)
        ptrs.append(cp[1:] + base)
        idx.append(np.asarray(h.row_idx[:cp[-1]]))
        vals.append(np.asarray(h.values[:cp[-1]]))
        base += int(cp[-1])
    n = parts[-1].n_v
    out = SparseMat(n_rows or parts[0].n_rows, n, np.concatenate(ptrs),
                    np.concatenate(idx) if idx else np.zeros(0, INDEX),
                    np.concatenate(vals) if vals else np.zeros(0), check=False)
    return out if renumbering is None else renumbering.restore(out)


def assemble_owned(parts, n_rows, n_vertices, renumbering=None):
    """Host SparseMat of the whole field from the ranks' owned parts (rank
    order = column order), in the mesh's vertex ids."""
    cnt = np.concatenate([c for c, _, _ in parts]).astype(np.int64)
    cp = np.concatenate([[0], np.cumsum(cnt)])
    out = SparseMat(n_rows, n_vertices, cp, np.concatenate([r for _, r, _ in parts]).astype(INDEX),
                    np.concatenate([v for _, _, v in parts]), check=False)
    return out if renumbering is None else renumbering.restore(out)


def gathered_field(ranks, transport, seeds, renumbering=None, precision="exact"):
    """The whole field on every rank (the all-gathered owned columns) as a
    LayeredField in the mesh's vertex ids: the input of the dual-mesh API
    (dual.py) and of any other whole-field consumer."""
    from .field import LayeredField
    steps = ranks[0].steps_done
    parts = transport.gather_owned(ranks, steps)
    phi = assemble_owned(parts, ranks[0].n_rows, ranks[0].n_v, renumbering)
    return LayeredField(phi, seeds, steps, precision=precision)


def dual_adjacency_partitioned(ranks, transport, mesh, threshold=0.25, renumbering=None):
    """``vertex_adjacency``, ``triangle_adjacency`` and ``confirm_candidates``
    (dual.py:85-233) of a partitioned field without gathering it (SURVEY
    8(e)): every rank runs the device products (ft_dual_products) on its owned
    + halo columns and the faces whose first vertex it owns, the four key sets
    are all-gathered and united -- a set union, so the result is exactly the
    single-GPU products -- and the order-dependent curation runs replicated.
    Returns ``(a_v, a_t, curated)``; ``build_dual`` then takes ``curated``.
    A skipped degenerate face or non-finite value (whose warnings the
    reference raises from the whole field) falls back to the gathered field."""
    from . import dual
    refresh_halo(ranks, transport)
    local = []
    for r in ranks:
        dphi = r.local_field(r.steps_done)
        faces, _, _, area, _, _, n_faces = r.lloyd_faces(mesh, renumbering)
        local.append(dual.product_keys(dphi, r.n_rows - 1, faces, area, n_faces, threshold))
    every = transport.gather_objects(local)
    union = tuple(np.unique(np.concatenate([k[i] for k in every])) for i in range(4))
    skipped = any(k[4] for k in every)
    n_cells = ranks[0].n_rows - 1
    if skipped:
        fld = gathered_field(ranks, transport, np.zeros(n_cells, dtype=np.int64), renumbering=renumbering)
        a_v = dual.vertex_adjacency(fld, threshold)
        a_t = dual.triangle_adjacency(fld, mesh, threshold)
        return a_v, a_t, dual.confirm_candidates(fld, mesh, a_v, a_t, threshold)
    pv, pt, px, tri, _ = dual.decode_products(union + (False,), n_cells)
    a_v = dual.AdjacencyMatrix(dual._pairs_matrix(n_cells, pv))
    a_v.provenance = {pair: "vertex-shared" for pair in a_v.pairs()}
    a_t = dual.AdjacencyMatrix(dual._pairs_matrix(n_cells, pt))
    return a_v, a_t, dual.curate(a_v, a_t, px, tri)


class PartitionedField:
    """A field that stays on the ranks between Lloyd iterations (the
    all-reduce exchange never assembles it): the LayeredField attributes a
    caller reads, and :meth:`gather` for the whole field on demand."""

    def __init__(self, ranks, transport, seeds, n_rows, steps, renumbering=None, precision="exact"):
        self.ranks = ranks
        self.transport = transport
        self.seed_vertices = np.asarray(seeds, dtype=np.int64)
        self.n_cells = n_rows - 1
        self.step_count = steps
        self.renumbering = renumbering
        self.precision = precision

    def gather(self):
        return gathered_field(self.ranks, self.transport, self.seed_vertices, self.renumbering, self.precision)


def refresh_halo(ranks, transport):
    """Bring every rank's halo up to date with its peers' final owned
    columns (the evolve loop skips the last step's unpack once it stops)."""
    stream = _stream_handle()
    for r in ranks:
        r.pack_final(r.steps_done, stream)
    transport.exchange(ranks)
    for r in ranks:
        r.unpack_final(r.steps_done, stream)


def _row_sums(dcsc, col_weight):
    """Per row: the sum over the row's entries of value * col_weight[column],
    in column order (deterministic: stable sort by row, sequential runs)."""
    torch = _torch()
    nnz = dcsc.nnz
    n_rows = dcsc.n_rows
    out = torch.zeros(n_rows, dtype=torch.float64, device=dcsc.values.device)
    if nnz == 0:
        return out
    cols = torch.repeat_interleave(torch.arange(dcsc.n_cols, device=out.device),
                                   (dcsc.col_ptr[1:] - dcsc.col_ptr[:-1]).long())
    rows = dcsc.row_idx[:nnz].long()
    prod = dcsc.values[:nnz].double() * col_weight[cols]
    rs, perm = torch.sort(rows, stable=True)
    pv = prod[perm].contiguous()
    head = torch.ones(nnz, dtype=torch.bool, device=out.device)
    head[1:] = rs[1:] != rs[:-1]
    starts = torch.nonzero(head).flatten()
    sums = torch.empty(starts.numel(), dtype=torch.float64, device=out.device)
    _check(_lib.lib().ft_segment_sums(ctypes.c_void_p(pv.data_ptr()), nnz, ctypes.c_void_p(starts.data_ptr()),
                                      starts.numel(), ctypes.c_void_p(sums.data_ptr()), _stream_handle()),
           "ft_segment_sums")
    out[rs[starts]] = sums
    return out


def _cell_areas_partitioned(ranks, transport, mesh, renumbering):
    """Field-weighted cell areas (lloyd.py:115-125) as per-rank partial sums
    over the owned vertices, all-reduced."""
    torch = _torch()
    parts = []
    for r in ranks:
        f = r.owned_field(r.steps_done)
        gids = np.arange(r.g_begin, r.g_begin + r.n_own)
        vid = renumbering.order[gids] if renumbering is not None else gids
        w = torch.from_numpy(np.asarray(mesh.vertex_area, dtype=np.float64)[vid]).to(r.device)
        parts.append(_row_sums(f, w))
    transport.all_reduce(parts, "sum")
    return parts[0].cpu().numpy()[1:]


def _reseed_allreduce(state, mesh, ranks, transport, renumbering):
    """The Lloyd reseed (lloyd.py:155-195) on a partitioned field: every rank
    sums approx_centroid's terms over its faces, the sums are all-reduced
    (8 doubles per cell), each rank back-projects through its faces and the
    best hit is chosen by all-reduces of (|t|, face id) -- smallest |t|,
    then the lowest face id, np.argmin's first occurrence.  The collision
    pass then runs replicated.  The centroid sums are taken in a different
    order than numpy's pairwise sums, so a point can differ from the
    single-GPU one in the last bits (the exact path is exchange="gather")."""
    torch = _torch()
    from . import lloyd as LL
    n = int(state.field.n_cells)
    old = np.asarray(state.seeds, dtype=np.int64)
    refresh_halo(ranks, transport)
    vp = ctypes.c_void_p
    lib = _lib.lib()
    st = _stream_handle()
    per = []
    for r in ranks:
        dm = LL.device_mesh(mesh)
        floc, fmesh, fid, area, bary, fnorm, nf = r.lloyd_faces(mesh, renumbering)
        lf = r.local_field(r.steps_done)
        cell_ptr, cell_faces, _ = LL.faces_by_cell_arrays(lf, floc, nf, 1, False)
        seeds_d = torch.from_numpy(old).to(r.device)
        sums = torch.zeros(max(n, 1) * 8, dtype=torch.float64, device=r.device)
        period = ctypes.cast(dm.period, ctypes.c_void_p) if dm.period is not None else None
        _check(lib.ft_lloyd_partials(vp(dm.positions.data_ptr()), dm.n_vertices, vp(fmesh.data_ptr()), nf,
                                     vp(area.data_ptr()), vp(bary.data_ptr()), vp(fnorm.data_ptr()), period, n,
                                     vp(cell_ptr.data_ptr()), vp(cell_faces.data_ptr()), vp(seeds_d.data_ptr()),
                                     vp(sums.data_ptr()), st), "ft_lloyd_partials")
        per.append((r, dm, fmesh, fid, nf, cell_ptr, cell_faces, sums, period))
    transport.all_reduce([x[7] for x in per], "sum")
    keys_t, keys_f, hits, statuses = [], [], [], []
    for r, dm, fmesh, fid, nf, cell_ptr, cell_faces, sums, period in per:
        point = torch.zeros(max(n, 1) * 3, dtype=torch.float64, device=r.device)
        normal = torch.zeros_like(point)
        status = torch.zeros(max(n, 1), dtype=torch.int32, device=r.device)
        _check(lib.ft_lloyd_finish(n, vp(sums.data_ptr()), vp(point.data_ptr()), vp(normal.data_ptr()),
                                   vp(status.data_ptr()), st), "ft_lloyd_finish")
        local = status.clone()
        hit = torch.full((max(n, 1),), -1, dtype=torch.int32, device=r.device)
        bt = torch.full((max(n, 1),), float("inf"), dtype=torch.float64, device=r.device)
        bf = torch.full((max(n, 1),), np.iinfo(np.int64).max, dtype=torch.int64, device=r.device)
        _check(lib.ft_lloyd_backproject_keys(vp(dm.positions.data_ptr()), dm.n_vertices, vp(fmesh.data_ptr()), nf,
                                             period, n, vp(cell_ptr.data_ptr()), vp(cell_faces.data_ptr()),
                                             vp(fid.data_ptr()), vp(point.data_ptr()), vp(normal.data_ptr()),
                                             vp(local.data_ptr()), vp(hit.data_ptr()), vp(bt.data_ptr()),
                                             vp(bf.data_ptr()), st), "ft_lloyd_backproject_keys")
        keys_t.append(bt)
        keys_f.append(bf)
        hits.append(hit)
        statuses.append(status)
    best_t = [t.clone() for t in keys_t]
    transport.all_reduce(best_t, "min")
    cand = [torch.where(t == b, f, torch.full_like(f, np.iinfo(np.int64).max))
            for t, b, f in zip(keys_t, best_t, keys_f)]
    transport.all_reduce(cand, "min")
    mine = [torch.where((f == c) & torch.isfinite(t), h.long(), torch.full_like(f, -1))
            for f, c, t, h in zip(keys_f, cand, keys_t, hits)]
    transport.all_reduce(mine, "max")
    status = statuses[0][:n].cpu().numpy()
    hit = mine[0][:n].cpu().numpy()
    fail = (status != LL.LLOYD_OK) | (hit < 0)
    candidates = np.where(fail, old, hit)

    def members(c):
        """The vertices of cell c (any stored phi), ascending, from every rank."""
        mine_v = []
        for r in ranks:
            f = r.owned_field(r.steps_done)
            cols = torch.repeat_interleave(torch.arange(r.n_own, device=r.device),
                                           (f.col_ptr[1:] - f.col_ptr[:-1]).long())
            sel = cols[f.row_idx[:f.nnz].long() == c + 1].cpu().numpy() + r.g_begin
            mine_v.append(renumbering.order[sel] if renumbering is not None else sel)
        allv = transport.gather_objects(mine_v)
        return np.sort(np.concatenate([np.asarray(v, dtype=np.int64) for v in allv]))

    taken, collisions = set(), 0
    seeds = np.empty(n, dtype=np.int64)
    for c in range(n):
        pick = int(candidates[c])
        if pick in taken:
            collisions += 1
            pick = int(old[c])
        if pick in taken:
            free = [int(v) for v in members(c) if int(v) not in taken]
            if not free:
                from .errors import VanishedCellError
                raise VanishedCellError(f"vanished-cell: no free vertex left for cell {c}")
            pick = free[0]
        taken.add(pick)
        seeds[c] = pick
    return seeds, {"reseed_misses": int(fail.sum()), "seed_collisions": collisions}


def lloyd_iterate_partitioned(state, mesh, lap, params, n_iter, transport, partition, local_ranks,
                              max_steps=1000, tol=1e-4, precision="exact", renumbering=None, device=None,
                              exchange="allreduce"):
    """:func:`lloyd.lloyd_iterate` (lloyd.py:198-229) with every evolve
    partitioned over the ranks (vertex row partition, NCCL halo exchange).
    ``local_ranks`` are the rank ids this process drives (one for a
    TorchTransport, all for a LoopbackTransport).

    ``exchange="allreduce"``: the field stays distributed; the
    reseed all-reduces the per-cell centroid sums and the best-hit keys and
    the cell areas of the history are all-reduced partial sums (a few KB per
    cell set per iteration); ``state.field`` is a :class:`PartitionedField`.
    ``exchange="gather"``: the owned fields are all-gathered and the
    single-GPU kernels reseed the whole field on every rank -- bitwise the
    seeds and history of ``lloyd_iterate``, at the cost of moving the field."""
    from . import lloyd as LL
    from .field import LayeredField, init_field
    if n_iter < 1:
        raise ShapeError("n_iter must be >= 1")
    if exchange not in ("allreduce", "gather"):
        raise ShapeError("exchange must be 'allreduce' or 'gather'")
    fresh = state.field is None or state.field.step_count == 0

    def run_evolve(seeds, fld=None):
        fld = fld if fld is not None else init_field(mesh, seeds, precision=precision)
        problems = [local_problem(fld.phi, lap, partition, q, renumbering=renumbering) for q in local_ranks]
        plans = build_plans(problems, transport)
        ranks = [DomainRank(pr, pl, precision=precision, device=device, renumbering=renumbering)
                 for pr, pl in zip(problems, plans)]
        steps, trace = evolve_partitioned(ranks, transport, params, max_steps=max_steps, tol=tol)
        if exchange == "gather":
            parts = transport.gather_owned(ranks, steps)
            phi = assemble_owned(parts, fld.phi.n_rows, mesh.n_vertices, renumbering)
            return LayeredField(phi, seeds, steps, precision=precision), trace, None
        return PartitionedField(ranks, transport, seeds, fld.phi.n_rows, steps, renumbering, precision), trace, ranks

    def record(trace, report, ranks):
        if exchange == "gather":
            return LL._history_entry(state, mesh, trace, report)
        areas = _cell_areas_partitioned(ranks, transport, mesh, renumbering)
        seeds = np.asarray(state.seeds, dtype=np.int64)
        rec = dict(iteration=state.iteration, seeds=seeds.tolist(),
                   seed_positions=mesh.positions[seeds].tolist(), cell_areas=areas.tolist(),
                   area_variance=float(np.var(areas)), steps=len(trace),
                   converged=bool(trace[-1].converged) if len(trace) else True)
        rec.update(report)
        return rec

    ranks = None
    trace = []
    if fresh:
        start = state.field if state.field is not None else None
        state.field, trace, ranks = run_evolve(np.asarray(state.seeds), start)
    elif exchange == "allreduce":
        raise ShapeError("the all-reduce exchange starts from an unstepped state")
    if not state.history:
        state.history.append(record(trace, {"reseed_misses": 0, "seed_collisions": 0}, ranks))
    for _ in range(n_iter):
        if exchange == "gather":
            seeds, report = LL._reseed(state, mesh)
        else:
            seeds, report = _reseed_allreduce(state, mesh, ranks, transport, renumbering)
        state.seeds = seeds
        state.iteration += 1
        state.field, trace, ranks = run_evolve(seeds)
        state.history.append(record(trace, report, ranks))
    return state
