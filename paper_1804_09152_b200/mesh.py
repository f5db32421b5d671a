"""Triangle meshes, order-identical synthetic generators, the Laplacian.

The mesh is the static input of the hot path.  Everything here is host-side
numpy, vectorised so the benchmark meshes (10M+ vertices) build in seconds,
and ORDER-IDENTICAL to the reference (pkg/src/fieldtess/mesh.py): same
vertex numbering, face list, edge list, one-ring order and Laplacian bytes
(pinned by SHA-256 digests in tests/golden/meshes.json).  Geometry uses the
same numpy reductions as the reference so derived areas are bitwise equal.

The icosphere generator is not capped at subdivision 7 (the reference's
limit, mesh.py:222-223): levels 8..12 are produced by the same midpoint
numbering rule, vectorised.

With a GPU the generators, the derived data and the uniform Laplacian are
built on the device instead (:mod:`devmesh`, ft_mesh.cu; same bytes) and
copied to the host only when a host attribute is first read.
"""

import warnings

import numpy as np

from .errors import (IsolatedVertexError, MeshFormatError,
                     NonTriangularFaceError, ShapeError)
from . import devmesh
from .sparse import INDEX, SparseMat, transpose


class TriMesh:
    """Indexed triangle mesh with precomputed derived data.

    Same constructor and attributes as the reference ``TriMesh``
    (mesh.py:20-162): face area / normal / barycenter, lumped vertex area,
    binary incidence ``incidence`` (n_v x n_f) and its transpose, sorted
    unique ``edges`` and the sorted one-ring (``neighbor_ptr`` /
    ``neighbor_idx``), optional torus lattice ``period_vectors``.
    """

    def __init__(self, positions, faces, period_vectors=None):
        self.positions = np.ascontiguousarray(positions, dtype=np.float64)
        self.faces = np.ascontiguousarray(faces, dtype=np.int32)
        if self.positions.ndim != 2 or self.positions.shape[1] != 3:
            raise ShapeError("positions must be (n_v, 3)")
        if self.faces.ndim != 2 or self.faces.shape[1] != 3:
            raise NonTriangularFaceError("faces must be (n_f, 3)")
        n_v = self.positions.shape[0]
        f = self.faces
        if f.size and (f.min() < 0 or f.max() >= n_v):
            raise MeshFormatError("face index out of range")
        if np.any((f[:, 0] == f[:, 1]) | (f[:, 1] == f[:, 2]) | (f[:, 0] == f[:, 2])):
            raise MeshFormatError("degenerate face (repeated vertex index)")
        self.period_vectors = (None if period_vectors is None
                               else np.asarray(period_vectors, dtype=np.float64))
        self._cache = {}
        self._topo = {}
        self._topology()

    @classmethod
    def _from_device(cls, positions, faces, period_vectors=None):
        """A generator's output built on the device (valid by construction):
        host positions / faces now, topology on the device (host copies on
        first access), geometry on first use."""
        self = cls.__new__(cls)
        self.positions = positions.cpu().numpy()
        self.faces = faces.cpu().numpy()
        self.period_vectors = (None if period_vectors is None
                               else np.asarray(period_vectors, dtype=np.float64))
        self._cache = {"dev_positions": positions, "dev_faces": faces}
        self._topo = {}
        self._topo_dev = devmesh.topology(self.positions.shape[0], faces)
        return self

    def device_arrays(self):
        """(positions, faces) device tensors of a device-built mesh, else None."""
        c = self._cache
        return (c["dev_positions"], c["dev_faces"]) if "dev_positions" in c else None

    def _topo_get(self, name):
        if name not in self._topo:
            self._topo[name] = self._topo_dev[name].cpu().numpy()
        return self._topo[name]

    edges = property(lambda self: self._topo_get("edges"), doc="sorted unique undirected edges (E, 2)")
    degree = property(lambda self: self._topo_get("degree"))
    neighbor_ptr = property(lambda self: self._topo_get("neighbor_ptr"))
    neighbor_idx = property(lambda self: self._topo_get("neighbor_idx"))

    # derived data (geometry and incidence are computed lazily: the Euler
    # step only needs the topology, and the torus geometry pass is the
    # expensive part at 10M+ vertices) -------------------------------------------

    def _geometry(self):
        if "face_area" in self._cache:
            return self._cache
        if "dev_positions" in self._cache:
            dev = self._device_geometry()
            for k in ("face_area", "face_normal", "face_barycenter", "vertex_area"):
                self._cache[k] = dev[k].cpu().numpy()
            return self._cache
        p, f = self.positions, self.faces
        e1 = self.wrap_deltas(p[f[:, 1]] - p[f[:, 0]])
        e2 = self.wrap_deltas(p[f[:, 2]] - p[f[:, 0]])
        cr = np.cross(e1, e2)
        nrm = np.linalg.norm(cr, axis=1)
        area = 0.5 * nrm
        safe = np.where(nrm == 0, 1, nrm)
        self._cache["face_area"] = area
        self._cache["face_normal"] = np.where(nrm[:, None] > 0, cr / safe[:, None], 0.0)
        self._cache["face_barycenter"] = p[f[:, 0]] + (e1 + e2) / 3.0
        # bincount adds in input order per bin, exactly like np.add.at
        self._cache["vertex_area"] = np.bincount(f.ravel(), weights=np.repeat(area / 3.0, 3),
                                                 minlength=p.shape[0]).astype(np.float64)
        return self._cache

    def _incidences(self):
        if "incidence" not in self._cache:
            n_v, n_f = self.positions.shape[0], self.faces.shape[0]
            inc = SparseMat(n_v, n_f, np.arange(0, 3 * n_f + 1, 3, dtype=INDEX),
                            np.sort(self.faces, axis=1).ravel().astype(INDEX),
                            np.ones(3 * n_f), check=False)
            self._cache["incidence"] = inc
            self._cache["incidence_t"] = transpose(inc)
        return self._cache

    def _device_geometry(self):
        """Device geometry tensors of a device-built mesh (computed once)."""
        c = self._cache
        if "dev_geometry" not in c:
            c["dev_geometry"] = devmesh.geometry(c["dev_positions"], c["dev_faces"], self.period_vectors,
                                                 self._quarter_r2() if self.periodic else 0.0)
        return c["dev_geometry"]

    def _geo(self, name):
        c = self._cache
        if name not in c:
            if "dev_positions" in c:
                c[name] = self._device_geometry()[name].cpu().numpy()
            else:
                self._geometry()
        return c[name]

    face_area = property(lambda self: self._geo("face_area"))
    face_normal = property(lambda self: self._geo("face_normal"))
    face_barycenter = property(lambda self: self._geo("face_barycenter"))
    vertex_area = property(lambda self: self._geo("vertex_area"))
    incidence = property(lambda self: self._incidences()["incidence"],
                         doc="binary vertex-face incidence (n_v x n_f), 3 per column")
    incidence_t = property(lambda self: self._incidences()["incidence_t"])

    def _topology(self):
        f = self.faces
        n_v = self.positions.shape[0]
        # unique undirected edges (lexicographic) and the sorted one-ring
        lo = np.concatenate([f[:, 0], f[:, 1], f[:, 2]]).astype(np.int64)
        hi = np.concatenate([f[:, 1], f[:, 2], f[:, 0]]).astype(np.int64)
        a, b = np.minimum(lo, hi), np.maximum(lo, hi)
        keys, counts = np.unique(a * max(n_v, 1) + b, return_counts=True)
        edges = np.stack([keys // max(n_v, 1), keys % max(n_v, 1)], axis=1)
        if np.any(counts > 2):
            warnings.warn(f"{int((counts > 2).sum())} non-manifold edge(s) (more than "
                          "2 incident faces); neighbors are treated uniformly",
                          RuntimeWarning, stacklevel=3)
        src = np.concatenate([edges[:, 0], edges[:, 1]])
        dst = np.concatenate([edges[:, 1], edges[:, 0]])
        order = np.argsort(src * max(n_v, 1) + dst, kind="stable")
        degree = np.bincount(src, minlength=n_v)
        ptr = np.zeros(n_v + 1, dtype=np.int64)
        np.cumsum(degree, out=ptr[1:])
        self._topo = {"edges": edges, "degree": degree, "neighbor_ptr": ptr,
                      "neighbor_idx": dst[order].astype(np.int32)}

    # queries ---------------------------------------------------------------

    @property
    def n_vertices(self):
        return self.positions.shape[0]

    @property
    def n_faces(self):
        return self.faces.shape[0]

    @property
    def n_edges(self):
        return self.edges.shape[0]

    @property
    def periodic(self):
        return self.period_vectors is not None

    def neighbors(self, v):
        return self.neighbor_idx[self.neighbor_ptr[v]:self.neighbor_ptr[v + 1]]

    def euler_characteristic(self):
        return self.n_vertices - self.n_edges + self.n_faces

    def mean_edge_length(self):
        d = self.wrap_deltas(self.positions[self.edges[:, 1]] - self.positions[self.edges[:, 0]])
        return float(np.linalg.norm(d, axis=1).mean())

    def bbox_diagonal(self):
        return float(np.linalg.norm(self.positions.max(axis=0) - self.positions.min(axis=0)))

    _WRAP_CHUNK = 1 << 20

    def wrap_deltas(self, deltas):
        """Shortest lattice representatives of difference vectors (identity on
        non-periodic meshes); mesh.py:136-157.  Row-wise, so large inputs go
        in chunks (identical results, cache-sized temporaries)."""
        if self.period_vectors is None:
            return deltas
        deltas = np.atleast_2d(np.asarray(deltas, dtype=np.float64))
        if deltas.shape[0] > self._WRAP_CHUNK:
            return np.concatenate([self._wrap(deltas[i:i + self._WRAP_CHUNK])
                                   for i in range(0, deltas.shape[0], self._WRAP_CHUNK)])
        return self._wrap(deltas)

    def _quarter_r2(self):
        """Squared quarter of the shortest nonzero lattice offset: a delta
        with lattice coordinate 0 shorter than this is its own shortest
        representative."""
        if not hasattr(self, "_wrap_r2"):
            offs = [np.array([di, dj]) @ self.period_vectors for di in (-1.0, 0.0, 1.0)
                    for dj in (-1.0, 0.0, 1.0) if (di, dj) != (0.0, 0.0)]
            self._wrap_r2 = (min(float(np.dot(o, o)) for o in offs) ** 0.5 / 4.0) ** 2
        return self._wrap_r2

    def _wrap(self, deltas):
        basis = self.period_vectors[:, :2].T
        frac = np.linalg.solve(basis, deltas[:, :2].T).T
        near = np.floor(frac + 0.5)
        # A row with lattice coordinate 0 that is shorter than a quarter of the
        # shortest lattice offset has (0, 0) as its strict minimum whatever the
        # rounding: its result is deltas - 0 = deltas.  Only the others (faces
        # across the seams) run the 9-candidate search.
        short = (near[:, 0] == 0) & (near[:, 1] == 0) & (np.einsum("ij,ij->i", deltas, deltas) < self._quarter_r2())
        if short.all():
            return deltas.copy()
        out = deltas.copy()
        rest = ~short
        out[rest] = self._wrap_search(deltas[rest], near[rest])
        return out

    def _wrap_search(self, deltas, near):
        best = best_d2 = None
        for di in (-1.0, 0.0, 1.0):
            for dj in (-1.0, 0.0, 1.0):
                cand = deltas - (near + [di, dj]) @ self.period_vectors
                d2 = np.einsum("ij,ij->i", cand, cand)
                if best is None:
                    best, best_d2 = cand, d2
                else:
                    # strict '<': the first minimal candidate wins
                    better = d2 < best_d2
                    best = np.where(better[:, None], cand, best)
                    best_d2 = np.where(better, d2, best_d2)
        return best

    def wrapped_distance(self, points, ref):
        return np.linalg.norm(self.wrap_deltas(np.atleast_2d(points) - np.asarray(ref)), axis=1)


# -- generators ------------------------------------------------------------------


def gen_periodic_grid(nx, ny, spacing=1.0):
    """Equilateral triangulated torus grid, vertex (i, j) -> j*nx + i, two
    faces per lattice cell; order-identical to mesh.py:168-199."""
    if nx < 3 or ny < 3:
        raise MeshFormatError("size too small: periodic grid needs nx, ny >= 3")
    s = float(spacing)
    a1 = np.array([s, 0.0, 0.0])
    a2 = np.array([0.5 * s, 0.5 * np.sqrt(3.0) * s, 0.0])
    if devmesh.enabled():
        pos, faces = devmesh.torus(int(nx), int(ny), s)
        return TriMesh._from_device(pos, faces, period_vectors=np.stack([nx * a1, ny * a2]))
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    positions = ii.reshape(-1, 1) * a1 + jj.reshape(-1, 1) * a2
    i = np.arange(nx, dtype=np.int64)[None, :]
    j = np.arange(ny, dtype=np.int64)[:, None]
    ip = (i + 1) % nx
    jp = (j + 1) % ny
    v00 = j * nx + i
    v10 = j * nx + ip
    v01 = jp * nx + i
    v11 = jp * nx + ip
    faces = np.empty((ny, nx, 2, 3), dtype=np.int32)
    faces[..., 0, 0], faces[..., 0, 1], faces[..., 0, 2] = v00, v10, v01
    faces[..., 1, 0], faces[..., 1, 1], faces[..., 1, 2] = v10, v11, v01
    return TriMesh(positions, faces.reshape(-1, 3), period_vectors=np.stack([nx * a1, ny * a2]))


_PHI_GOLD = (1.0 + np.sqrt(5.0)) / 2.0
_ICO_V = np.array([(-1, _PHI_GOLD, 0), (1, _PHI_GOLD, 0), (-1, -_PHI_GOLD, 0), (1, -_PHI_GOLD, 0),
                   (0, -1, _PHI_GOLD), (0, 1, _PHI_GOLD), (0, -1, -_PHI_GOLD), (0, 1, -_PHI_GOLD),
                   (_PHI_GOLD, 0, -1), (_PHI_GOLD, 0, 1), (-_PHI_GOLD, 0, -1), (-_PHI_GOLD, 0, 1)],
                  dtype=np.float64)
_ICO_F = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                   (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                   (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                   (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)


def _unit(v):
    # The reference normalises each new vertex with the 1-D np.linalg.norm,
    # i.e. sqrt(v.dot(v)) (a BLAS dot).  A batched (1x3)@(3x1) matmul goes
    # through the same dot kernel, so the result is bitwise equal; einsum or
    # an axis-norm round differently in ~10% of vertices.
    d = (v[:, None, :] @ v[:, :, None]).reshape(-1)
    return v / np.sqrt(d)[:, None]


def gen_icosphere(subdiv, max_subdiv=7):
    """Unit icosphere by midpoint subdivision (order-identical to
    mesh.py:216-246).  ``max_subdiv`` defaults to the reference's cap (7,
    mesh.py:222-223); the large benchmark meshes pass a higher cap (levels up
    to 12 = 167.8M vertices follow the same numbering rule).

    Per level, the new vertex of edge (i, j) gets the next id the first time
    the edge is met walking faces in order and, per face (i, j, k), edges
    (i,j), (j,k), (k,i); each face becomes (i,a,c), (j,b,a), (k,c,b), (a,b,c).
    """
    if not 0 <= subdiv <= max_subdiv:
        raise MeshFormatError(f"subdiv must be in [0, {max_subdiv}]")
    verts = _unit(_ICO_V.copy())
    faces = _ICO_F.copy()
    if devmesh.enabled():
        return TriMesh._from_device(*devmesh.icosphere(int(subdiv), verts, faces))
    for _ in range(subdiv):
        n_old = verts.shape[0]
        e0 = faces[:, [0, 1, 2]].ravel()
        e1 = faces[:, [1, 2, 0]].ravel()
        key = np.minimum(e0, e1) * n_old + np.maximum(e0, e1)
        uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
        rank = np.empty(uniq.size, dtype=np.int64)
        rank[np.argsort(first, kind="stable")] = np.arange(uniq.size)
        mid = (n_old + rank[inv]).reshape(-1, 3)          # a, b, c per face
        order = np.argsort(first, kind="stable")
        pa, pb = e0[first[order]], e1[first[order]]
        verts = np.concatenate([verts, _unit(verts[pa] + verts[pb])])
        i, j, k = faces[:, 0], faces[:, 1], faces[:, 2]
        a, b, c = mid[:, 0], mid[:, 1], mid[:, 2]
        faces = np.stack([np.stack([i, a, c], 1), np.stack([j, b, a], 1),
                          np.stack([k, c, b], 1), np.stack([a, b, c], 1)], 1).reshape(-1, 3)
    positions = verts / np.linalg.norm(verts, axis=1)[:, None]
    return TriMesh(positions, faces.astype(np.int32))


# -- Laplacian ---------------------------------------------------------------------


class Laplacian:
    """Mesh Laplacian with its transpose (mesh.py:364-376).  ``mat_t`` (L^T
    in CSC == L in CSR) is what the device step consumes."""

    def __init__(self, mat, mat_t, scheme):
        self._mat = mat
        self._mat_t = mat_t
        self.scheme = scheme
        self.device = None   # device-built: {"ptr", "idx", "val_t", "val", "n"} (host copies lazy)

    @classmethod
    def _from_device(cls, n_v, ptr, idx, val_t, val, scheme="uniform"):
        self = cls(None, None, scheme)
        self.device = {"n": int(n_v), "ptr": ptr, "idx": idx, "val_t": val_t, "val": val}
        return self

    def _host(self, which):
        d = self.device
        n = d["n"]
        nnz = int(d["idx"].numel()) if n else 0
        ptr, idx = d["ptr"].cpu().numpy(), d["idx"][:nnz].cpu().numpy()
        return SparseMat(n, n, ptr, idx, d[which][:nnz].cpu().numpy(), check=False)

    @property
    def mat(self):
        if self._mat is None and self.device is not None:
            self._mat = self._host("val")
        return self._mat

    @mat.setter
    def mat(self, m):
        self._mat = m

    @property
    def mat_t(self):
        if self._mat_t is None and self.device is not None:
            self._mat_t = self._host("val_t")
        return self._mat_t

    @mat_t.setter
    def mat_t(self, m):
        self._mat_t = m

    @property
    def n_vertices(self):
        return self.device["n"] if self.device is not None else self.mat_t.n_cols

    def __repr__(self):
        nnz = int(self.device["idx"].numel()) if self.device is not None else self.mat.nnz
        return f"Laplacian({self.scheme}, n={self.n_vertices}, nnz={nnz})"


def _csr_of_l(n_v, rows, cols, vals):
    """L in CSR (== L^T in CSC) from triplets with unique positions."""
    key = rows.astype(np.int64) * n_v + cols.astype(np.int64)
    order = np.argsort(key, kind="stable")
    ptr = np.zeros(n_v + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_v), out=ptr[1:])
    return SparseMat(n_v, n_v, ptr.astype(INDEX), cols[order].astype(INDEX),
                     vals[order], check=False)


def build_laplacian(mesh, scheme="uniform"):
    """``uniform``: L(i,j) = 1/deg(i) on edges, -1 on the diagonal.
    ``cotan-clamped``: clamped cotangent weights, rows rescaled to sum zero,
    diagonal -1, zero-weight vertices fall back to unit weights
    (mesh.py:379-431).  A device-built mesh gets its uniform Laplacian
    built on the device (ft_uniform_laplacian, same bytes)."""
    n_v = mesh.n_vertices
    topo = getattr(mesh, "_topo_dev", None)
    if scheme == "uniform" and topo is not None:
        deg = topo["degree"]
        if n_v and int(deg.min().item()) == 0:
            v = int((deg == 0).nonzero()[0, 0].item())
            raise IsolatedVertexError(f"isolated-vertex: vertex {v} has no edges")
        lap = Laplacian._from_device(n_v, *devmesh.uniform_laplacian(n_v, topo["neighbor_ptr"],
                                                                     topo["neighbor_idx"]))
        from .sparse import warm_pinned_results
        warm_pinned_results(n_v)     # the results' pinned host blocks, ahead of the first evolve
        if not mesh.periodic and n_v >= devmesh.LOCALITY_MIN_VERTICES:
            # the engine's locality order for long evolves (the caller's
            # numbering is kept at the API: field.evolve permutes in and out)
            lap.device["order"] = devmesh.morton_order_device(mesh._cache["dev_positions"])
        return lap
    deg = mesh.degree
    if np.any(deg == 0):
        raise IsolatedVertexError(
            f"isolated-vertex: vertex {int(np.flatnonzero(deg == 0)[0])} has no edges")
    ed = mesh.edges
    diag = np.arange(n_v)
    if scheme == "uniform":
        rows = np.concatenate([ed[:, 0], ed[:, 1], diag])
        cols = np.concatenate([ed[:, 1], ed[:, 0], diag])
        vals = np.concatenate([1.0 / deg[ed[:, 0]], 1.0 / deg[ed[:, 1]], -np.ones(n_v)])
    elif scheme == "cotan-clamped":
        wt = _cotan_edge_weights(mesh)
        keep = wt > 0
        rsum = np.zeros(n_v)
        np.add.at(rsum, ed[keep, 0], wt[keep])
        np.add.at(rsum, ed[keep, 1], wt[keep])
        dead = rsum == 0
        if dead.any():
            touch = dead[ed[:, 0]] | dead[ed[:, 1]]
            wt = np.where(touch, np.maximum(wt, 1.0), wt)
            keep = wt > 0
            rsum = np.zeros(n_v)
            np.add.at(rsum, ed[keep, 0], wt[keep])
            np.add.at(rsum, ed[keep, 1], wt[keep])
        e, w = ed[keep], wt[keep]
        rows = np.concatenate([e[:, 0], e[:, 1], diag])
        cols = np.concatenate([e[:, 1], e[:, 0], diag])
        vals = np.concatenate([w / rsum[e[:, 0]], w / rsum[e[:, 1]], -np.ones(n_v)])
    else:
        raise ShapeError(f"unknown Laplacian scheme: {scheme!r}")
    mat_t = _csr_of_l(n_v, rows, cols, vals)
    return Laplacian(mat=transpose(mat_t), mat_t=mat_t, scheme=scheme)


def _cotan_edge_weights(mesh):
    """Half-cotangent of the opposite angle summed per edge, clamped at 0
    (mesh.py:434-454).  Per-face loop with the same numpy operations as the
    reference so the weights are bitwise equal."""
    p, f = mesh.positions, mesh.faces
    n_v = mesh.n_vertices
    ekey = mesh.edges[:, 0] * n_v + mesh.edges[:, 1]
    out = np.zeros(mesh.n_edges)
    for face in f:
        pts = p[face]
        if mesh.periodic:
            pts = pts[0] + np.vstack([np.zeros(3), mesh.wrap_deltas(pts[1:] - pts[0])])
        for apex in range(3):
            i1, i2 = (apex + 1) % 3, (apex + 2) % 3
            u = pts[i1] - pts[apex]
            v = pts[i2] - pts[apex]
            cr = np.linalg.norm(np.cross(u, v))
            if cr <= 0:
                continue
            a, b = int(face[i1]), int(face[i2])
            k = np.searchsorted(ekey, min(a, b) * n_v + max(a, b))
            out[k] += 0.5 * (float(np.dot(u, v)) / cr)
    return np.maximum(out, 0.0)


# ---------------------------------------------------------------------------
# OBJ / OFF file plumbing (the reference's load_mesh / write_obj,
# mesh.py:252-358): same accepted inputs, error classes and messages.


def _parse_obj(lines):
    verts, faces = [], []
    for lineno, raw in enumerate(lines, 1):
        tok = raw.split()
        if not tok or tok[0].startswith("#"):
            continue
        try:
            if tok[0] == "v":
                verts.append([float(t) for t in tok[1:4]])
            elif tok[0] == "f":
                # "i", "i/t", "i//n", "i/t/n": the vertex index leads
                ids = [int(t.partition("/")[0]) for t in tok[1:]]
                if len(ids) != 3:
                    raise NonTriangularFaceError(f"non-triangular: line {lineno} has {len(ids)} vertices")
                if min(ids) <= 0:
                    raise MeshFormatError(f"line {lineno}: nonpositive OBJ index")
                faces.append([i - 1 for i in ids])
        except (ValueError, IndexError) as exc:
            raise MeshFormatError(f"line {lineno}: {exc}") from exc
    if not verts:
        raise MeshFormatError("no vertices found")
    if any(len(v) != 3 for v in verts):
        raise MeshFormatError("vertex record with fewer than 3 coordinates")
    return TriMesh(np.asarray(verts), np.asarray(faces, dtype=np.int32).reshape(-1, 3))


def _parse_off(lines):
    # tokens with their line numbers, comments stripped
    toks = [(t, ln) for ln, raw in enumerate(lines, 1) for t in raw.split("#", 1)[0].split()]
    if not toks or toks[0][0].upper() != "OFF":
        raise MeshFormatError("line 1: missing OFF header")
    it = iter(toks[1:])
    last = toks[-1][1]

    def nxt(kind):
        try:
            t, ln = next(it)
        except StopIteration:
            raise MeshFormatError(f"line {last}: truncated OFF file") from None
        try:
            return kind(t), ln
        except ValueError as exc:
            raise MeshFormatError(f"line {ln}: bad token {t!r}") from exc

    n_v, n_f = nxt(int)[0], nxt(int)[0]
    nxt(int)                                          # edge count (unused)
    verts = [[nxt(float)[0] for _ in range(3)] for _ in range(n_v)]
    faces = []
    for _ in range(n_f):
        k, ln = nxt(int)
        if k != 3:
            raise NonTriangularFaceError(f"non-triangular: line {ln} has {k} vertices")
        faces.append([nxt(int)[0] for _ in range(3)])
    return TriMesh(np.asarray(verts, dtype=np.float64).reshape(-1, 3),
                   np.asarray(faces, dtype=np.int32).reshape(-1, 3))


def load_mesh(path, fmt=None):
    """Load an ASCII OBJ (``v`` / ``f`` records; texture and normal indices
    ignored) or OFF triangle mesh; ``fmt`` defaults to the file extension.
    Non-triangle faces raise :class:`NonTriangularFaceError`, malformed
    records :class:`MeshFormatError` with the line number."""
    fmt = (fmt or str(path).rsplit(".", 1)[-1]).lower()
    if fmt not in ("obj", "off"):
        raise MeshFormatError(f"unknown mesh format: {fmt!r}")
    with open(path) as fh:
        lines = fh.readlines()
    return _parse_obj(lines) if fmt == "obj" else _parse_off(lines)


def write_obj(mesh_or_positions, path_or_faces, path=None, comments=()):
    """Write ASCII OBJ with 1-based face indices: ``write_obj(mesh, path)``
    or ``write_obj(positions, faces, path)``; coordinates with ``repr`` so
    they round-trip exactly."""
    if path is None:
        positions, faces, path = mesh_or_positions.positions, mesh_or_positions.faces, path_or_faces
    else:
        positions, faces = mesh_or_positions, path_or_faces
    out = [f"# {c}\n" for c in comments]
    out += [f"v {float(x)!r} {float(y)!r} {float(z)!r}\n" for x, y, z in np.asarray(positions).tolist()]
    out += [f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in np.asarray(faces).tolist()]
    with open(path, "w") as fh:
        fh.writelines(out)
