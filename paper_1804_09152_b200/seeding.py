"""Seed sampling: area-weighted random faces snapped to the nearest corner.

``sample_seed_vertices(mesh, count, rng_seed)`` returns exactly the seeds of
the reference's ``cli.sample_seed_vertices`` (pkg/src/fieldtess/cli.py:
183-215) -- same numpy PCG64 stream, same arithmetic -- without its
O(n_faces) cost per attempt (``rng.choice(n, p=...)`` rebuilds the CDF on
every call: ~55 min for 65,536 seeds at 10M vertices).

Replay: every attempt of the reference consumes three doubles of the
stream, in order -- the face draw (``choice`` with ``p`` draws one
``random()`` and searches the normalised CDF, side="right"), then
``sqrt(random())`` and ``random()``.  So attempts are drawn in batches of
3k doubles from the same Generator, the faces found with one
``searchsorted`` on the one CDF, the sample points and nearest corners
computed for the whole batch with the reference's operation order, and the
first occurrences kept in attempt order until ``count`` distinct vertices
are found.  The 200*count attempt cap and the error messages are the
reference's.
"""

import numpy as np

__all__ = ["sample_seed_vertices"]


def _face_cdf(mesh):
    # numpy Generator.choice(a, p=p): cdf = p.cumsum(); cdf /= cdf[-1]
    probs = mesh.face_area / mesh.face_area.sum()
    cdf = probs.cumsum()
    cdf /= cdf[-1]
    return cdf


def _batch_vertices(mesh, cdf, draws):
    """Seed vertex of each attempt; ``draws`` is (k, 3) stream doubles."""
    f = cdf.searchsorted(draws[:, 0], side="right")
    r1 = np.sqrt(draws[:, 1])
    r2 = draws[:, 2]
    tri = mesh.faces[f]
    pos = mesh.positions
    p0 = pos[tri[:, 0]]
    if mesh.periodic:
        e1 = mesh.wrap_deltas(pos[tri[:, 1]] - p0)
        e2 = mesh.wrap_deltas(pos[tri[:, 2]] - p0)
    else:
        e1 = pos[tri[:, 1]] - p0
        e2 = pos[tri[:, 2]] - p0
    # pt = p0 + (1 - r1) * e1 + (r1 * r2) * e2, left to right
    pt = (p0 + (1 - r1)[:, None] * e1) + (r1 * r2)[:, None] * e2
    corners = np.stack([p0, p0 + e1, p0 + e2], axis=1)          # (k, 3, 3)
    diff = corners - pt[:, None, :]
    # np.linalg.norm(x, axis=1) of a (3, 3): sqrt((x0^2 + x1^2) + x2^2)
    sq = diff * diff
    dist = np.sqrt((sq[:, :, 0] + sq[:, :, 1]) + sq[:, :, 2])
    return tri[np.arange(tri.shape[0]), np.argmin(dist, axis=1)].astype(np.int64)


def sample_seed_vertices(mesh, count, rng_seed):
    """Area-weighted random face sampling snapped to the nearest face vertex
    (identical to the reference's ``cli.sample_seed_vertices``)."""
    if count < 1:
        raise ValueError("seed count must be positive")
    if count > mesh.n_vertices:
        raise ValueError("more seeds than vertices")
    rng = np.random.default_rng(rng_seed)
    cdf = _face_cdf(mesh)
    limit = 200 * count
    taken = []
    seen = set()
    attempts = 0
    while len(taken) < count:
        k = min(max(2 * (count - len(taken)), 256), limit + 1 - attempts)
        if k <= 0:
            raise ValueError("could not draw distinct seed vertices")
        draws = rng.random(3 * k).reshape(k, 3)
        verts = _batch_vertices(mesh, cdf, draws)
        for v in verts.tolist():
            attempts += 1
            if attempts > limit:
                raise ValueError("could not draw distinct seed vertices")
            if v not in seen:
                seen.add(v)
                taken.append(v)
                if len(taken) == count:
                    break
    return np.asarray(taken, dtype=np.int64)
