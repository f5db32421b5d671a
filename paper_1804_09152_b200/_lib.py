"""ctypes binding of the C-ABI library ``libfieldtess_cuda.so``.

The library is the only compute backend: there is no CPU fallback.  If it is
missing or fails to load, every compute entry point raises immediately.
The structures mirror ``include/fieldtess_cuda.h`` field for field.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FT_LIB overrides the library path (A/B measurements of two builds)
LIB_PATH = os.environ.get("FT_LIB") or os.path.join(_HERE, "libfieldtess_cuda.so")

FT_OK = 0
FT_ERR_SHAPE = 1
FT_ERR_NUMERICAL = 2
FT_ERR_CAPACITY = 3
FT_ERR_CUDA = 4
FT_ERR_PATTERN = 5
FT_ERR_ARG = 6

FT_F64 = 0
FT_F32 = 1

FT_LAP_EXPLICIT = 0
FT_LAP_UNIFORM = 1
FT_LAP_PACKED = 2
FT_LAP_CHECK_FINITE = 4
FT_LAP_SYMMETRIC = 8
FT_HINT_DENSE_BAND = 16
FT_HINT_FOUR_ROW = 32

FT_PHASE_COLUMNS = 1
FT_PHASE_FINALIZE = 2

FT_STATUS_OK = 0
FT_STATUS_NAN = 1
FT_STATUS_PATTERN = 2
FT_STATUS_OVERFLOW = 3
FT_STATUS_CONVERGED = 4
FT_STATUS_MAXSTEPS = 5
FT_STATUS_OUT_OVERFLOW = 6
FT_STATUS_HALO_OVERFLOW = 7

FT_HALO_FORCE = 1

ABI_VERSION = 6


class FtParams(ctypes.Structure):
    _fields_ = [("w", ctypes.c_double), ("a", ctypes.c_double),
                ("e", ctypes.c_double), ("e_base", ctypes.c_double),
                ("mu", ctypes.c_double), ("dt", ctypes.c_double)]


class FtCsc(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int32), ("n_cols", ctypes.c_int32),
                ("col_ptr", ctypes.c_void_p), ("row_idx", ctypes.c_void_p),
                ("values", ctypes.c_void_p), ("capacity", ctypes.c_int64)]


class FtTiled(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int32), ("n_cols", ctypes.c_int32),
                ("sig", ctypes.c_void_p), ("aux", ctypes.c_void_p),
                ("v0", ctypes.c_void_p), ("v1", ctypes.c_void_p),
                ("pool_idx", ctypes.c_void_p), ("pool_val", ctypes.c_void_p),
                ("capacity", ctypes.c_int64)]


class FtDomain(ctypes.Structure):
    _fields_ = [("col_begin", ctypes.c_int32), ("col_count", ctypes.c_int32),
                ("step_capacity", ctypes.c_int64), ("report_ids", ctypes.c_void_p),
                ("out_id", ctypes.c_int32), ("pad", ctypes.c_int32)]


class FtStepStats(ctypes.Structure):
    _fields_ = [("max_delta", ctypes.c_double), ("base_mass", ctypes.c_double),
                ("nnz_phi", ctypes.c_int64), ("nnz_skel", ctypes.c_int64),
                ("status", ctypes.c_int32), ("nan_col", ctypes.c_int32),
                ("bad_col", ctypes.c_int32), ("bad_row", ctypes.c_int32),
                ("bad_is_lt", ctypes.c_int32), ("step", ctypes.c_int32),
                ("needed", ctypes.c_int64)]


STATS_BYTES = ctypes.sizeof(FtStepStats)
assert STATS_BYTES == 64

# numpy view of a device stats array copied to the host
import numpy as _np  # noqa: E402

STATS_DTYPE = _np.dtype([("max_delta", "<f8"), ("base_mass", "<f8"),
                         ("nnz_phi", "<i8"), ("nnz_skel", "<i8"),
                         ("status", "<i4"), ("nan_col", "<i4"),
                         ("bad_col", "<i4"), ("bad_row", "<i4"),
                         ("bad_is_lt", "<i4"), ("step", "<i4"),
                         ("needed", "<i8")])
assert STATS_DTYPE.itemsize == STATS_BYTES

# every symbol include/fieldtess_cuda.h declares
EXPORTS = ("ft_abi_version", "ft_last_error", "ft_workspace_bytes",
           "ft_workspace_init", "ft_tiled_from_csc",
           "ft_step", "ft_step_phases", "ft_step_run", "ft_compact",
           "ft_evolve", "ft_labels", "ft_faces_by_cell", "ft_lloyd_centroids",
           "ft_dual_products", "ft_domain_step", "ft_halo_bytes", "ft_halo_pack",
           "ft_halo_unpack", "ft_domain_combine", "ft_domain_control", "ft_laplacian_pack",
           "ft_point_triangle_distances", "ft_spgemm_count", "ft_spgemm_expand",
           "ft_segment_sums", "ft_skeleton", "ft_expand", "ft_normalize_columns",
           "ft_clique_triangles", "ft_lloyd_backproject", "ft_lloyd_partials", "ft_lloyd_finish",
           "ft_lloyd_backproject_keys", "ft_ico_flags", "ft_ico_midpoints", "ft_ico_children",
           "ft_renormalize", "ft_torus_grid", "ft_face_geometry", "ft_vertex_area", "ft_uniform_laplacian",
           "ft_wind_triangles")

_lib = None


class LibraryMissing(RuntimeError):
    """The CUDA library is not built or cannot be loaded (no CPU fallback)."""


def _declare(lib):
    vp = ctypes.c_void_p
    P = ctypes.POINTER
    lib.ft_abi_version.restype = ctypes.c_int
    lib.ft_last_error.restype = ctypes.c_char_p
    lib.ft_workspace_bytes.argtypes = [ctypes.c_int32]
    lib.ft_workspace_bytes.restype = ctypes.c_size_t
    lib.ft_workspace_init.argtypes = [vp, ctypes.c_size_t, vp]
    lib.ft_workspace_init.restype = ctypes.c_int
    lib.ft_tiled_from_csc.argtypes = [P(FtCsc), P(FtTiled), ctypes.c_int32, vp, ctypes.c_size_t,
                                      vp, vp]
    lib.ft_tiled_from_csc.restype = ctypes.c_int
    lib.ft_step.argtypes = [P(FtCsc), ctypes.c_int32, P(FtCsc), P(FtTiled), P(FtTiled), P(FtCsc),
                            ctypes.c_int32, P(FtParams), vp, ctypes.c_size_t, vp, vp]
    lib.ft_step.restype = ctypes.c_int
    lib.ft_step_phases.argtypes = [P(FtCsc), ctypes.c_int32, P(FtCsc), P(FtTiled), P(FtTiled), P(FtCsc),
                                   ctypes.c_int32, P(FtParams), vp, ctypes.c_size_t, vp,
                                   P(ctypes.c_float), vp]
    lib.ft_step_phases.restype = ctypes.c_int
    lib.ft_step_run.argtypes = [P(FtCsc), ctypes.c_int32, P(FtTiled), P(FtTiled), ctypes.c_int32,
                                ctypes.c_int32, P(FtParams), vp, ctypes.c_size_t, ctypes.c_int32,
                                vp, vp]
    lib.ft_step_run.restype = ctypes.c_int
    lib.ft_compact.argtypes = [P(FtTiled), P(FtCsc), ctypes.c_int32, vp, ctypes.c_size_t,
                               vp, vp]
    lib.ft_compact.restype = ctypes.c_int
    lib.ft_evolve.argtypes = [P(FtCsc), ctypes.c_int32, P(FtCsc), P(FtTiled), P(FtTiled),
                              P(FtCsc), ctypes.c_int32, P(FtParams), ctypes.c_int32,
                              ctypes.c_double, ctypes.c_double, vp, ctypes.c_size_t,
                              vp, vp, vp]
    lib.ft_evolve.restype = ctypes.c_int
    lib.ft_labels.argtypes = [P(FtCsc), ctypes.c_int32, vp, vp]
    lib.ft_labels.restype = ctypes.c_int
    i32 = ctypes.c_int32
    lib.ft_faces_by_cell.argtypes = [P(FtCsc), i32, i32, vp, vp, vp, vp, vp, vp, vp]
    lib.ft_faces_by_cell.restype = ctypes.c_int
    lib.ft_lloyd_centroids.argtypes = [vp, i32, vp, i32, vp, vp, vp, vp, i32, vp, vp, vp,
                                       vp, vp, vp, vp, vp]
    lib.ft_lloyd_centroids.restype = ctypes.c_int
    lib.ft_dual_products.argtypes = [P(FtCsc), i32, vp, vp, ctypes.c_double, vp, vp, vp, vp,
                                     ctypes.c_int64, vp, vp]
    lib.ft_dual_products.restype = ctypes.c_int
    lib.ft_domain_step.argtypes = [P(FtCsc), i32, P(FtTiled), P(FtTiled), i32, P(FtParams),
                                   P(FtDomain), vp, ctypes.c_size_t, vp, vp]
    lib.ft_domain_step.restype = ctypes.c_int
    lib.ft_halo_bytes.argtypes = [i32, i32, i32]
    lib.ft_halo_bytes.restype = ctypes.c_int64
    lib.ft_halo_pack.argtypes = [P(FtTiled), vp, i32, i32, i32, vp, vp, vp, vp, i32, vp]
    lib.ft_halo_pack.restype = ctypes.c_int
    lib.ft_halo_unpack.argtypes = [P(FtTiled), vp, i32, i32, i32, vp, ctypes.c_int64, vp, i32,
                                   P(FtTiled), vp, vp, vp]
    lib.ft_halo_unpack.restype = ctypes.c_int
    lib.ft_domain_combine.argtypes = [vp, i32, i32, i32, ctypes.c_double, ctypes.c_double, vp,
                                      vp, vp]
    lib.ft_domain_combine.restype = ctypes.c_int
    lib.ft_domain_control.argtypes = [vp, i32, vp, vp]
    lib.ft_domain_control.restype = ctypes.c_int
    lib.ft_laplacian_pack.argtypes = [P(FtCsc), i32, vp, vp, vp]
    lib.ft_laplacian_pack.restype = ctypes.c_int
    lib.ft_point_triangle_distances.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, vp]
    lib.ft_point_triangle_distances.restype = ctypes.c_int
    lib.ft_spgemm_count.argtypes = [P(FtCsc), P(FtCsc), ctypes.c_int64, vp, vp]
    lib.ft_spgemm_count.restype = ctypes.c_int
    lib.ft_spgemm_expand.argtypes = [P(FtCsc), P(FtCsc), ctypes.c_int64, vp, vp, vp, vp]
    lib.ft_spgemm_expand.restype = ctypes.c_int
    lib.ft_segment_sums.argtypes = [vp, ctypes.c_int64, vp, ctypes.c_int64, vp, vp]
    lib.ft_segment_sums.restype = ctypes.c_int
    lib.ft_skeleton.argtypes = [P(FtCsc), P(FtCsc), vp, vp, vp, vp]
    lib.ft_skeleton.restype = ctypes.c_int
    lib.ft_expand.argtypes = [P(FtCsc), vp, vp, vp, vp, vp]
    lib.ft_expand.restype = ctypes.c_int
    lib.ft_normalize_columns.argtypes = [P(FtCsc), vp, vp, vp]
    lib.ft_normalize_columns.restype = ctypes.c_int
    i64, f64 = ctypes.c_int64, ctypes.c_double
    lib.ft_ico_flags.argtypes = [i64, vp, vp, vp]
    lib.ft_ico_midpoints.argtypes = [i32, vp, vp, vp, i32, vp, vp, vp]
    lib.ft_ico_children.argtypes = [i32, vp, vp, vp, vp, vp, vp]
    lib.ft_renormalize.argtypes = [i32, vp, vp]
    lib.ft_torus_grid.argtypes = [i32, i32, f64, vp, vp, vp]
    lib.ft_face_geometry.argtypes = [i32, vp, vp, vp, f64, vp, vp, vp, vp, vp]
    lib.ft_vertex_area.argtypes = [i32, vp, vp, vp, vp, vp]
    lib.ft_uniform_laplacian.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp]
    for name in ("ft_ico_flags", "ft_ico_midpoints", "ft_ico_children", "ft_renormalize", "ft_torus_grid",
                 "ft_face_geometry", "ft_vertex_area", "ft_uniform_laplacian"):
        getattr(lib, name).restype = ctypes.c_int
    lib.ft_wind_triangles.argtypes = [ctypes.c_int64, vp]
    lib.ft_wind_triangles.restype = ctypes.c_int
    lib.ft_clique_triangles.argtypes = [i32, vp, vp, vp, vp, vp, vp]
    lib.ft_clique_triangles.restype = ctypes.c_int
    lib.ft_lloyd_backproject.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp]
    lib.ft_lloyd_backproject.restype = ctypes.c_int
    lib.ft_lloyd_partials.argtypes = [vp, i32, vp, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]
    lib.ft_lloyd_partials.restype = ctypes.c_int
    lib.ft_lloyd_finish.argtypes = [i32, vp, vp, vp, vp, vp]
    lib.ft_lloyd_finish.restype = ctypes.c_int
    lib.ft_lloyd_backproject_keys.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.ft_lloyd_backproject_keys.restype = ctypes.c_int


def lib():
    """The loaded library; raises :class:`LibraryMissing` loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is not built: run `make -C "
                f"{os.path.join(_HERE, 'csrc')}` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise LibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
        _declare(handle)
        if handle.ft_abi_version() != ABI_VERSION:
            raise LibraryMissing("libfieldtess_cuda.so ABI version mismatch")
        _lib = handle
    return _lib


def last_error():
    msg = lib().ft_last_error()
    return msg.decode() if msg else ""
