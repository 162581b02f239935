"""ctypes binding of libspfd_b200.so (include/spfd_b200.h).

The CUDA library is the only compute path: importing this module on a box
without the built library, or calling into it without a CUDA device, raises
immediately.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import EmptySystemError, LatticeError, ProjectionError, SingularPointError, SolverError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPFD_LIB") or os.path.join(_HERE, "libspfd_b200.so")  # SPFD_LIB: A/B builds

SPFD_OK = 0
SPFD_EINVAL = 1
SPFD_ENONFINITE = 2
SPFD_ENOTPOS = 3
SPFD_EEMPTY = 4
SPFD_ENOCONV = 5
SPFD_ECUDA = 6
SPFD_ENCCL = 7
SPFD_ENOMEM = 8
SPFD_EINCOMPAT = 9
SPFD_EPROJECTION = 10
SPFD_ELATTICE = 11
SPFD_ESINGULAR = 12

EXPORT_EDGE_CONDUCTANCE = 0
EXPORT_DOF_TO_NODE = 1
EXPORT_NODE_TO_DOF = 2
EXPORT_PINNED = 3
EXPORT_VOXEL_INDICES = 4
EXPORT_DIAGONAL = 5

METHOD_PCG = 0
METHOD_FGMRES = 1
SMOOTHER_JACOBI, SMOOTHER_CHEBYSHEV = 0, 1


class OpInfo(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int64 * 3),
        ("n_nodes", ctypes.c_int64),
        ("n_edges", ctypes.c_int64),
        ("n_dofs", ctypes.c_int64),
        ("n_conductive", ctypes.c_int64),
        ("n_components", ctypes.c_int64),
        ("n_cond_voxels", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("span_len", ctypes.c_int64),
        ("n_rows", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
    ]


class Config(ctypes.Structure):
    _fields_ = [
        ("rel_tol", ctypes.c_double),
        ("max_iters", ctypes.c_int32),
        ("restart", ctypes.c_int32),
        ("pre_sweeps", ctypes.c_int32),
        ("post_sweeps", ctypes.c_int32),
        ("jacobi_damping", ctypes.c_double),
        ("strength_threshold", ctypes.c_double),
        ("coarse_cap", ctypes.c_int32),
        ("max_levels", ctypes.c_int32),
        ("method", ctypes.c_int32),
        ("max_nrhs", ctypes.c_int32),
        ("smoother", ctypes.c_int32),
        ("cheb_degree", ctypes.c_int32),
    ]


class AmgInfo(ctypes.Structure):
    _fields_ = [
        ("n_levels", ctypes.c_int32),
        ("level_rows", ctypes.c_int64 * 32),
        ("level_nnz", ctypes.c_int64 * 32),
        ("prolong_nnz", ctypes.c_int64 * 32),
        ("setup_seconds", ctypes.c_double),
        ("device_bytes", ctypes.c_int64),
        ("structured", ctypes.c_int32),
        ("smoother", ctypes.c_int32),
        ("cheb_degree", ctypes.c_int32),
        ("cheb_lmax", ctypes.c_double * 32),
        ("restriction_csr", ctypes.c_int32),
    ]


class Box(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int64 * 3), ("spacing", ctypes.c_double * 3), ("origin", ctypes.c_double * 3)]


def make_box(dims, spacing, origin):
    b = Box()
    for a in range(3):
        b.dims[a] = int(dims[a])
        b.spacing[a] = float(spacing[a])
        b.origin[a] = float(origin[a])
    return b


class CleanInfo(ctypes.Structure):
    _fields_ = [
        ("rel_before", ctypes.c_double),
        ("rel_after", ctypes.c_double),
        ("solved", ctypes.c_int32),
        ("iterations", ctypes.c_int32),
        ("solve_rel_residual", ctypes.c_double),
        ("setup_seconds", ctypes.c_double),
    ]


class GaugeInfo(ctypes.Structure):
    _fields_ = [("rel_residual", ctypes.c_double), ("worst_face", ctypes.c_int64), ("worst_defect", ctypes.c_double)]


class Report(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("rel_residual", ctypes.c_double * 2),
        ("solve_seconds", ctypes.c_double),
        ("status", ctypes.c_int32),
    ]


_VP = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_D = ctypes.c_double

_SIGS = {
    "spfd_last_error": (ctypes.c_char_p, []),
    "spfd_version": (ctypes.c_char_p, []),
    "spfd_op_create": (_INT, [_VP, _VP, _VP, _VP, _I64, _INT, _VP, _VP]),
    "spfd_op_destroy": (_INT, [_VP]),
    "spfd_op_info_get": (_INT, [_VP, _VP]),
    "spfd_op_export": (_INT, [_VP, _INT, _VP, _VP]),
    "spfd_op_csr": (_INT, [_VP, _VP, _VP, _VP, _VP]),
    "spfd_stencil_apply": (_INT, [_VP, _VP, _VP, _INT, _VP]),
    "spfd_rhs_assemble": (_INT, [_VP, _VP, _VP, _INT, _VP]),
    "spfd_edge_voltages": (_INT, [_VP, _VP, _VP, _D, _VP, _INT, _VP]),
    "spfd_node_field": (_INT, [_VP, _VP, _VP, _INT, _VP]),
    "spfd_voxel_average": (_INT, [_VP, _VP, _VP, _INT, _VP]),
    "spfd_efield_voxavg": (_INT, [_VP, _VP, _VP, _D, _VP, _INT, _VP]),
    "spfd_amg_setup_op": (_INT, [_VP, _VP, _VP, _VP]),
    "spfd_amg_setup_csr": (_INT, [_I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "spfd_amg_destroy": (_INT, [_VP]),
    "spfd_amg_info_get": (_INT, [_VP, _VP]),
    "spfd_amg_level_csr": (_INT, [_VP, _INT, _INT, _VP, _VP, _VP, _VP]),
    "spfd_amg_level_agg": (_INT, [_VP, _INT, _VP, _VP]),
    "spfd_vcycle": (_INT, [_VP, _VP, _VP, _INT, _VP]),
    "spfd_solve": (_INT, [_VP, _VP, _VP, _INT, _VP, _VP, _VP, _VP]),
    "spfd_snapshot": (_INT, [_VP, _VP, _VP, _D, _VP, _VP, _INT, _VP, _VP, _VP]),
    "spfd_bench_kernel": (_INT, [_VP, _INT, _INT, _INT, _VP, _VP, _VP]),
    "spfd_iteration_bytes": (_INT, [_VP, _INT, _VP]),
    "spfd_set_fine_kernel": (_INT, [_INT]),
    "spfd_set_pcg_graph": (_INT, [_INT]),
    "spfd_launch_count": (ctypes.c_int64, []),
    "spfd_copy": (_INT, [_VP, _VP, _I64]),
    "spfd_nccl_unique_id": (_INT, [_VP]),
    "spfd_comm_init_nccl": (_INT, [_VP, _INT, _INT, _VP]),
    "spfd_comm_init_callbacks": (_INT, [_VP, _INT, _INT, _VP]),
    "spfd_comm_destroy": (_INT, [_VP]),
    "spfd_amg_distribute": (_INT, [_VP, _VP, _I64, _VP, _VP]),
    "spfd_field_create": (_INT, [_VP, _VP, _VP]),
    "spfd_field_destroy": (_INT, [_VP]),
    "spfd_coil_field": (_INT, [_I64, _VP, _INT, _VP, _D, _VP, _VP]),
    "spfd_field_interpolate": (_INT, [_VP, _VP, _VP, _VP, _VP]),
    "spfd_field_divergence": (_INT, [_VP, _VP, _VP, _VP]),
    "spfd_field_clean": (_INT, [_VP, _VP, _VP, _D, _VP, _VP]),
    "spfd_field_clean_batch": (_INT, [_VP, _INT, _VP, _VP, _D, _VP, _VP]),
    "spfd_field_gauge": (_INT, [_VP, _VP, _VP, _D, _VP, _VP]),
    "spfd_field_gauge_tree": (_INT, [_VP, _INT, _VP, _VP, _D, _VP, _VP]),
    "spfd_field_circulation": (_INT, [_VP, _VP, _VP, _VP, _VP]),
    "spfd_exposure_stats": (_INT, [_VP, _I64, _D, _VP, _VP, ctypes.c_int32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
}

EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                               ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p),
                               ctypes.POINTER(ctypes.c_int64))
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class CommCallbacks(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("exchange", EXCHANGE_FN), ("allgather", ALLGATHER_FN)]

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load():
    """Load libspfd_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib():
    return load()


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2010_12879_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def check(rc):
    """Map a status code onto the reference's exception classes."""
    if rc == SPFD_OK:
        return
    msg = (load().spfd_last_error() or b"").decode(errors="replace")
    if rc == SPFD_EINVAL:
        raise ValueError(msg)
    if rc in (SPFD_ENONFINITE, SPFD_ENOTPOS):
        raise SolverError(msg)
    if rc == SPFD_EEMPTY:
        raise EmptySystemError(msg)
    if rc == SPFD_ENOMEM:
        raise MemoryError(msg)
    if rc == SPFD_EPROJECTION:
        raise ProjectionError(msg)
    if rc == SPFD_ELATTICE:
        raise LatticeError(msg)
    if rc == SPFD_ESINGULAR:
        raise SingularPointError(msg)
    raise RuntimeError(f"spfd_b200 error {rc}: {msg}")


def make_config(cfg, method=None, max_nrhs=None):
    c = Config()
    c.rel_tol = float(cfg.rel_tol)
    c.max_iters = int(cfg.max_iters)
    c.restart = int(cfg.restart)
    c.pre_sweeps = int(cfg.pre_sweeps)
    c.post_sweeps = int(cfg.post_sweeps)
    c.jacobi_damping = float(cfg.jacobi_damping)
    c.strength_threshold = float(cfg.strength_threshold)
    c.coarse_cap = int(cfg.coarse_cap)
    c.max_levels = int(cfg.max_levels)
    m = method if method is not None else getattr(cfg, "method", "pcg")
    c.method = METHOD_FGMRES if m == "fgmres" else METHOD_PCG
    c.max_nrhs = int(max_nrhs if max_nrhs is not None else getattr(cfg, "max_nrhs", 2))
    c.smoother = SMOOTHER_CHEBYSHEV if getattr(cfg, "smoother", "jacobi") == "chebyshev" else SMOOTHER_JACOBI
    c.cheb_degree = int(getattr(cfg, "chebyshev_degree", 2))
    return c
