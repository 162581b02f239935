"""AMG-preconditioned Krylov solves on the GPU.

Drop-in for /root/reference/pkg/src/spfd/linsolve.py:26-298: `SolveConfig`,
`AmgLevel`, `AmgHierarchy`, `SolveReport`, `amg_setup`, `v_cycle`,
`fgmres_solve` keep their names, arguments, return types and error
behaviour.  `pcg_solve` is the B200 default method (the reference V-cycle is
symmetric).  All work runs in libspfd_b200.so:

* `amg_setup` on a `PoissonSystem` matrix keeps level 0 matrix-free (the
  7-point stencil in the row-span layout); on any other SPD scipy matrix it
  runs the same device setup on a CSR.  Aggregates, prolongators and coarse
  operators are identical to the reference's (plain_aggregation,
  _kernels.py:79-120; Galerkin products, linsolve.py:142-153).
* the Krylov loop, V-cycle and every reduction run on the device with a
  fixed reduction order: repeated solves are bitwise identical.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .errors import SolverError


@dataclass
class SolveConfig:
    """Solver parameters (linsolve.py:26-53) plus the B200 extensions
    `method` ("pcg" | "fgmres"), `max_nrhs` (1 or 2 batched right-hand
    sides, e.g. real/imaginary parts) and `smoother` ("jacobi", the
    reference's damped Jacobi, or "chebyshev": a degree-`chebyshev_degree`
    polynomial in D^-1 A on [beta/5, beta], beta = 1.1 x a power-iteration
    estimate of lambda_max per level; `pre_sweeps`/`post_sweeps` repeat it)."""

    rel_tol: float = 1e-12
    max_iters: int = 1000
    restart: int = 30
    pre_sweeps: int = 1
    post_sweeps: int = 1
    jacobi_damping: float = 2.0 / 3.0
    strength_threshold: float = 0.08
    coarse_cap: int = 500
    max_levels: int = 20
    threads: int | None = None
    trace: object = field(default=None, repr=False, compare=False)
    method: str = "pcg"
    max_nrhs: int = 2
    smoother: str = "jacobi"
    chebyshev_degree: int = 2

    def __post_init__(self):
        if not self.rel_tol > 0.0:
            raise ValueError("rel_tol must be positive")
        if self.restart < 1:
            raise ValueError("restart must be >= 1")
        if not 0.0 < self.jacobi_damping <= 1.0:
            raise ValueError("jacobi_damping must be in (0, 1]")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.coarse_cap < 1 or self.max_levels < 1:
            raise ValueError("coarse_cap and max_levels must be >= 1")
        if self.method not in ("pcg", "fgmres"):
            raise ValueError("method must be 'pcg' or 'fgmres'")
        if self.max_nrhs not in (1, 2):
            raise ValueError("max_nrhs must be 1 or 2")
        if self.smoother not in ("jacobi", "chebyshev"):
            raise ValueError("smoother must be 'jacobi' or 'chebyshev'")
        if not 1 <= self.chebyshev_degree <= 16:
            raise ValueError("chebyshev_degree must be in [1, 16]")


@dataclass
class SolveReport:
    """Observables of one solve (linsolve.py:92-103).  For a batched
    real/imag solve `rel_residual` is the worse of the two and
    `rel_residuals` holds both."""

    iterations: int
    rel_residual: float
    converged: bool
    setup_seconds: float
    solve_seconds: float
    level_sizes: list
    peak_matrix_memory_bytes: int
    threads: int | None = None
    rel_residuals: tuple = ()
    method: str = "pcg"


def _csr_bytes(rows: int, nnz: int) -> int:
    # scipy CSR with int32 indices: data + indices + indptr
    return 8 * nnz + 4 * nnz + 4 * (rows + 1)


class AmgLevel:
    """Lazy host view of one device level (linsolve.py:56-61)."""

    def __init__(self, h: "AmgHierarchy", index: int):
        # a weak reference: the hierarchy owns its levels, and a strong
        # back-reference would keep the device hierarchy alive until the
        # cycle collector runs instead of freeing it on the last `del`
        self._href = weakref.ref(h)
        self.index = index

    @property
    def _h(self) -> "AmgHierarchy":
        h = self._href()
        if h is None:
            raise ReferenceError("the AmgHierarchy of this level has been released")
        return h

    def _csr(self, which):
        h = self._h
        rows = h.level_sizes[self.index]
        if which == 0:
            nnz, shape = h._info.level_nnz[self.index], (rows, rows)
        else:
            if self.index >= h.n_levels - 1:
                return None
            nnz = h._info.prolong_nnz[self.index]
            nxt = h.level_sizes[self.index + 1]
            shape = (rows, nxt) if which == 1 else (nxt, rows)
        ip = torch.empty(shape[0] + 1, dtype=torch.int64, device="cuda")
        ix = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
        dv = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
        _lib.check(_lib.load().spfd_amg_level_csr(h.handle, self.index, which, _lib.ptr(ip), _lib.ptr(ix),
                                                  _lib.ptr(dv), _lib.stream_ptr()))
        return sp.csr_matrix((dv[:nnz].cpu().numpy(), ix[:nnz].cpu().numpy(), ip.cpu().numpy()), shape=shape)

    @cached_property
    def matrix(self):
        return self._csr(0)

    @cached_property
    def prolongation(self):
        return self._csr(1)

    @cached_property
    def restriction(self):
        return self._csr(2)

    @cached_property
    def dinv(self):
        return 1.0 / self.matrix.diagonal()

    @cached_property
    def aggregates(self):
        """Aggregate id per row (the reference's plain_aggregation output)."""
        out = torch.empty(max(self._h.level_sizes[self.index], 1), dtype=torch.int32, device="cuda")
        rc = _lib.load().spfd_amg_level_agg(self._h.handle, self.index, _lib.ptr(out), _lib.stream_ptr())
        if rc == _lib.SPFD_EINVAL:
            return None  # coarsest level: never aggregated
        _lib.check(rc)
        return out[:self._h.level_sizes[self.index]].cpu().numpy()


class AmgHierarchy:
    """Device AMG hierarchy handle (linsolve.py:64-89)."""

    def __init__(self, handle, cfg: SolveConfig, operator=None, fine_matrix=None):
        self.handle = handle
        self.operator = operator
        self._fine = fine_matrix
        info = _lib.AmgInfo()
        _lib.check(_lib.load().spfd_amg_info_get(handle, ctypes.byref(info)))
        self._info = info
        self.level_sizes = [int(info.level_rows[i]) for i in range(info.n_levels)]
        self.setup_seconds = float(info.setup_seconds)
        self.pre_sweeps = cfg.pre_sweeps
        self.post_sweeps = cfg.post_sweeps
        self.damping = cfg.jacobi_damping
        self.structured = bool(info.structured)
        self.device_bytes = int(info.device_bytes)
        self.restriction_csr = bool(info.restriction_csr & 1)    # fine restriction as R = P^T in CSR
        self.prolongation_csr = bool(info.restriction_csr & 2)   # fine prolongation as P in CSR
        self.smoother = "chebyshev" if info.smoother == _lib.SMOOTHER_CHEBYSHEV else "jacobi"
        self.chebyshev_degree = int(info.cheb_degree)
        # lambda_max(D^-1 A_l) estimates behind the Chebyshev intervals (levels < coarsest)
        self.chebyshev_lmax = ([float(info.cheb_lmax[i]) for i in range(info.n_levels - 1)]
                               if self.smoother == "chebyshev" else [])
        self.max_nrhs = cfg.max_nrhs
        self.coarse_lu = None  # the coarsest level is applied as a dense device inverse
        self.levels = [AmgLevel(self, i) for i in range(info.n_levels)]

    @property
    def n_levels(self) -> int:
        return len(self.level_sizes)

    @property
    def n(self) -> int:
        return self.level_sizes[0]

    def operator_complexity(self) -> float:
        nnz = [int(self._info.level_nnz[i]) for i in range(self.n_levels)]
        return sum(nnz) / max(nnz[0], 1)

    def matrix_memory_bytes(self) -> int:
        total = 0
        for i in range(self.n_levels):
            rows = self.level_sizes[i]
            total += _csr_bytes(rows, int(self._info.level_nnz[i]))
            if i < self.n_levels - 1:
                pn = int(self._info.prolong_nnz[i])
                total += _csr_bytes(rows, pn) + _csr_bytes(self.level_sizes[i + 1], pn)
        return total + self.level_sizes[-1] ** 2 * 8

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().spfd_amg_destroy(h)
            except Exception:
                pass
            self.handle = None


def _operator_of(a):
    op = getattr(a, "_spfd_op", None)
    if op is not None:
        return op
    from .fit_operators import PoissonSystem
    if isinstance(a, PoissonSystem):
        return a.operator
    return None


def amg_setup(a, cfg: SolveConfig | None = None) -> AmgHierarchy:
    """Build the smoothed-aggregation hierarchy on the GPU
    (linsolve.py:120-169).  Raises SolverError on a non-positive diagonal."""
    cfg = cfg or SolveConfig()
    _lib.require_cuda()
    lib = _lib.load()
    c = _lib.make_config(cfg)
    h = ctypes.c_void_p()
    op = _operator_of(a)
    if op is not None:
        _lib.check(lib.spfd_amg_setup_op(op.handle, ctypes.byref(c), _lib.stream_ptr(), ctypes.byref(h)))
        return AmgHierarchy(h, cfg, operator=op)
    m = sp.csr_matrix(a)
    if m.shape[0] != m.shape[1]:
        raise ValueError("matrix must be square")
    m.sum_duplicates()
    ip = torch.from_numpy(m.indptr.astype(np.int64)).cuda()
    ix = torch.from_numpy(m.indices.astype(np.int32)).cuda()
    dv = torch.from_numpy(m.data.astype(np.float64)).cuda()
    _lib.check(lib.spfd_amg_setup_csr(m.shape[0], m.nnz, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv),
                                      ctypes.byref(c), _lib.stream_ptr(), ctypes.byref(h)))
    return AmgHierarchy(h, cfg, fine_matrix=m)


def _as_planar(x, n):
    """-> (cuda (nrhs, n) tensor, was_numpy, squeeze)"""
    is_np = not isinstance(x, torch.Tensor)
    t = torch.as_tensor(np.asarray(x, dtype=np.float64)) if is_np else x
    squeeze = t.dim() == 1
    if squeeze:
        t = t.reshape(1, -1)
    if t.dim() != 2 or t.shape[1] != n or t.shape[0] not in (1, 2):
        raise ValueError(f"rhs has length {t.shape[-1] if t.dim() else 0}, expected {n}")
    return t.to(device="cuda", dtype=torch.float64).contiguous(), is_np, squeeze


def _back(t, is_np, squeeze):
    if squeeze:
        t = t[0]
    return t.cpu().numpy() if is_np else t


def v_cycle(hierarchy: AmgHierarchy, residual):
    """One V(pre, post) cycle (linsolve.py:179-197) on the GPU."""
    t, is_np, sq = _as_planar(residual, hierarchy.n)
    if t.shape[0] > hierarchy.max_nrhs:
        raise ValueError("more right-hand sides than the hierarchy was set up for")
    z = torch.empty_like(t)
    _lib.check(_lib.load().spfd_vcycle(hierarchy.handle, _lib.ptr(t), _lib.ptr(z), t.shape[0], _lib.stream_ptr()))
    return _back(z, is_np, sq)


def _solve(a, rhs, hierarchy: AmgHierarchy, cfg: SolveConfig, method: str):
    n = hierarchy.n
    if a is not None and tuple(a.shape) != (n, n):
        raise ValueError(f"matrix shape {tuple(a.shape)} does not match the hierarchy ({n})")
    shp = tuple(np.shape(rhs)) if not isinstance(rhs, torch.Tensor) else tuple(rhs.shape)
    if shp not in ((n,), (1, n), (2, n)):
        raise ValueError(f"rhs has length {shp[-1] if shp else 0}, expected {n}")
    b, is_np, sq = _as_planar(rhs, n)
    if b.shape[0] > hierarchy.max_nrhs:
        raise ValueError("more right-hand sides than the hierarchy was set up for")
    nrhs = b.shape[0]
    x = torch.empty_like(b)
    c = _lib.make_config(cfg, method=method)
    rep = _lib.Report()
    trace = None
    if cfg.trace is not None:
        trace = (ctypes.c_double * (cfg.max_iters * nrhs))()
    rc = _lib.load().spfd_solve(hierarchy.handle, _lib.ptr(b), _lib.ptr(x), nrhs, ctypes.byref(c),
                                ctypes.byref(rep), trace, _lib.stream_ptr())
    if rc == _lib.SPFD_ENONFINITE:
        raise SolverError("rhs contains non-finite values" if not torch.isfinite(b).all()
                          else "non-finite value in the Krylov iteration")
    _lib.check(rc)
    if trace is not None:
        for k in range(rep.iterations):
            est = max(trace[k * nrhs + c_] for c_ in range(nrhs))
            cfg.trace.write(f"iter {k + 1} rel_resid {est:.6e}\n")
    rels = tuple(float(rep.rel_residual[k]) for k in range(nrhs))
    vec_bytes = ((2 * cfg.restart + 1) if method == "fgmres" else 5) * n * 8 * nrhs
    report = SolveReport(
        iterations=int(rep.iterations),
        rel_residual=max(rels),
        converged=bool(rep.converged),
        setup_seconds=hierarchy.setup_seconds,
        solve_seconds=float(rep.solve_seconds),
        level_sizes=list(hierarchy.level_sizes),
        peak_matrix_memory_bytes=hierarchy.matrix_memory_bytes() + vec_bytes,
        threads=cfg.threads,
        rel_residuals=rels,
        method=method,
    )
    return _back(x, is_np, sq), report


def fgmres_solve(a, rhs, hierarchy: AmgHierarchy, cfg: SolveConfig | None = None):
    """Right-preconditioned FGMRES(m) with one V-cycle per iteration and
    true-residual restarts (linsolve.py:200-298).  Returns (x, SolveReport);
    `max_iters` is flagged in the report, non-finite input raises
    SolverError."""
    return _solve(a, rhs, hierarchy, cfg or SolveConfig(), "fgmres")


def pcg_solve(a, rhs, hierarchy: AmgHierarchy, cfg: SolveConfig | None = None):
    """AMG-preconditioned conjugate gradients (same report semantics)."""
    return _solve(a, rhs, hierarchy, cfg or SolveConfig(), "pcg")


def solve(a, rhs, hierarchy: AmgHierarchy, cfg: SolveConfig | None = None):
    """Dispatch on `cfg.method` (default PCG)."""
    cfg = cfg or SolveConfig()
    return _solve(a, rhs, hierarchy, cfg, cfg.method)
