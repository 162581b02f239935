"""Device-resident snapshot pipeline: assemble -> solve -> E-field.

Mirrors the hot stages of `run_pipeline` (/root/reference/pkg/src/spfd/
pipeline.py:158-175) and its setup-reuse seam (`_hierarchy`,
pipeline.py:136,162; `run_benchmark` hoisting, :277-288).  A `Session`
keeps the operator and AMG hierarchy resident on the GPU; each snapshot is
one C-ABI call (`spfd_snapshot`): RHS assembly, the Krylov solve and the
fused E-field / voxel average, with the real and imaginary parts batched.
Non-convergence raises PipelineError("solve") like the reference.
"""

from __future__ import annotations

import ctypes
import math
import time

import numpy as np
import torch

from . import _lib
from .errors import PipelineError
from .fit_operators import DeviceOperator
from .linsolve import AmgHierarchy, SolveConfig, SolveReport, amg_setup


class Session:
    """Operator + hierarchy for one (phantom, frequency), reused across
    snapshots (C5 of BASELINE.json)."""

    def __init__(self, model, frequency_hz: float, cfg: SolveConfig | None = None):
        self.cfg = cfg or SolveConfig(rel_tol=1e-8)
        self.frequency_hz = float(frequency_hz)
        self.omega = 2.0 * math.pi * self.frequency_hz
        t0 = time.perf_counter()
        self.op = DeviceOperator(model, frequency_hz, pin=True)
        self.assemble_seconds = time.perf_counter() - t0
        from .fit_operators import StencilMatrix  # noqa: F401
        self.hierarchy: AmgHierarchy = amg_setup(_OpRef(self.op), self.cfg)
        self._c = _lib.make_config(self.cfg)
        self._vox = None
        self._psi = None
        self._a_dev = None
        self.comm = None
        self.dof_range = (0, self.op.n_dofs)
        self.vox_range = (0, self.op.n_cond_voxels)

    def distribute(self, comm, replicate_below: int = 100_000):
        """Split the solve into z-slabs over `comm` (a distributed.Communicator):
        this rank then computes only its planes; `dof_range` / `vox_range`
        give the slices of psi / voxel |E| it produces."""
        rng = (ctypes.c_int64 * 6)()
        _lib.check(_lib.load().spfd_amg_distribute(self.hierarchy.handle, comm.handle, int(replicate_below), rng,
                                                   _lib.stream_ptr()))
        self.comm = comm
        self.dof_range = (int(rng[0]), int(rng[1]))
        self.vox_range = (int(rng[2]), int(rng[3]))
        self.plane_range = (int(rng[4]), int(rng[5]))
        return self

    def edge_slices(self):
        """Edge-index ranges this rank reads (all edges on one GPU): x- and
        y-edges of its node planes, z-edges of its planes and the one below."""
        nx, ny, nz = self.op.dims
        NX, NY = nx + 1, ny + 1
        if self.comm is None:
            return [(0, self.op.n_edges)]
        kb, ke = self.plane_range
        ex, ey = nx * NY * (nz + 1), NX * ny * (nz + 1)
        return [(nx * NY * kb, nx * NY * ke),
                (ex + NX * ny * kb, ex + NX * ny * ke),
                (ex + ey + NX * NY * max(kb - 1, 0), ex + ey + NX * NY * min(ke, nz))]

    @property
    def n_dofs(self) -> int:
        return self.op.n_dofs

    @property
    def n_cond_voxels(self) -> int:
        return self.op.n_cond_voxels

    def voxel_indices(self):
        return self.op.export(_lib.EXPORT_VOXEL_INDICES)

    def snapshot(self, a, keep_psi: bool = False, stream=None):
        """One snapshot from device-resident edge potentials `a`
        ((nrhs, n_edges) CUDA float64).  Returns (voxel |E| (nrhs, n_vox)
        CUDA tensor, SolveReport, psi or None)."""
        if not (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.float64):
            raise ValueError("snapshot() takes a CUDA float64 tensor; use snapshot_host() for numpy input")
        if a.dim() == 1:
            a = a.reshape(1, -1)
        nrhs = a.shape[0]
        if a.shape[1] != self.op.n_edges or nrhs not in (1, 2):
            raise ValueError(f"expected (nrhs<=2, {self.op.n_edges}) edge potentials, got {tuple(a.shape)}")
        a = a.contiguous()
        if self._vox is None or self._vox.shape[0] != nrhs:
            self._vox = torch.empty((nrhs, max(self.op.n_cond_voxels, 1)), dtype=torch.float64, device="cuda")
            self._psi = torch.empty((nrhs, max(self.op.n_dofs, 1)), dtype=torch.float64, device="cuda")
        rep = _lib.Report()
        _lib.check(_lib.load().spfd_snapshot(self.op.handle, self.hierarchy.handle, _lib.ptr(a), self.omega,
                                             _lib.ptr(self._psi) if keep_psi else ctypes.c_void_p(0),
                                             _lib.ptr(self._vox), nrhs, ctypes.byref(self._c), ctypes.byref(rep),
                                             _lib.stream_ptr(stream)))
        rels = tuple(float(rep.rel_residual[k]) for k in range(nrhs))
        report = SolveReport(iterations=int(rep.iterations), rel_residual=max(rels), converged=bool(rep.converged),
                             setup_seconds=self.hierarchy.setup_seconds, solve_seconds=float(rep.solve_seconds),
                             level_sizes=list(self.hierarchy.level_sizes),
                             peak_matrix_memory_bytes=self.hierarchy.matrix_memory_bytes(), rel_residuals=rels,
                             method=self.cfg.method)
        if not report.converged:
            raise PipelineError("solve", f"solver did not converge: residual {report.rel_residual:.3e} "
                                         f"after {report.iterations} iterations")
        vox = self._vox[:, :self.op.n_cond_voxels]
        psi = self._psi[:, :self.op.n_dofs] if keep_psi else None
        return vox, report, psi

    def snapshot_host(self, a_host, out=None):
        """End-to-end from host memory: H2D of the potentials, snapshot,
        D2H of the voxel field.  `a_host` is a numpy array or a (preferably
        pinned) CPU tensor; `out` an optional pinned CPU tensor
        (nrhs, n_vox) that receives the result.  Returns (numpy, report)."""
        a_t = a_host if isinstance(a_host, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(a_host, dtype=np.float64))
        if a_t.dim() == 1:
            a_t = a_t.reshape(1, -1)
        if self._a_dev is None or self._a_dev.shape != a_t.shape:
            self._a_dev = torch.empty(a_t.shape, dtype=torch.float64, device="cuda")
        nb = a_t.is_pinned()
        for e0, e1 in self.edge_slices():   # only the edges this rank's slab reads
            self._a_dev[:, e0:e1].copy_(a_t[:, e0:e1], non_blocking=nb)
        vox, rep, _ = self.snapshot(self._a_dev)
        v0, v1 = self.vox_range
        if out is None:
            out = torch.empty((vox.shape[0], v1 - v0), dtype=torch.float64, pin_memory=True)
        out.copy_(vox[:, v0:v1], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out.numpy(), rep

    def host_bytes(self, nrhs: int):
        """(H2D, D2H) bytes per snapshot_host call on this rank."""
        h2d = sum(e1 - e0 for e0, e1 in self.edge_slices()) * 8 * nrhs
        return h2d, (self.vox_range[1] - self.vox_range[0]) * 8 * nrhs


class _OpRef:
    """Minimal matrix-like object carrying the operator (selects the
    structured amg_setup path without materialising the host CSR)."""

    def __init__(self, op: DeviceOperator):
        self._spfd_op = op
        self.shape = (op.n_dofs, op.n_dofs)
