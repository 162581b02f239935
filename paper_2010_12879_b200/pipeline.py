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
        # node planes holding conductive nodes: only their edges are ever read
        # (RHS and E-field touch edges of conductive nodes only), so the host
        # path copies just those edge ranges
        zc = np.flatnonzero(np.asarray(model.voxel_kappa(self.frequency_hz) > 0).any(axis=(0, 1)))
        self.plane_range = (int(zc[0]), int(zc[-1]) + 2) if zc.size else (0, 0)

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
        """Edge-index ranges this rank reads: x- and y-edges of its node planes
        (one GPU: the planes holding conductive nodes), z-edges of those
        planes and the one below."""
        nx, ny, nz = self.op.dims
        NX, NY = nx + 1, ny + 1
        kb, ke = self.plane_range
        if ke <= kb:
            return [(0, self.op.n_edges)]
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

    def snapshot(self, a, keep_psi: bool = False, stream=None, vox_out=None, cfg: SolveConfig | None = None):
        """One snapshot from device-resident edge potentials `a`
        ((nrhs, n_edges) CUDA float64).  Returns (voxel |E| (nrhs, n_vox)
        CUDA tensor, SolveReport, psi or None).  `cfg` overrides the
        session's solver settings (tolerance, method) for this call."""
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
        vbuf = self._vox
        if vox_out is not None:
            if vox_out.shape != self._vox.shape or not vox_out.is_cuda or vox_out.dtype != torch.float64:
                raise ValueError("vox_out must be a CUDA float64 tensor shaped like the voxel field buffer")
            vbuf = vox_out
        rep = _lib.Report()
        c = self._c if cfg is None else _lib.make_config(cfg)
        _lib.check(_lib.load().spfd_snapshot(self.op.handle, self.hierarchy.handle, _lib.ptr(a), self.omega,
                                             _lib.ptr(self._psi) if keep_psi else ctypes.c_void_p(0),
                                             _lib.ptr(vbuf), nrhs, ctypes.byref(c), ctypes.byref(rep),
                                             _lib.stream_ptr(stream)))
        rels = tuple(float(rep.rel_residual[k]) for k in range(nrhs))
        report = SolveReport(iterations=int(rep.iterations), rel_residual=max(rels), converged=bool(rep.converged),
                             setup_seconds=self.hierarchy.setup_seconds, solve_seconds=float(rep.solve_seconds),
                             level_sizes=list(self.hierarchy.level_sizes),
                             peak_matrix_memory_bytes=self.hierarchy.matrix_memory_bytes(), rel_residuals=rels,
                             method=(cfg or self.cfg).method)
        if not report.converged:
            raise PipelineError("solve", f"solver did not converge: residual {report.rel_residual:.3e} "
                                         f"after {report.iterations} iterations")
        vox = vbuf[:, :self.op.n_cond_voxels]
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
            for c in range(a_t.shape[0]):   # contiguous 1-D ranges (a 2-D column slice is strided)
                self._a_dev[c, e0:e1].copy_(a_t[c, e0:e1], non_blocking=nb)
        vox, rep, _ = self.snapshot(self._a_dev)
        v0, v1 = self.vox_range
        if out is None:
            out = torch.empty((vox.shape[0], v1 - v0), dtype=torch.float64, pin_memory=True)
        out.copy_(vox[:, v0:v1], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out.numpy(), rep

    def snapshots_host(self, inputs, outs=None):
        """A stream of snapshots from host memory (the real-time use case,
        BASELINE config C5), pipelined: the H2D copy of snapshot i+1 and the
        D2H copy of result i-1 run on copy streams while snapshot i solves.
        Every snapshot's potentials are copied in and its voxel field copied
        out.  `inputs`: sequence of (preferably pinned) CPU tensors (nrhs,
        n_edges); `outs`: optional sequence of pinned CPU tensors (nrhs,
        n_vox of this rank).  Returns (outs, reports)."""
        inputs = [a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
                  for a in inputs]
        inputs = [a.reshape(1, -1) if a.dim() == 1 else a for a in inputs]
        if not inputs:
            return [], []
        shape = tuple(inputs[0].shape)
        if any(tuple(a.shape) != shape for a in inputs):
            raise ValueError("all snapshots of a stream must have the same shape")
        v0, v1 = self.vox_range
        nrhs = shape[0]
        if outs is None:
            outs = [torch.empty((nrhs, v1 - v0), dtype=torch.float64, pin_memory=True) for _ in inputs]
        if self._vox is None or self._vox.shape[0] != nrhs:
            self._vox = torch.empty((nrhs, max(self.op.n_cond_voxels, 1)), dtype=torch.float64, device="cuda")
            self._psi = torch.empty((nrhs, max(self.op.n_dofs, 1)), dtype=torch.float64, device="cuda")
        if getattr(self, "_stream_bufs", None) is None or self._stream_bufs[0].shape != shape:
            self._stream_bufs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(2)]
            self._stream_vox = [torch.empty_like(self._vox) for _ in range(2)]
            self._h2d_stream = torch.cuda.Stream()
            self._d2h_stream = torch.cuda.Stream()
        bufs, voxb = self._stream_bufs, self._stream_vox
        hs, ds = self._h2d_stream, self._d2h_stream
        compute = torch.cuda.current_stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_out = [None, None]
        slices = self.edge_slices()

        def h2d(i):
            b = i % 2
            with torch.cuda.stream(hs):
                hs.wait_stream(compute)          # buffer b's previous snapshot is done with it
                for e0, e1 in slices:
                    for c in range(nrhs):
                        bufs[b][c, e0:e1].copy_(inputs[i][c, e0:e1], non_blocking=inputs[i].is_pinned())
                ev_in[b].record(hs)

        reports = []
        h2d(0)
        for i in range(len(inputs)):
            b = i % 2
            if i + 1 < len(inputs):
                h2d(i + 1)
            compute.wait_event(ev_in[b])
            if ev_out[b] is not None:
                compute.wait_event(ev_out[b])    # result i-2 has left voxb[b]
            _, rep, _ = self.snapshot(bufs[b], vox_out=voxb[b])
            reports.append(rep)
            with torch.cuda.stream(ds):
                ds.wait_stream(compute)
                outs[i].copy_(voxb[b][:, v0:v1], non_blocking=True)
                ev_out[b] = torch.cuda.Event()
                ev_out[b].record(ds)
        ds.synchronize()
        hs.synchronize()
        return outs, reports

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


# ---------------------------------------------------------------------------
# end-to-end pipeline (pipeline.py:46-195 of the reference) on the device
# ---------------------------------------------------------------------------

from dataclasses import dataclass, replace  # noqa: E402
from dataclasses import field as dataclass_field  # noqa: E402

STEP_NAMES = ("interpolate", "gauge", "assemble", "solve", "efield", "report")


@dataclass
class PipelineConfig:
    """Inputs and knobs for one exposure computation (pipeline.py:46-84).
    Exactly one field source (`field_path`, `coil`, `uniform_b`) and exactly
    one phantom (`phantom_path`, `model`)."""

    phantom_path: str | None = None
    model: object = None
    field_path: str | None = None
    coil: object = None
    uniform_b: tuple | None = None
    frequency_hz: float = 85e3
    solve: SolveConfig = dataclass_field(default_factory=SolveConfig)
    clean_fluxes: bool = True
    clean_tol: float = 1e-10
    gauge_tol: float = 1e-10
    tree_kind: str = "comb"
    coil_lattice_dims: tuple = (17, 17, 17)
    out_report: str | None = None
    out_field: str | None = None
    latency_budget_s: float = 5.0
    report_rms: bool = False

    def __post_init__(self):
        if not self.latency_budget_s > 0.0:
            raise ValueError("latency budget must be positive")
        if not self.frequency_hz > 0.0:
            raise ValueError("frequency must be positive")
        if sum(x is not None for x in (self.field_path, self.coil, self.uniform_b)) != 1:
            raise ValueError("exactly one of field_path, coil, uniform_b must be set")
        if (self.phantom_path is None) == (self.model is None):
            raise ValueError("exactly one of phantom_path, model must be set")


@dataclass
class PipelineTiming:
    """Per-stage seconds (device work synchronised at every stage end)."""

    interpolate: float = 0.0
    gauge: float = 0.0
    assemble: float = 0.0
    solve: float = 0.0
    efield: float = 0.0
    report: float = 0.0
    total: float = 0.0
    budget_met: bool = True

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name in STEP_NAMES}


def _load_inputs(cfg: PipelineConfig):
    from .field_source import Lattice, UniformField, sample_on_lattice
    from .fit_operators import StaggeredGrid
    from .formats import load_model, load_samples
    model = cfg.model if cfg.model is not None else load_model(cfg.phantom_path)
    grid = StaggeredGrid.from_model(model)
    if cfg.field_path is not None:
        samples = load_samples(cfg.field_path)
    elif cfg.uniform_b is not None:
        samples = sample_on_lattice(UniformField(cfg.uniform_b), Lattice.covering(grid, (2, 2, 2)), cfg.frequency_hz)
    else:
        samples = sample_on_lattice(cfg.coil, Lattice.covering(grid, cfg.coil_lattice_dims), cfg.frequency_hz)
    return model, grid, samples


class _Stage:
    def __init__(self, timing: PipelineTiming, step: str):
        self.timing, self.step = timing, step

    def __enter__(self):
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, exc_type, exc, tb):
        if exc is None:
            torch.cuda.synchronize()
        setattr(self.timing, self.step, time.perf_counter() - self.t0)
        if exc is not None and not isinstance(exc, PipelineError):
            from .errors import SpfdError
            if isinstance(exc, (SpfdError, ValueError, OSError)):
                raise PipelineError(self.step, str(exc)) from exc
        return False


class PipelineState:
    """Device state a repeated pipeline reuses: the operator of the phantom
    and its AMG hierarchy (the reference hoists only the hierarchy,
    pipeline.py:277-288; the operator depends on phantom and frequency only)."""

    def __init__(self, model, frequency_hz: float, cfg: SolveConfig):
        self.op = DeviceOperator(model, frequency_hz, pin=True)
        self.hierarchy = amg_setup(_OpRef(self.op), replace(cfg, max_nrhs=1))
        self.vox_index = self.op.export(_lib.EXPORT_VOXEL_INDICES)


def run_pipeline(cfg: PipelineConfig, *, _hierarchy=None, _state: PipelineState | None = None):
    """Execute the full chain on the device; returns (ExposureReport,
    PipelineTiming) like pipeline.py:158-195.  Stage failures are re-raised
    as PipelineError carrying the stage name."""
    from .dosimetry import build_exposure_report
    from .errors import SpfdError
    from .field_source import field_ops
    from .formats import write_field_dump, write_report
    from .gauging import build_tree
    from .linsolve import solve as _solve
    try:
        model, grid, samples = _load_inputs(cfg)
    except (SpfdError, ValueError, OSError) as exc:
        raise PipelineError("load", str(exc)) from exc
    timing = PipelineTiming()
    ops = field_ops(grid, cfg.solve)
    with _Stage(timing, "interpolate"):
        flux = ops.interpolate(samples.lattice, samples.b)
        if cfg.clean_fluxes:
            flux = ops.clean(flux, cfg.clean_tol)
    with _Stage(timing, "gauge"):
        tree = build_tree(grid, cfg.tree_kind)
        a = ops.gauge(flux, cfg.gauge_tol, tree=tree.kind)
    with _Stage(timing, "assemble"):
        state = _state if _state is not None else PipelineState(model, cfg.frequency_hz, cfg.solve)
        rhs = state.op.rhs(a)
    with _Stage(timing, "solve"):
        h = _hierarchy if _hierarchy is not None else state.hierarchy
        psi, rep = _solve(None, rhs, h, cfg.solve)
        if not rep.converged:
            raise PipelineError("solve", f"solver did not converge: residual {rep.rel_residual:.3e} "
                                         f"after {rep.iterations} iterations")
    with _Stage(timing, "efield"):
        omega = 2.0 * math.pi * cfg.frequency_hz
        vox = state.op.efield_voxavg(a, psi, omega)[0]
    with _Stage(timing, "report"):
        report = build_exposure_report(vox, state.vox_index, model, cfg.frequency_hz, dof_count=state.op.n_dofs,
                                       solver=rep, rms=cfg.report_rms, rel_tol=cfg.solve.rel_tol)
        if cfg.out_report:
            write_report(report, cfg.out_report)
        if cfg.out_field:
            write_field_dump(model, report.voxel_field, report.voxel_indices, cfg.out_field)
    timing.total = sum(timing.as_dict().values())
    timing.budget_met = timing.total <= cfg.latency_budget_s
    return report, timing


@dataclass(frozen=True)
class StepStats:
    mean: float
    stddev: float
    min: float
    max: float


def summarize_runs(samples: dict) -> dict:
    """Per-step mean / sample stddev (n-1) / min / max (pipeline.py:209-222)."""
    out = {}
    for step, values in samples.items():
        arr = np.asarray(values, dtype=np.float64)
        if arr.size < 2:
            raise ValueError(f"step '{step}' needs at least 2 runs, got {arr.size}")
        out[step] = StepStats(float(arr.mean()), float(arr.std(ddof=1)), float(arr.min()), float(arr.max()))
    return out


@dataclass
class BenchmarkResult:
    steps: dict
    runs: int
    setup_seconds: float
    iterations: list
    report: object = None

    def to_csv(self) -> str:
        rows = ["step,mean_s,stddev_s,min_s,max_s"]
        for name in (*STEP_NAMES, "total"):
            s = self.steps[name]
            rows.append(f"{name},{s.mean:.9f},{s.stddev:.9f},{s.min:.9f},{s.max:.9f}")
        return "\n".join(rows) + "\n"

    def to_text(self) -> str:
        w = max(len(n) for n in (*STEP_NAMES, "total"))
        rows = [f"{'step':<{w}}  {'mean [s]':>12}  {'stddev [s]':>12}  {'min [s]':>12}  {'max [s]':>12}"]
        for name in (*STEP_NAMES, "total"):
            s = self.steps[name]
            rows.append(f"{name:<{w}}  {s.mean:>12.6f}  {s.stddev:>12.6f}  {s.min:>12.6f}  {s.max:>12.6f}")
        rows.append(f"amg setup (once): {self.setup_seconds:.6f} s")
        rows.append(f"solver iterations per run: {self.iterations}")
        return "\n".join(rows)


def run_benchmark(cfg: PipelineConfig, runs: int = 5, timings_override: dict | None = None):
    """Repeat the timed stages `runs` times on identical inputs with the
    operator and hierarchy built once up front (pipeline.py:256-306)."""
    if runs < 2:
        raise ValueError("need at least 2 runs for a sample standard deviation")
    if timings_override is not None:
        samples = dict(timings_override)
        if "total" not in samples:
            n = len(next(iter(samples.values())))
            samples["total"] = [sum(samples[s][i] for s in samples if s != "total") for i in range(n)]
        return BenchmarkResult(summarize_runs(samples), runs, 0.0, [])
    bench_cfg = replace(cfg, out_report=None, out_field=None)
    model, _, _ = _load_inputs(bench_cfg)
    in_memory = replace(bench_cfg, model=model, phantom_path=None)
    t0 = time.perf_counter()
    state = PipelineState(model, cfg.frequency_hz, cfg.solve)
    torch.cuda.synchronize()
    setup_seconds = time.perf_counter() - t0
    run_pipeline(in_memory, _state=state)          # warm-up (cleaning hierarchy, caches)
    samples: dict = {name: [] for name in (*STEP_NAMES, "total")}
    iterations = []
    report = None
    for _ in range(runs):
        report, timing = run_pipeline(in_memory, _state=state)
        for name in STEP_NAMES:
            samples[name].append(getattr(timing, name))
        samples["total"].append(timing.total)
        iterations.append(report.solver.iterations)
    return BenchmarkResult(summarize_runs(samples), runs, setup_seconds, iterations, report)
