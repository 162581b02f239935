"""Electric field reconstruction and voxel averaging on the GPU.

Drop-in for /root/reference/pkg/src/spfd/dosimetry.py:27-116
(`edge_voltages`, `node_field_strength`, `voxel_average`, `corner_mean`);
every stage is bit-identical to the reference.  `efield_voxel_average` is
the fused device path used by the pipeline: vector potential + solved
potential -> voxel |E| without materialising edge voltages or the node box.
Inputs may be numpy arrays (numpy is returned) or CUDA tensors (tensors are
returned); a leading axis of 2 carries real/imaginary parts.
"""

from __future__ import annotations

import weakref

import numpy as np
import torch

from .fit_operators import DeviceOperator, PoissonSystem, StaggeredGrid

_OP_CACHE: dict = {}


def _operator_for(model, frequency_hz, system=None) -> DeviceOperator:
    if system is not None:
        return system.operator
    # models are frozen dataclasses holding arrays (unhashable): key by id
    # and keep a weak reference to detect reuse of the id after collection
    key = (id(model), float(frequency_hz))
    hit = _OP_CACHE.get(key)
    if hit is not None and hit[0]() is model:
        return hit[1]
    op = DeviceOperator(model, frequency_hz, pin=True)
    try:
        _OP_CACHE[key] = (weakref.ref(model), op)
    except TypeError:
        pass
    return op


def _ret(t, like_numpy, squeeze):
    if squeeze:
        t = t[0]
    return t.cpu().numpy() if like_numpy else t


def _is_np(x):
    return not isinstance(x, torch.Tensor)


def edge_voltages(vector_potential, potential_reduced, system: PoissonSystem, omega: float):
    """omega * (a + grad psi) on every edge (dosimetry.py:27-47)."""
    grid = system.grid
    shp = tuple(np.shape(vector_potential))
    if shp[-1:] != (grid.n_edges,):
        raise ValueError(f"vector potential has length {shp[-1] if shp else 0}, expected {grid.n_edges}")
    squeeze = len(shp) == 1
    out = system.operator.edge_voltages(vector_potential, potential_reduced, omega)
    return _ret(out, _is_np(vector_potential), squeeze)


def node_field_strength(voltages, grid: StaggeredGrid, model, frequency_hz: float, system=None):
    """Per-node |E| (dosimetry.py:50-85), shape node_dims (or (2, *node_dims))."""
    shp = tuple(np.shape(voltages))
    if shp[-1:] != (grid.n_edges,):
        raise ValueError(f"edge voltages have length {shp[-1] if shp else 0}, expected {grid.n_edges}")
    op = _operator_for(model, frequency_hz, system)
    out = op.node_field(voltages)
    nd = grid.node_dims
    if _is_np(voltages):
        arr = out.cpu().numpy()
        arr = np.stack([a.reshape(nd, order="F") for a in arr])
        return arr[0] if len(shp) == 1 else arr
    return out[0] if len(shp) == 1 else out


def voxel_average(node_field, grid: StaggeredGrid, model, frequency_hz: float, system=None):
    """Eight-corner mean on conductive voxels (dosimetry.py:88-104).
    Returns (values, x-fastest voxel indices)."""
    op = _operator_for(model, frequency_hz, system)
    is_np = _is_np(node_field)
    if is_np:
        nf = np.asarray(node_field, dtype=np.float64)
        batched = nf.ndim == 4 or (nf.ndim == 2 and nf.shape[0] == 2)
        if nf.ndim == 4:
            flat = np.stack([a.ravel(order="F") for a in nf])
        elif nf.ndim == 3:
            flat = nf.ravel(order="F")[None]
        else:
            flat = nf.reshape(-1, grid.n_nodes)
        vals = op.voxel_average(flat)
    else:
        batched = node_field.dim() == 2 and node_field.shape[0] == 2
        vals = op.voxel_average(node_field.reshape(-1, grid.n_nodes))
    idx = op.export(4)
    out = vals if batched else vals[0]
    if is_np:
        return out.cpu().numpy(), idx.cpu().numpy()
    return out, idx


def corner_mean(node_field: np.ndarray) -> np.ndarray:
    """Eight-corner mean of a node array, one value per voxel
    (dosimetry.py:107-116).  Host helper with the reference's summation order."""
    acc = np.zeros(tuple(n - 1 for n in node_field.shape), dtype=np.float64)
    for di in (0, 1):
        for dj in (0, 1):
            for dk in (0, 1):
                acc += node_field[di:di + acc.shape[0], dj:dj + acc.shape[1], dk:dk + acc.shape[2]]
    return acc * 0.125


def efield_voxel_average(system: PoissonSystem, vector_potential, potential_reduced, omega: float):
    """Fused device chain a, psi -> voxel-averaged |E| (per rhs); equals
    voxel_average(node_field_strength(edge_voltages(...)))."""
    shp = tuple(np.shape(vector_potential))
    squeeze = len(shp) == 1
    out = system.operator.efield_voxavg(vector_potential, potential_reduced, omega)
    return _ret(out, _is_np(vector_potential), squeeze)


# ---------------------------------------------------------------------------
# exposure statistics (dosimetry.py:119-234)
# ---------------------------------------------------------------------------

import ctypes  # noqa: E402
import math  # noqa: E402
from dataclasses import dataclass  # noqa: E402
from dataclasses import field as dataclass_field  # noqa: E402

from . import _lib  # noqa: E402

RMS_FACTOR = 1.0 / math.sqrt(2.0)
FREE_SPACE_ID = 0


def _stats(values, scale, vox_index, ids_box, n_ids):
    """Device statistics: (scaled values, counts, means, maxima, p99s, (p99, max))."""
    v = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(values, np.float64))
    v = v.to(device="cuda", dtype=torch.float64).contiguous()
    n = v.numel()
    if n == 0:
        raise ValueError("percentile of an empty array")
    scaled = torch.empty_like(v)
    cnt = np.zeros(n_ids, np.int64)
    mean = np.zeros(n_ids)
    mx = np.zeros(n_ids)
    p99 = np.zeros(n_ids)
    glob = np.zeros(2)
    f64p = ctypes.POINTER(ctypes.c_double)
    _lib.check(_lib.load().spfd_exposure_stats(
        _lib.ptr(v), n, float(scale), _lib.ptr(vox_index), _lib.ptr(ids_box), int(n_ids), _lib.ptr(scaled),
        cnt.ctypes.data_as(ctypes.c_void_p), mean.ctypes.data_as(f64p), mx.ctypes.data_as(f64p),
        p99.ctypes.data_as(f64p), glob.ctypes.data_as(f64p), _lib.stream_ptr()))
    return scaled, cnt, mean, mx, p99, glob


def percentile99(values) -> float:
    """Nearest-rank 99th percentile: sorted element at index ceil(0.99 n) - 1
    (dosimetry.py:119-127), by a device radix sort."""
    _lib.require_cuda()
    n = int(np.prod(np.shape(values)))
    if n == 0:
        raise ValueError("percentile of an empty array")
    zeros = torch.zeros(n, dtype=torch.int64, device="cuda")
    ids = torch.zeros(1, dtype=torch.int16, device="cuda")
    vals = values.reshape(-1) if isinstance(values, torch.Tensor) else np.asarray(values, np.float64).ravel()
    return float(_stats(vals, 1.0, zeros, ids, 1)[5][0])


def scale_reference_field(e, frequency_hz: float, ref_frequency_hz: float, kappa: float, ref_kappa: float):
    """(f / f_ref) * (kappa(f_ref) / kappa(f)) * e (dosimetry.py:130-146)."""
    for name, v in (("frequency_hz", frequency_hz), ("ref_frequency_hz", ref_frequency_hz), ("kappa", kappa),
                    ("ref_kappa", ref_kappa)):
        if not float(v) > 0.0:
            raise ValueError(f"{name} must be positive, got {v}")
    factor = (frequency_hz / ref_frequency_hz) * (ref_kappa / kappa)
    return e * factor


@dataclass(frozen=True)
class TissueStats:
    name: str
    count: int
    mean: float
    max: float
    p99: float


@dataclass
class ExposureReport:
    """Voxel-averaged |E| statistics over the conductive voxels (dosimetry.py:158-176)."""

    frequency_hz: float
    voxel_field: object         # V/m per conductive voxel (numpy or CUDA tensor)
    voxel_indices: object       # x-fastest voxel linear indices
    percentile99_vpm: float
    max_vpm: float
    per_tissue: dict            # tissue ID -> TissueStats
    dof_count: int
    solver: object = None
    rms: bool = False
    rel_tol: float | None = None
    extra: dict = dataclass_field(default_factory=dict)

    @property
    def n_voxels(self) -> int:
        return int(self.voxel_field.numel() if isinstance(self.voxel_field, torch.Tensor) else self.voxel_field.size)


@dataclass(frozen=True)
class LimitCheck:
    passed: bool
    margin: float


def check_limits(report: ExposureReport, limit_vpm: float) -> LimitCheck:
    """Compare the 99th percentile against a limit, inclusive (dosimetry.py:185-192)."""
    if not limit_vpm > 0.0:
        raise ValueError("limit must be positive")
    p99 = report.percentile99_vpm
    if p99 == 0.0:
        return LimitCheck(True, math.inf)
    return LimitCheck(p99 <= limit_vpm, limit_vpm / p99)


def _ids_box(model):
    from .voxel_model import ids_fortran_flat
    cache = getattr(model, "_spfd_ids_dev", None)
    if cache is None:
        cache = torch.from_numpy(ids_fortran_flat(model).view(np.int16)).cuda()
        try:
            object.__setattr__(model, "_spfd_ids_dev", cache)
        except Exception:
            pass
    return cache


def build_exposure_report(voxel_values, voxel_indices, model, frequency_hz: float, *, dof_count: int, solver=None,
                          rms: bool = False, rel_tol: float | None = None) -> ExposureReport:
    """Exposure statistics on the device (dosimetry.py:195-234): optional RMS
    scaling, global nearest-rank p99 and max, per-tissue count / mean / max /
    p99 (free space excluded).  p99 and max are exact selections; the mean
    is a deterministic device sum (≈1e-16 relative to numpy's pairwise sum)."""
    _lib.require_cuda()
    as_np = not isinstance(voxel_values, torch.Tensor)
    idx = voxel_indices if isinstance(voxel_indices, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(voxel_indices, np.int64))
    idx = idx.to(device="cuda", dtype=torch.int64).contiguous()
    n = idx.numel()
    if n == 0:
        empty = np.zeros(0) if as_np else torch.zeros(0, dtype=torch.float64, device="cuda")
        return ExposureReport(float(frequency_hz), empty, voxel_indices, 0.0, 0.0, {}, int(dof_count), solver, rms,
                              rel_tol)
    n_ids = int(max(model.tissue_table)) + 1
    scaled, cnt, mean, mx, p99, glob = _stats(voxel_values, RMS_FACTOR if rms else 1.0, idx, _ids_box(model), n_ids)
    per_tissue = {}
    for tid in np.flatnonzero(cnt):
        tid = int(tid)
        if tid == FREE_SPACE_ID:
            continue
        per_tissue[tid] = TissueStats(name=model.tissue_table[tid].name, count=int(cnt[tid]), mean=float(mean[tid]),
                                      max=float(mx[tid]), p99=float(p99[tid]))
    return ExposureReport(
        frequency_hz=float(frequency_hz),
        voxel_field=scaled.cpu().numpy() if as_np else scaled,
        voxel_indices=voxel_indices,
        percentile99_vpm=float(glob[0]),
        max_vpm=float(glob[1]),
        per_tissue=per_tissue,
        dof_count=int(dof_count),
        solver=solver,
        rms=rms,
        rel_tol=rel_tol,
    )
