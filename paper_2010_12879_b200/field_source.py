"""Flux-density sources, face-flux interpolation and divergence cleaning on
the GPU.

Drop-in for /root/reference/pkg/src/spfd/field_source.py:31-329: the same
classes (`Lattice`, `FieldSampleSet`, `CoilSpec`, `UniformField`) and
functions (`coil_field`, `sample_on_lattice`, `interpolate_to_faces`,
`divergence_clean`).  The compute runs in libspfd_b200.so:

* `coil_field`: Biot-Savart per lattice point (k_coil_field);
* `interpolate_to_faces`: trilinear midpoint fluxes, bit-identical to the
  reference (k_interp_faces);
* `divergence_clean`: cell divergence (bit-identical), then the l2-minimal
  projection with the hot path's own AMG + Krylov solver on div divᵀ (the
  hierarchy is built once per grid and kept).

numpy in -> numpy out; CUDA tensors in -> CUDA tensors out.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import LatticeError
from .fit_operators import StaggeredGrid
from .linsolve import SolveConfig

MU_0 = 4e-7 * np.pi  # vacuum permeability (T*m/A)

_WIRE_EPS = 1e-12  # evaluation closer than this to a wire segment is singular


@dataclass(frozen=True)
class Lattice:
    """Regular Cartesian sampling lattice (field_source.py:31-73)."""

    origin: tuple
    spacing: tuple
    dims: tuple

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        spacing = tuple(float(s) for s in self.spacing)
        origin = tuple(float(o) for o in self.origin)
        if any(n < 1 for n in dims):
            raise ValueError(f"lattice dims must be >= 1, got {dims}")
        if any(not s > 0.0 for s in spacing):
            raise ValueError(f"lattice spacing must be positive, got {spacing}")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "origin", origin)

    @property
    def n_points(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def points(self) -> np.ndarray:
        """All lattice points, x-fastest, shape (n_points, 3)."""
        axes = [self.origin[a] + np.arange(self.dims[a]) * self.spacing[a] for a in range(3)]
        i, j, k = np.meshgrid(axes[0], axes[1], axes[2], indexing="ij")
        return np.stack([i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")], axis=1)

    @classmethod
    def covering(cls, grid: StaggeredGrid, dims=(2, 2, 2)) -> "Lattice":
        """Lattice spanning the grid bounding box with the given point counts."""
        dims = tuple(int(n) for n in dims)
        extent = [grid.dims[a] * grid.spacing[a] for a in range(3)]
        spacing = tuple(extent[a] / (dims[a] - 1) if dims[a] > 1 else max(extent[a], 1.0) for a in range(3))
        return cls(grid.origin, spacing, dims)

    def box(self):
        return _lib.make_box(self.dims, self.spacing, self.origin)


@dataclass(frozen=True)
class FieldSampleSet:
    """Single-phase flux density amplitudes sampled on a regular lattice
    (field_source.py:76-106).  `b` may be a numpy array or a CUDA tensor."""

    frequency_hz: float
    lattice: Lattice
    positions: np.ndarray  # (n, 3) meters
    b: object              # (n, 3) tesla

    def __post_init__(self):
        pos = np.asarray(self.positions, dtype=np.float64)
        b = self.b if isinstance(self.b, torch.Tensor) else np.asarray(self.b, dtype=np.float64)
        n = self.lattice.n_points
        if pos.shape != (n, 3) or tuple(b.shape) != (n, 3):
            raise LatticeError(f"sample count mismatch: lattice has {n} points, "
                               f"got {pos.shape[0]} positions / {b.shape[0]} values")
        if not float(self.frequency_hz) > 0.0:
            raise ValueError("frequency must be positive")
        expected = self.lattice.points()
        if pos.size and np.max(np.abs(pos - expected)) > 1e-9:
            raise LatticeError("sample positions do not lie on the declared lattice")
        pos.flags.writeable = False
        if isinstance(b, np.ndarray):
            b.flags.writeable = False
        object.__setattr__(self, "positions", pos)
        object.__setattr__(self, "b", b)
        object.__setattr__(self, "frequency_hz", float(self.frequency_hz))

    def component_grid(self, comp: int):
        b = self.b if isinstance(self.b, np.ndarray) else self.b.cpu().numpy()
        return b[:, comp].reshape(self.lattice.dims, order="F")


@dataclass(frozen=True)
class CoilSpec:
    """Circular loop approximated by straight segments (field_source.py:109-152)."""

    center: tuple
    axis: tuple
    radius_m: float
    current_a: float
    segments: int = 256

    def __post_init__(self):
        center = tuple(float(c) for c in self.center)
        axis = np.asarray(self.axis, dtype=np.float64)
        norm = float(np.linalg.norm(axis))
        if norm == 0.0:
            raise ValueError("coil axis must be a nonzero vector")
        if not self.radius_m > 0.0:
            raise ValueError("coil radius must be positive")
        if self.segments < 8:
            raise ValueError("need at least 8 segments")
        object.__setattr__(self, "center", center)
        object.__setattr__(self, "axis", tuple(axis / norm))
        object.__setattr__(self, "radius_m", float(self.radius_m))
        object.__setattr__(self, "current_a", float(self.current_a))
        object.__setattr__(self, "segments", int(self.segments))

    def vertices(self) -> np.ndarray:
        """Closed polygon vertices, shape (segments + 1, 3)."""
        n = np.asarray(self.axis)
        ref = np.array([0.0, 0.0, 1.0])
        if abs(float(n @ ref)) > 0.9:
            ref = np.array([1.0, 0.0, 0.0])
        u = np.cross(n, ref)
        u /= np.linalg.norm(u)
        v = np.cross(n, u)
        theta = 2.0 * np.pi * np.arange(self.segments + 1) / self.segments
        return np.asarray(self.center) + self.radius_m * (np.cos(theta)[:, None] * u + np.sin(theta)[:, None] * v)


@dataclass(frozen=True)
class UniformField:
    """Spatially constant flux density amplitude."""

    b: tuple

    def __post_init__(self):
        object.__setattr__(self, "b", tuple(float(c) for c in self.b))


def _dev(x):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.require(x, np.float64, ["C", "W"])).cuda()


def coil_field(coil: CoilSpec, points, chunk: int = 16384):
    """Biot-Savart flux density of the polygonized loop (field_source.py:163-197).
    Accepts (3,) or (n, 3); raises SingularPointError on the wire."""
    _lib.require_cuda()
    as_np = not isinstance(points, torch.Tensor)
    pts = _dev(points)
    single = pts.dim() == 1
    pts = pts.reshape(-1, pts.shape[-1]) if pts.dim() else pts
    if pts.dim() != 2 or pts.shape[1] != 3:
        raise ValueError("points must have shape (3,) or (n, 3)")
    verts = _dev(coil.vertices())
    out = torch.empty_like(pts)
    scale = MU_0 * coil.current_a / (4.0 * np.pi)
    _lib.check(_lib.load().spfd_coil_field(pts.shape[0], _lib.ptr(pts), coil.segments, _lib.ptr(verts), scale,
                                           _lib.ptr(out), _lib.stream_ptr()))
    out = out[0] if single else out
    return out.cpu().numpy() if as_np else out


def _evaluate_source(source, points):
    if isinstance(source, CoilSpec):
        return coil_field(source, points)
    if isinstance(source, UniformField):
        return np.broadcast_to(np.asarray(source.b), (points.shape[0], 3)).copy()
    raise TypeError(f"unsupported field source {type(source).__name__}")


def sample_on_lattice(source, lattice: Lattice, frequency_hz: float) -> FieldSampleSet:
    """Evaluate a synthetic source at every lattice point (field_source.py:208-212)."""
    points = lattice.points()
    return FieldSampleSet(frequency_hz, lattice, points, _evaluate_source(source, points))


# ---------------------------------------------------------------------------
# device handle per grid (workspace + the cleaning hierarchy)
# ---------------------------------------------------------------------------

def _cfg_key(cfg: SolveConfig):
    return (cfg.max_iters, cfg.restart, cfg.pre_sweeps, cfg.post_sweeps, cfg.jacobi_damping, cfg.strength_threshold,
            cfg.coarse_cap, cfg.max_levels, cfg.method, cfg.smoother, cfg.chebyshev_degree)


class FieldOps:
    """libspfd_b200 field handle for one grid: interpolation, divergence,
    cleaning (AMG on div divᵀ built on first use and kept), comb gauging."""

    def __init__(self, grid: StaggeredGrid, cfg: SolveConfig | None = None):
        _lib.require_cuda()
        self._lib = _lib.load()
        self.grid = grid
        self.cfg = cfg or SolveConfig()
        self._c = _lib.make_config(self.cfg, max_nrhs=1)
        self._box = grid.box()
        h = ctypes.c_void_p()
        _lib.check(self._lib.spfd_field_create(ctypes.byref(self._box), ctypes.byref(self._c), ctypes.byref(h)))
        self.handle = h
        self.last_clean = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                self._lib.spfd_field_destroy(h)
            except Exception:
                pass
            self.handle = None

    def interpolate(self, lattice: Lattice, b, out=None, stream=None):
        b = _dev(b)
        if tuple(b.shape) != (lattice.n_points, 3):
            raise LatticeError(f"sample count mismatch: lattice has {lattice.n_points} points, got {tuple(b.shape)}")
        out = torch.empty(self.grid.n_faces, dtype=torch.float64, device="cuda") if out is None else out
        box = lattice.box()
        _lib.check(self._lib.spfd_field_interpolate(self.handle, ctypes.byref(box), _lib.ptr(b), _lib.ptr(out),
                                                    _lib.stream_ptr(stream)))
        return out

    def divergence(self, flux, out=None, stream=None):
        flux = _dev(flux)
        out = torch.empty(self.grid.n_cells, dtype=torch.float64, device="cuda") if out is None else out
        _lib.check(self._lib.spfd_field_divergence(self.handle, _lib.ptr(flux), _lib.ptr(out), _lib.stream_ptr(stream)))
        return out

    def clean(self, flux, tol: float = 1e-10, out=None, stream=None):
        """Divergence cleaning of one (n_faces,) or a batch of two (2, n_faces)
        flux vectors (one batched Krylov solve); `last_clean` holds the info
        (a list for a batch)."""
        flux = _dev(flux)
        out = torch.empty_like(flux) if out is None else out
        if flux.dim() == 2:
            nrhs = flux.shape[0]
            if nrhs not in (1, 2) or flux.shape[1] != self.grid.n_faces or tuple(out.shape) != tuple(flux.shape):
                raise ValueError(f"expected (1 or 2, {self.grid.n_faces}) flux vectors")
            infos = (_lib.CleanInfo * nrhs)()
            _lib.check(self._lib.spfd_field_clean_batch(self.handle, nrhs, _lib.ptr(flux), _lib.ptr(out), float(tol),
                                                        infos, _lib.stream_ptr(stream)))
            self.last_clean = list(infos)
            return out
        info = _lib.CleanInfo()
        _lib.check(self._lib.spfd_field_clean(self.handle, _lib.ptr(flux), _lib.ptr(out), float(tol),
                                              ctypes.byref(info), _lib.stream_ptr(stream)))
        self.last_clean = info
        return out

    def gauge(self, flux, tol: float = 1e-10, out=None, stream=None, tree: str = "comb"):
        from .errors import IncompatibleFluxError
        if tree not in ("comb", "bfs"):
            raise ValueError(f"unknown tree kind {tree!r}")
        flux = _dev(flux)
        out = torch.empty(self.grid.n_edges, dtype=torch.float64, device="cuda") if out is None else out
        info = _lib.GaugeInfo()
        rc = self._lib.spfd_field_gauge_tree(self.handle, 0 if tree == "comb" else 1, _lib.ptr(flux), _lib.ptr(out),
                                             float(tol), ctypes.byref(info), _lib.stream_ptr(stream))
        if rc == _lib.SPFD_EINCOMPAT:
            raise IncompatibleFluxError(info.rel_residual, int(info.worst_face), info.worst_defect)
        _lib.check(rc)
        self.last_gauge = info
        return out

    def circulation(self, a, flux, out=None, stream=None):
        a, flux = _dev(a), _dev(flux)
        out = torch.empty(self.grid.n_faces, dtype=torch.float64, device="cuda") if out is None else out
        _lib.check(self._lib.spfd_field_circulation(self.handle, _lib.ptr(a), _lib.ptr(flux), _lib.ptr(out),
                                                    _lib.stream_ptr(stream)))
        return out


_FIELD_CACHE: dict = {}


def field_ops(grid: StaggeredGrid, cfg: SolveConfig | None = None) -> FieldOps:
    """Cached FieldOps per (grid, solver settings)."""
    cfg = cfg or SolveConfig()
    key = (grid.dims, grid.spacing, grid.origin, _cfg_key(cfg))
    ops = _FIELD_CACHE.get(key)
    if ops is None:
        ops = _FIELD_CACHE[key] = FieldOps(grid, cfg)
    return ops


def _ret(t, as_np):
    return t.cpu().numpy() if as_np else t


def interpolate_to_faces(samples: FieldSampleSet, grid: StaggeredGrid):
    """Integrated flux through every grid face (field_source.py:254-272),
    bit-identical to the reference."""
    as_np = not isinstance(samples.b, torch.Tensor)
    return _ret(field_ops(grid).interpolate(samples.lattice, samples.b), as_np)


def face_fluxes_from_callable(grid: StaggeredGrid, fn) -> np.ndarray:
    """Face fluxes from a direct field evaluation ``fn(points (n,3)) -> (n,3)``
    (field_source.py:275-285; `fn` is user host code)."""
    fluxes = np.empty(grid.n_faces, dtype=np.float64)
    for axis in range(3):
        xs, ys, zs = grid.face_center_axes(axis)
        i, j, k = np.meshgrid(xs, ys, zs, indexing="ij")
        pts = np.stack([i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")], axis=1)
        vals = np.asarray(fn(pts))[:, axis]
        lo = grid.face_offsets[axis]
        fluxes[lo:lo + grid.face_counts[axis]] = vals * grid.face_area(axis)
    return fluxes


def divergence(fluxes, grid: StaggeredGrid):
    """build_divergence(grid) @ fluxes on the device (bit-identical)."""
    as_np = not isinstance(fluxes, torch.Tensor)
    return _ret(field_ops(grid).divergence(fluxes), as_np)


def divergence_clean(fluxes, grid: StaggeredGrid, tol: float = 1e-10, cfg: SolveConfig | None = None):
    """Project face fluxes onto the discretely solenoidal subspace
    (field_source.py:292-329).  Returns the input unchanged (a copy) when the
    relative cell-outflux norm is already <= tol; raises ProjectionError when
    the projection fails."""
    as_np = not isinstance(fluxes, torch.Tensor)
    n = int(np.prod(np.shape(fluxes)))
    if n != grid.n_faces:
        raise ValueError(f"flux vector has length {n}, expected {grid.n_faces}")
    return _ret(field_ops(grid, cfg).clean(fluxes, tol), as_np)
