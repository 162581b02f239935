"""Voxel body model (host data; the hot path consumes ``tissue_ids`` and the
per-tissue conductivity LUT).

Same constructor, attributes and conductivity semantics as the reference
(/root/reference/pkg/src/spfd/voxel_model.py:30-163).  Any object with
``dims``, ``spacing``, ``origin``, ``tissue_ids`` and a ``tissue_table``
mapping id -> object with ``conductivity.at(f)`` is accepted by the solver
API, so reference VoxelModel instances work unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import exp, log

import numpy as np

from .errors import GeometryError, PhantomFormatError, UnknownTissueError

FREE_SPACE_ID = 0


@dataclass(frozen=True)
class ConductivitySamples:
    """Sampled conductivity curve kappa(f) (voxel_model.py:30-87)."""

    frequencies_hz: np.ndarray
    kappas_spm: np.ndarray

    def __post_init__(self):
        f = np.asarray(self.frequencies_hz, dtype=np.float64).copy()
        k = np.asarray(self.kappas_spm, dtype=np.float64).copy()
        if f.ndim != 1 or f.size == 0 or k.shape != f.shape:
            raise ValueError("need at least one (frequency, kappa) sample")
        if not np.all(np.isfinite(f)) or not np.all(f > 0.0):
            raise ValueError("sample frequencies must be finite and positive")
        if np.any(np.diff(f) <= 0.0):
            raise ValueError("sample frequencies must be strictly increasing")
        if not np.all(np.isfinite(k)) or np.any(k < 0.0):
            raise ValueError("conductivities must be finite and >= 0")
        f.flags.writeable = False
        k.flags.writeable = False
        object.__setattr__(self, "frequencies_hz", f)
        object.__setattr__(self, "kappas_spm", k)

    @classmethod
    def constant(cls, kappa: float, frequency_hz: float = 1e3) -> "ConductivitySamples":
        return cls(np.array([frequency_hz]), np.array([float(kappa)]))

    @classmethod
    def from_pairs(cls, pairs) -> "ConductivitySamples":
        arr = np.asarray(list(pairs), dtype=np.float64).reshape(-1, 2)
        return cls(arr[:, 0].copy(), arr[:, 1].copy())

    def at(self, frequency_hz: float) -> float:
        """Log-log interpolation, clamped, exact at the samples."""
        f = float(frequency_hz)
        if not f > 0.0:
            raise ValueError("frequency must be positive")
        fs, ks = self.frequencies_hz, self.kappas_spm
        j = int(np.searchsorted(fs, f))
        if j < fs.size and fs[j] == f:
            return float(ks[j])
        if f < fs[0]:
            return float(ks[0])
        if f > fs[-1]:
            return float(ks[-1])
        k0, k1 = float(ks[j - 1]), float(ks[j])
        t = (log(f) - log(fs[j - 1])) / (log(fs[j]) - log(fs[j - 1]))
        if k0 > 0.0 and k1 > 0.0:
            return exp((1.0 - t) * log(k0) + t * log(k1))
        return (1.0 - t) * k0 + t * k1


@dataclass(frozen=True)
class Tissue:
    name: str
    conductivity: ConductivitySamples


@dataclass(frozen=True)
class VoxelModel:
    """Uniform Cartesian tissue-id grid with a conductivity table."""

    dims: tuple
    spacing: tuple
    origin: tuple
    tissue_ids: np.ndarray
    tissue_table: dict

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        spacing = tuple(float(s) for s in self.spacing)
        origin = tuple(float(o) for o in self.origin)
        if len(dims) != 3 or any(n < 1 for n in dims):
            raise ValueError(f"dims must be three integers >= 1, got {dims}")
        if len(spacing) != 3 or any(not s > 0.0 for s in spacing):
            raise ValueError(f"spacing must be three positive reals, got {spacing}")
        ids = np.asarray(self.tissue_ids)
        if ids.dtype != np.uint16:
            ids = ids.astype(np.uint16)
        if ids.shape != dims:
            ids = ids.reshape(dims, order="F")
        for tid in np.unique(ids):
            if int(tid) not in self.tissue_table:
                raise PhantomFormatError(f"tissue ID {int(tid)} has no table entry")
        fs = self.tissue_table.get(FREE_SPACE_ID)
        if fs is not None and np.any(fs.conductivity.kappas_spm != 0.0):
            raise PhantomFormatError("tissue ID 0 is reserved for free space (kappa == 0)")
        ids = np.ascontiguousarray(ids)
        ids.flags.writeable = False
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "origin", origin)
        object.__setattr__(self, "tissue_ids", ids)

    @property
    def n_voxels(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def kappa_lut(self, frequency_hz: float) -> np.ndarray:
        return kappa_lut(self, frequency_hz)

    def voxel_kappa(self, frequency_hz: float) -> np.ndarray:
        return self.kappa_lut(frequency_hz)[self.tissue_ids]

    def conductive_mask(self, frequency_hz: float) -> np.ndarray:
        return self.voxel_kappa(frequency_hz) > 0.0


def kappa_lut(model, frequency_hz: float) -> np.ndarray:
    """Conductivity per tissue id (voxel_model.py:155-158)."""
    ids = np.asarray(model.tissue_ids)
    lut = np.zeros(int(ids.max()) + 1, dtype=np.float64)
    for tid, tissue in model.tissue_table.items():
        if tid < lut.size:
            lut[tid] = tissue.conductivity.at(frequency_hz)
    return lut


def kappa_at(model, tissue_id: int, frequency_hz: float) -> float:
    try:
        tissue = model.tissue_table[int(tissue_id)]
    except KeyError:
        raise UnknownTissueError(f"unknown tissue ID {tissue_id}") from None
    return tissue.conductivity.at(frequency_hz)


def ids_fortran_flat(model) -> np.ndarray:
    """Tissue ids flattened x-fastest (the device layout)."""
    return np.ascontiguousarray(np.asarray(model.tissue_ids, dtype=np.uint16).ravel(order="F"))


def _table(kappas, names, f_sample):
    table = {FREE_SPACE_ID: Tissue("free_space", ConductivitySamples.constant(0.0, f_sample))}
    for i, k in enumerate(kappas):
        samples = k if isinstance(k, ConductivitySamples) else ConductivitySamples.constant(float(k), f_sample)
        table[i + 1] = Tissue(names[i], samples)
    return table


def make_phantom(kind, dims, spacing, *, origin=(0.0, 0.0, 0.0), center_m=None, radius_m=None,
                 height_m=None, axis="z", size_m=None, layers=1, kappa_spm=0.2, tissue_name="tissue",
                 sample_frequency_hz=1e3) -> VoxelModel:
    """Analytic phantoms with the reference's inside-test and id layout
    (voxel_model.py:321-423): 'sphere', 'cylinder', 'block', 'layered-block'."""
    dims = tuple(int(n) for n in dims)
    spacing = tuple(float(v) for v in np.broadcast_to(np.asarray(spacing, dtype=np.float64), (3,)))
    origin = tuple(float(v) for v in np.broadcast_to(np.asarray(origin, dtype=np.float64), (3,)))
    extent = tuple(origin[a] + dims[a] * spacing[a] for a in range(3))
    if center_m is None:
        center_m = tuple(0.5 * (origin[a] + extent[a]) for a in range(3))
    center_m = tuple(float(v) for v in np.broadcast_to(np.asarray(center_m, dtype=np.float64), (3,)))
    ax = "xyz".index(axis)

    def bounds(lo, hi):
        for a in range(3):
            if lo[a] < origin[a] - 1e-12 or hi[a] > extent[a] + 1e-12:
                raise GeometryError(f"{kind} phantom exceeds grid bounds on axis {'xyz'[a]}")

    X, Y, Z = (origin[a] + (np.arange(dims[a]) + 0.5) * spacing[a] - center_m[a] for a in range(3))
    X, Y, Z = X[:, None, None], Y[None, :, None], Z[None, None, :]
    kappas, names = [kappa_spm], [tissue_name]
    if kind == "sphere":
        r = float(radius_m)
        bounds([c - r for c in center_m], [c + r for c in center_m])
        inside = X * X + Y * Y + Z * Z < r * r
    elif kind == "cylinder":
        r = float(radius_m)
        h = float(height_m) if height_m is not None else extent[ax] - origin[ax]
        half = [r, r, r]
        half[ax] = 0.5 * h
        bounds([center_m[a] - half[a] for a in range(3)], [center_m[a] + half[a] for a in range(3)])
        coords = (X, Y, Z)
        trans = [coords[a] for a in range(3) if a != ax]
        inside = (trans[0] ** 2 + trans[1] ** 2 < r * r) & (np.abs(coords[ax]) < 0.5 * h)
    elif kind in ("block", "layered-block"):
        if size_m is None:
            size_m = tuple(extent[a] - origin[a] for a in range(3))
        size_m = tuple(float(v) for v in np.broadcast_to(np.asarray(size_m, dtype=np.float64), (3,)))
        half = [0.5 * s for s in size_m]
        bounds([center_m[a] - half[a] for a in range(3)], [center_m[a] + half[a] for a in range(3)])
        inside = (np.abs(X) < half[0]) & (np.abs(Y) < half[1]) & (np.abs(Z) < half[2])
        if kind == "layered-block":
            layers = int(layers)
            kappas = [kappa_spm] * layers if np.ndim(kappa_spm) == 0 else list(kappa_spm)
            if len(kappas) != layers:
                raise ValueError("need one kappa per layer")
            names = [f"{tissue_name}_{i + 1}" for i in range(layers)]
            rel = ((X, Y, Z)[ax] + half[ax]) / (2.0 * half[ax] / layers)
            idx = np.clip(np.floor(rel).astype(np.int64), 0, layers - 1)
            ids = np.where(inside, (idx + 1).astype(np.uint16), np.uint16(0))
            return VoxelModel(dims, spacing, origin, ids, _table(kappas, names, sample_frequency_hz))
    else:
        raise ValueError(f"unknown phantom kind {kind!r}")
    ids = np.where(inside, np.uint16(1), np.uint16(0))
    return VoxelModel(dims, spacing, origin, ids, _table(kappas, names, sample_frequency_hz))
