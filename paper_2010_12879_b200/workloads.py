"""Synthetic workloads C1-C5 (BASELINE.json `configs`).

Host-side input builders only (phantom tissue ids + edge vector potentials);
nothing here is on the timed hot path.

* C1  64^3 homogeneous box (0.2 S/m), uniform B.
* C2  128^3 layered block (skin/fat/muscle/bone = 0.17/0.04/0.35/0.02 S/m
      along z, voxel_model.py:403-417 layout) with a coil-like magnetic
      dipole source below the block.
* C3  Duke-sized layered elliptic cylinder, 160x112x860 voxels at 2 mm,
      8,913,552 DOFs; re = uniform B_z 1 uT, im = uniform B_x 0.5 uT.
* C4  the same body at 1 mm (320x224x1720, 70,668,030 DOFs).
* C5  C3 with 100 seeded random field directions (setup reuse).

Uniform fields use the comb-tree gauge (gauging.py:34-71) in closed form:
a_x(i,j,k) = -j*Bz*dx*dy + k*By*dx*dz, a_y(i,j,k) = -k*Bx*dy*dz, a_z = 0,
which is the prefix-scan solution of the tree-cotree elimination for
constant face fluxes.  The dipole potential is sampled at edge midpoints,
a = A(mid) . t * length, so curl a is exactly solenoidal (no cleaning).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .voxel_model import ConductivitySamples, Tissue, VoxelModel, make_phantom

MU0 = 4e-7 * math.pi
FREQ_HZ = 85e3
SEED = 20240817


@dataclass
class Workload:
    name: str
    model: VoxelModel
    frequency_hz: float
    a: np.ndarray  # (nrhs, n_edges) edge vector potential(s)

    @property
    def omega(self) -> float:
        return 2.0 * math.pi * self.frequency_hz


def _table(kappas, names):
    t = {0: Tissue("free_space", ConductivitySamples.constant(0.0))}
    for i, (k, n) in enumerate(zip(kappas, names)):
        t[i + 1] = Tissue(n, ConductivitySamples.constant(k))
    return t


def box_model(dims, kappa=0.2, spacing=0.002) -> VoxelModel:
    ids = np.ones(tuple(dims), dtype=np.uint16)
    return VoxelModel(tuple(dims), (spacing,) * 3, (0.0, 0.0, 0.0), ids, _table([kappa], ["tissue"]))


def layered_block_model(n=128, spacing=0.002) -> VoxelModel:
    # 0.2048 m block in a 0.256 m box at 128^3, scaled with n
    return make_phantom("layered-block", (n, n, n), spacing, layers=4, kappa_spm=[0.17, 0.04, 0.35, 0.02],
                        size_m=(0.0016 * n,) * 3)


def duke_like_model(spacing=0.002) -> VoxelModel:
    """Layered elliptic cylinder."""
    scale = 0.002 / spacing
    dims = (int(round(160 * scale)), int(round(112 * scale)), int(round(860 * scale)))
    c = [n * spacing / 2 for n in dims]
    x = (np.arange(dims[0]) + 0.5) * spacing - c[0]
    y = (np.arange(dims[1]) + 0.5) * spacing - c[1]
    z = (np.arange(dims[2]) + 0.5) * spacing - c[2]
    rho = np.sqrt((x[:, None] / 0.150) ** 2 + (y[None, :] / 0.095) ** 2)
    plane = np.zeros(rho.shape, dtype=np.uint16)
    plane[rho < 1.0] = 1          # skin
    plane[rho < 0.96] = 2         # fat
    plane[rho < 0.85] = 3         # muscle
    plane[rho < 0.25] = 4         # bone
    inz = np.abs(z) < 0.78
    ids = np.where(inz[None, None, :], plane[:, :, None], np.uint16(0)).astype(np.uint16)
    table = _table([0.10, 0.04, 0.35, 0.02], ["skin", "fat", "muscle", "bone"])
    return VoxelModel(dims, (spacing,) * 3, (0.0, 0.0, 0.0), ids, table)


def uniform_potential(dims, spacing, b) -> np.ndarray:
    """Comb-gauge edge vector potential of a uniform flux density b."""
    nx, ny, nz = (int(d) for d in dims)
    dx, dy, dz = (float(s) for s in (spacing if np.ndim(spacing) else (spacing,) * 3))
    bx, by, bz = (float(v) for v in b)
    j = np.arange(ny + 1, dtype=np.float64)
    k = np.arange(nz + 1, dtype=np.float64)
    ax_jk = (-j[:, None] * (bz * dx * dy)) + k[None, :] * (by * dx * dz)      # (ny+1, nz+1)
    ax = np.broadcast_to(ax_jk[None, :, :], (nx, ny + 1, nz + 1))
    ay_k = -k * (bx * dy * dz)
    ay = np.broadcast_to(ay_k[None, None, :], (nx + 1, ny, nz + 1))
    az_n = (nx + 1) * (ny + 1) * nz
    return np.concatenate([ax.ravel(order="F"), ay.ravel(order="F"), np.zeros(az_n)])


def dipole_potential(dims, spacing, moment, center, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Edge line integrals (midpoint rule) of the dipole vector potential
    A = mu0/(4 pi) m x (r - r0) / |r - r0|^3."""
    nx, ny, nz = (int(d) for d in dims)
    s = [float(v) for v in (spacing if np.ndim(spacing) else (spacing,) * 3)]
    m = np.asarray(moment, dtype=np.float64)
    r0 = np.asarray(center, dtype=np.float64)
    out = []
    for axis in range(3):
        ed = [nx + 1, ny + 1, nz + 1]
        ed[axis] -= 1
        coords = []
        for a in range(3):
            v = origin[a] + np.arange(ed[a]) * s[a]
            if a == axis:
                v = v + 0.5 * s[a]
            coords.append(v - r0[a])
        X, Y, Z = coords[0][:, None, None], coords[1][None, :, None], coords[2][None, None, :]
        r3 = (X * X + Y * Y + Z * Z) ** 1.5
        comp = [m[1] * Z - m[2] * Y, m[2] * X - m[0] * Z, m[0] * Y - m[1] * X][axis]
        out.append((MU0 / (4 * math.pi) * comp / r3 * s[axis]).ravel(order="F"))
    return np.concatenate(out)


def c1(n=64) -> Workload:
    model = box_model((n, n, n), 0.2, 0.002)
    a = np.stack([uniform_potential(model.dims, 0.002, (0, 0, 1e-6)),
                  uniform_potential(model.dims, 0.002, (0.5e-6, 0, 0))])
    return Workload(f"C1 box {n}^3 uniform B", model, FREQ_HZ, a)


def c2(n=128) -> Workload:
    model = layered_block_model(n)
    ext = n * 0.002
    m_mag = 100.0 * math.pi * 0.15 ** 2  # I * area of the survey's R=0.15 m, 100 A coil
    center = (ext / 2, ext / 2, -0.05)
    a = np.stack([dipole_potential(model.dims, 0.002, (0, 0, m_mag), center),
                  dipole_potential(model.dims, 0.002, (0.5 * m_mag, 0, 0), center)])
    return Workload(f"C2 layered {n}^3 dipole", model, FREQ_HZ, a)


def c3(spacing=0.002) -> Workload:
    model = duke_like_model(spacing)
    a = np.stack([uniform_potential(model.dims, spacing, (0, 0, 1e-6)),
                  uniform_potential(model.dims, spacing, (0.5e-6, 0, 0))])
    tag = "2 mm" if spacing == 0.002 else f"{spacing * 1e3:g} mm"
    return Workload(f"C3 Duke-like {tag}", model, FREQ_HZ, a)


def c4() -> Workload:
    w = c3(0.001)
    w.name = "C4 Duke-like 1 mm"
    return w


def unit_potentials(model) -> np.ndarray:
    """(3, E) potentials of unit uniform B along x, y, z (C5 basis)."""
    return np.stack([uniform_potential(model.dims, model.spacing, e) for e in np.eye(3)])


def snapshot_fields(count=100, seed=SEED, magnitude=1e-6) -> np.ndarray:
    """C5: B_s = 1 uT (sin t cos p, sin t sin p, cos t) at seeded angles."""
    rng = np.random.default_rng(seed)
    th = np.arccos(rng.uniform(-1.0, 1.0, count))
    ph = rng.uniform(0.0, 2 * math.pi, count)
    return magnitude * np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], axis=1)


def small_box(n=12, kappa=0.2) -> Workload:
    model = box_model((n, n, n), kappa, 0.002)
    a = np.stack([uniform_potential(model.dims, 0.002, (0, 0, 1e-6)),
                  uniform_potential(model.dims, 0.002, (0.5e-6, 0.2e-6, 0))])
    return Workload(f"box {n}^3", model, FREQ_HZ, a)


def c2_small() -> Workload:
    """C2 geometry at 48^3 (multi-process tests)."""
    return c2(48)
