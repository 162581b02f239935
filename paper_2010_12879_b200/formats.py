"""File formats around the hot path: the phantom
file, the field-sample file, the exposure report and the full-grid field
dump.  Host I/O only; byte-compatible with the reference's writers and
readers (voxel_model.py:175-298, field_source.py:330-397,
dosimetry.py:236-312) so files move freely between the two packages.

Phantom / dump file: UTF-8 ``key = value`` header lines, ``END_HEADER\\n``,
then a little-endian payload (u16 tissue ids, or f64 |E| with NaN in free
space), x-fastest.  Sample file: four header lines then one
``x y z bx by bz`` line per lattice point.  Report: ``key = value`` lines
and one ``tissue id name count mean max p99`` line per tissue.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import FieldFormatError, LatticeError, PhantomFormatError

HEADER_END = b"END_HEADER\n"
FORMAT_VERSION = 1
_BASE_KEYS = ("format_version", "dims", "spacing_m", "origin_m")


def _r(x) -> str:
    """Round-trip float text (Python repr)."""
    return repr(float(x))


def _join(vals, fmt=_r) -> str:
    return " ".join(fmt(v) for v in vals)


# ---------------------------------------------------------------- phantom --

def encode_header(model) -> bytes:
    """Canonical phantom header bytes including the END_HEADER marker."""
    out = [f"format_version = {FORMAT_VERSION}",
           f"dims = {_join(model.dims, str)}",
           f"spacing_m = {_join(model.spacing)}",
           f"origin_m = {_join(model.origin)}"]
    for tid in sorted(model.tissue_table):
        t = model.tissue_table[tid]
        c = t.conductivity
        samples = " ".join(f"{_r(f)}:{_r(k)}" for f, k in zip(c.frequencies_hz, c.kappas_spm))
        out.append(f"tissue = {tid} {t.name} {samples}".rstrip())
    return ("\n".join(out) + "\n").encode("utf-8") + HEADER_END


def _triple(text: str, cast, key: str):
    toks = text.split()
    if len(toks) != 3:
        raise PhantomFormatError(f"header key '{key}' needs three values, got {text!r}")
    try:
        return tuple(cast(t) for t in toks)
    except ValueError:
        raise PhantomFormatError(f"bad value for header key '{key}': {text!r}") from None


def _tissue(text: str):
    from .voxel_model import ConductivitySamples, Tissue
    toks = text.split()
    if len(toks) < 2:
        raise PhantomFormatError(f"bad tissue line: {text!r}")
    try:
        tid = int(toks[0])
    except ValueError:
        raise PhantomFormatError(f"bad tissue ID in: {text!r}") from None
    pairs = []
    for tok in toks[2:]:
        f, _, k = tok.partition(":")
        try:
            pairs.append((float(f), float(k)))
        except ValueError:
            raise PhantomFormatError(f"bad conductivity sample {tok!r}") from None
    if not pairs:
        raise PhantomFormatError(f"tissue {tid} has no conductivity samples")
    try:
        return tid, Tissue(toks[1], ConductivitySamples.from_pairs(pairs))
    except ValueError as exc:
        raise PhantomFormatError(f"tissue {tid}: {exc}") from None


def parse_header(data: bytes, where: str = "phantom"):
    """-> (dims, spacing, origin, tissue_table, payload bytes)."""
    cut = data.find(HEADER_END)
    if cut < 0:
        raise PhantomFormatError(f"{where}: missing END_HEADER")
    try:
        text = data[:cut].decode("utf-8")
    except UnicodeDecodeError:
        raise PhantomFormatError(f"{where}: header is not valid UTF-8") from None
    base: dict = {}
    tissues: dict = {}
    for raw in text.splitlines():
        line = raw.strip()
        if not line:
            continue
        key, sep, value = line.partition(" = ")
        key = key.strip()
        if not sep:
            raise PhantomFormatError(f"malformed header line: {raw!r}")
        if key == "tissue":
            tid, t = _tissue(value)
            if tid in tissues:
                raise PhantomFormatError(f"duplicate tissue ID {tid}")
            tissues[tid] = t
        elif key in _BASE_KEYS:
            if key in base:
                raise PhantomFormatError(f"duplicate header key '{key}'")
            base[key] = value
        else:
            raise PhantomFormatError(f"unknown header key '{key}'")
    missing = [k for k in _BASE_KEYS if k not in base]
    if missing:
        raise PhantomFormatError(f"missing header key '{missing[0]}'")
    if base["format_version"].strip() != str(FORMAT_VERSION):
        raise PhantomFormatError(f"unsupported format_version {base['format_version']!r}")
    return (_triple(base["dims"], int, "dims"), _triple(base["spacing_m"], float, "spacing_m"),
            _triple(base["origin_m"], float, "origin_m"), tissues, data[cut + len(HEADER_END):])


def save_model(model, path) -> None:
    Path(path).write_bytes(encode_header(model) + np.asarray(model.tissue_ids).ravel(order="F").astype("<u2").tobytes())


def load_model(path):
    from .voxel_model import VoxelModel
    dims, spacing, origin, tissues, payload = parse_header(Path(path).read_bytes(), str(path))
    want = 2 * dims[0] * dims[1] * dims[2]
    if len(payload) != want:
        raise PhantomFormatError(f"payload size mismatch: expected {want} bytes, got {len(payload)}")
    ids = np.frombuffer(payload, dtype="<u2").reshape(dims, order="F")
    return VoxelModel(dims, spacing, origin, ids, tissues)


# ---------------------------------------------------------------- samples --

_SAMPLE_KEYS = ("frequency_hz", "lattice_dims", "lattice_origin_m", "lattice_spacing_m")


def save_samples(samples, path) -> None:
    lat = samples.lattice
    b = samples.b if isinstance(samples.b, np.ndarray) else samples.b.cpu().numpy()
    rows = [f"frequency_hz = {_r(samples.frequency_hz)}",
            f"lattice_dims = {_join(lat.dims, str)}",
            f"lattice_origin_m = {_join(lat.origin)}",
            f"lattice_spacing_m = {_join(lat.spacing)}"]
    rows += [_join((*p, *v)) for p, v in zip(samples.positions, b)]
    Path(path).write_text("\n".join(rows) + "\n", encoding="utf-8")


def load_samples(path):
    from .field_source import FieldSampleSet, Lattice
    head: dict = {}
    vals = []
    for raw in Path(path).read_text(encoding="utf-8").splitlines():
        line = raw.strip()
        if not line:
            continue
        if " = " in line:
            key, _, value = line.partition(" = ")
            key = key.strip()
            if key in head:
                raise FieldFormatError(f"duplicate header key '{key}'")
            head[key] = value
            continue
        toks = line.split()
        if len(toks) != 6:
            raise FieldFormatError(f"bad sample line: {raw!r}")
        try:
            vals.append([float(t) for t in toks])
        except ValueError:
            raise FieldFormatError(f"bad sample line: {raw!r}") from None
    for key in _SAMPLE_KEYS:
        if key not in head:
            raise FieldFormatError(f"missing header key '{key}'")
    try:
        freq = float(head["frequency_hz"])
        dims = tuple(int(v) for v in head["lattice_dims"].split())
        origin = tuple(float(v) for v in head["lattice_origin_m"].split())
        spacing = tuple(float(v) for v in head["lattice_spacing_m"].split())
        if not (len(dims) == len(origin) == len(spacing) == 3):
            raise ValueError
    except ValueError:
        raise FieldFormatError("malformed lattice header") from None
    lat = Lattice(origin, spacing, dims)
    if len(vals) != lat.n_points:
        raise FieldFormatError(f"sample count mismatch: header implies {lat.n_points}, got {len(vals)}")
    arr = np.asarray(vals, dtype=np.float64).reshape(-1, 6)
    try:
        return FieldSampleSet(freq, lat, arr[:, :3], arr[:, 3:])
    except LatticeError as exc:
        raise FieldFormatError(str(exc)) from None


# ----------------------------------------------------------------- report --

def write_report(report, path) -> None:
    s = report.solver
    rows = [f"p99_vpm = {_r(report.percentile99_vpm)}",
            f"max_vpm = {_r(report.max_vpm)}",
            f"n_voxels = {report.n_voxels}",
            f"frequency_hz = {_r(report.frequency_hz)}",
            f"solver_iterations = {s.iterations if s else 0}",
            f"solve_seconds = {_r(s.solve_seconds if s else 0.0)}",
            f"setup_seconds = {_r(s.setup_seconds if s else 0.0)}",
            f"dof_count = {report.dof_count}",
            f"rms = {int(report.rms)}"]
    if report.rel_tol is not None:
        rows.append(f"rel_tol = {_r(report.rel_tol)}")
    rows += [f"{k} = {v}" for k, v in report.extra.items()]
    for tid in sorted(report.per_tissue):
        t = report.per_tissue[tid]
        rows.append(f"tissue {tid} {t.name} {t.count} {_r(t.mean)} {_r(t.max)} {_r(t.p99)}")
    Path(path).write_text("\n".join(rows) + "\n", encoding="utf-8")


def read_report(path) -> dict:
    out: dict = {"tissue": []}
    for raw in Path(path).read_text(encoding="utf-8").splitlines():
        line = raw.strip()
        if not line:
            continue
        if line.startswith("tissue "):
            out["tissue"].append(line.split()[1:])
            continue
        key, _, value = line.partition(" = ")
        out[key.strip()] = value.strip()
    return out


# ------------------------------------------------------------- field dump --

@dataclass(frozen=True)
class FieldDump:
    dims: tuple
    spacing: tuple
    origin: tuple
    values: np.ndarray  # (nx, ny, nz), NaN in free space


def write_field_dump(model, voxel_values, voxel_indices, path) -> None:
    vals = voxel_values if isinstance(voxel_values, np.ndarray) else voxel_values.cpu().numpy()
    idx = voxel_indices if isinstance(voxel_indices, np.ndarray) else voxel_indices.cpu().numpy()
    full = np.full(model.n_voxels, np.nan)
    full[idx] = vals
    Path(path).write_bytes(encode_header(model) + full.astype("<f8").tobytes())


def load_field_dump(path) -> FieldDump:
    dims, spacing, origin, _, payload = parse_header(Path(path).read_bytes(), str(path))
    n = dims[0] * dims[1] * dims[2]
    if len(payload) != 8 * n:
        raise PhantomFormatError(f"payload size mismatch: expected {8 * n} bytes, got {len(payload)}")
    return FieldDump(dims, spacing, origin, np.frombuffer(payload, dtype="<f8").reshape(dims, order="F"))
