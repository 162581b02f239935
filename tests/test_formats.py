"""CPU: the file formats (phantom, field samples, report, field dump) are
byte-compatible with the reference's writers (golden bytes from
tests/golden/make_golden.py pipeline_case)."""

import os
import types

import numpy as np
import pytest

from conftest import load_golden


def two_blobs():
    from paper_2010_12879_b200.voxel_model import ConductivitySamples, Tissue, VoxelModel
    dims = (14, 9, 8)
    ids = np.zeros(dims, dtype=np.uint16)
    ids[1:6, 1:8, 1:7] = 1
    ids[8:13, 2:7, 2:6] = 2
    ids[3, 4, 3] = 0
    table = {0: Tissue("free_space", ConductivitySamples.constant(0.0)),
             1: Tissue("a", ConductivitySamples.from_pairs([(1e3, 0.1), (1e6, 0.4)])),
             2: Tissue("b", ConductivitySamples.constant(0.05))}
    return VoxelModel(dims, (0.002, 0.0025, 0.003), (0.0, 0.0, 0.0), ids, table)


@pytest.fixture(scope="module")
def g():
    return load_golden("field_pipeline")


def test_phantom_bytes_and_roundtrip(g, tmp_path):
    from paper_2010_12879_b200.formats import load_model, save_model
    m = two_blobs()
    p = tmp_path / "m.phantom"
    save_model(m, p)
    assert p.read_bytes() == g["phantom_bytes"].tobytes()
    m2 = load_model(p)
    assert m2.dims == m.dims and np.array_equal(m2.tissue_ids, m.tissue_ids)
    assert sorted(m2.tissue_table) == [0, 1, 2]
    assert np.array_equal(m2.tissue_table[1].conductivity.kappas_spm, m.tissue_table[1].conductivity.kappas_spm)


def test_phantom_format_errors(g, tmp_path):
    from paper_2010_12879_b200.errors import PhantomFormatError
    from paper_2010_12879_b200.formats import load_model
    raw = g["phantom_bytes"].tobytes()
    for bad in (raw[:-2], raw.replace(b"END_HEADER\n", b""), raw.replace(b"format_version = 1", b"format_version = 2"),
                raw.replace(b"dims = 14 9 8", b"dims = 14 9"), b"bogus = 1\n" + raw):
        p = tmp_path / "bad.phantom"
        p.write_bytes(bad)
        with pytest.raises(PhantomFormatError):
            load_model(p)


def test_samples_roundtrip(g, tmp_path):
    from paper_2010_12879_b200.formats import load_samples, save_samples
    p = tmp_path / "s.txt"
    p.write_bytes(g["samples_bytes"].tobytes())
    s = load_samples(p)
    assert s.lattice.dims == (3, 3, 2)
    q = tmp_path / "s2.txt"
    save_samples(s, q)
    assert q.read_bytes() == g["samples_bytes"].tobytes()


def test_samples_format_errors(g, tmp_path):
    from paper_2010_12879_b200.errors import FieldFormatError
    from paper_2010_12879_b200.formats import load_samples
    text = g["samples_bytes"].tobytes().decode()
    lines = text.splitlines()
    for bad in ("\n".join(lines[:-1]), "\n".join(lines[1:]), "\n".join(lines + ["1 2 3"]),
                "\n".join(lines[:1] + lines)):
        p = tmp_path / "bad.txt"
        p.write_text(bad + "\n")
        with pytest.raises(FieldFormatError):
            load_samples(p)


def test_report_and_dump_bytes(g, tmp_path):
    from paper_2010_12879_b200.dosimetry import ExposureReport, TissueStats
    from paper_2010_12879_b200.formats import load_field_dump, read_report, write_field_dump, write_report
    p = tmp_path / "r0.txt"
    p.write_bytes(g["report_bytes"].tobytes())
    parsed = read_report(p)
    solver = types.SimpleNamespace(iterations=int(parsed["solver_iterations"]),
                                   solve_seconds=float(parsed["solve_seconds"]),
                                   setup_seconds=float(parsed["setup_seconds"]))
    names = {1: "a", 2: "b"}
    per = {int(t): TissueStats(names[int(t)], int(c), float(m), float(x), float(q))
           for t, c, m, x, q in zip(g["tids"], g["t_count"], g["t_mean"], g["t_max"], g["t_p99"])}
    rep = ExposureReport(85e3, g["vox"], g["vox_idx"], float(g["p99"]), float(g["max"]), per, int(g["dofs"]),
                         solver, True, float(parsed["rel_tol"]))
    q = tmp_path / "r.txt"
    write_report(rep, q)
    assert q.read_bytes() == g["report_bytes"].tobytes()
    d = tmp_path / "f.dump"
    write_field_dump(two_blobs(), g["vox"], g["vox_idx"], d)
    assert d.read_bytes() == g["dump_bytes"].tobytes()
    fd = load_field_dump(d)
    assert fd.dims == (14, 9, 8) and np.isnan(fd.values).sum() == 14 * 9 * 8 - g["vox"].size
