"""GPU: the device `run_pipeline` / `run_benchmark` against the reference's
run_pipeline (golden field_pipeline.npz: coil source on a 5x5x5 lattice,
divergence cleaning, comb gauge, solve at rel_tol 1e-12, E-field, RMS
report; and a uniform-field run).  Voxel |E| within 1e-7 of the reference's
maximum (two solves at 1e-12 plus 1e-16-level Biot-Savart differences),
statistics within the same bound, counts exact."""

import numpy as np
import pytest

from conftest import load_golden
from test_formats import two_blobs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return load_golden("field_pipeline")


def _coil(g):
    from paper_2010_12879_b200.field_source import CoilSpec
    return CoilSpec(tuple(g["coil_center"]), tuple(g["coil_axis"]), float(g["coil_radius"]),
                    float(g["coil_current"]), int(g["coil_segments"]))


def test_run_pipeline_coil_matches_reference(g, tmp_path):
    from paper_2010_12879_b200.formats import load_field_dump, read_report
    from paper_2010_12879_b200.pipeline import PipelineConfig, run_pipeline
    cfg = PipelineConfig(model=two_blobs(), coil=_coil(g), frequency_hz=85e3, coil_lattice_dims=(5, 5, 5),
                         report_rms=True, out_report=str(tmp_path / "r.txt"), out_field=str(tmp_path / "f.dump"))
    rep, timing = run_pipeline(cfg)
    assert np.array_equal(rep.voxel_indices.cpu().numpy(), g["vox_idx"])
    vmax = float(np.abs(g["vox"]).max())
    assert np.abs(rep.voxel_field.cpu().numpy() - g["vox"]).max() <= 1e-7 * vmax
    assert abs(rep.percentile99_vpm - float(g["p99"])) <= 1e-7 * vmax
    assert abs(rep.max_vpm - float(g["max"])) <= 1e-7 * vmax
    assert rep.dof_count == int(g["dofs"])
    assert sorted(rep.per_tissue) == list(g["tids"])
    for t, c, m, x, p in zip(g["tids"], g["t_count"], g["t_mean"], g["t_max"], g["t_p99"]):
        s = rep.per_tissue[int(t)]
        assert s.count == int(c)
        for a, b in ((s.mean, m), (s.max, x), (s.p99, p)):
            assert abs(a - float(b)) <= 1e-7 * vmax
    assert timing.total > 0 and timing.budget_met
    r = read_report(tmp_path / "r.txt")
    assert float(r["p99_vpm"]) == rep.percentile99_vpm and r["rms"] == "1"
    fd = load_field_dump(tmp_path / "f.dump")
    assert np.nanmax(fd.values) == rep.max_vpm


def test_run_pipeline_uniform_matches_reference(g):
    from paper_2010_12879_b200.pipeline import PipelineConfig, run_pipeline
    rep, _ = run_pipeline(PipelineConfig(model=two_blobs(), uniform_b=(0.0, 0.0, 1e-6), frequency_hz=85e3))
    vmax = float(np.abs(g["u_vox"]).max())
    assert np.abs(rep.voxel_field.cpu().numpy() - g["u_vox"]).max() <= 1e-7 * vmax
    assert abs(rep.percentile99_vpm - float(g["u_p99"])) <= 1e-7 * vmax


def test_pipeline_stage_errors(g):
    from paper_2010_12879_b200.errors import PipelineError
    from paper_2010_12879_b200.pipeline import PipelineConfig, run_pipeline
    with pytest.raises(ValueError):
        PipelineConfig(model=two_blobs(), uniform_b=(0, 0, 1e-6), coil=_coil(g))
    with pytest.raises(PipelineError) as ei:
        run_pipeline(PipelineConfig(model=two_blobs(), uniform_b=(0, 0, 1e-6), tree_kind="nope"))
    assert ei.value.step == "gauge"


def test_run_benchmark(g):
    from paper_2010_12879_b200.pipeline import STEP_NAMES, PipelineConfig, run_benchmark
    res = run_benchmark(PipelineConfig(model=two_blobs(), coil=_coil(g), coil_lattice_dims=(5, 5, 5)), runs=3)
    assert res.runs == 3 and len(res.iterations) == 3 and len(set(res.iterations)) == 1
    assert set(res.steps) == set(STEP_NAMES) | {"total"}
    assert "amg setup" in res.to_text() and res.to_csv().startswith("step,mean_s")


@pytest.mark.parametrize("case", ["c1", "sphere8_uniform", "layered_dipole", "two_blobs"])
def test_snapshot_host_matches_device(case):
    """The host path copies only the edge ranges of the planes that hold
    conductive nodes; its result equals the device-resident snapshot's bit
    for bit (the untouched edges are never read), with the plane range
    covering every conductive voxel."""
    import torch
    from conftest import golden_model
    from paper_2010_12879_b200 import Session, SolveConfig, workloads
    if case == "c1":
        w = workloads.c1(24)
        model, freq, a = w.model, w.frequency_hz, w.a
    else:
        d = load_golden(case)
        model, freq = golden_model(d), float(d["freq"])
        a = np.stack([d["a"], 0.5 * d["a"]])
    sess = Session(model, freq, SolveConfig(rel_tol=1e-10))
    kb, ke = sess.plane_range
    zc = np.flatnonzero((model.voxel_kappa(freq) > 0).any(axis=(0, 1)))
    assert kb == zc[0] and ke == zc[-1] + 2
    vox_d, rep_d, _ = sess.snapshot(torch.from_numpy(np.ascontiguousarray(a)).cuda())
    vox_d = vox_d.cpu().numpy().copy()
    pinned = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    vox_h, rep_h = sess.snapshot_host(pinned)
    assert rep_h.iterations == rep_d.iterations
    assert np.array_equal(vox_h, vox_d)
    h2d, _ = sess.host_bytes(a.shape[0])
    assert h2d <= a.size * 8


def test_snapshots_host_stream_matches_single_snapshots():
    """The pipelined host stream (copy-in of i+1 and copy-out of i-1 overlap
    the solve of i) returns, per snapshot, exactly the device snapshot's
    voxel field (different inputs, odd count, double-buffer reuse)."""
    import torch
    from paper_2010_12879_b200 import Session, SolveConfig, workloads
    w = workloads.c1(20)
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10))
    ins = [torch.from_numpy(np.ascontiguousarray(w.a * s)).pin_memory() for s in (1.0, -0.5, 2.0, 0.25, 3.0)]
    ref = []
    for a in ins:
        vox, rep, _ = sess.snapshot(a.cuda())
        ref.append((vox.cpu().numpy().copy(), rep.iterations))
    outs, reps = sess.snapshots_host(ins)
    assert len(outs) == len(ins) == len(reps)
    for (v, its), o, r in zip(ref, outs, reps):
        assert r.iterations == its
        assert np.array_equal(o.numpy(), v)
