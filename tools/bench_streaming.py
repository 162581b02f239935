"""C5: 100 successive measured-field snapshots on the 2 mm phantom reusing
one setup (BASELINE.json configs[4]; the paper's real-time use case,
PAPER.md:50, "< 5 s" per snapshot).

Each snapshot is the reference's run_pipeline chain (pipeline.py:136-195)
with the hierarchy reused (`_hierarchy`, pipeline.py:136,162):

    sampled B on a lattice (host, pinned)  --H2D-->
    interpolate_to_faces (field_source.py:254-272)
    divergence_clean on S S^T (field_source.py:292-329, AMG reused; the re
    and im sets in one batched solve)
    gauge_vector_potential, comb tree (gauging.py:137-172)
    assemble RHS + AMG-PCG to 1e-8 + E-field / voxel average (one spfd_snapshot)
    --D2H--> voxel |E|

A snapshot is complex: real and imaginary sample sets (two coil currents in
quadrature), batched as the rhs pair of the solve.  The "measured" samples
are synthetic: a 0.15 m, 100 A charger coil beside the body at a seeded
position per snapshot (a person moving past a fixed charger), evaluated with
Biot-Savart on a 17 x 13 x 87 lattice (2 cm) covering the phantom and
prepared before timing (they are the sensor input, not part of the work).
No library GEMM or host compute in the timed loop.

--mode uniform keeps the round-1 closed-form uniform-B snapshots (no field
stages) for comparison.
"""

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2010_12879_b200 import Session, SolveConfig, workloads  # noqa: E402


def measured_samples(grid, count, seed=workloads.SEED, lat_dims=(17, 13, 87)):
    from paper_2010_12879_b200.field_source import CoilSpec, Lattice, coil_field
    lattice = Lattice.covering(grid, lat_dims)
    pts = lattice.points()
    ext = [grid.dims[a] * grid.spacing[a] for a in range(3)]
    rng = np.random.default_rng(seed)
    zs = rng.uniform(0.15, ext[2] - 0.15, count)
    ys = rng.uniform(0.3 * ext[1], 0.7 * ext[1], count)
    out = []
    for s in range(count):
        # pad beside the body (outside the grid box, so the lattice never
        # touches the wire); the quadrature current feeds a tilted second loop
        re = CoilSpec(center=(ext[0] + 0.03, ys[s], zs[s]), axis=(1.0, 0.0, 0.0), radius_m=0.15, current_a=100.0,
                      segments=256)
        im = CoilSpec(center=(ext[0] + 0.03, ys[s], zs[s]), axis=(1.0, 0.3, 0.0), radius_m=0.15, current_a=50.0,
                      segments=256)
        b = np.stack([coil_field(re, pts), coil_field(im, pts)])
        out.append(torch.from_numpy(b).pin_memory())
    return lattice, out


def run_measured(count, rel_tol, clean_tol, gauge_tol):
    from paper_2010_12879_b200.field_source import FieldOps
    from paper_2010_12879_b200.fit_operators import StaggeredGrid
    model = workloads.duke_like_model(0.002)
    grid = StaggeredGrid.from_model(model)
    t0 = time.perf_counter()
    sess = Session(model, workloads.FREQ_HZ, SolveConfig(rel_tol=rel_tol))
    ops = FieldOps(grid, SolveConfig())
    torch.cuda.synchronize()
    setup_wall = time.perf_counter() - t0
    lattice, samples = measured_samples(grid, count + 2)
    n_vox = sess.n_cond_voxels
    outs = [torch.empty((2, n_vox), dtype=torch.float64, pin_memory=True) for _ in range(count)]
    b_dev = torch.empty(samples[0].shape, dtype=torch.float64, device="cuda")
    a = torch.empty((2, grid.n_edges), dtype=torch.float64, device="cuda")
    fl = torch.empty((2, grid.n_faces), dtype=torch.float64, device="cuda")
    fc = torch.empty((2, grid.n_faces), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    names = ("h2d", "interpolate", "clean", "gauge", "rhs+solve+efield", "d2h")
    # the voxel field leaves on a copy stream while the next snapshot runs
    # (two device result buffers, as Session.snapshots_host)
    d2h = torch.cuda.Stream()
    voxb = [torch.empty((2, n_vox), dtype=torch.float64, device="cuda") for _ in range(2)]
    out_ev = [None, None]

    def one(i, out, ev=None):
        if ev:
            ev[0].record(stream)
        b_dev.copy_(samples[i], non_blocking=True)
        if ev:
            ev[1].record(stream)
        for c in range(2):
            ops.interpolate(lattice, b_dev[c], out=fl[c])
        if ev:
            ev[2].record(stream)
        ops.clean(fl, clean_tol, out=fc)          # re and im in one batched projection solve
        infos = ops.last_clean
        if ev:
            ev[3].record(stream)
        for c in range(2):
            ops.gauge(fc[c], gauge_tol, out=a[c])
        if ev:
            ev[4].record(stream)
        b = i % 2
        if out_ev[b] is not None:
            stream.wait_event(out_ev[b])           # result i-2 has left voxb[b]
        vox, rep, _ = sess.snapshot(a, vox_out=voxb[b])
        if ev:
            ev[5].record(stream)
        with torch.cuda.stream(d2h):
            d2h.wait_stream(stream)
            out.copy_(voxb[b], non_blocking=True)
            out_ev[b] = torch.cuda.Event(enable_timing=True)
            out_ev[b].record(d2h)
        if ev:
            ev[6] = out_ev[b]
        return rep, infos

    # warm-up (cleaning hierarchy built on first use: reported as setup)
    t0 = time.perf_counter()
    one(count, outs[0])
    torch.cuda.synchronize()
    clean_setup_wall = time.perf_counter() - t0
    one(count + 1, outs[0])
    torch.cuda.synchronize()
    torch.cuda.synchronize()
    per, stages, its, clean_its, wall = [], {n: [] for n in names}, [], [], []
    evs = []
    w0 = time.perf_counter()
    for i in range(count):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        rep, infos = one(i, outs[i], ev)
        evs.append(ev)
        its.append(rep.iterations)
        clean_its.append([int(x.iterations) for x in infos])
    torch.cuda.synchronize()
    wall_total = (time.perf_counter() - w0) * 1e3
    for i, ev in enumerate(evs):
        # snapshot i spans its start to the next snapshot's start (its copy-out
        # overlaps the next snapshot); the last one ends when its copy-out does
        per.append(ev[0].elapsed_time(evs[i + 1][0]) if i + 1 < count else ev[0].elapsed_time(ev[6]))
        for k, n in enumerate(names):
            stages[n].append(ev[k].elapsed_time(ev[k + 1]))
    wall = [wall_total / count]
    return {
        "config": "C5 Duke-like 2 mm (8,913,552 DOFs), 100 measured-field snapshots (coil samples on a 17x13x87 "
                  "lattice, re+im), one setup reused",
        "mode": "measured", "snapshots": count,
        "setup_s_device": sess.hierarchy.setup_seconds, "setup_s_wall_incl_assembly": setup_wall,
        "clean_setup_s_wall": clean_setup_wall,
        "per_snapshot_ms_mean": statistics.mean(per), "per_snapshot_ms_stdev": statistics.stdev(per),
        "per_snapshot_ms_min": min(per), "per_snapshot_ms_max": max(per),
        "per_snapshot_wall_ms_mean": statistics.mean(wall),
        "stage_ms_mean": {n: round(statistics.mean(v), 3) for n, v in stages.items()},
        "pcg_iterations_mean": statistics.mean(its),
        "clean_iterations_mean": statistics.mean(x for c in clean_its for x in c),
        "total_s": sum(per) / 1e3,
        "h2d_bytes_per_snapshot": int(samples[0].numel() * 8), "d2h_bytes_per_snapshot": int(2 * n_vox * 8),
        "timing": "CUDA events: a snapshot runs from its start to the next snapshot's start (host samples in -> "
                  "voxel |E| out; the copy-out of snapshot i overlaps snapshot i+1 on a copy stream, the last one "
                  "is waited for); stage times per event pair; the cleaning and gauging calls read their residual "
                  "checks back to the host",
    }


def run_uniform(count, rel_tol):
    model = workloads.duke_like_model(0.002)
    t0 = time.perf_counter()
    sess = Session(model, workloads.FREQ_HZ, SolveConfig(rel_tol=rel_tol))
    torch.cuda.synchronize()
    setup_wall = time.perf_counter() - t0
    unit = workloads.unit_potentials(model)          # (3, E), gauged once
    fields = workloads.snapshot_fields(count)         # (count, 3)
    # per-snapshot potentials prepared on the host before timing (linearity)
    pots = [torch.from_numpy(np.ascontiguousarray(fields[s:s + 2] @ unit)).pin_memory() for s in range(0, count, 2)]
    a = torch.empty((2, unit.shape[1]), dtype=torch.float64, device="cuda")
    a.copy_(pots[0])
    sess.snapshot(a)
    times, iters = [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for p in pots:
        ev[0].record()
        a.copy_(p, non_blocking=True)
        vox, rep, _ = sess.snapshot(a)
        ev[1].record()
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]) / 2.0)
        iters.append(rep.iterations)
    return {
        "config": "C5 Duke-like 2 mm, 100 uniform-B snapshots at seeded random directions, one AMG setup",
        "mode": "uniform", "snapshots": count, "setup_s_device": sess.hierarchy.setup_seconds,
        "setup_s_wall_incl_assembly": setup_wall,
        "per_snapshot_ms_mean": statistics.mean(times), "per_snapshot_ms_stdev": statistics.stdev(times),
        "per_snapshot_ms_min": min(times), "per_snapshot_ms_max": max(times),
        "pcg_iterations_mean": statistics.mean(iters), "total_s": sum(times) / 1e3,
        "note": "two snapshots per call (batched rhs pair), potentials copied in from pinned host memory; "
                "time per snapshot = call time / 2",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="measured", choices=["measured", "uniform"])
    ap.add_argument("--count", type=int, default=100)
    ap.add_argument("--rel-tol", type=float, default=1e-8)
    ap.add_argument("--clean-tol", type=float, default=1e-10)
    ap.add_argument("--gauge-tol", type=float, default=1e-10)
    args = ap.parse_args()
    if args.mode == "measured":
        line = run_measured(args.count, args.rel_tol, args.clean_tol, args.gauge_tol)
    else:
        line = run_uniform(args.count, args.rel_tol)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
