"""C5: 100 successive field snapshots on the 2 mm phantom reusing one AMG
setup (BASELINE.json configs[4]).  Snapshots are processed two at a time
(batched as the rhs pair); prints setup time and per-snapshot time."""

import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2010_12879_b200 import Session, SolveConfig, workloads  # noqa: E402


def main(count=100):
    model = workloads.duke_like_model(0.002)
    t0 = time.perf_counter()
    sess = Session(model, workloads.FREQ_HZ, SolveConfig(rel_tol=1e-8))
    torch.cuda.synchronize()
    setup_wall = time.perf_counter() - t0
    unit = torch.from_numpy(workloads.unit_potentials(model)).cuda()  # (3, E)
    fields = torch.from_numpy(workloads.snapshot_fields(count)).cuda()  # (count, 3)
    a = torch.empty((2, unit.shape[1]), dtype=torch.float64, device="cuda")
    # warm-up
    torch.matmul(fields[:2], unit, out=a)
    sess.snapshot(a)
    times, iters = [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for s in range(0, count, 2):
        ev[0].record()
        torch.matmul(fields[s:s + 2], unit, out=a)       # a_s = sum_i B_s,i a_i (linearity)
        vox, rep, _ = sess.snapshot(a)
        ev[1].record()
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]) / 2.0)
        iters.append(rep.iterations)
    line = {
        "config": "C5 Duke-like 2 mm, 100 uniform-B snapshots at seeded random directions, one AMG setup",
        "snapshots": count, "setup_s_device": sess.hierarchy.setup_seconds, "setup_s_wall_incl_assembly": setup_wall,
        "per_snapshot_ms_mean": statistics.mean(times), "per_snapshot_ms_stdev": statistics.stdev(times),
        "per_snapshot_ms_min": min(times), "per_snapshot_ms_max": max(times),
        "pcg_iterations_mean": statistics.mean(iters), "total_s": sum(times) / 1e3,
        "note": "two snapshots per call (batched rhs pair); time per snapshot = call time / 2",
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
