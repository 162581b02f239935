"""Benchmark: Poisson solve time of the Duke-sized 2 mm synthetic phantom.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A step is one complex snapshot through the device-resident hot path
(`Session.snapshot` -> one `spfd_snapshot` C-ABI call): RHS assembly from
the real/imag edge vector potentials, AMG-PCG to rel.res 1e-8 for both
parts, fused E-field + voxel average.  The AMG setup is hoisted (reported
as `setup_s`), as in the reference's run_benchmark (pipeline.py:277-288).
`value` is seconds per step (device time, CUDA events, max over ranks).
`e2e` is the same step through the public API from pinned host memory
(H2D of both edge potentials, D2H of both voxel |E| arrays).

`--impl reference` times the reference algorithm on the host CPU (the
numpy/scipy oracle port, oracle/; the reference itself is Python and
cannot travel to the GPU box) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Poisson solve time (s), 8.9M-DOF 2mm phantom, rel.res 1e-8; HBM GB/s vs peak"
REL_TOL = 1e-8
FALLBACK_HBM = 6650.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        loaded = [v for v in sm if smax and v > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_workload(name):
    from paper_2010_12879_b200 import workloads
    if name == "C1":
        return workloads.c1()
    if name == "C2":
        return workloads.c2()
    if name == "C3":
        return workloads.c3()
    if name == "C4":
        return workloads.c4()
    raise SystemExit(f"unknown config {name}")


# --------------------------------------------------------------------------
# CPU reference (oracle port) on a bounded sample
# --------------------------------------------------------------------------

def cpu_sample_model():
    """z-slab of the C3 phantom: the full 160x112 cross-section, 100 voxel
    layers from the middle of the body (~1.14M DOFs)."""
    import numpy as np
    from paper_2010_12879_b200 import workloads
    from paper_2010_12879_b200.voxel_model import VoxelModel
    full = workloads.duke_like_model(0.002)
    ids = np.array(full.tissue_ids[:, :, 380:480])
    return VoxelModel(ids.shape, full.spacing, (0.0, 0.0, 0.0), ids, full.tissue_table), full


def cpu_reference(steps, warmup, n_full_dofs=8_913_552, nrhs=2, log=print):
    """Time the reference algorithm (oracle port: assemble_poisson,
    amg_setup hoisted, fgmres_solve to 1e-8) on the slab sample; scale per
    DOF to the full C3 phantom and to both rhs."""
    import numpy as np
    import oracle
    from paper_2010_12879_b200 import workloads
    try:
        from threadpoolctl import threadpool_info
        blas_threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        blas_threads = os.cpu_count() or 1
    model, full = cpu_sample_model()
    kappa = model.voxel_kappa(workloads.FREQ_HZ)
    a = workloads.uniform_potential(model.dims, model.spacing, (0.0, 0.0, 1e-6))
    t0 = time.perf_counter()
    sysd = oracle.assemble(kappa, model.spacing, a)
    t_asm = time.perf_counter() - t0
    cfg = oracle.OracleSolveConfig(rel_tol=REL_TOL)
    t0 = time.perf_counter()
    h = oracle.amg_setup(sysd["matrix"], cfg)
    t_setup = time.perf_counter() - t0
    n_s = sysd["matrix"].shape[0]
    times, its = [], []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        _, it, rel, conv = oracle.fgmres(sysd["matrix"], sysd["rhs"], h, cfg)
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
            its.append(it)
        log(f"[cpu] fgmres sample {k}: {dt:.3f}s, {it} it, rel {rel:.2e}")
    t = statistics.mean(times)
    scale = n_full_dofs / n_s * nrhs
    return {
        "value": t * scale,
        "unit": "s",
        "cores": int(blas_threads),
        "kind": "port",
        "sample": (f"oracle FGMRES(30)+SA-AMG to rel.res {REL_TOL:g} on a 160x112x100 z-slab of the C3 phantom "
                   f"({n_s} DOFs, {statistics.mean(its):.1f} it, {t:.3f}s mean of {len(times)}), scaled x{scale:.2f} "
                   f"= (C3 DOFs / slab DOFs) x 2 rhs; scipy sparse kernels single-threaded, BLAS {blas_threads} threads; "
                   f"setup {t_setup:.2f}s and assembly {t_asm:.2f}s not included"),
        "sample_solve_s": t,
        "sample_dofs": n_s,
        "sample_iters": statistics.mean(its),
        "sample_setup_s": t_setup,
    }


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="host = gloo host-callback transport (testing several ranks on one GPU)")
    ap.add_argument("--replicate-below", type=int, default=100_000,
                    help="coarse levels with fewer rows are solved redundantly on every rank")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    log = (lambda *a: print(*a, file=sys.stderr, flush=True))

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference(args.steps, args.warmup, log=log)
        line = {
            "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["sample_solve_s"] * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Duke-like layered elliptic cylinder, uniform B)",
            "config": {"workload": "C3 Duke-like 2 mm, 8,913,552 DOFs, complex (re/im) rhs", "rel_tol": REL_TOL,
                       "parallelism": "host CPU"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2010_12879_b200 import Session, SolveConfig, _lib

    ndev = torch.cuda.device_count()
    dev = local % ndev if args.transport == "host" else local
    torch.cuda.set_device(dev)
    if world > 1:
        if args.transport == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    w = build_workload(args.config)
    log(f"[bench] rank {rank}: {w.name}, building operator + AMG")
    cfg = SolveConfig(rel_tol=REL_TOL, max_nrhs=2)
    t0 = time.perf_counter()
    sess = Session(w.model, w.frequency_hz, cfg)
    torch.cuda.synchronize()
    setup_wall = time.perf_counter() - t0
    h = sess.hierarchy
    log(f"[bench] dofs {sess.n_dofs} levels {h.level_sizes} setup {h.setup_seconds:.3f}s (device) "
        f"{setup_wall:.3f}s wall incl. assembly")
    if world > 1:
        from paper_2010_12879_b200.distributed import Communicator
        comm = Communicator.nccl() if args.transport == "nccl" else Communicator.host()
        sess.distribute(comm, replicate_below=args.replicate_below)
        log(f"[bench] rank {rank}: planes {sess.plane_range} dofs {sess.dof_range} voxels {sess.vox_range}")
    a_host = torch.from_numpy(np.ascontiguousarray(w.a)).pin_memory()
    a_dev = a_host.to("cuda")
    lib = _lib.load()
    lib.spfd_launch_count.restype = __import__("ctypes").c_int64

    reports = []
    for _ in range(args.warmup):
        _, rep, _ = sess.snapshot(a_dev)
        reports.append(rep)
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = lib.spfd_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")
    e0.record(stream)
    its = []
    for _ in range(args.steps):
        _, rep, _ = sess.snapshot(a_dev)
        its.append(rep.iterations)
        reports.append(rep)
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    launches = (lib.spfd_launch_count() - n0) // args.steps
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        t = t.cuda() if args.transport == "nccl" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop()
    solve_s = statistics.mean(r.solve_seconds for r in reports[args.warmup:])

    # e2e through the public API from pinned host memory
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    v0, v1 = sess.vox_range
    out_host = torch.empty((w.a.shape[0], v1 - v0), dtype=torch.float64, pin_memory=True)
    # single snapshots, each copy in -> solve -> copy out serialised
    e2.record(stream)
    for _ in range(args.steps):
        vox_host, rep = sess.snapshot_host(a_host, out=out_host)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_single_ms = e2.elapsed_time(e3) / args.steps
    if world > 1:
        t = torch.tensor([e2e_single_ms], dtype=torch.float64)
        t = t.cuda() if args.transport == "nccl" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_single_ms = float(t.item())
    # the public streaming API (C5 use case): every step's potentials copied in
    # and voxel field copied out, transfers overlapping the neighbouring solves
    outs = [torch.empty((w.a.shape[0], v1 - v0), dtype=torch.float64, pin_memory=True) for _ in range(args.steps)]
    sess.snapshots_host([a_host] * 2, outs[:2])   # warm the copy streams / buffers
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2.record(stream)
    sess.snapshots_host([a_host] * args.steps, outs)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64)
        t = t.cuda() if args.transport == "nccl" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d, d2h = sess.host_bytes(w.a.shape[0])
    if world > 1:
        t = torch.tensor([h2d, d2h], dtype=torch.float64)
        t = t.cuda() if args.transport == "nccl" else t
        dist.all_reduce(t)
        h2d, d2h = int(t[0].item()), int(t[1].item())

    # roofline of the dominant kernel (fine-level matrix-free SpMV, both rhs)
    import ctypes
    kms, kbytes = ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.spfd_bench_kernel(h.handle, 0, args.kernel_reps, 2, ctypes.byref(kms), ctypes.byref(kbytes),
                                     _lib.stream_ptr()))
    peak, peak_src = _peaks()
    achieved = kbytes.value / (kms.value * 1e-3) / 1e9
    extra = {}
    for which, name in ((1, "fine_presmooth_defect"), (2, "fine_postsmooth"), (3, "vcycle")):
        m_, b_ = ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.spfd_bench_kernel(h.handle, which, args.kernel_reps, 2, ctypes.byref(m_), ctypes.byref(b_),
                                         _lib.stream_ptr()))
        extra[name] = {"ms": round(m_.value, 4)}
        if b_.value > 0:
            extra[name]["gbs"] = round(b_.value / (m_.value * 1e-3) / 1e9, 1)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{args.config}_fine_spmv_dram_bytes")

    it_mean = statistics.mean(its)
    n_dofs = sess.n_dofs
    line = {
        "metric": METRIC,
        "value": ms / 1e3,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (Duke-like layered elliptic cylinder, uniform B re/im, comb-gauge edge potentials)",
        "config": {
            "workload": f"{args.config} {w.name}: {n_dofs} DOFs, complex (re/im) rhs batched",
            "rel_tol": REL_TOL, "method": "AMG-PCG (SA-AMG V(1,1), reference aggregation)",
            "parallelism": (f"z-slab decomposition over {world} GPUs (NCCL send/recv halos, allgathered dots; "
                            f"coarse levels < {args.replicate_below} rows replicated)") if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (fine-level working set >> 126 MB)",
            "step": "rhs assembly + solve to 1e-8 (both rhs) + fused E-field/voxel average",
        },
        "solve_s": solve_s,
        "iterations": it_mean,
        "dof_iter_per_s": n_dofs * it_mean * 2 / (ms / 1e3),
        "setup_s": h.setup_seconds,
        "levels": h.level_sizes,
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "fine-level matrix-free 7-point SpMV (k_span<2,0,true>), both rhs",
                     "bytes_per_launch": kbytes.value, "ms_per_launch": round(kms.value, 4), "peak_source": peak_src},
        "kernels": extra,
        "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "Session.snapshots_host: stream of `steps` snapshots from pinned host memory, each copied in and "
                       "its voxel |E| copied out; transfers overlap the neighbouring snapshots' solves",
                "single_snapshot_s": e2e_single_ms / 1e3},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(args.cpu_steps, 1, log=log)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
