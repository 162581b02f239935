"""Time the FGMRES path (the reference's default solver) on C3 against PCG:
rhs pairs through Session.snapshot and a single rhs through fgmres_solve."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_12879_b200 import Session, SolveConfig, workloads

w = workloads.c3()
for method in ("pcg", "fgmres"):
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-8, method=method))
    a = torch.from_numpy(w.a).cuda()
    for _ in range(2):
        sess.snapshot(a)
    torch.cuda.synchronize()
    t = time.perf_counter()
    n = 3
    for _ in range(n):
        vox, rep, _ = sess.snapshot(a)
    torch.cuda.synchronize()
    print(method, "ms per snapshot pair", (time.perf_counter() - t) / n * 1e3, "iterations", rep.iterations,
          "rel", rep.rel_residuals, flush=True)
    a1 = a[:1].contiguous()
    for _ in range(2):  # warm the single-rhs path (its graph / workspaces)
        sess.snapshot(a1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        vox, rep, _ = sess.snapshot(a1)
    torch.cuda.synchronize()
    print(method, "ms per single-rhs snapshot", (time.perf_counter() - t) / n * 1e3, "iterations", rep.iterations,
          flush=True)
    del sess
