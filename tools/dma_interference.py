"""Does a concurrent H2D stream slow the solve?  C3 snapshot loop timed alone
and while a copy stream keeps moving the snapshot's input from pinned host
memory (as Session.snapshots_host does)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2010_12879_b200 import Session, SolveConfig, workloads
w = workloads.c3()
sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-8, max_nrhs=2))
a_host = torch.from_numpy(np.ascontiguousarray(w.a)).pin_memory()
a_dev = a_host.to("cuda")
dst = torch.empty_like(a_dev)
for _ in range(3):
    sess.snapshot(a_dev)
torch.cuda.synchronize()
def timed(copy):
    cs = torch.cuda.Stream()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if copy:
        with torch.cuda.stream(cs):
            for _ in range(40):
                dst.copy_(a_host, non_blocking=True)
    e0.record(st)
    for _ in range(10):
        sess.snapshot(a_dev)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10
r = {"alone_ms": timed(False), "with_h2d_ms": timed(True), "alone2_ms": timed(False)}
print(json.dumps(r))
