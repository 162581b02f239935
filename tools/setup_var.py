"""Setup-time spread on C3: one operator, N hierarchy setups (device-timed)."""
import os, statistics, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_12879_b200 import Session, SolveConfig, amg_setup, workloads
from paper_2010_12879_b200.pipeline import _OpRef
w = workloads.c3()
cfg = SolveConfig(rel_tol=1e-8, max_nrhs=2)
sess = Session(w.model, w.frequency_hz, cfg)
t = [sess.hierarchy.setup_seconds]
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    h = amg_setup(_OpRef(sess.op), cfg)
    t.append(h.setup_seconds)
    del h
print(json.dumps({"first_s": t[0], "repeats_s": t[1:], "median_repeat_s": statistics.median(t[1:]),
                  "keep_mb": os.environ.get("SPFD_POOL_KEEP_MB", "4096")}))
