"""C3 setup time (operator + AMG hierarchy on device), repeated in one process."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_12879_b200 import Session, SolveConfig, workloads
m = workloads.duke_like_model(0.002)
for k in range(3):
    t = time.perf_counter()
    s = Session(m, workloads.FREQ_HZ, SolveConfig(rel_tol=1e-8))
    torch.cuda.synchronize()
    print(os.environ.get("TAG", ""), "setup device", round(s.hierarchy.setup_seconds, 3), "wall", round(time.perf_counter() - t, 3), flush=True)
    del s
