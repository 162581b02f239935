import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2010_12879_b200 import Session, SolveConfig, workloads, _lib
kind, graph, name = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
_lib.check(_lib.lib().spfd_set_fine_kernel(kind))
_lib.check(_lib.lib().spfd_set_pcg_graph(graph))
w = getattr(workloads, name)()
for rep_i in range(2):
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-8))
    print("session", flush=True)
    vox, rep, _ = sess.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
    torch.cuda.synchronize()
    print(kind, graph, name, rep.iterations, rep.rel_residual, flush=True)
