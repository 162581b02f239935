import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2010_12879_b200 as p
from paper_2010_12879_b200 import workloads
w = workloads.c1(48)
grid = p.StaggeredGrid.from_model(w.model)
system = p.assemble_poisson(w.model, grid, w.a[0], w.frequency_hz)
h = p.amg_setup(system.matrix, p.SolveConfig(rel_tol=1e-8))
rng = np.random.default_rng(1)
r = rng.standard_normal((2, h.n))
z = p.v_cycle(h, r)
x, rep = p.solve(system.matrix, system.rhs, h, p.SolveConfig(rel_tol=1e-10))
np.save(sys.argv[1], np.concatenate([z.ravel(), x.ravel(), [rep.iterations]]))
print(h.level_sizes, rep.iterations)
