import sys, os, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import load_golden, golden_csr, golden_model
import paper_2010_12879_b200 as p
import oracle
d = load_golden("box16_uniform")
model = golden_model(d)
g = p.StaggeredGrid.from_model(model)
system = p.assemble_poisson(model, g, d["a"], float(d["freq"]))
a = golden_csr(d, "matrix")
for structured in (True, False):
    h = p.amg_setup(system.matrix if structured else a, p.SolveConfig(rel_tol=1e-12))
    z = p.v_cycle(h, d["vcycle_in"])
    print("structured", structured, h.level_sizes, np.linalg.norm(z - d["vcycle_out"]) / np.linalg.norm(d["vcycle_out"]))
# 2-level variants via coarse_cap
for cap in (700, 40):
    h = p.amg_setup(a, p.SolveConfig(coarse_cap=cap))
    ho = oracle.amg_setup(a, oracle.OracleSolveConfig(coarse_cap=cap))
    z = p.v_cycle(h, d["vcycle_in"]); zo = oracle.v_cycle(ho, d["vcycle_in"])
    print("csr cap", cap, h.level_sizes, np.linalg.norm(z - zo) / np.linalg.norm(zo))
    h = p.amg_setup(system.matrix, p.SolveConfig(coarse_cap=cap))
    z = p.v_cycle(h, d["vcycle_in"])
    print("st cap", cap, h.level_sizes, np.linalg.norm(z - zo) / np.linalg.norm(zo))
