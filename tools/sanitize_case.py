"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): operator + AMG setup (union-find components,
event-driven aggregation, ESC SpGEMM), the graph PCG snapshot, the device
FGMRES graph and host loop, a generic-CSR hierarchy, and the field chain
(interpolate, batched cleaning, comb gauge)."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2010_12879_b200 as p  # noqa: E402
from paper_2010_12879_b200 import Session, SolveConfig, workloads  # noqa: E402


def step(msg):
    print(f"[sanitize] {msg}", flush=True)


STEPS = set((os.environ.get("SANITIZE_STEPS") or "snapshot,generic,field").split(","))


def main():
    sess = vox = psi = None
    if "snapshot" in STEPS:
        step("snapshot: setup")
        w = workloads.small_box(12)
        sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10))
        a = torch.from_numpy(w.a).cuda()
        step("snapshot: solve")
        vox, rep, psi = sess.snapshot(a, keep_psi=True)
        assert rep.converged
    w2 = workloads.c2(24)   # layered block + free space + dipole
    grid = p.StaggeredGrid.from_model(w2.model)
    system = h = hc = x = r = ops = None
    if "generic" in STEPS:
        step("generic solves")
        system = p.assemble_poisson(w2.model, grid, w2.a[0], w2.frequency_hz)
        step("generic: amg_setup")
        h = p.amg_setup(system.matrix, SolveConfig())
        # SANITIZE_NO_GRAPHS=1: host-loop Krylov only (the graph and host-loop paths
        # run the same kernels; tested bit-identical in tests/test_gpu_kernels.py)
        for mode in (("0",) if os.environ.get("SANITIZE_NO_GRAPHS") else ("1", "0")):
            step(f"generic: fgmres graph={mode}")
            os.environ["SPFD_FGMRES_GRAPH"] = mode
            x, r = p.solve(system.matrix, np.stack([system.rhs, 0.5 * system.rhs]), h,
                           SolveConfig(rel_tol=1e-10, method="fgmres"))
            assert r.converged
        step("generic: pcg")
        x, r = p.solve(system.matrix, system.rhs, h, SolveConfig(rel_tol=1e-10, method="pcg"))
        step("generic: csr setup + fgmres")
        hc = p.amg_setup(system.matrix.tocsr().copy(), SolveConfig())   # generic CSR path
        x, r = p.fgmres_solve(system.matrix, system.rhs, hc, SolveConfig(rel_tol=1e-10))
        assert r.converged
    if "field" in STEPS:
        step("field chain")
        from paper_2010_12879_b200.field_source import CoilSpec, FieldOps, Lattice, coil_field
        ops = FieldOps(grid, SolveConfig())
        lat = Lattice.covering(grid, (5, 5, 5))
        coil = CoilSpec(center=(0.03, 0.03, -0.05), axis=(0.0, 0.0, 1.0), radius_m=0.05, current_a=10.0,
                        segments=64)
        b = torch.from_numpy(coil_field(coil, lat.points())).cuda()
        f = torch.stack([ops.interpolate(lat, b), ops.interpolate(lat, 0.5 * b)])
        fc = ops.clean(f, 1e-10)
        for c in range(2):
            ops.gauge(fc[c], 1e-10)
    torch.cuda.synchronize()
    # release every library handle before exit so the leak check sees only
    # real leaks (interpreter shutdown does not run these destructors)
    import gc
    from paper_2010_12879_b200 import dosimetry, field_source
    del sess, h, hc, ops, system, x, r, vox, psi
    field_source._FIELD_CACHE.clear()
    dosimetry._OP_CACHE.clear()
    gc.collect()
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
