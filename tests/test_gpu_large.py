"""GPU parity at the benchmark configurations (BASELINE.json configs).

C1/C2: the whole snapshot (RHS, AMG-PCG to 1e-8, E-field, voxel average)
against the CPU oracle run on the same inputs (oracle FGMRES to 1e-8):
RHS bit-exact, voxel |E| within max|dE|/max|E| <= 1e-5.
C3 (8.9 M DOFs): size-independent properties -- DOF count, the true
residual recomputed on the host CSR, and the device E-field chain equal bit
for bit to the oracle chain evaluated on the device potential.
"""

import math

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _snapshot(w, tol=1e-8):
    from paper_2010_12879_b200 import Session, SolveConfig
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=tol))
    vox, rep, psi = sess.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
    return sess, vox.cpu().numpy(), rep, psi.cpu().numpy()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_snapshot_matches_oracle(name):
    from paper_2010_12879_b200 import workloads
    w = getattr(workloads, name)()
    sess, vox, rep, psi = _snapshot(w)
    assert rep.converged and rep.rel_residual <= 1e-8
    kappa = w.model.voxel_kappa(w.frequency_hz)
    rhs_dev = sess.op.rhs(w.a).cpu().numpy()
    for c in range(2):
        sysd = oracle.assemble(kappa, w.model.spacing, w.a[c])
        assert sysd["matrix"].shape[0] == sess.n_dofs
        assert np.array_equal(rhs_dev[c], sysd["rhs"])           # bit-exact RHS
        a = sysd["matrix"]
        rel = np.linalg.norm(sysd["rhs"] - a @ psi[c]) / np.linalg.norm(sysd["rhs"])
        assert rel <= 1e-8                                      # independent residual
        cfg = oracle.OracleSolveConfig(rel_tol=1e-8)
        h = oracle.amg_setup(a, cfg)
        if c == 0:   # the device hierarchy is the reference's, level by level
            hd = sess.hierarchy
            assert hd.level_sizes == h["sizes"]
            for lvl in range(len(h["sizes"]) - 1):
                assert np.array_equal(hd.levels[lvl].aggregates, h["levels"][lvl]["agg"]), lvl
        x, its, rel_o, conv = oracle.fgmres(a, sysd["rhs"], h, cfg)
        assert conv
        v = oracle.edge_voltages(w.a[c], x, sysd["dof_to_node"], w.model.dims, w.omega)
        nf = oracle.node_field(v, sysd["w"], w.model.dims, w.model.spacing)
        ref, _ = oracle.voxel_average(nf, kappa)
        err = np.abs(vox[c] - ref).max() / np.abs(ref).max()
        assert err <= 1e-5, err                                 # SURVEY §8(c) contract


@pytest.mark.slow
def test_c3_full_size_properties():
    from paper_2010_12879_b200 import workloads
    w = workloads.c3()
    sess, vox, rep, psi = _snapshot(w)
    assert sess.n_dofs == 8_913_552
    assert sess.n_cond_voxels == 8_711_040
    assert rep.converged
    a = sess.op.csr_host()
    rhs = sess.op.rhs(w.a).cpu().numpy()
    dof_to_node = sess.op.export(1).cpu().numpy()
    w_edges = sess.op.export(0).cpu().numpy()
    kappa = w.model.voxel_kappa(w.frequency_hz)
    for c in range(2):
        rel = np.linalg.norm(rhs[c] - a @ psi[c]) / np.linalg.norm(rhs[c])
        assert rel <= 1e-8, rel
        # the E-field chain on the device potential equals the oracle chain bit for bit
        v = oracle.edge_voltages(w.a[c], psi[c], dof_to_node, w.model.dims, w.omega)
        nf = oracle.node_field(v, w_edges, w.model.dims, w.model.spacing)
        ref, _ = oracle.voxel_average(nf, kappa)
        assert np.array_equal(vox[c], ref)
    # uniform B_z in a z-aligned cylinder: |E| grows with the radius, bounded by pi f B rho_max
    assert np.all(np.isfinite(vox)) and vox.max() < math.pi * w.frequency_hz * 1e-6 * 0.16 * 1.5
