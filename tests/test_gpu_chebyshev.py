"""Chebyshev smoother (north_star (2): "Chebyshev/Jacobi smoother"; the
reference itself has damped Jacobi only, linsolve.py:184-197).

The device V-cycle with the Chebyshev smoother is checked against the
oracle's restatement (oracle.with_chebyshev, Saad alg. 12.1 on
[beta/5, beta], beta = 1.1 lambda_max) fed the device's per-level
lambda_max estimates: <= 1e-11 relative (the fine level's transfers are
matrix-free on the device, CSR in the oracle).  The estimates themselves
are bounded against the exact lambda_max(D^-1 A) (power iteration
approaches it from below).  Krylov solves with the Chebyshev V-cycle meet
the tolerance with at most the Jacobi iteration count; the graph and
host-loop PCG give the same bits."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import golden_cases, golden_model, load_golden

pytestmark = pytest.mark.gpu

CASES = golden_cases("model")


def _setup(d, **kw):
    import paper_2010_12879_b200 as p
    model = golden_model(d)
    grid = p.StaggeredGrid.from_model(model)
    system = p.assemble_poisson(model, grid, d["a"], float(d["freq"]))
    cfg = p.SolveConfig(rel_tol=1e-11, smoother="chebyshev", **kw)
    return p, system, cfg, p.amg_setup(system.matrix, cfg)


def _lmax_exact(a):
    d = 1.0 / np.sqrt(a.diagonal())
    s = sp.diags(d) @ a @ sp.diags(d)
    if s.shape[0] < 400:
        return float(np.linalg.eigvalsh(s.toarray()).max())
    return float(spla.eigsh(s, k=1, which="LA", tol=1e-10)[0][0])


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("degree,sweeps", [(2, (1, 1)), (3, (1, 1)), (2, (2, 1))])
def test_vcycle_matches_oracle(case, degree, sweeps, rng):
    import oracle
    d = load_golden(case)
    p, system, cfg, h = _setup(d, chebyshev_degree=degree, pre_sweeps=sweeps[0], post_sweeps=sweeps[1])
    if h.n_levels < 2:
        pytest.skip("single level: the dense inverse, no smoother")
    assert h.smoother == "chebyshev" and h.chebyshev_degree == degree
    assert len(h.chebyshev_lmax) == h.n_levels - 1
    ho = oracle.amg_setup(system.matrix, oracle.OracleSolveConfig(pre_sweeps=sweeps[0], post_sweeps=sweeps[1]))
    assert ho["sizes"] == h.level_sizes
    hc = oracle.with_chebyshev(ho, h.chebyshev_lmax, degree)
    for _ in range(2):
        r = rng.standard_normal(h.n)
        z = p.v_cycle(h, r)
        zo = oracle.v_cycle(hc, r)
        assert np.linalg.norm(z - zo) <= 1e-11 * np.linalg.norm(zo)


@pytest.mark.parametrize("case", CASES)
def test_lmax_estimates(case):
    import oracle
    d = load_golden(case)
    p, system, cfg, h = _setup(d)
    ho = oracle.amg_setup(system.matrix)
    for l, est in enumerate(h.chebyshev_lmax):
        exact = _lmax_exact(ho["levels"][l]["A"])
        assert 0.85 * exact <= est <= exact * (1 + 1e-9), (l, est, exact)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("method", ["pcg", "fgmres"])
def test_solve_converges(case, method):
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    _, system, _, h = _setup(d)
    if not np.any(system.rhs):
        pytest.skip("zero rhs")
    cfg = p.SolveConfig(rel_tol=1e-11, smoother="chebyshev", method=method)
    x, rep = p.solve(system.matrix, system.rhs, h, cfg)
    assert rep.converged and rep.rel_residual <= 1e-11
    res = np.linalg.norm(system.rhs - system.matrix @ x) / np.linalg.norm(system.rhs)
    assert res <= 1e-11
    hj = p.amg_setup(system.matrix, p.SolveConfig(rel_tol=1e-11))
    xj, repj = p.solve(system.matrix, system.rhs, hj, p.SolveConfig(rel_tol=1e-11, method=method))
    assert rep.iterations <= repj.iterations + 1
    assert np.linalg.norm(x - xj) <= 1e-8 * np.linalg.norm(xj)


def test_graph_matches_host_loop_and_snapshot():
    import torch
    import paper_2010_12879_b200 as p
    from paper_2010_12879_b200 import Session, _lib, workloads
    w = workloads.c1()
    outs = []
    try:
        for mode in (1, 0):
            _lib.check(_lib.lib().spfd_set_pcg_graph(mode))
            sess = Session(w.model, w.frequency_hz, p.SolveConfig(rel_tol=1e-10, smoother="chebyshev"))
            vox, rep, psi = sess.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
            assert rep.converged
            outs.append((rep.iterations, psi.cpu().numpy(), vox.cpu().numpy()))
    finally:
        _lib.check(_lib.lib().spfd_set_pcg_graph(-1))
    assert outs[0][0] == outs[1][0] and np.array_equal(outs[0][1], outs[1][1])
    sj = Session(w.model, w.frequency_hz, p.SolveConfig(rel_tol=1e-10))
    vj, repj, _ = sj.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
    assert outs[0][0] < repj.iterations
    e = np.abs(outs[0][2] - vj.cpu().numpy()).max() / np.abs(vj.cpu().numpy()).max()
    assert e <= 1e-7, e
