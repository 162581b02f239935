"""GPU A/B of the fine-level stencil kernels: flat and with the tile's L2
bulk prefetch (every stencil mode bit-identical, so V-cycles give the same
bits; Krylov solves agree to tolerance), plus the graph / host-loop and
block / MGS solver A/B tests.

Every stencil mode must be bit-identical between the two kernels, so a
V-cycle (pre-smooth+defect, restriction input, matrix-free prolongation,
post-smooth: modes 1-4) gives the same bits.  A Krylov solve is compared to
tolerance only: its dot products are reduced per CTA, and the two kernels
cut the positions into CTAs differently (fixed order within each kernel, so
each is bitwise reproducible on its own).  Cases: every golden phantom
(spheres, cylinders, cavities, separate bodies), C1 and C2, with sweep
variants."""

import numpy as np
import pytest
import torch

from conftest import golden_cases, golden_model, load_golden

pytestmark = pytest.mark.gpu

FLAT, PF = 2, 3
KINDS = (PF, FLAT)


def _set_kernel(kind):
    from paper_2010_12879_b200 import _lib
    _lib.check(_lib.lib().spfd_set_fine_kernel(kind))


@pytest.fixture(autouse=True)
def _restore():
    yield
    _set_kernel(-1)


def _hier(model, freq, a, cfg):
    import paper_2010_12879_b200 as p
    grid = p.StaggeredGrid.from_model(model)
    system = p.assemble_poisson(model, grid, a, freq)
    return system, p.amg_setup(system.matrix, cfg)


@pytest.mark.parametrize("case", golden_cases("model"))
@pytest.mark.parametrize("sweeps", [(1, 1), (2, 2), (1, 0)])
def test_vcycle_bitwise(case, sweeps, rng):
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    cfg = p.SolveConfig(rel_tol=1e-10, pre_sweeps=sweeps[0], post_sweeps=sweeps[1])
    system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
    r = rng.standard_normal((2, h.n))
    out = []
    for kind in KINDS:
        _set_kernel(kind)
        out.append(p.v_cycle(h, r))
    for k in range(1, len(KINDS)):
        assert np.array_equal(out[0], out[k]), KINDS[k]


@pytest.mark.parametrize("case", golden_cases("model"))
@pytest.mark.parametrize("method", ["pcg", "fgmres"])
def test_solve_agrees(case, method):
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    cfg = p.SolveConfig(rel_tol=1e-12, method=method)
    system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
    if not np.any(system.rhs):
        pytest.skip("zero rhs")
    res = []
    for kind in KINDS:
        _set_kernel(kind)
        x, rep = p.solve(system.matrix, system.rhs, h, cfg)
        assert rep.converged
        res.append((rep.iterations, x))
    for k in range(1, len(KINDS)):
        assert abs(res[0][0] - res[k][0]) <= 1
        assert np.linalg.norm(res[0][1] - res[k][1]) <= 1e-10 * np.linalg.norm(res[0][1])


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_configs_vcycle_bitwise_and_snapshot(name, rng):
    import paper_2010_12879_b200 as p
    from paper_2010_12879_b200 import Session, workloads
    w = getattr(workloads, name)()
    cfg = p.SolveConfig(rel_tol=1e-8)
    system, h = _hier(w.model, w.frequency_hz, w.a[0], cfg)
    r = rng.standard_normal((2, h.n))
    z = []
    snaps = []
    for kind in KINDS:
        _set_kernel(kind)
        z.append(p.v_cycle(h, r))
        sess = Session(w.model, w.frequency_hz, cfg)
        vox, rep, _ = sess.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
        snaps.append((rep.iterations, vox.cpu().numpy()))
    for k in range(1, len(KINDS)):
        assert np.array_equal(z[0], z[k]), KINDS[k]
    for k in range(1, len(KINDS)):
        assert abs(snaps[0][0] - snaps[k][0]) <= 1
        e = np.abs(snaps[0][1] - snaps[k][1]).max() / np.abs(snaps[0][1]).max()
        assert e <= 1e-6, e


def _set_graph(mode):
    from paper_2010_12879_b200 import _lib
    _lib.check(_lib.lib().spfd_set_pcg_graph(mode))


@pytest.mark.parametrize("case", golden_cases("model"))
def test_pcg_graph_matches_host_loop(case):
    """The graph-captured PCG (device-side WHILE node) runs the host loop's
    kernels in the same order: same iteration count, same bits, same trace."""
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    out = []
    try:
        for mode in (0, 1):
            _set_graph(mode)
            import io
            trace = io.StringIO()
            cfg = p.SolveConfig(rel_tol=1e-11, method="pcg", trace=trace)
            system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
            if not np.any(system.rhs):
                pytest.skip("zero rhs")
            b = np.stack([system.rhs, 0.25 * system.rhs[::-1].copy()])
            x, rep = p.solve(system.matrix, b, h, cfg)
            out.append((rep.iterations, x, trace.getvalue(), rep.converged))
    finally:
        _set_graph(-1)
    assert out[0][0] == out[1][0] and out[0][3] and out[1][3]
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


def test_pcg_graph_max_iters_and_restart():
    import paper_2010_12879_b200 as p
    d = load_golden(golden_cases("model")[0])
    for mode in (0, 1):
        _set_graph(mode)
        try:
            cfg = p.SolveConfig(rel_tol=1e-14, max_iters=3, method="pcg")
            system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
            x, rep = p.solve(system.matrix, system.rhs, h, cfg)
            assert rep.iterations == 3 and not rep.converged
        finally:
            _set_graph(-1)


@pytest.mark.parametrize("case", golden_cases("model"))
def test_fgmres_batched_pair_matches_single(case):
    """FGMRES on a rhs pair (one Arnoldi process, batched V-cycle/SpMV, CGS2
    block orthogonalisation) against two single-rhs solves (the reference's
    MGS): iteration counts within one, potentials within 1e-9, both true
    residuals met, trace per rhs."""
    import io
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    cfg = p.SolveConfig(rel_tol=1e-12, method="fgmres")
    system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
    if not np.any(system.rhs):
        pytest.skip("zero rhs")
    b = np.stack([system.rhs, 0.25 * system.rhs[::-1].copy()])
    tr = io.StringIO()
    cfg_t = p.SolveConfig(rel_tol=1e-12, method="fgmres", trace=tr)
    x2, rep2 = p.solve(system.matrix, b, h, cfg_t)
    assert rep2.converged and rep2.rel_residual <= 1e-12
    assert tr.getvalue().count("iter") == rep2.iterations
    its = []
    for c in range(2):
        x1, rep1 = p.solve(system.matrix, b[c], h, cfg)
        assert rep1.converged
        its.append(rep1.iterations)
        assert np.linalg.norm(x2[c] - x1) <= 1e-9 * np.linalg.norm(x1)
    assert abs(rep2.iterations - max(its)) <= 1


@pytest.mark.parametrize("case", golden_cases("model"))
def test_fgmres_block_single_rhs_matches_mgs(case, monkeypatch):
    """Single-rhs FGMRES: the block (Gram-corrected CGS2) Arnoldi against the
    reference's modified Gram-Schmidt (SPFD_FGMRES_BATCH=0)."""
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    cfg = p.SolveConfig(rel_tol=1e-12, method="fgmres")
    system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
    if not np.any(system.rhs):
        pytest.skip("zero rhs")
    xb, rb = p.solve(system.matrix, system.rhs, h, cfg)
    monkeypatch.setenv("SPFD_FGMRES_BATCH", "0")
    xm, rm = p.solve(system.matrix, system.rhs, h, cfg)
    assert rb.converged and rm.converged
    assert abs(rb.iterations - rm.iterations) <= 1
    assert np.linalg.norm(xb - xm) <= 1e-9 * np.linalg.norm(xm)


def test_level1_morton_renumbering_is_bitwise_neutral(monkeypatch, rng):
    """The solve layout renumbers level 1 along a Morton curve (rows and
    columns permuted, each row's entry order kept): V-cycle and PCG give the
    same bits as the reference numbering (SPFD_MORTON=0), and the exported
    level-1 matrices are the reference's."""
    import paper_2010_12879_b200 as p
    from paper_2010_12879_b200 import workloads
    w = workloads.c1(40)
    grid = p.StaggeredGrid.from_model(w.model)
    system = p.assemble_poisson(w.model, grid, w.a[0], w.frequency_hz)
    cfg = p.SolveConfig(rel_tol=1e-10)
    r = rng.standard_normal((2, system.matrix.shape[0]))
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SPFD_MORTON", flag)
        h = p.amg_setup(system.matrix, cfg)
        assert h.n_levels >= 3
        z = p.v_cycle(h, r)
        x, rep = p.solve(system.matrix, system.rhs, h, cfg)
        lv = h.levels[1]
        out.append((z, x, rep.iterations, lv.matrix.toarray() if lv.matrix.shape[0] < 4000 else lv.matrix,
                    lv.prolongation, lv.restriction))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1]) and out[0][2] == out[1][2]
    for k in (4, 5):
        a, b = out[0][k], out[1][k]
        assert (a != b).nnz == 0
    a, b = out[0][3], out[1][3]
    assert np.array_equal(a, b) if isinstance(a, np.ndarray) else (a != b).nnz == 0


@pytest.mark.parametrize("case", golden_cases("model"))
@pytest.mark.parametrize("nrhs", [1, 2])
def test_fgmres_graph_matches_host_loop(case, nrhs, monkeypatch):
    """FGMRES with the restart cycle as one device graph (Givens rotations,
    convergence decisions and the back substitution on the device) against
    the host-driven loop: same iteration counts, same trace length, the same
    potentials to rounding, true residuals met; repeated graph solves are
    bitwise identical."""
    import io
    import paper_2010_12879_b200 as p
    d = load_golden(case)
    cfg = p.SolveConfig(rel_tol=1e-12, method="fgmres")
    system, h = _hier(golden_model(d), float(d["freq"]), d["a"], cfg)
    if not np.any(system.rhs):
        pytest.skip("zero rhs")
    b = np.stack([system.rhs, 0.25 * system.rhs[::-1].copy()])[:nrhs]
    out = []
    for mode in ("1", "0", "1"):
        monkeypatch.setenv("SPFD_FGMRES_GRAPH", mode)
        tr = io.StringIO()
        x, rep = p.solve(system.matrix, b, h, p.SolveConfig(rel_tol=1e-12, method="fgmres", trace=tr))
        assert rep.converged and rep.rel_residual <= 1e-12
        out.append((rep.iterations, x, tr.getvalue().count("iter")))
    assert out[0][0] == out[1][0] and out[0][2] == out[1][2] == out[0][0]
    assert np.linalg.norm(out[0][1] - out[1][1]) <= 1e-12 * np.linalg.norm(out[1][1])
    assert np.array_equal(out[0][1], out[2][1])


def test_fgmres_graph_restarts_and_max_iters(monkeypatch):
    """Restart cycles (restart=3 needs several) and the max_iters flag on the
    device FGMRES, against the host loop."""
    import paper_2010_12879_b200 as p
    from paper_2010_12879_b200 import workloads
    w = workloads.c1(24)
    grid = p.StaggeredGrid.from_model(w.model)
    system = p.assemble_poisson(w.model, grid, w.a[0], w.frequency_hz)
    h = p.amg_setup(system.matrix, p.SolveConfig())
    for cfg in (p.SolveConfig(rel_tol=1e-12, method="fgmres", restart=3),
                p.SolveConfig(rel_tol=1e-14, method="fgmres", max_iters=4, restart=3)):
        res = []
        for mode in ("1", "0"):
            monkeypatch.setenv("SPFD_FGMRES_GRAPH", mode)
            x, rep = p.solve(system.matrix, system.rhs, h, cfg)
            res.append((rep.iterations, rep.converged, x))
        assert res[0][:2] == res[1][:2]
        assert np.linalg.norm(res[0][2] - res[1][2]) <= 1e-10 * np.linalg.norm(res[1][2])
    assert res[0][0] == 4 and not res[0][1]


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_fine_transfers_csr_vs_matrix_free(name, monkeypatch, rng):
    """The fine-level restriction R d and prolongation x0 + P e run on the
    reference's R = P^T and P as CSRs over span positions by default
    (SPFD_RSPAN / SPFD_PSPAN) and matrix-free through the aggregates when
    disabled: the same V-cycle to rounding (different summation orders), the
    same PCG iteration counts and solutions to the solve tolerance; the info
    flags report the layout in use."""
    import paper_2010_12879_b200 as p
    from paper_2010_12879_b200 import workloads
    w = getattr(workloads, name)()
    grid = p.StaggeredGrid.from_model(w.model)
    system = p.assemble_poisson(w.model, grid, w.a[0], w.frequency_hz)
    cfg = p.SolveConfig(rel_tol=1e-10)
    r = rng.standard_normal((2, system.matrix.shape[0]))
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SPFD_RSPAN", flag)
        monkeypatch.setenv("SPFD_PSPAN", flag)
        h = p.amg_setup(system.matrix, cfg)
        assert h.restriction_csr == (flag == "1") and h.prolongation_csr == (flag == "1")
        z = p.v_cycle(h, r)
        x, rep = p.solve(system.matrix, system.rhs, h, cfg)
        assert rep.converged
        out[flag] = (z, x, rep.iterations)
    z1, x1, i1 = out["1"]
    z0, x0, i0 = out["0"]
    assert np.linalg.norm(z1 - z0) <= 1e-13 * np.linalg.norm(z0)
    assert i1 == i0
    assert np.linalg.norm(x1 - x0) <= 1e-9 * np.linalg.norm(x0)
