"""GPU parity: the CUDA path (through the C-ABI) against golden vectors
produced by the reference and against the CPU oracle.

Bit-exact: conductances, DOF maps, pinned nodes, the CSR matrix, the RHS,
the stencil product, aggregates, P, R and every Galerkin coarse operator,
and the E-field chain.  Tolerance (stated per test): iterative solutions.
"""

import io
import math

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_cases, golden_csr, golden_model, load_golden

pytestmark = pytest.mark.gpu

MODEL_CASES = golden_cases("model")


def _pkg():
    import paper_2010_12879_b200 as p
    return p


def _same_csr(a, b, exact=True):
    a = sp.csr_matrix(a)
    b = sp.csr_matrix(b)
    a.sort_indices()
    b.sort_indices()
    assert a.shape == b.shape
    assert np.array_equal(a.indptr, b.indptr)
    assert np.array_equal(a.indices, b.indices)
    if exact:
        assert np.array_equal(a.data, b.data), np.abs(a.data - b.data).max()
    else:
        assert np.allclose(a.data, b.data, rtol=1e-14, atol=0)


def _system(d):
    p = _pkg()
    model = golden_model(d)
    grid = p.StaggeredGrid.from_model(model)
    return p.assemble_poisson(model, grid, d["a"], float(d["freq"])), model, grid


@pytest.mark.parametrize("case", MODEL_CASES)
def test_operator_bit_exact(case):
    d = load_golden(case)
    system, _, _ = _system(d)
    assert np.array_equal(system.edge_conductance, d["w"])
    _same_csr(system.matrix, golden_csr(d, "matrix"))
    assert np.array_equal(system.rhs, d["rhs"])
    assert np.array_equal(system.dof_to_node, d["dof_to_node"])
    assert np.array_equal(system.pinned_nodes, d["pinned"])
    assert system.n_components == int(d["n_components"])
    assert system.n_conductive_nodes == int(d["n_conductive"])


@pytest.mark.parametrize("case", MODEL_CASES)
def test_stencil_matches_reference_csr_matvec(case, rng):
    d = load_golden(case)
    system, _, _ = _system(d)
    a = golden_csr(d, "matrix")
    x = rng.standard_normal((2, a.shape[0]))
    y = system.operator.stencil(x).cpu().numpy()
    assert np.array_equal(y[0], a @ x[0])   # same products, same order
    assert np.array_equal(y[1], a @ x[1])


@pytest.mark.parametrize("case", MODEL_CASES)
def test_amg_hierarchy_matches_reference(case):
    p = _pkg()
    d = load_golden(case)
    system, _, _ = _system(d)
    h = p.amg_setup(system.matrix, p.SolveConfig(rel_tol=1e-12))
    assert h.structured
    assert h.level_sizes == list(d["amg_sizes"])
    for l, lv in enumerate(h.levels):
        _same_csr(lv.matrix, golden_csr(d, f"A{l}"))
        if l < h.n_levels - 1:
            assert np.array_equal(lv.aggregates, d[f"agg{l}"])
            _same_csr(lv.prolongation, golden_csr(d, f"P{l}"))
            _same_csr(lv.restriction, golden_csr(d, f"R{l}"))
    # V-cycle: the coarsest solve is a dense inverse here (LU in the reference)
    z = p.v_cycle(h, d["vcycle_in"])
    assert np.linalg.norm(z - d["vcycle_out"]) <= 1e-12 * np.linalg.norm(d["vcycle_out"])


@pytest.mark.parametrize("case", MODEL_CASES)
@pytest.mark.parametrize("method", ["fgmres", "pcg"])
def test_solve_matches_reference(case, method):
    p = _pkg()
    d = load_golden(case)
    if "psi" not in d:
        pytest.skip("zero rhs")
    system, _, _ = _system(d)
    cfg = p.SolveConfig(rel_tol=1e-12, method=method)
    h = p.amg_setup(system.matrix, cfg)
    x, rep = p.solve(system.matrix, system.rhs, h, cfg)
    a = golden_csr(d, "matrix")
    rel = np.linalg.norm(system.rhs - a @ x) / np.linalg.norm(system.rhs)
    assert rep.converged and rel <= 1e-12
    assert rep.rel_residual == pytest.approx(rel, rel=1e-6, abs=1e-15)
    if method == "fgmres":
        assert abs(rep.iterations - int(d["fgmres_iters"])) <= 1
    # tolerance: both sides at 1e-12 -> potentials agree to ~1e-10
    assert np.linalg.norm(x - d["psi"]) <= 1e-9 * np.linalg.norm(d["psi"])


@pytest.mark.parametrize("case", MODEL_CASES)
def test_efield_chain_bit_exact(case):
    p = _pkg()
    d = load_golden(case)
    if "psi" not in d:
        pytest.skip("zero rhs")
    system, model, grid = _system(d)
    omega = float(d["omega"])
    v = p.edge_voltages(d["a"], d["psi"], system, omega)
    assert np.array_equal(v, d["volts"])
    nf = p.node_field_strength(v, grid, model, float(d["freq"]))
    assert np.array_equal(nf.ravel(order="F"), d["node_field"])
    vals, idx = p.voxel_average(nf, grid, model, float(d["freq"]))
    assert np.array_equal(idx, d["vox_idx"])
    assert np.array_equal(vals, d["vox"])
    fused = p.efield_voxel_average(system, d["a"], d["psi"], omega)
    assert np.array_equal(fused, d["vox"])


def test_generic_csr_laplacian():
    p = _pkg()
    d = load_golden("laplacian12")
    a = golden_csr(d, "A0")
    h = p.amg_setup(a)
    assert not h.structured
    assert h.level_sizes == list(d["amg_sizes"])
    assert np.array_equal(h.levels[0].aggregates, d["agg0"])
    _same_csr(h.levels[0].prolongation, golden_csr(d, "P0"))
    _same_csr(h.levels[1].matrix, golden_csr(d, "A1"))
    x, rep = p.fgmres_solve(a, d["b"], h)
    assert rep.converged
    assert np.linalg.norm(x - d["x"]) <= 1e-9 * np.linalg.norm(d["x"])


# --------------------------------------------------------------------------
# the reference's own linsolve tests (test_linsolve.py:20-193), on device
# --------------------------------------------------------------------------

def laplacian_3d(n):
    t = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    e = sp.identity(n)
    return (sp.kron(sp.kron(t, e), e) + sp.kron(sp.kron(e, t), e) + sp.kron(sp.kron(e, e), t)).tocsr()


def cube_system(n, kappa=0.2, spacing=0.002):
    p = _pkg()
    from paper_2010_12879_b200 import workloads
    model = workloads.box_model((n, n, n), kappa, spacing)
    g = p.StaggeredGrid.from_model(model)
    return p.assemble_poisson(model, g, np.zeros(g.n_edges), 85e3)


class TestReferenceLinsolve:
    def test_single_entry(self):
        p = _pkg()
        h = p.amg_setup(sp.csr_matrix(np.array([[2.0]])))
        assert h.level_sizes == [1]
        assert np.allclose(p.v_cycle(h, np.array([4.0])), [2.0])

    def test_level1_band_and_complexity(self):
        p = _pkg()
        a = laplacian_3d(16)
        h = p.amg_setup(a)
        n = a.shape[0]
        assert len(h.level_sizes) >= 2 and n / 20 <= h.level_sizes[1] <= n / 4
        for m in (16, 32):
            assert p.amg_setup(laplacian_3d(m)).operator_complexity() <= 2.5

    def test_sizes_decreasing_and_capped(self):
        p = _pkg()
        h = p.amg_setup(laplacian_3d(12), p.SolveConfig(coarse_cap=100))
        s = h.level_sizes
        assert all(x > y for x, y in zip(s, s[1:])) and s[-1] <= 100

    def test_galerkin_and_transpose(self, rng):
        p = _pkg()
        h = p.amg_setup(laplacian_3d(10))
        lv = h.levels[0]
        x = rng.standard_normal(h.level_sizes[1])
        lhs = h.levels[1].matrix @ x
        rhs = lv.restriction @ (lv.matrix @ (lv.prolongation @ x))
        assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
        diff = (lv.restriction - lv.prolongation.T).tocsr()
        diff.eliminate_zeros()
        assert diff.nnz == 0

    def test_stagnation_direct(self):
        p = _pkg()
        a = sp.diags(np.linspace(1.0, 2.0, 800)).tocsr()
        h = p.amg_setup(a)
        assert h.level_sizes == [800]
        assert np.allclose(p.v_cycle(h, np.ones(800)), 1.0 / np.linspace(1.0, 2.0, 800))

    def test_vcycle_zero_and_homogeneous(self, rng):
        p = _pkg()
        h = p.amg_setup(laplacian_3d(8))
        assert np.all(p.v_cycle(h, np.zeros(512)) == 0.0)
        r = rng.standard_normal(512)
        a1, b1 = p.v_cycle(h, 3.0 * r), 3.0 * p.v_cycle(h, r)
        assert np.linalg.norm(a1 - b1) <= 1e-13 * np.linalg.norm(b1)

    def test_error_contraction_16cube(self, rng):
        p = _pkg()
        system = cube_system(16)
        a = system.matrix
        h = p.amg_setup(a)
        b = rng.standard_normal(a.shape[0])
        exact = np.linalg.solve(a.toarray(), b)
        x = np.zeros_like(b)
        prev = math.sqrt((exact - x) @ (a @ (exact - x)))
        for _ in range(5):
            x = x + p.v_cycle(h, b - a @ x)
            cur = math.sqrt((exact - x) @ (a @ (exact - x)))
            assert cur / prev <= 0.7
            prev = cur

    def test_zero_rhs_and_identity(self, rng):
        p = _pkg()
        a = laplacian_3d(6)
        x, rep = p.fgmres_solve(a, np.zeros(a.shape[0]), p.amg_setup(a))
        assert np.all(x == 0.0) and rep.iterations == 0 and rep.converged
        eye = sp.identity(40, format="csr")
        rhs = rng.standard_normal(40)
        x, rep = p.fgmres_solve(eye, rhs, p.amg_setup(eye))
        assert rep.iterations == 1 and np.allclose(x, rhs, rtol=1e-14)

    def test_dense_oracle_8cube(self, rng):
        p = _pkg()
        system = cube_system(8)
        a = system.matrix
        rhs = rng.standard_normal(a.shape[0])
        for method in ("fgmres", "pcg"):
            x, rep = p.solve(a, rhs, p.amg_setup(a), p.SolveConfig(method=method))
            assert rep.converged
            exact = np.linalg.solve(a.toarray(), rhs)
            assert np.linalg.norm(x - exact) <= 1e-9 * np.linalg.norm(exact)

    def test_max_iters_flagged(self, rng):
        p = _pkg()
        a = laplacian_3d(12)
        rhs = rng.standard_normal(a.shape[0])
        cfg = p.SolveConfig(max_iters=2, rel_tol=1e-14)
        for method in ("fgmres", "pcg"):
            cfg.method = method
            x, rep = p.solve(a, rhs, p.amg_setup(a, cfg), cfg)
            assert not rep.converged and rep.iterations == 2 and np.all(np.isfinite(x))
            assert np.linalg.norm(rhs - a @ x) < np.linalg.norm(rhs)

    def test_nonfinite_rhs(self):
        p = _pkg()
        a = laplacian_3d(4)
        rhs = np.zeros(a.shape[0])
        rhs[0] = np.nan
        with pytest.raises(p.SolverError):
            p.fgmres_solve(a, rhs, p.amg_setup(a))

    def test_bitwise_deterministic(self, rng):
        p = _pkg()
        system = cube_system(10)
        rhs = rng.standard_normal(system.n_dofs)
        for method in ("fgmres", "pcg"):
            cfg = p.SolveConfig(method=method)
            h = p.amg_setup(system.matrix, cfg)
            x1, r1 = p.solve(system.matrix, rhs, h, cfg)
            x2, r2 = p.solve(system.matrix, rhs, h, cfg)
            assert np.array_equal(x1, x2) and r1.iterations == r2.iterations

    def test_trace_and_report(self, rng):
        p = _pkg()
        a = laplacian_3d(8)
        stream = io.StringIO()
        cfg = p.SolveConfig(trace=stream)
        _, rep = p.fgmres_solve(a, rng.standard_normal(a.shape[0]), p.amg_setup(a, cfg), cfg)
        lines = stream.getvalue().strip().splitlines()
        assert lines and all(ln.startswith("iter ") and "rel_resid" in ln for ln in lines)
        assert rep.level_sizes[0] == a.shape[0]
        assert rep.peak_matrix_memory_bytes > a.data.nbytes
        assert rep.setup_seconds >= 0.0 and rep.solve_seconds > 0.0

    def test_nonpositive_diagonal(self):
        p = _pkg()
        a = sp.csr_matrix(np.array([[1.0, 0.0], [0.0, -1.0]]))
        with pytest.raises(p.SolverError):
            p.amg_setup(a)


def test_empty_system():
    p = _pkg()
    from paper_2010_12879_b200.voxel_model import ConductivitySamples, Tissue, VoxelModel
    m = VoxelModel((2, 2, 2), (0.002,) * 3, (0.0,) * 3, np.zeros((2, 2, 2), dtype=np.uint16),
                   {0: Tissue("free_space", ConductivitySamples.constant(0.0))})
    g = p.StaggeredGrid.from_model(m)
    with pytest.raises(p.EmptySystemError):
        p.assemble_poisson(m, g, np.zeros(g.n_edges), 85e3)
