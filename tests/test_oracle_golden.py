"""CPU: pin the oracle against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  Integer/index data and every
floating value the reference computes with a fixed operation order must
match bit for bit; iterative solutions to the solve tolerance."""

import math

import numpy as np
import pytest

import oracle
from conftest import golden_cases, golden_csr, golden_kappa, load_golden

MODEL_CASES = golden_cases("model")


def _same_csr(a, b):
    a.sort_indices()
    b.sort_indices()
    assert a.shape == b.shape
    assert np.array_equal(a.indptr, b.indptr)
    assert np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)


@pytest.mark.parametrize("case", MODEL_CASES)
def test_conductance_and_assembly_bit_exact(case):
    d = load_golden(case)
    kappa = golden_kappa(d)
    sysd = oracle.assemble(kappa, d["spacing"], d["a"])
    assert np.array_equal(sysd["w"], d["w"])
    _same_csr(sysd["matrix"], golden_csr(d, "matrix"))
    assert np.array_equal(sysd["rhs"], d["rhs"])
    assert np.array_equal(sysd["dof_to_node"], d["dof_to_node"])
    assert np.array_equal(sysd["pinned"], d["pinned"])
    assert np.array_equal(sysd["labels"], d["labels"])
    assert sysd["n_components"] == int(d["n_components"])
    # the RHS-only helper (second rhs of a pair without re-assembly) is the same bincount
    assert np.array_equal(oracle.assemble_rhs(sysd, kappa.shape, d["a"]), d["rhs"])


@pytest.mark.parametrize("case", MODEL_CASES)
def test_amg_hierarchy_bit_exact(case):
    d = load_golden(case)
    a = golden_csr(d, "matrix")
    h = oracle.amg_setup(a, oracle.OracleSolveConfig(rel_tol=1e-12))
    assert h["sizes"] == list(d["amg_sizes"])
    for l, lv in enumerate(h["levels"]):
        _same_csr(lv["A"], golden_csr(d, f"A{l}"))
        if lv["P"] is not None:
            assert np.array_equal(lv["agg"], d[f"agg{l}"])
            _same_csr(lv["P"], golden_csr(d, f"P{l}"))
            _same_csr(lv["R"], golden_csr(d, f"R{l}"))
    # the V-cycle itself (same LAPACK factorisation -> identical)
    z = oracle.v_cycle(h, d["vcycle_in"])
    assert np.allclose(z, d["vcycle_out"], rtol=1e-13, atol=0)


@pytest.mark.parametrize("case", [c for c in MODEL_CASES if c != "box6_random" or True])
def test_solve_and_efield(case):
    d = load_golden(case)
    if "psi" not in d:
        pytest.skip("zero rhs case")
    a = golden_csr(d, "matrix")
    cfg = oracle.OracleSolveConfig(rel_tol=1e-12)
    h = oracle.amg_setup(a, cfg)
    x, its, rel, conv = oracle.fgmres(a, d["rhs"], h, cfg)
    assert conv and rel <= 1e-12
    assert its == int(d["fgmres_iters"])
    assert np.array_equal(x, d["psi"])  # same ops, same order
    # PCG with the same V-cycle reaches the same solution
    xp, itp, relp, convp = oracle.pcg(a, d["rhs"], h, cfg)
    assert convp and np.linalg.norm(xp - d["psi"]) <= 1e-9 * np.linalg.norm(d["psi"])
    # E-field chain from the golden potential: bit-exact
    dims = tuple(int(v) for v in d["dims"])
    v = oracle.edge_voltages(d["a"], d["psi"], d["dof_to_node"], dims, float(d["omega"]))
    assert np.array_equal(v, d["volts"])
    nf = oracle.node_field(v, d["w"], dims, d["spacing"])
    assert np.array_equal(nf.ravel(order="F"), d["node_field"])
    vals, idx = oracle.voxel_average(nf, golden_kappa(d))
    assert np.array_equal(idx, d["vox_idx"])
    assert np.array_equal(vals, d["vox"])


def test_laplacian_hierarchy_and_solve():
    d = load_golden("laplacian12")
    import scipy.sparse as sp
    n = 12
    t = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    e = sp.identity(n)
    a = (sp.kron(sp.kron(t, e), e) + sp.kron(sp.kron(e, t), e) + sp.kron(sp.kron(e, e), t)).tocsr()
    h = oracle.amg_setup(a)
    assert h["sizes"] == list(d["amg_sizes"])
    assert np.array_equal(h["levels"][0]["agg"], d["agg0"])
    _same_csr(h["levels"][1]["A"], golden_csr(d, "A1"))
    x, its, rel, conv = oracle.fgmres(a, d["b"], h)
    assert conv and np.array_equal(x, d["x"])


def test_kappa_log_interpolation():
    # two_blobs tissue 1 is sampled at 1 kHz / 1 MHz; 85 kHz is interpolated
    d = load_golden("two_blobs")
    k = oracle.kappa_at([1e3, 1e6], [0.1, 0.4], 85e3)
    assert k == d["lut"][1]
    assert oracle.kappa_at([1e3], [0.3], 5.0) == 0.3


def test_comb_gauge_reproduces_fluxes():
    dims = (5, 4, 3)
    s = (0.002, 0.003, 0.004)
    flux = oracle.uniform_face_fluxes(dims, s, (0.3e-6, -0.7e-6, 1e-6))
    a = oracle.comb_gauge(dims, flux)
    # circulation of a around every z-face equals its flux
    nx, ny, nz = dims
    off, cnt = oracle.edge_offsets(dims)
    ax = a[:cnt[0]].reshape((nx, ny + 1, nz + 1), order="F")
    ay = a[off[1]:off[1] + cnt[1]].reshape((nx + 1, ny, nz + 1), order="F")
    circ = ax[:, :-1, :] + ay[1:, :, :] - ax[:, 1:, :] - ay[:-1, :, :]
    assert np.allclose(circ, 1e-6 * s[0] * s[1], rtol=1e-12)


def test_workload_dof_counts():
    from paper_2010_12879_b200 import workloads
    m = workloads.layered_block_model(128)
    kappa = m.voxel_kappa(85e3)
    nodes = oracle.node_conductive_mask(kappa)
    assert int(nodes.sum()) - 1 == 1_092_726
    assert int((kappa > 0).sum()) == 1_061_208
    m3 = workloads.duke_like_model(0.002)
    k3 = m3.voxel_kappa(85e3)
    assert int((k3 > 0).sum()) == 8_711_040
    assert int(oracle.node_conductive_mask(k3).sum()) - 1 == 8_913_552
    assert math.isclose(m3.tissue_table[3].conductivity.at(85e3), 0.35)
