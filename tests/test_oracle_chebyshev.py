"""CPU: the oracle's Chebyshev smoother restatement (Saad alg. 12.1, the
[beta/5, beta] interval) -- symmetric V-cycle, preconditioned CG
convergence, coefficient recurrence against the closed form of the scaled
Chebyshev polynomial, and the config validation of the host mirror."""

import numpy as np
import pytest

from conftest import golden_cases, golden_csr, load_golden


def _lap(n):
    import scipy.sparse as sp
    t = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    e = sp.identity(n)
    return (sp.kron(sp.kron(t, e), e) + sp.kron(sp.kron(e, t), e) + sp.kron(sp.kron(e, e), t)).tocsr()


def test_polynomial_matches_chebyshev_closed_form():
    """After one degree-k sweep from 0 the error operator is
    I - q(D^-1 A) D^-1 A = T_k((beta+alpha-2t)/(beta-alpha)) / T_k((beta+alpha)/(beta-alpha))."""
    import oracle
    lmax, k = 2.0, 4
    beta = 1.1 * lmax
    alpha = 0.2 * beta
    c0, steps = oracle.chebyshev_coefficients(lmax, k)
    for t in np.linspace(alpha, beta, 7):
        # scalar problem a = t (D = 1): error after the sweep for b = t x*, x* = 1
        x = c0 * t
        d = x
        for c1, c2 in steps:
            d = c1 * d + c2 * (t - t * x)
            x = x + d
        err = 1.0 - x
        s0 = (beta + alpha) / (beta - alpha)
        ref = np.cos(k * np.arccos((beta + alpha - 2 * t) / (beta - alpha))) / np.cosh(k * np.arccosh(s0))
        assert abs(err - ref) <= 1e-12


@pytest.mark.parametrize("degree", [1, 2, 3])
def test_cycle_symmetric_and_pcg(degree):
    import oracle
    rng = np.random.default_rng(5)
    a = _lap(12)
    h = oracle.amg_setup(a, oracle.OracleSolveConfig(coarse_cap=50))
    lm = [oracle.power_lmax(lv["A"], lv["dinv"]) for lv in h["levels"][:-1]]
    hc = oracle.with_chebyshev(h, lm, degree)
    x, y = rng.standard_normal((2, a.shape[0]))
    assert abs(x @ oracle.v_cycle(hc, y) - y @ oracle.v_cycle(hc, x)) <= 1e-12 * abs(x @ oracle.v_cycle(hc, x))
    b = rng.standard_normal(a.shape[0])
    sol, its, rel, conv = oracle.pcg(a, b, hc, oracle.OracleSolveConfig(rel_tol=1e-10))
    _, its_j, _, _ = oracle.pcg(a, b, h, oracle.OracleSolveConfig(rel_tol=1e-10))
    assert conv and rel <= 1e-10
    if degree >= 2:
        assert its <= its_j


@pytest.mark.parametrize("case", golden_cases("model")[:3])
def test_power_lmax_below_exact(case):
    import oracle
    d = load_golden(case)
    a = golden_csr(d, "matrix")
    lam = oracle.power_lmax(a, 1.0 / a.diagonal())
    dh = 1.0 / np.sqrt(a.diagonal())
    exact = np.linalg.eigvalsh((a.multiply(dh[:, None]).multiply(dh[None, :])).toarray()).max() \
        if a.shape[0] < 3000 else None
    if exact is not None:
        assert 0.8 * exact <= lam <= exact * (1 + 1e-12)


def test_config_validation():
    from paper_2010_12879_b200 import SolveConfig
    with pytest.raises(ValueError):
        SolveConfig(smoother="gauss-seidel")
    with pytest.raises(ValueError):
        SolveConfig(smoother="chebyshev", chebyshev_degree=0)
    c = SolveConfig(smoother="chebyshev", chebyshev_degree=3)
    from paper_2010_12879_b200 import _lib
    m = _lib.make_config(c)
    assert m.smoother == _lib.SMOOTHER_CHEBYSHEV and m.cheb_degree == 3
