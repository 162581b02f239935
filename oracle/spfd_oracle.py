"""Numpy/scipy restatement of the reference SPFD hot path (CPU oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Arrays follow the
reference conventions: voxel arrays are indexed [i, j, k] with shape
``dims``; flat node / edge / voxel vectors are x-fastest (``order="F"``);
edges are three orientation blocks x, y, z
(/root/reference/pkg/src/spfd/fit_operators.py:1-16).
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

__all__ = [
    "OracleSolveConfig", "kappa_at", "edge_dims", "edge_offsets", "n_edges", "kappa_lut",
    "voxel_kappa", "edge_conductance", "node_conductive_mask",
    "component_labels", "assemble", "assemble_rhs", "strength_graph", "plain_aggregation",
    "amg_setup", "v_cycle", "fgmres", "pcg", "edge_voltages", "node_field",
    "voxel_average", "comb_gauge", "uniform_face_fluxes", "node_index", "coil_field",
    "interpolate_to_faces", "divergence_matrix", "divergence_clean", "circulation_residual", "comb_tree_mask",
    "eliminate_cotree_edges", "percentile99", "exposure_stats", "bfs_tree_mask", "bfs_gauge",
    "power_lmax", "chebyshev_coefficients", "with_chebyshev",
]


# --------------------------------------------------------------------------
# index spaces (fit_operators.py:57-124)
# --------------------------------------------------------------------------

def node_dims(dims):
    return tuple(int(d) + 1 for d in dims)


def edge_dims(dims, axis):
    d = list(node_dims(dims))
    d[axis] = int(dims[axis])
    return tuple(d)


def edge_offsets(dims):
    c = [int(np.prod(edge_dims(dims, a))) for a in range(3)]
    return (0, c[0], c[0] + c[1]), tuple(c)


def n_edges(dims):
    off, c = edge_offsets(dims)
    return off[2] + c[2]


def node_index(dims, i, j, k):
    nd = node_dims(dims)
    return i + nd[0] * (j + nd[1] * np.asarray(k))


def _edge_endpoints(dims):
    """(tail, head) node per edge in canonical order (fit_operators.py:167-184)."""
    tails, heads = [], []
    for a in range(3):
        ed = edge_dims(dims, a)
        ii, jj, kk = (np.arange(ed[0]), np.arange(ed[1]), np.arange(ed[2]))
        I, J, K = np.meshgrid(ii, jj, kk, indexing="ij")
        I, J, K = I.ravel(order="F"), J.ravel(order="F"), K.ravel(order="F")
        t = node_index(dims, I, J, K)
        step = [I, J, K]
        step[a] = step[a] + 1
        tails.append(t)
        heads.append(node_index(dims, *step))
    return np.concatenate(tails), np.concatenate(heads)


# --------------------------------------------------------------------------
# conductivities (voxel_model.py:62-87, 153-159)
# --------------------------------------------------------------------------

def kappa_at(freqs, kappas, f):
    """Log-log piecewise-linear kappa(f), clamped, exact at samples
    (voxel_model.py:62-87)."""
    freqs = np.asarray(freqs, dtype=np.float64)
    kappas = np.asarray(kappas, dtype=np.float64)
    f = float(f)
    pos = int(np.searchsorted(freqs, f))
    if pos < freqs.size and freqs[pos] == f:
        return float(kappas[pos])
    if f < freqs[0]:
        return float(kappas[0])
    if f > freqs[-1]:
        return float(kappas[-1])
    lo_k, hi_k = float(kappas[pos - 1]), float(kappas[pos])
    t = (math.log(f) - math.log(freqs[pos - 1])) / (math.log(freqs[pos]) - math.log(freqs[pos - 1]))
    if lo_k > 0.0 and hi_k > 0.0:
        return math.exp((1.0 - t) * math.log(lo_k) + t * math.log(hi_k))
    return (1.0 - t) * lo_k + t * hi_k


def kappa_lut(table, f, max_id):
    """LUT indexed by tissue id (voxel_model.py:155-158).  ``table`` maps
    id -> (freqs, kappas)."""
    lut = np.zeros(int(max_id) + 1, dtype=np.float64)
    for tid, (fr, ka) in table.items():
        if tid < lut.size:
            lut[tid] = kappa_at(fr, ka, f)
    return lut


def voxel_kappa(ids, lut):
    return np.asarray(lut, dtype=np.float64)[np.asarray(ids)]


# --------------------------------------------------------------------------
# edge conductance (fit_operators.py:289-324)
# --------------------------------------------------------------------------

def _around_edge_sum(kappa, axis):
    """Sum of the <=4 voxels around each edge of one orientation, absent
    voxels as 0, accumulated in the reference's (da, db) order
    (fit_operators.py:289-308)."""
    t0, t1 = [a for a in range(3) if a != axis]
    padw = [(0, 0)] * 3
    padw[t0] = (1, 1)
    padw[t1] = (1, 1)
    padded = np.pad(kappa, padw)
    total = None
    for da in (0, 1):
        for db in (0, 1):
            sel = [slice(None)] * 3
            sel[t0] = slice(da, padded.shape[t0] - 1 + da)
            sel[t1] = slice(db, padded.shape[t1] - 1 + db)
            piece = padded[tuple(sel)]
            total = piece.copy() if total is None else total + piece
    return total


def edge_conductance(kappa, spacing):
    """w_e = mean4(kappa) * dual_area / length (fit_operators.py:311-324)."""
    dims = kappa.shape
    off, cnt = edge_offsets(dims)
    w = np.empty(off[2] + cnt[2], dtype=np.float64)
    s = [float(v) for v in spacing]
    for a in range(3):
        t0, t1 = [b for b in range(3) if b != a]
        geom = (s[t0] * s[t1]) / s[a]
        blk = (_around_edge_sum(kappa, a) * 0.25) * geom
        w[off[a]:off[a] + cnt[a]] = blk.ravel(order="F")
    return w


# --------------------------------------------------------------------------
# conductive nodes and components (voxel_model.py:448-511)
# --------------------------------------------------------------------------

def node_conductive_mask(kappa):
    """Nodes touching a conductive voxel (voxel_model.py:459-467)."""
    cond = np.pad(kappa > 0.0, 1)
    out = np.zeros(tuple(n + 1 for n in kappa.shape), dtype=bool)
    for di in (0, 1):
        for dj in (0, 1):
            for dk in (0, 1):
                out |= cond[di:di + out.shape[0], dj:dj + out.shape[1], dk:dk + out.shape[2]]
    return out


def component_labels(kappa):
    """Per-node component label over conductive edges, ranked by lowest node
    index, -1 elsewhere (voxel_model.py:470-511).  A conductive edge is one
    with a conductive voxel among its <=4 neighbours, i.e. w > 0."""
    dims = kappa.shape
    nn = int(np.prod(node_dims(dims)))
    around = [(_around_edge_sum((kappa > 0.0).astype(np.float64), a) > 0.0).ravel(order="F")
              for a in range(3)]
    tails, heads = _edge_endpoints(dims)
    mask = np.concatenate(around)
    labels = np.full(nn, -1, dtype=np.int32)
    if not mask.any():
        return labels
    g = sp.coo_matrix((np.ones(int(mask.sum()), dtype=np.int8),
                       (tails[mask], heads[mask])), shape=(nn, nn))
    _, raw = connected_components(g, directed=False)
    cond = node_conductive_mask(kappa).ravel(order="F")
    kept = raw[cond]
    uniq, first = np.unique(kept, return_index=True)
    order = np.empty(uniq.size, dtype=np.int32)
    order[np.argsort(first, kind="stable")] = np.arange(uniq.size, dtype=np.int32)
    labels[cond] = order[np.searchsorted(uniq, kept)]
    return labels


# --------------------------------------------------------------------------
# Poisson assembly (fit_operators.py:367-457)
# --------------------------------------------------------------------------

def assemble(kappa, spacing, a_edges, pin=True):
    """Reduced system A psi = rhs on free conductive nodes.

    The COO triplets are emitted in the reference order (diagonal from
    tails, diagonal from heads, then the two off-diagonal halves) so the
    CSR duplicate summation reproduces the reference bit for bit
    (fit_operators.py:421-441).
    """
    dims = kappa.shape
    a_edges = np.asarray(a_edges, dtype=np.float64)
    w = edge_conductance(kappa, spacing)
    if a_edges.shape != w.shape:
        raise ValueError("vector potential has the wrong length")
    labels = component_labels(kappa)
    cond = np.flatnonzero(labels >= 0)
    if cond.size == 0:
        raise ValueError("empty system")
    _, first = np.unique(labels[cond], return_index=True)
    pinned = cond[np.sort(first)]
    free = labels >= 0
    if pin:
        free[pinned] = False
    nn = labels.size
    node_to_dof = np.full(nn, -1, dtype=np.int64)
    dof_to_node = np.flatnonzero(free)
    node_to_dof[dof_to_node] = np.arange(dof_to_node.size)
    n = dof_to_node.size

    tails, heads = _edge_endpoints(dims)
    on = w > 0.0
    t, h, we = tails[on], heads[on], w[on]
    dt, dh = node_to_dof[t], node_to_dof[h]
    kt, kh = dt >= 0, dh >= 0
    both = kt & kh
    r = np.concatenate([dt[kt], dh[kh], dt[both], dh[both]])
    c = np.concatenate([dt[kt], dh[kh], dh[both], dt[both]])
    v = np.concatenate([we[kt], we[kh], -we[both], -we[both]])
    mat = sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr()
    mat.sort_indices()

    flow = we * a_edges[on]
    rhs_nodes = np.bincount(t, weights=flow, minlength=nn)
    rhs_nodes -= np.bincount(h, weights=flow, minlength=nn)
    return dict(matrix=mat, rhs=rhs_nodes[dof_to_node], node_to_dof=node_to_dof,
                dof_to_node=dof_to_node, pinned=pinned, w=w, labels=labels,
                n_conductive=int(cond.size), n_components=int(pinned.size))


def assemble_rhs(sysd, dims, a_edges):
    """RHS of an already assembled system for another vector potential
    (fit_operators.py:438-441: the same bincount over active edges, no
    re-assembly of the matrix)."""
    w = sysd["w"]
    a_edges = np.asarray(a_edges, dtype=np.float64)
    if a_edges.shape != w.shape:
        raise ValueError("vector potential has the wrong length")
    tails, heads = _edge_endpoints(dims)
    on = w > 0.0
    t, h = tails[on], heads[on]
    flow = w[on] * a_edges[on]
    nn = sysd["labels"].size
    rhs_nodes = np.bincount(t, weights=flow, minlength=nn)
    rhs_nodes -= np.bincount(h, weights=flow, minlength=nn)
    return rhs_nodes[sysd["dof_to_node"]]


# --------------------------------------------------------------------------
# AMG (linsolve.py:26-197, _kernels.py:79-120)
# --------------------------------------------------------------------------

@dataclass
class OracleSolveConfig:
    """Same fields and defaults as the reference SolveConfig (linsolve.py:26-41)."""
    rel_tol: float = 1e-12
    max_iters: int = 1000
    restart: int = 30
    pre_sweeps: int = 1
    post_sweeps: int = 1
    jacobi_damping: float = 2.0 / 3.0
    strength_threshold: float = 0.08
    coarse_cap: int = 500
    max_levels: int = 20
    trace: object = field(default=None, repr=False)


def strength_graph(a, theta):
    """Strong off-diagonal couplings |a_ij| >= theta*sqrt|a_ii|*sqrt|a_jj|
    (linsolve.py:106-117).  Returns (indptr, cols, |a_ij|) as int64/f64."""
    n = a.shape[0]
    root_diag = np.sqrt(np.abs(a.diagonal()))
    row_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.indptr))
    cols = a.indices.astype(np.int64)
    mag = np.abs(a.data)
    keep = (row_of != cols) & (mag >= theta * root_diag[row_of] * root_diag[cols])
    counts = np.bincount(row_of[keep], minlength=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols[keep], mag[keep]


_AGG_LIB = None


def _agg_lib():
    global _AGG_LIB
    if _AGG_LIB is None:
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "_build", "liboracle_agg.so")
        if not os.path.exists(path):
            build_oracle()
        lib = ctypes.CDLL(path)
        lib.oracle_plain_aggregation.restype = ctypes.c_int64
        lib.oracle_plain_aggregation.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p]
        _AGG_LIB = lib
    return _AGG_LIB


def build_oracle():
    """Compile oracle/agg.c with gcc into oracle/_build/."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    os.makedirs(os.path.join(here, "_build"), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o",
                           os.path.join(here, "_build", "liboracle_agg.so"),
                           os.path.join(here, "agg.c")])


def plain_aggregation(indptr, cols, strengths, n):
    """C restatement of _kernels.py:79-120 (see oracle/agg.c)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    strengths = np.ascontiguousarray(strengths, dtype=np.float64)
    agg = np.empty(int(n), dtype=np.int32)
    k = _agg_lib().oracle_plain_aggregation(indptr.ctypes.data, cols.ctypes.data,
                                            strengths.ctypes.data, int(n), agg.ctypes.data)
    return agg, int(k)


def _dinv(a):
    d = a.diagonal()
    if np.any(d <= 0.0):
        raise ValueError("matrix has a non-positive diagonal entry")
    return 1.0 / d


def amg_setup(a, cfg=None):
    """Smoothed-aggregation hierarchy (linsolve.py:120-169).

    Returns dict(levels=[dict(A, dinv, P, R, agg)], lu, sizes, seconds)."""
    cfg = cfg or OracleSolveConfig()
    t0 = time.perf_counter()
    a = sp.csr_matrix(a)
    a.sort_indices()
    levels = [dict(A=a, dinv=_dinv(a), P=None, R=None, agg=None)]
    depth = 0
    while levels[-1]["A"].shape[0] > cfg.coarse_cap and len(levels) < cfg.max_levels:
        fine = levels[-1]["A"]
        n = fine.shape[0]
        sip, sj, sv = strength_graph(fine, cfg.strength_threshold * 0.5 ** depth)
        agg, n_agg = plain_aggregation(sip, sj, sv, n)
        if n_agg >= n:
            break
        tent = sp.csr_matrix((np.ones(n), agg.astype(np.int64), np.arange(n + 1, dtype=np.int64)),
                             shape=(n, n_agg))
        sm = fine @ tent
        sm.data *= np.repeat(cfg.jacobi_damping * levels[-1]["dinv"], np.diff(sm.indptr))
        p = (tent - sm).tocsr()
        p.sort_indices()
        r = p.T.tocsr()
        r.sort_indices()
        coarse = (r @ (fine @ p)).tocsr()
        coarse.sort_indices()
        levels[-1].update(P=p, R=r, agg=agg)
        levels.append(dict(A=coarse, dinv=_dinv(coarse), P=None, R=None, agg=None))
        depth += 1
    lu = sla.lu_factor(levels[-1]["A"].toarray())
    return dict(levels=levels, lu=lu, sizes=[lv["A"].shape[0] for lv in levels],
                seconds=time.perf_counter() - t0, pre=cfg.pre_sweeps,
                post=cfg.post_sweeps, omega=cfg.jacobi_damping)


def _cycle(h, lvl, r):
    if lvl == len(h["levels"]) - 1:
        return sla.lu_solve(h["lu"], r)
    L = h["levels"][lvl]
    a = L["A"]
    wd = h["omega"] * L["dinv"]
    x = wd * r
    for _ in range(h["pre"] - 1):
        x += wd * (r - a @ x)
    d = r - a @ x
    x += L["P"] @ _cycle(h, lvl + 1, L["R"] @ d)
    for _ in range(h["post"]):
        x += wd * (r - a @ x)
    return x


def v_cycle(h, r):
    """V(pre, post) cycle (linsolve.py:179-197); with_chebyshev(h, ...)
    switches the smoother."""
    if h.get("smoother") == "chebyshev":
        return _cycle_cheb(h, 0, np.asarray(r, dtype=np.float64))
    return _cycle(h, 0, np.asarray(r, dtype=np.float64))


# --------------------------------------------------------------------------
# Chebyshev smoother -- NOT in the reference (its V-cycle is damped Jacobi,
# linsolve.py:184-197); north_star (2) names it as an option.  Restatement of
# the standard polynomial smoother in D^-1 A (Saad, Iterative Methods for
# Sparse Linear Systems, alg. 12.1) on [beta/5, beta], beta = 1.1 lambda_max
# estimate (lower end 0.2 beta: measured on the golden phantoms, degree 2
# takes 9-11 PCG iterations against 16-19 with Jacobi; PyAMG's beta/30
# interval needs degree 3 to beat Jacobi), used to check the device smoother.
# --------------------------------------------------------------------------

def power_lmax(a, dinv, iters=20, x0=None):
    """||D^-1 A x|| power iteration from x0 (normalised), as the device does."""
    n = a.shape[0]
    x = np.ones(n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = dinv * (a @ x)
        lam = float(np.linalg.norm(y))
        x = y / lam
    return lam


def chebyshev_coefficients(lmax, degree):
    beta = 1.1 * lmax
    alpha = 0.2 * beta
    theta, delta = 0.5 * (beta + alpha), 0.5 * (beta - alpha)
    sigma = theta / delta
    rho = 1.0 / sigma
    steps = []
    for _ in range(1, degree):
        rn = 1.0 / (2.0 * sigma - rho)
        steps.append((rn * rho, 2.0 * rn / delta))
        rho = rn
    return 1.0 / theta, steps


def with_chebyshev(h, lmax, degree=2):
    """Copy of hierarchy h using the Chebyshev smoother with the given
    per-level lambda_max estimates (e.g. the device's)."""
    g = dict(h)
    g.update(smoother="chebyshev", cheb_lmax=list(lmax), cheb_degree=int(degree))
    return g


def _cheb_sweep(a, dinv, coef, b, x):
    c0, steps = coef
    t = b if x is None else b - a @ x
    d = c0 * (dinv * t)
    x = d.copy() if x is None else x + d
    for c1, c2 in steps:
        t = b - a @ x
        d = c1 * d + c2 * (dinv * t)
        x = x + d
    return x


def _cycle_cheb(h, lvl, r):
    if lvl == len(h["levels"]) - 1:
        return sla.lu_solve(h["lu"], r)
    L = h["levels"][lvl]
    a, dinv = L["A"], L["dinv"]
    coef = chebyshev_coefficients(h["cheb_lmax"][lvl], h["cheb_degree"])
    x = None
    for _ in range(h["pre"]):
        x = _cheb_sweep(a, dinv, coef, r, x)
    if x is None:
        x = np.zeros_like(r)
    d = r - a @ x
    x = x + L["P"] @ _cycle_cheb(h, lvl + 1, L["R"] @ d)
    for _ in range(h["post"]):
        x = _cheb_sweep(a, dinv, coef, r, x)
    return x


def fgmres(a, b, h, cfg=None):
    """Right-preconditioned FGMRES(m) with true-residual restarts
    (linsolve.py:200-298).  Returns (x, iterations, rel_residual, converged)."""
    cfg = cfg or OracleSolveConfig()
    b = np.asarray(b, dtype=np.float64)
    n = a.shape[0]
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, 0.0, True
    m = cfg.restart
    its = 0
    while its < cfg.max_iters:
        res = b - a @ x
        beta = float(np.linalg.norm(res))
        if beta / bnorm <= cfg.rel_tol:
            return x, its, beta / bnorm, True
        V = np.empty((m + 1, n))
        Z = np.empty((m, n))
        H = np.zeros((m + 1, m))
        cs = np.empty(m)
        sn = np.empty(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = res / beta
        j = 0
        while j < m and its < cfg.max_iters:
            Z[j] = _cycle(h, 0, V[j])
            w = a @ Z[j]
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w -= H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            if not math.isfinite(hn):
                raise FloatingPointError("non-finite Arnoldi value")
            for i in range(j):
                u, v = H[i, j], H[i + 1, j]
                H[i, j], H[i + 1, j] = cs[i] * u + sn[i] * v, -sn[i] * u + cs[i] * v
            den = math.hypot(H[j, j], hn)
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, hn / den)
            H[j, j] = cs[j] * H[j, j] + sn[j] * hn
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            j += 1
            est = abs(g[j]) / bnorm
            if cfg.trace is not None:
                cfg.trace.write(f"iter {its} rel_resid {est:.6e}\n")
            if hn == 0.0 or est <= cfg.rel_tol:
                break
            if j < m:
                V[j] = w / hn
        if j > 0:
            y = sla.solve_triangular(H[:j, :j], g[:j], lower=False)
            x = x + Z[:j].T @ y
    rel = float(np.linalg.norm(b - a @ x)) / bnorm
    return x, its, rel, rel <= cfg.rel_tol


def pcg(a, b, h, cfg=None):
    """Preconditioned CG with the same V-cycle (the reference
    V-cycle is symmetric, so PCG is admissible).  Convergence on the true
    residual at exit; returns (x, iterations, rel_residual, converged)."""
    cfg = cfg or OracleSolveConfig()
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, 0.0, True
    r = b.copy()
    z = v_cycle(h, r)
    p = z.copy()
    rho = float(r @ z)
    its = 0
    while its < cfg.max_iters:
        q = a @ p
        alpha = rho / float(p @ q)
        x += alpha * p
        r -= alpha * q
        its += 1
        if float(np.linalg.norm(r)) / bnorm <= cfg.rel_tol:
            break
        z = v_cycle(h, r)
        rho_new = float(r @ z)
        p = z + (rho_new / rho) * p
        rho = rho_new
    rel = float(np.linalg.norm(b - a @ x)) / bnorm
    return x, its, rel, rel <= cfg.rel_tol


# --------------------------------------------------------------------------
# E-field chain (dosimetry.py:27-116)
# --------------------------------------------------------------------------

def edge_voltages(a_edges, psi_dofs, dof_to_node, dims, omega):
    """omega * (a + psi[head] - psi[tail]) on every edge (dosimetry.py:27-47)."""
    full = np.zeros(int(np.prod(node_dims(dims))))
    full[dof_to_node] = psi_dofs
    tails, heads = _edge_endpoints(dims)
    return omega * (np.asarray(a_edges, dtype=np.float64) + full[heads] - full[tails])


def node_field(volts, w, dims, spacing):
    """Per-node |E|: per-axis mean of conductive incident edge fields
    (dosimetry.py:50-85).  Returns shape node_dims."""
    off, cnt = edge_offsets(dims)
    nd = node_dims(dims)
    acc = np.zeros(nd)
    for a in range(3):
        ed = edge_dims(dims, a)
        ev = volts[off[a]:off[a] + cnt[a]].reshape(ed, order="F")
        on = (w[off[a]:off[a] + cnt[a]] > 0.0).astype(np.float64).reshape(ed, order="F")
        val = ev * on / float(spacing[a])
        num = np.zeros(nd)
        den = np.zeros(nd)
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[a] = slice(None, -1)
        hi[a] = slice(1, None)
        num[tuple(lo)] += val
        num[tuple(hi)] += val
        den[tuple(lo)] += on
        den[tuple(hi)] += on
        comp = num / np.maximum(den, 1.0)
        comp[den == 0.0] = 0.0
        acc += comp * comp
    return np.sqrt(acc)


def voxel_average(node_vals, kappa):
    """Eight-corner mean over conductive voxels, x-fastest
    (dosimetry.py:88-116).  Returns (values, voxel_indices)."""
    nf = np.asarray(node_vals, dtype=np.float64).reshape(node_dims(kappa.shape), order="F") \
        if np.ndim(node_vals) == 1 else np.asarray(node_vals, dtype=np.float64)
    s = kappa.shape
    acc = np.zeros(s)
    for di in (0, 1):
        for dj in (0, 1):
            for dk in (0, 1):
                acc += nf[di:di + s[0], dj:dj + s[1], dk:dk + s[2]]
    acc *= 0.125
    idx = np.flatnonzero((kappa > 0.0).ravel(order="F"))
    return acc.ravel(order="F")[idx], idx


# --------------------------------------------------------------------------
# input generation helpers (upstream of the hot path)
# --------------------------------------------------------------------------

def uniform_face_fluxes(dims, spacing, b):
    """Face fluxes of a uniform B (B_axis * face area)."""
    out = []
    s = [float(v) for v in spacing]
    for a in range(3):
        t0, t1 = [c for c in range(3) if c != a]
        fd = list(dims)
        fd[a] += 1
        out.append(np.full(int(np.prod(fd)), float(b[a]) * s[t0] * s[t1]))
    return np.concatenate(out)


def comb_gauge(dims, fluxes):
    """Comb-tree gauge as three prefix scans (equivalent to
    gauging.py:34-71 + _kernels.py:12-76 up to rounding)."""
    nx, ny, nz = [int(d) for d in dims]
    fcount = [(nx + 1) * ny * nz, nx * (ny + 1) * nz, nx * ny * (nz + 1)]
    bx = fluxes[:fcount[0]].reshape((nx + 1, ny, nz), order="F")
    by = fluxes[fcount[0]:fcount[0] + fcount[1]].reshape((nx, ny + 1, nz), order="F")
    bz = fluxes[fcount[0] + fcount[1]:].reshape((nx, ny, nz + 1), order="F")
    ax = np.zeros((nx, ny + 1, nz + 1))
    ay = np.zeros((nx + 1, ny, nz + 1))
    az = np.zeros((nx + 1, ny + 1, nz))
    ax[:, 1:, 0] = -np.cumsum(bz[:, :, 0], axis=1)
    ax[:, :, 1:] = ax[:, :, :1] + np.cumsum(by, axis=2)
    ay[:, :, 1:] = -np.cumsum(bx, axis=2)
    return np.concatenate([ax.ravel(order="F"), ay.ravel(order="F"), az.ravel(order="F")])


def bfs_tree_mask(dims):
    """Tree edges of the BFS spanning tree from node 0 (gauging.py:74-119).
    On the full node box the level-synchronous BFS with its direction order
    (+x first) reaches every node with i > 0 through its -x neighbour, nodes
    (0, j > 0, k) through -y and (0, 0, k > 0) through -z: all x-edges, the
    y-edges of the plane i = 0 and the z-edges of the line i = j = 0."""
    nx, ny, nz = [int(n) for n in dims]
    m = np.zeros(n_edges(dims), bool)
    eoff = edge_offsets(dims)[0]
    ey, ez = edge_dims(dims, 1), edge_dims(dims, 2)
    m[eoff[0]:eoff[1]] = True
    j, k = np.meshgrid(np.arange(ny), np.arange(nz + 1), indexing="ij")
    m[eoff[1] + (ey[0] * (j + ey[1] * k)).ravel()] = True
    m[eoff[2] + ez[0] * ez[1] * np.arange(nz)] = True
    return m


def bfs_gauge(dims, fluxes):
    """BFS-tree gauge as three prefix scans along x (the FIFO elimination
    _kernels.py:12-76 with the BFS tree, up to rounding): z-faces give
    a_y(i+1) = a_y(i) + b_z(i), x-faces of the plane i = 0 give a_z(0, j+1)
    = a_z(0, j) + b_x(0, j), y-faces give a_z(i+1) = a_z(i) - b_y(i);
    tree edges are 0."""
    nx, ny, nz = [int(d) for d in dims]
    fcount = [(nx + 1) * ny * nz, nx * (ny + 1) * nz, nx * ny * (nz + 1)]
    bx = fluxes[:fcount[0]].reshape((nx + 1, ny, nz), order="F")
    by = fluxes[fcount[0]:fcount[0] + fcount[1]].reshape((nx, ny + 1, nz), order="F")
    bz = fluxes[fcount[0] + fcount[1]:].reshape((nx, ny, nz + 1), order="F")
    ax = np.zeros((nx, ny + 1, nz + 1))
    ay = np.zeros((nx + 1, ny, nz + 1))
    az = np.zeros((nx + 1, ny + 1, nz))
    ay[1:] = np.cumsum(bz, axis=0)
    az[0, 1:] = np.cumsum(bx[0], axis=0)
    az[1:] = az[:1] - np.cumsum(by, axis=0)
    return np.concatenate([ax.ravel(order="F"), ay.ravel(order="F"), az.ravel(order="F")])


# --------------------------------------------------------------------------
# rows f1-f4: sources, interpolation, cleaning, gauging, statistics
# --------------------------------------------------------------------------

def face_dims(dims, axis):
    d = [int(n) for n in dims]
    d[axis] += 1
    return tuple(d)


def face_center_axes(dims, spacing, origin, axis):
    """fit_operators.py:156-165."""
    d = face_dims(dims, axis)
    out = []
    for a in range(3):
        if a == axis:
            out.append(origin[a] + np.arange(d[a]) * spacing[a])
        else:
            out.append(origin[a] + (np.arange(d[a]) + 0.5) * spacing[a])
    return out


def coil_field(verts, current_a, points):
    """Biot-Savart of a closed polyline (field_source.py:163-197)."""
    pts = np.atleast_2d(np.asarray(points, np.float64))
    p1 = verts[:-1]
    seg = verts[1:] - p1
    seg_len2 = np.einsum("sj,sj->s", seg, seg)
    a = pts[:, None, :] - p1[None, :, :]
    b = a - seg[None, :, :]
    la = np.sqrt(np.einsum("nsj,nsj->ns", a, a))
    lb = np.sqrt(np.einsum("nsj,nsj->ns", b, b))
    cross = np.cross(a, b)
    denom = la * lb * ((la + lb) ** 2 - seg_len2[None, :])
    coeff = 2.0 * (la + lb) / denom
    return (4e-7 * np.pi * current_a / (4.0 * np.pi)) * np.einsum("ns,nsj->nj", coeff, cross)


def _axis_params(coords, origin, spacing, n):
    """field_source.py:218-233."""
    u = (coords - origin) / spacing
    if n == 1:
        return np.zeros(coords.shape, np.int64), np.zeros_like(coords), 0
    i0 = np.clip(np.floor(u).astype(np.int64), 0, n - 2)
    return i0, u - i0, 1


def interpolate_to_faces(dims, spacing, origin, lat_dims, lat_spacing, lat_origin, b):
    """Trilinear midpoint face fluxes (field_source.py:235-272)."""
    out = []
    for axis in range(3):
        comp = b[:, axis].reshape(tuple(lat_dims), order="F")
        xs, ys, zs = face_center_axes(dims, spacing, origin, axis)
        ix, tx, sx = _axis_params(xs, lat_origin[0], lat_spacing[0], lat_dims[0])
        iy, ty, sy = _axis_params(ys, lat_origin[1], lat_spacing[1], lat_dims[1])
        iz, tz, sz = _axis_params(zs, lat_origin[2], lat_spacing[2], lat_dims[2])
        vals = np.zeros((xs.size, ys.size, zs.size))
        for dx in (0, 1):
            wx = (tx if dx else 1.0 - tx)[:, None, None]
            for dy in (0, 1):
                wy = (ty if dy else 1.0 - ty)[None, :, None]
                for dz in (0, 1):
                    wz = (tz if dz else 1.0 - tz)[None, None, :]
                    corner = comp[(ix + dx * sx)[:, None, None], (iy + dy * sy)[None, :, None],
                                  (iz + dz * sz)[None, None, :]]
                    vals += wx * wy * wz * corner
        t = [a for a in range(3) if a != axis]
        out.append((vals * (spacing[t[0]] * spacing[t[1]])).ravel(order="F"))
    return np.concatenate(out)


def divergence_matrix(dims):
    """Cell net-outflux operator (fit_operators.py:227-244,276-286)."""
    nx, ny, nz = [int(n) for n in dims]
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    i, j, k = i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")
    fx, fy = (nx + 1) * ny * nz, nx * (ny + 1) * nz
    fi = lambda a, ii, jj, kk: ([0, fx, fx + fy][a] + ii + face_dims(dims, a)[0] * (jj + face_dims(dims, a)[1] * kk))
    faces = np.stack([fi(0, i + 1, j, k), fi(0, i, j, k), fi(1, i, j + 1, k), fi(1, i, j, k),
                      fi(2, i, j, k + 1), fi(2, i, j, k)], axis=1)
    signs = np.tile(np.array([1, -1, 1, -1, 1, -1], np.float64), (faces.shape[0], 1))
    nc = nx * ny * nz
    nf = fx + fy + nx * ny * (nz + 1)
    m = sp.coo_matrix((signs.ravel(), (np.repeat(np.arange(nc), 6), faces.ravel())), shape=(nc, nf)).tocsr()
    m.sort_indices()
    return m


def divergence_clean(dims, fluxes, tol=1e-10):
    """l2-minimal solenoidal projection (field_source.py:292-329) with a
    direct sparse solve of (div divT) phi = div f (test oracle)."""
    from scipy.sparse.linalg import spsolve
    div = divergence_matrix(dims)
    fn = float(np.linalg.norm(fluxes))
    if fn == 0.0:
        return fluxes.copy()
    defect = div @ fluxes
    if float(np.linalg.norm(defect)) / fn <= tol:
        return fluxes.copy()
    phi = spsolve((div @ div.T).tocsc(), defect)
    return fluxes - div.T @ phi


def face_edge_incidence(dims):
    """(edges, signs) per face, right-handed (fit_operators.py:186-224)."""
    nx, ny, nz = [int(n) for n in dims]
    eoff = edge_offsets(dims)[0]
    all_e, all_s = [], []
    for axis in range(3):
        e1, e2 = (axis + 1) % 3, (axis + 2) % 3
        d = face_dims(dims, axis)
        i, j, k = np.meshgrid(np.arange(d[0]), np.arange(d[1]), np.arange(d[2]), indexing="ij")
        base = [i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")]

        def eidx(a, c):
            ed = edge_dims(dims, a)
            return eoff[a] + c[0] + ed[0] * (c[1] + ed[1] * c[2])

        def sh(c, a):
            c = [x.copy() for x in c]
            c[a] = c[a] + 1
            return c
        all_e.append(np.stack([eidx(e1, base), eidx(e2, sh(base, e1)), eidx(e1, sh(base, e2)), eidx(e2, base)], 1))
        all_s.append(np.tile(np.array([1, 1, -1, -1], np.int8), (all_e[-1].shape[0], 1)))
    return np.concatenate(all_e), np.concatenate(all_s)


def circulation_residual(values, fluxes, dims):
    """gauging.py:127-134."""
    edges, signs = face_edge_incidence(dims)
    return np.einsum("fm,fm->f", values[edges], signs.astype(np.float64)) - fluxes


def comb_tree_mask(dims):
    """Tree edges of the comb tree (gauging.py:34-71)."""
    nx, ny, nz = [int(n) for n in dims]
    m = np.zeros(n_edges(dims), bool)
    eoff = edge_offsets(dims)[0]
    ex, ey, ez = (edge_dims(dims, a) for a in range(3))
    m[eoff[0] + np.arange(nx)] = True
    i, j = np.meshgrid(np.arange(nx + 1), np.arange(ny), indexing="ij")
    m[eoff[1] + (i + ey[0] * j).ravel()] = True
    m[eoff[2]:] = True
    return m


def eliminate_cotree_edges(dims, fluxes, known):
    """FIFO greedy face elimination (_kernels.py:12-76), pure Python loops:
    small cases only.  Returns (values, undetermined)."""
    edges, signs = face_edge_incidence(dims)
    known = known.astype(np.uint8).copy()
    values = np.zeros(known.size)
    counts = (4 - known[edges].sum(axis=1)).astype(np.int64)
    nf = edges.shape[0]
    incident = [[] for _ in range(known.size)]
    for f in range(nf):
        for m in range(4):
            incident[edges[f, m]].append(f)
    undetermined = int((known == 0).sum())
    queue = [f for f in range(nf) if counts[f] == 1]
    head = 0
    while head < len(queue):
        f = queue[head]
        head += 1
        if counts[f] != 1:
            continue
        acc, ue, us = 0.0, -1, 0.0
        for m in range(4):
            e, s = edges[f, m], float(signs[f, m])
            if known[e]:
                acc += s * values[e]
            else:
                ue, us = e, s
        values[ue] = (fluxes[f] - acc) / us
        known[ue] = 1
        undetermined -= 1
        for g in incident[ue]:
            counts[g] -= 1
            if counts[g] == 1:
                queue.append(g)
    return values, undetermined


def percentile99(values):
    """Nearest-rank p99 (dosimetry.py:119-127)."""
    values = np.asarray(values)
    n = values.size
    idx = -((-99 * n) // 100) - 1
    return float(np.partition(values, idx)[idx])


def exposure_stats(values, tissue_of_value, rms=False):
    """build_exposure_report statistics (dosimetry.py:195-234):
    scaled values, global (p99, max), {tid: (count, mean, max, p99)}."""
    v = np.asarray(values, np.float64)
    if rms:
        v = v * (1.0 / math.sqrt(2.0))
    per = {}
    for tid in np.unique(tissue_of_value):
        if int(tid) == 0:
            continue
        sel = v[tissue_of_value == tid]
        per[int(tid)] = (int(sel.size), float(sel.mean()), float(sel.max()), percentile99(sel))
    return v, (percentile99(v), float(v.max())), per
