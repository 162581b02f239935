"""CPU: pin the oracle's restatement of rows f1-f4 (sources, interpolation,
divergence cleaning, comb-tree gauging, exposure statistics) against golden
vectors produced by the reference (tests/golden/make_golden.py field_case)."""

import numpy as np
import pytest

import oracle
from conftest import golden_csr, load_golden


@pytest.fixture(scope="module")
def g():
    return load_golden("field_coil")


def _grid(g):
    return tuple(int(v) for v in g["grid_dims"]), g["grid_spacing"], g["grid_origin"]


def test_coil_field_matches_reference(g):
    b = oracle.coil_field(g["coil_vertices"], float(g["coil_current"]), g["points"])
    assert np.allclose(b, g["b"], rtol=1e-13, atol=1e-13 * np.abs(g["b"]).max())


def test_interpolation_bit_exact(g):
    dims, h, o = _grid(g)
    f = oracle.interpolate_to_faces(dims, h, o, g["lat_dims"], g["lat_spacing"], g["lat_origin"], g["b"])
    assert np.array_equal(f, g["flux"])


def test_divergence_bit_exact(g):
    dims, _, _ = _grid(g)
    assert np.array_equal(oracle.divergence_matrix(dims) @ g["flux"], g["div"])


def test_normal_matrix_and_aggregates(g):
    dims, _, _ = _grid(g)
    d = oracle.divergence_matrix(dims)
    n = (d @ d.T).tocsr()
    n.sort_indices()
    ref = golden_csr(g, "normal")
    assert np.array_equal(n.indptr, ref.indptr) and np.array_equal(n.indices, ref.indices)
    assert np.array_equal(n.data, ref.data)
    h = oracle.amg_setup(n)
    assert list(h["sizes"]) == list(g["normal_sizes"])
    assert np.array_equal(h["levels"][0]["agg"], g["normal_agg0"])


def test_cleaning_projection(g):
    dims, _, _ = _grid(g)
    c = oracle.divergence_clean(dims, g["flux"], 1e-10)
    fn = np.linalg.norm(g["flux"])
    assert np.linalg.norm(c - g["clean"]) <= 1e-9 * fn
    assert np.linalg.norm(oracle.divergence_matrix(dims) @ c) <= 1e-10 * fn


def test_fifo_elimination_bit_exact(g):
    dims, _, _ = _grid(g)
    mask = oracle.comb_tree_mask(dims)
    assert np.array_equal(mask, g["tree_mask"])
    vals, und = oracle.eliminate_cotree_edges(dims, g["clean"], mask)
    assert und == 0
    assert np.array_equal(vals, g["a"])
    assert np.array_equal(oracle.circulation_residual(vals, g["clean"], dims), g["circ"])


def test_comb_scan_equals_fifo_to_rounding(g):
    dims, _, _ = _grid(g)
    a = oracle.comb_gauge(dims, g["clean"])
    assert np.abs(a - g["a"]).max() <= 1e-12 * np.abs(g["a"]).max()
    ua = oracle.comb_gauge(dims, g["uniform_flux"])
    assert np.abs(ua - g["uniform_a"]).max() <= 1e-14 * np.abs(g["uniform_a"]).max()


def test_exposure_stats(g):
    ids = g["st_ids"][g["st_idx"]]
    v, (p99, mx), per = oracle.exposure_stats(g["st_vals"], ids, rms=True)
    assert np.array_equal(v, g["st_scaled"])
    assert p99 == float(g["st_p99"]) and mx == float(g["st_max"])
    assert sorted(per) == list(g["st_tids"])
    for t, c, m, x, p in zip(g["st_tids"], g["st_count"], g["st_mean"], g["st_tmax"], g["st_tp99"]):
        assert per[int(t)] == (int(c), float(m), float(x), float(p))
    assert oracle.percentile99(g["st_vals"]) == float(g["p99_plain"])


def test_bfs_tree_and_gauge_match_reference():
    """BFS spanning tree (gauging.py:74-119) and the FIFO elimination with it
    (_kernels.py:12-76): the closed-form tree equals the reference's, the
    oracle's FIFO restatement reproduces the reference potential bit for
    bit, and the x-scan form agrees to rounding."""
    b = load_golden("field_bfs")
    dims = tuple(int(v) for v in b["grid_dims"])
    mask = oracle.bfs_tree_mask(dims)
    assert np.array_equal(mask, b["tree_mask"])
    v, und = oracle.eliminate_cotree_edges(dims, b["clean"], mask)
    assert und == 0 and np.array_equal(v, b["a"])
    scale = np.abs(b["a"]).max()
    assert np.abs(oracle.bfs_gauge(dims, b["clean"]) - b["a"]).max() <= 1e-14 * scale
    assert np.abs(oracle.bfs_gauge(dims, b["uniform_flux"]) - b["uniform_a"]).max() <= 1e-14 * np.abs(b["uniform_a"]).max()


def test_bfs_spanning_tree_host_arrays():
    """The package's BFS SpanningTree metadata (mask, parent node / edge) is
    the reference's (host index bookkeeping; the gauge itself runs on the
    device)."""
    from paper_2010_12879_b200.fit_operators import StaggeredGrid
    from paper_2010_12879_b200.gauging import build_tree
    b = load_golden("field_bfs")
    grid = StaggeredGrid(tuple(int(v) for v in b["grid_dims"]), tuple(b["grid_spacing"]), tuple(b["grid_origin"]))
    t = build_tree(grid, "bfs")
    assert np.array_equal(t.edge_mask, b["tree_mask"])
    assert np.array_equal(t.parent_node, b["parent_node"])
    assert np.array_equal(t.parent_edge, b["parent_edge"])
    assert t.n_tree_edges == int(b["tree_mask"].sum())
