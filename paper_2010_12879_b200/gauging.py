"""Tree-cotree gauging on the GPU.

Drop-in for /root/reference/pkg/src/spfd/gauging.py:20-172.  With the comb
tree (the pipeline default, gauging.py:34-71) the greedy face elimination
(_kernels.py:12-76) unrolls into three column prefix scans, which
libspfd_b200.so runs as sequential-per-column scans (k_gauge_ax0,
k_gauge_kscan), followed by the reference's postcondition: the circulation
residual over every face against `tol` (IncompatibleFluxError).  The result
equals the reference's FIFO elimination up to rounding (the FIFO may reach
an edge through a different face; SURVEY P7 measured 9e-16) and equals the
numpy cumsum formulation (`oracle.comb_gauge`) bit for bit.

The BFS tree (gauging.py:74-119) spans the full node box, where the
level-synchronous BFS from node 0 (+x pass first) always produces the same
shape: every x-edge, the y-edges of the plane i = 0 and the z-edges of the
line i = j = 0.  Its FIFO elimination unrolls into running sums along x
(k_gauge_xscan, k_gauge_bfs_az0), equal to `oracle.bfs_gauge` bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from .field_source import _dev, field_ops
from .fit_operators import StaggeredGrid


@dataclass(frozen=True)
class SpanningTree:
    """Spanning tree of the grid node graph (gauging.py:20-31).  For the
    comb tree the per-edge / per-node arrays are materialised lazily on the
    host (they are not needed by the device gauge)."""

    grid: StaggeredGrid
    kind: str = "comb"
    root: int = 0

    @cached_property
    def _arrays(self):
        if self.kind == "bfs":
            return self._bfs_arrays()
        g = self.grid
        nx, ny, nz = g.dims
        mask = np.zeros(g.n_edges, dtype=bool)
        parent_node = np.full(g.n_nodes, -1, dtype=np.int64)
        parent_edge = np.full(g.n_nodes, -1, dtype=np.int64)
        if nx > 0:
            i = np.arange(nx)
            e = g.edge_index(0, i, 0, 0)
            mask[e] = True
            parent_node[g.node_index(i + 1, 0, 0)] = g.node_index(i, 0, 0)
            parent_edge[g.node_index(i + 1, 0, 0)] = e
        if ny > 0:
            i, j = np.meshgrid(np.arange(nx + 1), np.arange(ny), indexing="ij")
            i, j = i.ravel(order="F"), j.ravel(order="F")
            e = g.edge_index(1, i, j, 0)
            mask[e] = True
            parent_node[g.node_index(i, j + 1, 0)] = g.node_index(i, j, 0)
            parent_edge[g.node_index(i, j + 1, 0)] = e
        if nz > 0:
            i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz), indexing="ij")
            i, j, k = i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")
            e = g.edge_index(2, i, j, k)
            mask[e] = True
            parent_node[g.node_index(i, j, k + 1)] = g.node_index(i, j, k)
            parent_edge[g.node_index(i, j, k + 1)] = e
        return mask, parent_node, parent_edge

    def _bfs_arrays(self):
        # node (i, j, k): i > 0 via its -x neighbour, else j > 0 via -y, else -z
        g = self.grid
        nx, ny, nz = g.dims
        mask = np.zeros(g.n_edges, dtype=bool)
        parent_node = np.full(g.n_nodes, -1, dtype=np.int64)
        parent_edge = np.full(g.n_nodes, -1, dtype=np.int64)
        i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
        i, j, k = i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")
        node = g.node_index(i, j, k)
        sel = i > 0
        e = g.edge_index(0, i[sel] - 1, j[sel], k[sel])
        parent_node[node[sel]] = g.node_index(i[sel] - 1, j[sel], k[sel])
        parent_edge[node[sel]] = e
        sel = (i == 0) & (j > 0)
        e2 = g.edge_index(1, i[sel], j[sel] - 1, k[sel])
        parent_node[node[sel]] = g.node_index(i[sel], j[sel] - 1, k[sel])
        parent_edge[node[sel]] = e2
        sel = (i == 0) & (j == 0) & (k > 0)
        e3 = g.edge_index(2, i[sel], j[sel], k[sel] - 1)
        parent_node[node[sel]] = g.node_index(i[sel], j[sel], k[sel] - 1)
        parent_edge[node[sel]] = e3
        mask[np.concatenate([e, e2, e3])] = True
        return mask, parent_node, parent_edge

    @property
    def edge_mask(self) -> np.ndarray:
        return self._arrays[0]

    @property
    def parent_node(self) -> np.ndarray:
        return self._arrays[1]

    @property
    def parent_edge(self) -> np.ndarray:
        return self._arrays[2]

    @property
    def n_tree_edges(self) -> int:
        nx, ny, nz = self.grid.dims
        return (nx + 1) * (ny + 1) * (nz + 1) - 1  # a spanning tree of the node box


def build_comb_tree(grid: StaggeredGrid) -> SpanningTree:
    """Deterministic comb tree rooted at node (0, 0, 0) (gauging.py:34-71):
    x-edges on the line (., 0, 0), y-edges in the plane (., ., 0), every z-edge."""
    return SpanningTree(grid, "comb")


def build_bfs_tree(grid: StaggeredGrid) -> SpanningTree:
    """Breadth-first spanning tree from node 0 with the reference's
    deterministic frontier order (gauging.py:74-119)."""
    return SpanningTree(grid, "bfs")


def build_tree(grid: StaggeredGrid, kind: str = "comb") -> SpanningTree:
    if kind == "comb":
        return build_comb_tree(grid)
    if kind == "bfs":
        return build_bfs_tree(grid)
    raise ValueError(f"unknown tree kind {kind!r}")


def circulation_residual(values, fluxes, grid: StaggeredGrid):
    """Per-face circulation defect (gauging.py:127-134)."""
    as_np = not isinstance(values, torch.Tensor)
    out = field_ops(grid).circulation(values, fluxes)
    return out.cpu().numpy() if as_np else out


def gauge_vector_potential(fluxes, grid: StaggeredGrid, tree: SpanningTree, tol: float = 1e-10):
    """Edge vector potential with zero tree-edge entries reproducing the
    fluxes (gauging.py:137-172).  Raises IncompatibleFluxError when the
    relative circulation residual exceeds `tol`."""
    as_np = not isinstance(fluxes, torch.Tensor)
    n = int(np.prod(np.shape(fluxes)))
    if n != grid.n_faces:
        raise ValueError(f"flux vector has length {n}, expected {grid.n_faces}")
    if tree.kind not in ("comb", "bfs") or tree.grid != grid:
        raise ValueError("gauge_vector_potential needs a comb or BFS tree of this grid (build_tree(grid, kind))")
    out = field_ops(grid).gauge(_dev(fluxes), tol, tree=tree.kind)
    return out.cpu().numpy() if as_np else out
