"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes tests/golden/<case>.npz.  The GPU box never reads /root/reference;
it only reads these committed fixtures.  Every array comes straight from the
reference package (`spfd`): conductances, the assembled CSR matrix and RHS,
DOF maps, the AMG hierarchy (aggregates, P, R, coarse operators), the
FGMRES solution at rel_tol 1e-12, and the E-field chain.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import scipy.sparse as sp  # noqa: E402
from spfd import dosimetry as rd  # noqa: E402
from spfd import field_source as rf  # noqa: E402
from spfd import fit_operators as ro  # noqa: E402
from spfd import gauging as rg  # noqa: E402
from spfd import linsolve as rl  # noqa: E402
from spfd import voxel_model as rv  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FREQ = 85e3


def block(dims, kappa=0.2, spacing=0.002):
    ids = np.ones(dims, dtype=np.uint16)
    table = {0: rv.Tissue("free_space", rv.ConductivitySamples.constant(0.0)),
             1: rv.Tissue("tissue", rv.ConductivitySamples.constant(kappa))}
    return rv.VoxelModel(dims, (spacing,) * 3, (0.0, 0.0, 0.0), ids, table)


def two_blobs():
    """Two separate conductive bodies, an internal cavity and a row with two
    spans: exercises multi-component pinning and holes."""
    dims = (14, 9, 8)
    ids = np.zeros(dims, dtype=np.uint16)
    ids[1:6, 1:8, 1:7] = 1
    ids[8:13, 2:7, 2:6] = 2
    ids[3, 4, 3] = 0          # cavity inside body 1
    table = {0: rv.Tissue("free_space", rv.ConductivitySamples.constant(0.0)),
             1: rv.Tissue("a", rv.ConductivitySamples.from_pairs([(1e3, 0.1), (1e6, 0.4)])),
             2: rv.Tissue("b", rv.ConductivitySamples.constant(0.05))}
    return rv.VoxelModel(dims, (0.002, 0.0025, 0.003), (0.0, 0.0, 0.0), ids, table)


def reference_potential(model, b):
    """Uniform field through the reference's own chain: lattice sampling,
    face interpolation, comb-tree gauging (pipeline.py:105-156)."""
    grid = ro.StaggeredGrid.from_model(model)
    lattice = rf.Lattice.covering(grid, (2, 2, 2))
    samples = rf.sample_on_lattice(rf.UniformField(b), lattice, FREQ)
    flux = rf.interpolate_to_faces(samples, grid)
    flux = rf.divergence_clean(flux, grid, 1e-10)
    tree = rg.build_tree(grid, "comb")
    return rg.gauge_vector_potential(flux, grid, tree, 1e-10)


def dipole_potential(model, moment, center):
    grid = ro.StaggeredGrid.from_model(model)
    out = []
    for axis in range(3):
        ed = grid.edge_dims(axis)
        c = []
        for a in range(3):
            v = np.arange(ed[a]) * model.spacing[a]
            if a == axis:
                v = v + 0.5 * model.spacing[a]
            c.append(v - center[a])
        X, Y, Z = c[0][:, None, None], c[1][None, :, None], c[2][None, None, :]
        r3 = (X * X + Y * Y + Z * Z) ** 1.5
        m = moment
        comp = [m[1] * Z - m[2] * Y, m[2] * X - m[0] * Z, m[0] * Y - m[1] * X][axis]
        out.append((1e-7 * comp / r3 * model.spacing[axis]).ravel(order="F"))
    return np.concatenate(out)


def csr_parts(prefix, m, d):
    m = sp.csr_matrix(m)
    d[prefix + "_indptr"] = m.indptr.astype(np.int64)
    d[prefix + "_indices"] = m.indices.astype(np.int32)
    d[prefix + "_data"] = m.data.astype(np.float64)
    d[prefix + "_shape"] = np.array(m.shape, dtype=np.int64)


def hierarchy_parts(h, d, max_levels_store=10):
    d["amg_sizes"] = np.array(h.level_sizes, dtype=np.int64)
    for l, lv in enumerate(h.levels[:max_levels_store]):
        csr_parts(f"A{l}", lv.matrix, d)
        if lv.prolongation is not None:
            csr_parts(f"P{l}", lv.prolongation, d)
            csr_parts(f"R{l}", lv.restriction, d)


def aggregates(h, cfg):
    """Re-run the reference's strength graph + plain_aggregation per level."""
    from spfd._kernels import plain_aggregation
    out = []
    for l, lv in enumerate(h.levels[:-1]):
        ip, ix, sv = rl._strength_graph(lv.matrix, cfg.strength_threshold * 0.5 ** l)
        agg, _ = plain_aggregation(ip, ix, sv, lv.matrix.shape[0])
        out.append(agg.astype(np.int32))
    return out


def model_case(name, model, a, solve=True, store_amg=True):
    grid = ro.StaggeredGrid.from_model(model)
    d = {}
    d["dims"] = np.array(model.dims, dtype=np.int64)
    d["spacing"] = np.array(model.spacing, dtype=np.float64)
    d["ids"] = np.asarray(model.tissue_ids, dtype=np.uint16).ravel(order="F")
    lut = np.zeros(int(model.tissue_ids.max()) + 1)
    for tid, t in model.tissue_table.items():
        if tid < lut.size:
            lut[tid] = t.conductivity.at(FREQ)
    d["lut"] = lut
    d["freq"] = np.array(FREQ)
    d["a"] = np.asarray(a, dtype=np.float64)
    system = ro.assemble_poisson(model, grid, a, FREQ)
    d["w"] = system.edge_conductance
    csr_parts("matrix", system.matrix, d)
    d["rhs"] = system.rhs
    d["dof_to_node"] = system.dof_to_node.astype(np.int64)
    d["pinned"] = system.pinned_nodes.astype(np.int64)
    d["n_components"] = np.array(system.n_components)
    d["n_conductive"] = np.array(system.n_conductive_nodes)
    labels = rv.conductive_component_labels(model, FREQ)
    d["labels"] = labels.astype(np.int32)
    cfg = rl.SolveConfig(rel_tol=1e-12)
    h = rl.amg_setup(system.matrix, cfg)
    if store_amg:
        hierarchy_parts(h, d)
        for l, agg in enumerate(aggregates(h, cfg)):
            d[f"agg{l}"] = agg
    if solve and system.rhs.any():
        psi, rep = rl.fgmres_solve(system.matrix, system.rhs, h, cfg)
        d["psi"] = psi
        d["fgmres_iters"] = np.array(rep.iterations)
        omega = 2 * math.pi * FREQ
        v = rd.edge_voltages(a, psi, system, omega)
        nf = rd.node_field_strength(v, grid, model, FREQ)
        vals, idx = rd.voxel_average(nf, grid, model, FREQ)
        d["omega"] = np.array(omega)
        d["volts"] = v
        d["node_field"] = nf.ravel(order="F")
        d["vox"] = vals
        d["vox_idx"] = idx.astype(np.int64)
    # a random residual through the reference V-cycle
    rng = np.random.default_rng(20240817)
    r = rng.standard_normal(system.n_dofs)
    d["vcycle_in"] = r
    d["vcycle_out"] = rl.v_cycle(h, r)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, "dofs", system.n_dofs, "levels", h.level_sizes, "bytes",
          os.path.getsize(os.path.join(OUT, f"{name}.npz")))


def matrix_case(name, a):
    d = {}
    cfg = rl.SolveConfig(rel_tol=1e-12)
    h = rl.amg_setup(a, cfg)
    hierarchy_parts(h, d)
    for l, agg in enumerate(aggregates(h, cfg)):
        d[f"agg{l}"] = agg
    rng = np.random.default_rng(20240817)
    b = rng.standard_normal(a.shape[0])
    x, rep = rl.fgmres_solve(a, b, h, cfg)
    d["b"] = b
    d["x"] = x
    d["fgmres_iters"] = np.array(rep.iterations)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, "n", a.shape[0], "levels", h.level_sizes)


def laplacian_3d(n):
    d = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    eye = sp.identity(n)
    return (sp.kron(sp.kron(d, eye), eye) + sp.kron(sp.kron(eye, d), eye)
            + sp.kron(sp.kron(eye, eye), d)).tocsr()


def field_case(name):
    """Rows f1-f4 through the reference: coil Biot-Savart samples on a lattice
    that does not cover the grid (extrapolation), face interpolation, the
    divergence and its cleaning, comb-tree gauging (FIFO elimination), the
    circulation residual, the cleaning hierarchy's aggregates, and the
    exposure report of a voxel field."""
    grid = ro.StaggeredGrid((12, 10, 8), (0.002, 0.0025, 0.003), (0.001, -0.002, 0.0005))
    axis = (0.2, 0.1, 1.0)
    coil = rf.CoilSpec(center=(0.012, 0.01, -0.02), axis=axis, radius_m=0.03, current_a=5.0, segments=64)
    lattice = rf.Lattice((0.004, -0.001, 0.002), (0.006, 0.007, 0.008), (4, 4, 3))
    samples = rf.sample_on_lattice(coil, lattice, FREQ)
    d = {"grid_dims": np.array(grid.dims, np.int64), "grid_spacing": np.array(grid.spacing),
         "grid_origin": np.array(grid.origin), "lat_dims": np.array(lattice.dims, np.int64),
         "lat_spacing": np.array(lattice.spacing), "lat_origin": np.array(lattice.origin),
         "coil_center": np.array(coil.center), "coil_axis": np.array(axis),
         "coil_radius": np.array(coil.radius_m), "coil_current": np.array(coil.current_a),
         "coil_segments": np.array(coil.segments), "coil_vertices": coil.vertices(),
         "points": samples.positions, "b": samples.b}
    flux = rf.interpolate_to_faces(samples, grid)
    div = ro.build_divergence(grid)
    d["flux"] = flux
    d["div"] = div @ flux
    clean = rf.divergence_clean(flux, grid, 1e-10)
    d["clean"] = clean
    d["clean_div_rel"] = np.array(np.linalg.norm(div @ clean) / np.linalg.norm(flux))
    tree = rg.build_tree(grid, "comb")
    a = rg.gauge_vector_potential(clean, grid, tree, 1e-10)
    d["a"] = a
    d["tree_mask"] = tree.edge_mask
    d["circ"] = rg.circulation_residual(a, clean, grid)
    try:
        rg.gauge_vector_potential(flux, grid, tree, 1e-10)
        d["uncleaned_raises"] = np.array(0)
    except Exception:
        d["uncleaned_raises"] = np.array(1)
    normal = (div @ div.T).tocsr()
    cfg = rl.SolveConfig()
    h = rl.amg_setup(normal, cfg)
    d["normal_sizes"] = np.array(h.level_sizes, np.int64)
    for l, agg in enumerate(aggregates(h, cfg)):
        d[f"normal_agg{l}"] = agg
    csr_parts("normal", h.levels[0].matrix, d)
    # a uniform field: the cleaning is a no-op and the gauge is exact
    usamp = rf.sample_on_lattice(rf.UniformField((0.3e-6, -0.2e-6, 1e-6)), rf.Lattice.covering(grid, (2, 2, 2)), FREQ)
    uflux = rf.interpolate_to_faces(usamp, grid)
    d["uniform_flux"] = uflux
    d["uniform_a"] = rg.gauge_vector_potential(uflux, grid, tree, 1e-10)
    # exposure report of a voxel field with ties, three tissues + free space
    rng = np.random.default_rng(7)
    m = rv.make_phantom("layered-block", (10, 9, 8), 0.002, layers=3, kappa_spm=[0.2, 0.05, 0.4],
                        size_m=(0.016, 0.014, 0.012))
    ids = m.tissue_ids.ravel(order="F")
    idx = np.flatnonzero(ids > 0)
    vals = np.round(rng.gamma(2.0, 1.5, idx.size), 2)
    rep = rd.build_exposure_report(vals, idx, m, FREQ, dof_count=123, rms=True)
    d["st_ids"] = ids.astype(np.uint16)
    d["st_dims"] = np.array(m.dims, np.int64)
    d["st_idx"] = idx.astype(np.int64)
    d["st_vals"] = vals
    d["st_scaled"] = rep.voxel_field
    d["st_p99"] = np.array(rep.percentile99_vpm)
    d["st_max"] = np.array(rep.max_vpm)
    tids = sorted(rep.per_tissue)
    d["st_tids"] = np.array(tids, np.int64)
    d["st_count"] = np.array([rep.per_tissue[t].count for t in tids], np.int64)
    d["st_mean"] = np.array([rep.per_tissue[t].mean for t in tids])
    d["st_tmax"] = np.array([rep.per_tissue[t].max for t in tids])
    d["st_tp99"] = np.array([rep.per_tissue[t].p99 for t in tids])
    d["p99_plain"] = np.array(rd.percentile99(vals))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, "faces", grid.n_faces, "normal levels", h.level_sizes)


def bfs_case(name):
    """The BFS spanning tree (gauging.py:74-119) and the reference's FIFO
    cotree elimination with it (_kernels.py:12-76) on the field_coil grid:
    the tree's mask / parents, the gauged potential of the cleaned coil
    fluxes and of a uniform field, and the circulation residuals."""
    grid = ro.StaggeredGrid((12, 10, 8), (0.002, 0.0025, 0.003), (0.001, -0.002, 0.0005))
    coil = rf.CoilSpec(center=(0.012, 0.01, -0.02), axis=(0.2, 0.1, 1.0), radius_m=0.03, current_a=5.0, segments=64)
    lattice = rf.Lattice((0.004, -0.001, 0.002), (0.006, 0.007, 0.008), (4, 4, 3))
    samples = rf.sample_on_lattice(coil, lattice, FREQ)
    clean = rf.divergence_clean(rf.interpolate_to_faces(samples, grid), grid, 1e-10)
    tree = rg.build_tree(grid, "bfs")
    d = {"grid_dims": np.array(grid.dims, np.int64), "grid_spacing": np.array(grid.spacing),
         "grid_origin": np.array(grid.origin), "clean": clean, "tree_mask": tree.edge_mask,
         "parent_node": tree.parent_node, "parent_edge": tree.parent_edge}
    d["a"] = rg.gauge_vector_potential(clean, grid, tree, 1e-10)
    d["circ"] = rg.circulation_residual(d["a"], clean, grid)
    usamp = rf.sample_on_lattice(rf.UniformField((0.3e-6, -0.2e-6, 1e-6)), rf.Lattice.covering(grid, (2, 2, 2)), FREQ)
    d["uniform_flux"] = rf.interpolate_to_faces(usamp, grid)
    d["uniform_a"] = rg.gauge_vector_potential(d["uniform_flux"], grid, tree, 1e-10)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, "tree edges", int(tree.edge_mask.sum()))


def pipeline_case(name):
    """The reference's run_pipeline end to end (coil source sampled on a
    5x5x5 lattice, cleaning, comb gauge, solve, E-field, report) plus the
    byte images of its file formats."""
    import tempfile
    from spfd import pipeline as rp
    m = two_blobs()
    coil = rf.CoilSpec(center=(0.014, 0.011, -0.01), axis=(0.3, -0.2, 1.0), radius_m=0.02, current_a=20.0, segments=48)
    cfg = rp.PipelineConfig(model=m, coil=coil, frequency_hz=FREQ, coil_lattice_dims=(5, 5, 5), report_rms=True)
    rep, _ = rp.run_pipeline(cfg)
    d = {"coil_center": np.array(coil.center), "coil_axis": np.array((0.3, -0.2, 1.0)),
         "coil_radius": np.array(coil.radius_m), "coil_current": np.array(coil.current_a),
         "coil_segments": np.array(coil.segments), "vox": rep.voxel_field, "vox_idx": rep.voxel_indices,
         "p99": np.array(rep.percentile99_vpm), "max": np.array(rep.max_vpm), "dofs": np.array(rep.dof_count),
         "iters": np.array(rep.solver.iterations)}
    tids = sorted(rep.per_tissue)
    d["tids"] = np.array(tids, np.int64)
    d["t_count"] = np.array([rep.per_tissue[t].count for t in tids], np.int64)
    d["t_mean"] = np.array([rep.per_tissue[t].mean for t in tids])
    d["t_max"] = np.array([rep.per_tissue[t].max for t in tids])
    d["t_p99"] = np.array([rep.per_tissue[t].p99 for t in tids])
    uni = rp.PipelineConfig(model=m, uniform_b=(0.0, 0.0, 1e-6), frequency_hz=FREQ)
    urep, _ = rp.run_pipeline(uni)
    d["u_vox"] = urep.voxel_field
    d["u_p99"] = np.array(urep.percentile99_vpm)
    # file formats: phantom, samples, report and field dump bytes
    with tempfile.TemporaryDirectory() as tmp:
        rv.save_model(m, os.path.join(tmp, "m.phantom"))
        samples = rf.sample_on_lattice(coil, rf.Lattice.covering(ro.StaggeredGrid.from_model(m), (3, 3, 2)), FREQ)
        rf.save_samples(samples, os.path.join(tmp, "s.txt"))
        rd.write_report(rep, os.path.join(tmp, "r.txt"))
        rd.write_field_dump(m, rep.voxel_field, rep.voxel_indices, os.path.join(tmp, "f.dump"))
        for key, fn in (("phantom_bytes", "m.phantom"), ("samples_bytes", "s.txt"), ("report_bytes", "r.txt"),
                        ("dump_bytes", "f.dump")):
            with open(os.path.join(tmp, fn), "rb") as fh:
                d[key] = np.frombuffer(fh.read(), np.uint8)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(name, "dofs", rep.dof_count, "iters", rep.solver.iterations, "p99", rep.percentile99_vpm)


def main():
    rng = np.random.default_rng(20240817)
    m = block((6, 6, 6))
    g = ro.StaggeredGrid.from_model(m)
    model_case("box6_random", m, rng.standard_normal(g.n_edges))

    m = rv.make_phantom("sphere", (8, 8, 8), 0.002, radius_m=0.006)
    model_case("sphere8_uniform", m, reference_potential(m, (0.0, 0.0, 1e-6)))

    m = rv.make_phantom("layered-block", (14, 12, 16), 0.002, layers=4,
                        kappa_spm=[0.17, 0.04, 0.35, 0.02], size_m=(0.02, 0.016, 0.024))
    model_case("layered_dipole", m, dipole_potential(m, (0.0, 0.0, 7.0), (0.014, 0.012, -0.05)))

    m = two_blobs()
    g = ro.StaggeredGrid.from_model(m)
    model_case("two_blobs", m, rng.standard_normal(g.n_edges))

    m = block((16, 16, 16))
    model_case("box16_uniform", m, reference_potential(m, (0.3e-6, -0.2e-6, 1e-6)))

    m = rv.make_phantom("cylinder", (20, 20, 12), 0.002, radius_m=0.016, kappa_spm=0.3)
    model_case("cylinder_uniform", m, reference_potential(m, (0.0, 0.0, 1e-6)))

    matrix_case("laplacian12", laplacian_3d(12))

    field_case("field_coil")
    pipeline_case("field_pipeline")
    bfs_case("field_bfs")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "field":
        field_case("field_coil")
        pipeline_case("field_pipeline")
    elif len(sys.argv) > 1 and sys.argv[1] == "bfs":
        bfs_case("field_bfs")
    else:
        main()
