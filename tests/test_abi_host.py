"""CPU: the C-ABI library loads and exports the header's symbols; host-side
logic (config validation, grid index maps, phantoms, synthetic sources)
matches the reference / oracle; the product path refuses to run without a
GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, cuda_ok, load_golden

HEADER = os.path.join(ROOT, "include", "spfd_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spfd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_function():
    from paper_2010_12879_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "build() must produce libspfd_b200.so"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/spfd_b200.h but not exported"
    # the Python binding declares a signature for every header function
    assert set(names) == set(_lib.EXPORTED_SYMBOLS)
    assert b"sm_100a" in _lib.load().spfd_version()


def test_error_mapping():
    from paper_2010_12879_b200 import _lib
    from paper_2010_12879_b200.errors import EmptySystemError, SolverError
    with pytest.raises(ValueError):
        _lib.check(_lib.SPFD_EINVAL)
    with pytest.raises(SolverError):
        _lib.check(_lib.SPFD_ENONFINITE)
    with pytest.raises(SolverError):
        _lib.check(_lib.SPFD_ENOTPOS)
    with pytest.raises(EmptySystemError):
        _lib.check(_lib.SPFD_EEMPTY)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.SPFD_ECUDA)
    _lib.check(_lib.SPFD_OK)


@pytest.mark.skipif(cuda_ok(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2010_12879_b200 import workloads
    from paper_2010_12879_b200.fit_operators import DeviceOperator
    with pytest.raises(RuntimeError, match="CUDA"):
        DeviceOperator(workloads.box_model((4, 4, 4)), 85e3)


def test_config_validation():
    from paper_2010_12879_b200 import SolveConfig
    for bad in (dict(rel_tol=0.0), dict(restart=0), dict(jacobi_damping=1.5), dict(max_iters=0),
                dict(coarse_cap=0), dict(method="gmres"), dict(max_nrhs=3)):
        with pytest.raises(ValueError):
            SolveConfig(**bad)
    c = SolveConfig()
    assert (c.rel_tol, c.max_iters, c.restart, c.pre_sweeps, c.post_sweeps) == (1e-12, 1000, 30, 1, 1)
    assert (c.jacobi_damping, c.strength_threshold, c.coarse_cap, c.max_levels) == (2.0 / 3.0, 0.08, 500, 20)


def test_config_struct_layout():
    from paper_2010_12879_b200 import SolveConfig, _lib
    c = _lib.make_config(SolveConfig(method="fgmres", max_nrhs=1))
    assert c.method == _lib.METHOD_FGMRES and c.max_nrhs == 1
    # the C struct is 8+4*4+8+8+6*4 with natural alignment
    assert ctypes.sizeof(_lib.Config) == 64
    assert _lib.Config.cheb_degree.offset == 60
    assert ctypes.sizeof(_lib.Report) == 40


def test_grid_index_maps_match_oracle():
    from paper_2010_12879_b200 import StaggeredGrid
    g = StaggeredGrid((5, 4, 3), (0.002, 0.003, 0.004))
    off, cnt = oracle.edge_offsets(g.dims)
    assert g.edge_offsets == off and g.edge_counts == cnt
    assert g.n_edges == oracle.n_edges(g.dims)
    assert g.n_nodes == 6 * 5 * 4
    assert g.node_index(2, 3, 1) == oracle.node_index(g.dims, 2, 3, 1)
    assert g.edge_index(1, 2, 3, 1) == off[1] + 2 + 6 * (3 + 4 * 1)
    v = np.arange(g.n_edges, dtype=float)
    bx, by, bz = g.edge_blocks(v)
    assert bx.shape == (5, 5, 4) and by.shape == (6, 4, 4) and bz.shape == (6, 5, 3)
    assert np.array_equal(g.merge_edge_blocks((bx, by, bz)), v)


@pytest.mark.parametrize("case,kind,kw", [
    ("sphere8_uniform", "sphere", dict(dims=(8, 8, 8), spacing=0.002, radius_m=0.006)),
    ("layered_dipole", "layered-block", dict(dims=(14, 12, 16), spacing=0.002, layers=4,
                                             kappa_spm=[0.17, 0.04, 0.35, 0.02], size_m=(0.02, 0.016, 0.024))),
    ("cylinder_uniform", "cylinder", dict(dims=(20, 20, 12), spacing=0.002, radius_m=0.016, kappa_spm=0.3)),
])
def test_make_phantom_matches_reference_ids(case, kind, kw):
    from paper_2010_12879_b200 import make_phantom
    d = load_golden(case)
    dims = kw.pop("dims")
    sp_ = kw.pop("spacing")
    m = make_phantom(kind, dims, sp_, **kw)
    assert np.array_equal(np.asarray(m.tissue_ids).ravel(order="F"), d["ids"])
    lut = m.kappa_lut(float(d["freq"]))
    assert np.array_equal(lut[: d["lut"].size], d["lut"])


def test_conductivity_log_interpolation_matches_reference():
    from paper_2010_12879_b200 import ConductivitySamples
    d = load_golden("two_blobs")
    s = ConductivitySamples.from_pairs([(1e3, 0.1), (1e6, 0.4)])
    assert s.at(85e3) == d["lut"][1]
    assert s.at(10.0) == 0.1 and s.at(1e9) == 0.4 and s.at(1e6) == 0.4


def test_uniform_potential_is_comb_gauge():
    from paper_2010_12879_b200 import workloads
    dims, s, b = (7, 5, 6), (0.002, 0.002, 0.002), (0.3e-6, -0.2e-6, 1e-6)
    a = workloads.uniform_potential(dims, s, b)
    ref = oracle.comb_gauge(dims, oracle.uniform_face_fluxes(dims, s, b))
    assert np.allclose(a, ref, rtol=1e-12, atol=1e-24)


def test_dipole_potential_symmetry():
    from paper_2010_12879_b200 import workloads
    dims = (6, 6, 6)
    a = workloads.dipole_potential(dims, 0.002, (0, 0, 1.0), (0.006, 0.006, -0.02))
    nx = 6
    ax = a[: nx * 7 * 7].reshape((6, 7, 7), order="F")
    # m along z, centred in x/y: A_x is antisymmetric in y about the centre
    assert np.allclose(ax[:, ::-1, :], -ax, atol=1e-18)


def test_snapshot_fields_unit_norm():
    from paper_2010_12879_b200 import workloads
    f = workloads.snapshot_fields(100)
    assert f.shape == (100, 3)
    assert np.allclose(np.linalg.norm(f, axis=1), 1e-6)
    assert np.array_equal(f, workloads.snapshot_fields(100))


def _header_struct_fields(name):
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    end = re.search(r"\}\s*" + name + ";", text)
    assert end, name
    start = text.rindex("typedef struct {", 0, end.start())
    body = text[start + len("typedef struct {"):end.start()]
    fields = []
    for line in body.split(";"):
        line = line.strip()
        if not line:
            continue
        fields.append(re.sub(r"\[.*\]", "", line.split()[-1]))
    return fields


@pytest.mark.parametrize("cname,pyname", [("spfd_config", "Config"), ("spfd_report", "Report"),
                                          ("spfd_amg_info", "AmgInfo"), ("spfd_op_info", "OpInfo")])
def test_ctypes_structs_match_header(cname, pyname):
    """Every ctypes mirror of a header struct lists the same fields in the same
    order (a drifted mirror would let the library write past the Python
    object)."""
    from paper_2010_12879_b200 import _lib
    py = [f[0] for f in getattr(_lib, pyname)._fields_]
    assert py == _header_struct_fields(cname)


def test_integration_doc_config_stub_matches_header():
    """INTEGRATION.md's reference-side ctypes stub declares spfd_config with
    the header's fields (the maintainer copies it verbatim)."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text[text.index("class Config(ctypes.Structure):"):text.index("class Report(ctypes.Structure):")]
    names = re.findall(r'\("([a-z_0-9]+)",', block)
    assert names == _header_struct_fields("spfd_config")
