"""Shared fixtures.  `gpu` tests need a CUDA device and the built library;
everything else runs on CPU (oracle vs golden vectors, host logic, ABI)."""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libspfd_b200.so")
    config.addinivalue_line("markers", "slow: large configuration (C3-sized)")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def golden_cases(kind="model"):
    names = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
    if kind == "model":
        return [n for n in names if not n.startswith(("laplacian", "field"))]
    if kind == "field":
        return [n for n in names if n.startswith("field")]
    return [n for n in names if n.startswith("laplacian")]


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_csr(d, prefix):
    import scipy.sparse as sp
    return sp.csr_matrix((d[prefix + "_data"], d[prefix + "_indices"], d[prefix + "_indptr"]),
                         shape=tuple(d[prefix + "_shape"]))


def golden_kappa(d):
    dims = tuple(int(v) for v in d["dims"])
    return d["lut"][d["ids"]].reshape(dims, order="F")


def golden_model(d):
    """VoxelModel with a constant-kappa table equal to the golden LUT."""
    from paper_2010_12879_b200.voxel_model import ConductivitySamples, Tissue, VoxelModel
    dims = tuple(int(v) for v in d["dims"])
    ids = d["ids"].reshape(dims, order="F")
    table = {i: Tissue(f"t{i}", ConductivitySamples.constant(float(k))) for i, k in enumerate(d["lut"])}
    return VoxelModel(dims, tuple(float(s) for s in d["spacing"]), (0.0, 0.0, 0.0), ids, table)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
