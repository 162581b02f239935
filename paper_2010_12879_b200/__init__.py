"""B200-native SPFD Poisson hot path (arXiv 2010.12879), drop-in for the
reference package's solver/operator API (`spfd`).

The compute runs in libspfd_b200.so (hand-written sm_100a CUDA, C-ABI in
include/spfd_b200.h); this package is the host-side mirror of the
reference interface.  Importing works without a GPU (for building and
introspection); every compute call requires CUDA and fails loudly otherwise.
"""

from .dosimetry import corner_mean, edge_voltages, efield_voxel_average, node_field_strength, voxel_average
from .errors import EmptySystemError, PipelineError, SolverError, SpfdError
from .fit_operators import (DeviceOperator, PoissonSystem, StaggeredGrid, StencilMatrix, assemble_poisson,
                            edge_conductance)
from .gauging import SpanningTree, build_bfs_tree, build_comb_tree, gauge_vector_potential
from .linsolve import (AmgHierarchy, AmgLevel, SolveConfig, SolveReport, amg_setup, fgmres_solve, pcg_solve,
                       solve, v_cycle)
from .pipeline import Session
from .voxel_model import ConductivitySamples, Tissue, VoxelModel, kappa_at, make_phantom

__version__ = "0.1.0"

__all__ = [
    "AmgHierarchy", "AmgLevel", "ConductivitySamples", "DeviceOperator", "EmptySystemError", "PipelineError",
    "SpanningTree", "build_bfs_tree", "build_comb_tree", "gauge_vector_potential",
    "PoissonSystem", "Session", "SolveConfig", "SolveReport", "SolverError", "SpfdError", "StaggeredGrid",
    "StencilMatrix", "Tissue", "VoxelModel", "amg_setup", "assemble_poisson", "corner_mean", "edge_conductance",
    "edge_voltages", "efield_voxel_average", "fgmres_solve", "kappa_at", "make_phantom", "node_field_strength",
    "pcg_solve", "solve", "v_cycle", "voxel_average",
]
