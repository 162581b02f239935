"""Staggered-grid index spaces and the device-assembled Poisson system.

Drop-in for the reference's `StaggeredGrid`, `edge_conductance`,
`PoissonSystem` and `assemble_poisson`
(/root/reference/pkg/src/spfd/fit_operators.py:31-457).  The operator lives
on the GPU (`DeviceOperator`, a handle of libspfd_b200.so): conductances,
component labelling and pinning, DOF numbering, the matrix-free 7-point
stencil and the RHS are computed there.  Host-side numpy/scipy views
(`matrix`, `rhs`, `dof_to_node`, ...) are materialised lazily from the
device on first access and are bit-identical to the reference's arrays.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .voxel_model import ids_fortran_flat, kappa_lut


@dataclass(frozen=True)
class StaggeredGrid:
    """Node/edge/face/cell index structure (fit_operators.py:31-124)."""

    dims: tuple
    spacing: tuple
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        spacing = tuple(float(s) for s in self.spacing)
        if len(dims) != 3 or any(n < 0 for n in dims):
            raise ValueError(f"dims must be three integers >= 0, got {dims}")
        if len(spacing) != 3 or any(not s > 0.0 for s in spacing):
            raise ValueError(f"spacing must be positive, got {spacing}")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "origin", tuple(float(o) for o in self.origin))

    @classmethod
    def from_model(cls, model) -> "StaggeredGrid":
        return cls(model.dims, model.spacing, getattr(model, "origin", (0.0, 0.0, 0.0)))

    @property
    def node_dims(self):
        return tuple(n + 1 for n in self.dims)

    @property
    def n_nodes(self) -> int:
        a, b, c = self.node_dims
        return a * b * c

    def edge_dims(self, axis: int):
        d = list(self.node_dims)
        d[axis] = self.dims[axis]
        return tuple(d)

    @cached_property
    def edge_counts(self):
        return tuple(int(np.prod(self.edge_dims(a))) for a in range(3))

    @cached_property
    def edge_offsets(self):
        ex, ey, _ = self.edge_counts
        return (0, ex, ex + ey)

    @property
    def n_edges(self) -> int:
        return sum(self.edge_counts)

    @property
    def n_cells(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    def node_index(self, i, j, k):
        nx1, ny1, _ = self.node_dims
        return i + nx1 * (j + ny1 * np.asarray(k))

    def edge_index(self, axis: int, i, j, k):
        d = self.edge_dims(axis)
        return self.edge_offsets[axis] + i + d[0] * (j + d[1] * np.asarray(k))

    def cell_index(self, i, j, k):
        nx, ny, _ = self.dims
        return i + nx * (j + ny * np.asarray(k))

    def edge_blocks(self, vec):
        out = []
        for a in range(3):
            lo = self.edge_offsets[a]
            out.append(vec[lo:lo + self.edge_counts[a]].reshape(self.edge_dims(a), order="F"))
        return tuple(out)

    def merge_edge_blocks(self, blocks) -> np.ndarray:
        return np.concatenate([np.asarray(b).ravel(order="F") for b in blocks])

    def face_area(self, axis: int) -> float:
        s = self.spacing
        t = [a for a in range(3) if a != axis]
        return s[t[0]] * s[t[1]]

    # -- faces (fit_operators.py:72-165) -------------------------------------

    def face_dims(self, axis: int):
        d = list(self.dims)
        d[axis] = self.dims[axis] + 1
        return tuple(d)

    @cached_property
    def face_counts(self):
        return tuple(int(np.prod(self.face_dims(a))) for a in range(3))

    @cached_property
    def face_offsets(self):
        fx, fy, _ = self.face_counts
        return (0, fx, fx + fy)

    @property
    def n_faces(self) -> int:
        return sum(self.face_counts)

    def face_index(self, axis: int, i, j, k):
        d = self.face_dims(axis)
        return self.face_offsets[axis] + i + d[0] * (j + d[1] * np.asarray(k))

    def face_blocks(self, vec):
        out = []
        for a in range(3):
            lo = self.face_offsets[a]
            out.append(vec[lo:lo + self.face_counts[a]].reshape(self.face_dims(a), order="F"))
        return tuple(out)

    def merge_face_blocks(self, blocks) -> np.ndarray:
        return np.concatenate([np.asarray(b).ravel(order="F") for b in blocks])

    def face_center_axes(self, axis: int):
        """Per-axis 1-d center coordinates of the faces with the given normal."""
        d = self.face_dims(axis)
        out = []
        for a in range(3):
            if a == axis:
                out.append(self.origin[a] + np.arange(d[a]) * self.spacing[a])
            else:
                out.append(self.origin[a] + (np.arange(d[a]) + 0.5) * self.spacing[a])
        return tuple(out)

    def box(self):
        """The grid as a C-ABI `spfd_box`."""
        return _lib.make_box(self.dims, self.spacing, self.origin)


# ---------------------------------------------------------------------------
# device operator
# ---------------------------------------------------------------------------

def _cuda(t, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (no copy if already there)."""
    if isinstance(t, torch.Tensor):
        t = t.to(device="cuda", dtype=dtype) if dtype is not None else t.to("cuda")
        return t.contiguous()
    arr = np.ascontiguousarray(t)
    out = torch.from_numpy(arr)
    if dtype is not None:
        out = out.to(dtype)
    return out.to("cuda", non_blocking=False).contiguous()


class DeviceOperator:
    """GPU-resident assembled operator for one (model, frequency, pin)."""

    def __init__(self, model, frequency_hz: float, pin: bool = True):
        _lib.require_cuda()
        self._lib = _lib.load()
        self.dims = tuple(int(n) for n in model.dims)
        self.spacing = tuple(float(s) for s in model.spacing)
        self.frequency_hz = float(frequency_hz)
        self.pin = bool(pin)
        lut = kappa_lut(model, frequency_hz)
        ids = ids_fortran_flat(model)
        self._ids = _cuda(ids.view(np.int16))
        self._lut = _cuda(lut)
        h = ctypes.c_void_p()
        d = (ctypes.c_int64 * 3)(*self.dims)
        s = (ctypes.c_double * 3)(*self.spacing)
        _lib.check(self._lib.spfd_op_create(d, s, _lib.ptr(self._ids), _lib.ptr(self._lut), lut.size,
                                            1 if pin else 0, _lib.stream_ptr(), ctypes.byref(h)))
        self.handle = h
        info = _lib.OpInfo()
        _lib.check(self._lib.spfd_op_info_get(h, ctypes.byref(info)))
        self.info = info
        self.n_dofs = int(info.n_dofs)
        self.n_nodes = int(info.n_nodes)
        self.n_edges = int(info.n_edges)
        self.n_conductive = int(info.n_conductive)
        self.n_components = int(info.n_components)
        self.n_cond_voxels = int(info.n_cond_voxels)
        self.nnz = int(info.nnz)
        self.span_len = int(info.span_len)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.spfd_op_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- exports ---------------------------------------------------------
    def export(self, what: int) -> torch.Tensor:
        sizes = {
            _lib.EXPORT_EDGE_CONDUCTANCE: (self.n_edges, torch.float64),
            _lib.EXPORT_DOF_TO_NODE: (self.n_dofs, torch.int64),
            _lib.EXPORT_NODE_TO_DOF: (self.n_nodes, torch.int64),
            _lib.EXPORT_PINNED: (self.n_components, torch.int64),
            _lib.EXPORT_VOXEL_INDICES: (self.n_cond_voxels, torch.int64),
            _lib.EXPORT_DIAGONAL: (self.n_dofs, torch.float64),
        }
        n, dt = sizes[what]
        out = torch.empty(max(n, 1), dtype=dt, device="cuda")
        _lib.check(self._lib.spfd_op_export(self.handle, what, _lib.ptr(out), _lib.stream_ptr()))
        return out[:n]

    def csr_device(self):
        ip = torch.empty(self.n_dofs + 1, dtype=torch.int64, device="cuda")
        ix = torch.empty(max(self.nnz, 1), dtype=torch.int32, device="cuda")
        dv = torch.empty(max(self.nnz, 1), dtype=torch.float64, device="cuda")
        _lib.check(self._lib.spfd_op_csr(self.handle, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), _lib.stream_ptr()))
        return ip, ix[:self.nnz], dv[:self.nnz]

    def csr_host(self) -> sp.csr_matrix:
        ip, ix, dv = self.csr_device()
        m = StencilMatrix((dv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()),
                          shape=(self.n_dofs, self.n_dofs))
        m._spfd_op = self
        return m

    # -- compute -----------------------------------------------------------
    def _planar(self, x, length):
        t = _cuda(x, torch.float64)
        if t.dim() == 1:
            t = t.reshape(1, -1)
        if t.shape[-1] != length or t.shape[0] not in (1, 2):
            raise ValueError(f"expected shape (n,) or (nrhs<=2, n) with n={length}, got {tuple(t.shape)}")
        return t.contiguous()

    def stencil(self, x):
        t = self._planar(x, self.n_dofs)
        y = torch.empty_like(t)
        _lib.check(self._lib.spfd_stencil_apply(self.handle, _lib.ptr(t), _lib.ptr(y), t.shape[0], _lib.stream_ptr()))
        return y

    def rhs(self, a):
        t = self._planar(a, self.n_edges)
        out = torch.empty((t.shape[0], self.n_dofs), dtype=torch.float64, device="cuda")
        _lib.check(self._lib.spfd_rhs_assemble(self.handle, _lib.ptr(t), _lib.ptr(out), t.shape[0],
                                               _lib.stream_ptr()))
        return out

    def edge_voltages(self, a, psi, omega):
        at = self._planar(a, self.n_edges)
        pt = self._planar(psi, self.n_dofs)
        if at.shape[0] != pt.shape[0]:
            raise ValueError("vector potential and potential have different nrhs")
        out = torch.empty_like(at)
        _lib.check(self._lib.spfd_edge_voltages(self.handle, _lib.ptr(at), _lib.ptr(pt), float(omega), _lib.ptr(out),
                                                at.shape[0], _lib.stream_ptr()))
        return out

    def node_field(self, v):
        vt = self._planar(v, self.n_edges)
        out = torch.empty((vt.shape[0], self.n_nodes), dtype=torch.float64, device="cuda")
        _lib.check(self._lib.spfd_node_field(self.handle, _lib.ptr(vt), _lib.ptr(out), vt.shape[0], _lib.stream_ptr()))
        return out

    def voxel_average(self, node):
        nt = self._planar(node, self.n_nodes)
        out = torch.empty((nt.shape[0], max(self.n_cond_voxels, 1)), dtype=torch.float64, device="cuda")
        _lib.check(self._lib.spfd_voxel_average(self.handle, _lib.ptr(nt), _lib.ptr(out), nt.shape[0],
                                                _lib.stream_ptr()))
        return out[:, :self.n_cond_voxels]

    def efield_voxavg(self, a, psi, omega):
        at = self._planar(a, self.n_edges)
        pt = self._planar(psi, self.n_dofs)
        out = torch.empty((at.shape[0], max(self.n_cond_voxels, 1)), dtype=torch.float64, device="cuda")
        _lib.check(self._lib.spfd_efield_voxavg(self.handle, _lib.ptr(at), _lib.ptr(pt), float(omega), _lib.ptr(out),
                                                at.shape[0], _lib.stream_ptr()))
        return out[:, :self.n_cond_voxels]


class StencilMatrix(sp.csr_matrix):
    """scipy CSR view of the device operator; carries the operator handle so
    `amg_setup(system.matrix)` selects the matrix-free structured path."""

    _spfd_op = None


# ---------------------------------------------------------------------------
# reference API
# ---------------------------------------------------------------------------

def edge_conductance(model, grid: StaggeredGrid, frequency_hz: float) -> np.ndarray:
    """Edge conductances (fit_operators.py:311-324), computed on the GPU."""
    op = DeviceOperator(model, frequency_hz, pin=False)
    return op.export(_lib.EXPORT_EDGE_CONDUCTANCE).cpu().numpy()


class PoissonSystem:
    """Reduced SPD system on free conductive nodes (fit_operators.py:336-364).

    Host arrays are lazy views of the device operator; `rhs_device` /
    `operator` give the resident tensors/handle used by the solver.
    """

    def __init__(self, op: DeviceOperator, rhs_device: torch.Tensor, grid: StaggeredGrid, frequency_hz: float):
        self.operator = op
        self.rhs_device = rhs_device  # (nrhs, n_dofs)
        self.grid = grid
        self.frequency_hz = float(frequency_hz)
        self.n_conductive_nodes = op.n_conductive
        self.n_components = op.n_components

    @property
    def n_dofs(self) -> int:
        return self.operator.n_dofs

    @cached_property
    def matrix(self) -> sp.csr_matrix:
        return self.operator.csr_host()

    @cached_property
    def rhs(self) -> np.ndarray:
        r = self.rhs_device.cpu().numpy()
        return r[0].copy() if r.shape[0] == 1 else r

    @cached_property
    def dof_to_node(self) -> np.ndarray:
        return self.operator.export(_lib.EXPORT_DOF_TO_NODE).cpu().numpy()

    @cached_property
    def node_to_dof(self) -> np.ndarray:
        return self.operator.export(_lib.EXPORT_NODE_TO_DOF).cpu().numpy()

    @cached_property
    def pinned_nodes(self) -> np.ndarray:
        return self.operator.export(_lib.EXPORT_PINNED).cpu().numpy()

    @cached_property
    def edge_conductance(self) -> np.ndarray:
        return self.operator.export(_lib.EXPORT_EDGE_CONDUCTANCE).cpu().numpy()

    def expand(self, reduced) -> np.ndarray:
        full = np.zeros(self.grid.n_nodes, dtype=np.float64)
        full[self.dof_to_node] = reduced
        return full


def assemble_poisson(model, grid: StaggeredGrid, vector_potential, frequency_hz: float, *, pin: bool = True,
                     use_triple_product: bool = False) -> PoissonSystem:
    """Assemble the conductivity-weighted Poisson system on the GPU
    (fit_operators.py:367-457).  `vector_potential` is one edge vector
    (n_edges,) or a stacked real/imag pair (2, n_edges), numpy or torch.
    `use_triple_product` is accepted for API compatibility: the device path
    always forms G^T M G through the stencil (both reference paths agree,
    test_fit_operators.py:162-172)."""
    n_edges = grid.n_edges
    shape = tuple(vector_potential.shape)
    if shape not in ((n_edges,), (1, n_edges), (2, n_edges)):
        raise ValueError(f"vector potential has length {shape[-1] if shape else 0}, expected {n_edges}")
    op = DeviceOperator(model, frequency_hz, pin=pin)
    rhs = op.rhs(vector_potential) if op.n_dofs > 0 else torch.zeros((1, 0), dtype=torch.float64, device="cuda")
    return PoissonSystem(op, rhs, grid, frequency_hz)
