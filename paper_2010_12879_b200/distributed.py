"""Multi-GPU z-slab decomposition of the snapshot solve.

One process per GPU.  `torch.distributed` is only the plumbing that hands
the 128-byte NCCL unique id to every rank (and, for tests, the gloo
transport); the halo planes, coarse halos and dot-product allgathers of the
solve itself run inside libspfd_b200.so on the solve stream.

    comm = Communicator.nccl()                 # after dist.init_process_group("nccl")
    sess = Session(model, f, cfg)              # identical operator + hierarchy on every rank
    sess.distribute(comm)                      # rank r owns node planes [k_r, k_{r+1})
    vox, rep, _ = sess.snapshot(a_dev)         # valid on sess.vox_range

`Communicator.host()` routes the same messages through host callbacks over
any torch.distributed group (gloo), which lets several processes share one
GPU in tests.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


class HostTransport:
    """Message protocol of the host transport, independent of where the
    bytes live: `exchange` posts every send/recv of one group at once, so
    the order in which ranks call it cannot deadlock; `allgather` is
    rank-ordered.  Buffers are CPU uint8 tensors."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def exchange(self, ops):
        """ops: list of (peer, kind, tensor) with kind 0 = send, 1 = recv."""
        reqs = []
        for peer, kind, t in ops:
            gpeer = dist.get_global_rank(self.group, peer) if self.group is not None else peer
            if kind == 0:
                reqs.append(dist.isend(t, gpeer, group=self.group))
            else:
                reqs.append(dist.irecv(t, gpeer, group=self.group))
        for r in reqs:
            r.wait()

    def allgather(self, send):
        out = [torch.empty_like(send) for _ in range(self.size)]
        dist.all_gather(out, send, group=self.group)
        return torch.cat(out)


def _nccl_library_hint():
    """Point the library's NCCL loader (dlopen, csrc/comm.cu) at the
    nvidia-nccl wheel PyTorch uses, unless SPFD_NCCL_LIB is already set."""
    if os.environ.get("SPFD_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        for base in list(getattr(nvidia.nccl, "__path__", [])):
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["SPFD_NCCL_LIB"] = cand
                return
    except ImportError:
        pass


class Communicator:
    """Owns a spfd_comm_t handle."""

    def __init__(self, handle, rank, size, keep=None):
        self.handle = handle
        self.rank = rank
        self.size = size
        self._keep = keep  # callbacks must outlive the handle

    @classmethod
    def nccl(cls, group=None):
        """NCCL transport; rank 0 creates the unique id, torch.distributed
        broadcasts it."""
        _nccl_library_hint()
        lib = _lib.load()
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            _lib.check(lib.spfd_nccl_unique_id(buf))
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            uid_d = uid.cuda()
            dist.broadcast(uid_d, dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = uid_d.cpu()
        else:
            dist.broadcast(uid, dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = (ctypes.c_uint8 * 128)(*uid.tolist())
        h = ctypes.c_void_p()
        _lib.check(lib.spfd_comm_init_nccl(raw, rank, size, ctypes.byref(h)))
        return cls(h, rank, size)

    @classmethod
    def host(cls, group=None):
        """Host-callback transport over a torch.distributed group (gloo)."""
        lib = _lib.load()
        tr = HostTransport(group)

        def exchange(user, n, peer, kind, buf, nbytes):
            try:
                ops, recvs = [], []
                for i in range(n):
                    t = torch.empty(int(nbytes[i]), dtype=torch.uint8)
                    if kind[i] == 0:
                        _lib.check(lib.spfd_copy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(buf[i]), t.numel()))
                    else:
                        recvs.append((t, buf[i]))
                    ops.append((int(peer[i]), int(kind[i]), t))
                tr.exchange(ops)
                for t, dst in recvs:
                    _lib.check(lib.spfd_copy(ctypes.c_void_p(dst), ctypes.c_void_p(t.data_ptr()), t.numel()))
                return 0
            except Exception:  # pragma: no cover - surfaced as SPFD_ENCCL
                return 1

        def allgather(user, send, recv, nbytes):
            try:
                t = torch.empty(int(nbytes), dtype=torch.uint8)
                _lib.check(lib.spfd_copy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(send), t.numel()))
                out = tr.allgather(t).contiguous()
                _lib.check(lib.spfd_copy(ctypes.c_void_p(recv), ctypes.c_void_p(out.data_ptr()), out.numel()))
                return 0
            except Exception:  # pragma: no cover
                return 1

        cb = _lib.CommCallbacks(None, _lib.EXCHANGE_FN(exchange), _lib.ALLGATHER_FN(allgather))
        h = ctypes.c_void_p()
        _lib.check(lib.spfd_comm_init_callbacks(ctypes.byref(cb), tr.rank, tr.size, ctypes.byref(h)))
        return cls(h, tr.rank, tr.size, keep=(cb, exchange, allgather))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().spfd_comm_destroy(h)
            except Exception:
                pass
            self.handle = None


def slab_planes(node_plane_positions: np.ndarray, size: int) -> list:
    """Plane boundaries balanced by span positions -- the same rule as
    amg_distribute (dist.cuh): rank p starts at the first plane whose first
    position reaches p*L/size, each rank keeping at least one plane.
    `node_plane_positions` is the first position of every plane plus L."""
    pos = np.asarray(node_plane_positions, dtype=np.int64)
    nz = pos.size - 1
    L = int(pos[-1])
    kb = [0]
    for p in range(1, size):
        target = L * p // size
        k = kb[-1] + 1
        while k < nz - (size - p) and pos[k] < target:
            k += 1
        kb.append(k)
    kb.append(nz)
    return kb
