"""Multi-process (world_size 2) tests of the z-slab decomposition.

CPU (gloo): the host-transport message protocol and the slab balancing
rule.  GPU (gloo host transport, both ranks sharing cuda:0): the full
distributed snapshot against the single-GPU snapshot -- same iteration
count, voxel |E| within the solve tolerance -- with level 1 distributed
and with level 1 replicated.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, size, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=size)


def _transport_worker(rank, size, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2010_12879_b200.distributed import HostTransport
    _init(rank, size, port)
    tr = HostTransport()
    peer = 1 - rank
    send = torch.arange(10, dtype=torch.uint8) + 10 * rank
    recv = torch.empty(10, dtype=torch.uint8)
    # both ranks post (send, recv) in the same order: must not deadlock
    tr.exchange([(peer, 0, send), (peer, 1, recv)])
    g = tr.allgather(torch.full((4,), rank + 1, dtype=torch.uint8))
    torch.save({"recv": recv, "gather": g}, os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


def test_host_transport_protocol_gloo():
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_transport_worker, args=(2, _port(), out), nprocs=2, join=True)
        r0 = torch.load(os.path.join(out, "r0.pt"))
        r1 = torch.load(os.path.join(out, "r1.pt"))
    assert torch.equal(r0["recv"], torch.arange(10, dtype=torch.uint8) + 10)
    assert torch.equal(r1["recv"], torch.arange(10, dtype=torch.uint8))
    assert r0["gather"].tolist() == [1, 1, 1, 1, 2, 2, 2, 2] == r1["gather"].tolist()


def test_slab_balancing_rule():
    from paper_2010_12879_b200.distributed import slab_planes
    # 100 planes, the body (positions) in planes 10..90 only
    per = np.array([0] * 10 + [50] * 80 + [0] * 10)
    pos = np.concatenate([[0], np.cumsum(per)])
    for size in (2, 4, 8):
        kb = slab_planes(pos, size)
        assert kb[0] == 0 and kb[-1] == 100 and all(a < b for a, b in zip(kb, kb[1:]))
        counts = [pos[kb[p + 1]] - pos[kb[p]] for p in range(size)]
        assert max(counts) - min(counts) <= 50  # balanced to one plane


def _solve_worker(rank, size, port, out, name, replicate_below, transport="host", method="pcg"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2010_12879_b200 import Session, SolveConfig, workloads
    from paper_2010_12879_b200.distributed import Communicator
    if transport == "nccl":  # one GPU per rank
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=size,
                                device_id=torch.device("cuda", rank))
    else:
        torch.cuda.set_device(0)
        _init(rank, size, port)
    w = getattr(workloads, name)()
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10, method=method))
    a = torch.from_numpy(w.a).cuda()
    comm = Communicator.host() if transport == "host" else Communicator.nccl()
    sess.distribute(comm, replicate_below=replicate_below)
    vox, rep, psi = sess.snapshot(a, keep_psi=True)
    v0, v1 = sess.vox_range
    d0, d1 = sess.dof_range
    torch.save({"vox": vox[:, v0:v1].cpu(), "vr": (v0, v1), "psi": psi[:, d0:d1].cpu(), "dr": (d0, d1),
                "it": rep.iterations, "rel": rep.rel_residuals}, os.path.join(out, f"s{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _small_layered():
    from paper_2010_12879_b200 import workloads
    return workloads.c2(48)


@pytest.mark.gpu
@pytest.mark.parametrize("replicate_below,method", [(1000, "pcg"), (10**9, "pcg"), (1000, "fgmres")])
def test_distributed_snapshot_matches_single_gpu(replicate_below, method):
    """Two ranks reproduce the single-GPU snapshot; for FGMRES the batched
    Arnoldi process runs on the ranks' own positions with rank-ordered
    reductions of every inner product (fgmres_dist)."""
    from paper_2010_12879_b200 import Session, SolveConfig, workloads
    w = workloads.c2(48)
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10, method=method))
    vox, rep, psi = sess.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
    vox, psi = vox.cpu().numpy(), psi.cpu().numpy()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_solve_worker, args=(2, _port(), out, "c2_small", replicate_below, "host", method), nprocs=2,
                 join=True)
        parts = [torch.load(os.path.join(out, f"s{r}.pt")) for r in range(2)]
    assert parts[0]["vr"][1] == parts[1]["vr"][0] and parts[1]["vr"][1] == vox.shape[1]
    assert parts[0]["dr"][1] == parts[1]["dr"][0] and parts[1]["dr"][1] == psi.shape[1]
    vd = np.concatenate([p["vox"].numpy() for p in parts], axis=1)
    pd = np.concatenate([p["psi"].numpy() for p in parts], axis=1)
    for p in parts:
        assert abs(p["it"] - rep.iterations) <= 1
        assert max(p["rel"]) <= 1e-10
    # both solves at rel.res 1e-10 (psi ~1e-11, E ~1e-8)
    assert np.linalg.norm(pd - psi) <= 1e-8 * np.linalg.norm(psi)
    assert np.abs(vd - vox).max() <= 1e-7 * np.abs(vox).max()


def _nccl_single_worker(rank, size, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2010_12879_b200 import Session, SolveConfig, workloads
    from paper_2010_12879_b200.distributed import Communicator
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=size,
                            device_id=torch.device("cuda", 0))
    w = workloads.c2_small()
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10))
    a = torch.from_numpy(w.a).cuda()
    ref, rep0, _ = sess.snapshot(a)
    ref = ref.cpu()
    sess2 = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10))
    sess2.distribute(Communicator.nccl(), replicate_below=1000)   # NCCL transport, one rank
    vox, rep, _ = sess2.snapshot(a)
    torch.save({"ref": ref, "vox": vox.cpu(), "it": (rep0.iterations, rep.iterations)}, os.path.join(out, "n.pt"))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_transport_single_rank():
    """The NCCL transport (dlopen, comm init, grouped send/recv, allgather)
    on one rank: the distributed code path must reproduce the plain solve."""
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_nccl_single_worker, args=(1, _port(), out), nprocs=1, join=True)
        d = torch.load(os.path.join(out, "n.pt"))
    assert d["it"][0] == d["it"][1]
    assert torch.allclose(d["vox"], d["ref"], rtol=1e-10, atol=0)


@pytest.mark.gpu
def test_nccl_batch_graph_is_exact(monkeypatch, capfd):
    """On the stream-ordered NCCL transport the distributed PCG replays each
    full batch of iterations as one captured CUDA graph; it must give the
    launched batches' iterations and bits (SPFD_DIST_GRAPH=0)."""
    res = {}
    monkeypatch.setenv("SPFD_DEBUG", "1")
    for graph in ("0", "1"):
        monkeypatch.setenv("SPFD_DIST_GRAPH", graph)
        capfd.readouterr()
        with tempfile.TemporaryDirectory() as out:
            mp.spawn(_nccl_single_worker, args=(1, _port(), out), nprocs=1, join=True)
            res[graph] = torch.load(os.path.join(out, "n.pt"))
        captured = "distributed batch graph captured" in capfd.readouterr().err
        assert captured == (graph == "1")
    assert res["0"]["it"] == res["1"]["it"]
    assert torch.equal(res["0"]["vox"], res["1"]["vox"])


@pytest.mark.gpu
def test_distributed_iteration_batching_is_exact(monkeypatch):
    """The distributed PCG queues several iterations per host read, with the
    convergence test on the device freezing the iterations behind a stop:
    batches of 1 and 4 give the same iteration count and the same bits."""
    res = {}
    for batch in ("1", "4"):
        monkeypatch.setenv("SPFD_DIST_BATCH", batch)
        with tempfile.TemporaryDirectory() as out:
            mp.spawn(_solve_worker, args=(2, _port(), out, "c2_small", 1000), nprocs=2, join=True)
            res[batch] = [torch.load(os.path.join(out, f"s{r}.pt")) for r in range(2)]
    for r in range(2):
        assert res["1"][r]["it"] == res["4"][r]["it"]
        assert torch.equal(res["1"][r]["psi"], res["4"][r]["psi"])
        assert torch.equal(res["1"][r]["vox"], res["4"][r]["vox"])


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_distributed_nccl_two_gpus():
    """Two ranks on two GPUs over NCCL (NVLink): the z-slab solve against
    the single-GPU snapshot (same bar as the host-transport test)."""
    from paper_2010_12879_b200 import Session, SolveConfig, workloads
    w = workloads.c2_small()
    sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-10))
    vox, rep, psi = sess.snapshot(torch.from_numpy(w.a).cuda(), keep_psi=True)
    vox, psi = vox.cpu().numpy(), psi.cpu().numpy()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_solve_worker, args=(2, _port(), out, "c2_small", 1000, "nccl"), nprocs=2, join=True)
        parts = [torch.load(os.path.join(out, f"s{r}.pt")) for r in range(2)]
    vd = np.concatenate([p["vox"].numpy() for p in parts], axis=1)
    pd = np.concatenate([p["psi"].numpy() for p in parts], axis=1)
    for p in parts:
        assert abs(p["it"] - rep.iterations) <= 1 and max(p["rel"]) <= 1e-10
    assert np.linalg.norm(pd - psi) <= 1e-8 * np.linalg.norm(psi)
    assert np.abs(vd - vox).max() <= 1e-7 * np.abs(vox).max()
