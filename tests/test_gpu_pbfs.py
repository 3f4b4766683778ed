"""The §8(b) multi-GPU boundary: gr_comm + gr_graph_create_partitioned +
collective gr_bfs, whose whole level loop (advance, exchange over peer
memory, pull-shard all-gather, per-level counter exchange, direction rule)
runs in one persistent kernel per rank (csrc/pbfs.cu).

Every partitioned BFS is compared element by element with the CPU oracle's
FIFO BFS plus its O(m) certificate on the parents. Loopback
groups (P virtual ranks in one launch on one GPU) exercise the multi-rank
logic; a world-size-1 NCCL group exercises the real-rank path."""
import os
import socket

import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mg():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    from paper_1501_05387_b200 import multigpu
    return multigpu


def _loopback_graphs(mg, g, P, keep_order=False):
    comms = mg.Comm.loopback(P)
    parts = []
    for r in range(P):
        v0, v1, Rl, Cl, _ = mg.partition_csr(g.R, g.C, P, r)
        parts.append(mg.PartitionedGraph(comms[r], Rl.cuda(), Cl.cuda(), g.n, keep_order=keep_order))
    return comms, parts


def _close(comms, parts):
    for p in parts:
        p.close()
    for c in comms:
        c.close()


def _run_check(parts, g, srcs, directions=("auto", "push", "pull"), **kw):
    R, C, _ = g.numpy()
    for s in srcs:
        ref, _ = oracle.bfs(R, C, s)
        for d in directions:
            outs = [p.bfs(s, direction=d, **kw) for p in parts]  # the last call runs every rank
            depth = torch.cat([o[0] for o in outs]).cpu().numpy()
            pred = torch.cat([o[1] for o in outs]).cpu().numpy()
            bad = np.flatnonzero(depth != ref)
            assert bad.size == 0, (len(parts), s, d, bad[:5], depth[bad[:5]], ref[bad[:5]])
            assert oracle.check_bfs(R, C, s, depth, pred) == [], (len(parts), s, d)
            st = parts[0].run_stats()
            # an isolated source has an empty frontier: no level runs
            assert st["num_levels"] == (int(ref.max()) + 1 if R[s + 1] > R[s] else 0)
            assert sum(p.run_stats()["reached"] for p in parts) == int((ref >= 0).sum())
            assert sum(p.run_stats()["reached_edges"] for p in parts) == oracle.reached_edges(R, ref, -1)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_loopback_rmat(mg, P):
    g = gg.rmat(14, 16, seed=5)
    comms, parts = _loopback_graphs(mg, g, P)
    _run_check(parts, g, [0] + gg.sources(g, 2))
    _close(comms, parts)


@pytest.mark.parametrize("P", [2, 5])
def test_loopback_kron_and_mesh(mg, P):
    """Kronecker (hubs: remote-heavy pushes, pull levels) and a road-like mesh
    (hundreds of levels: many barriers, tiny exchanges)."""
    for g, srcs in ((gg.kronecker(16, 16, seed=2), None), (gg.make_config("c4_road", shrink=6), None)):
        comms, parts = _loopback_graphs(mg, g, P)
        _run_check(parts, g, gg.sources(g, 2), directions=("auto", "push"))
        _close(comms, parts)


def test_loopback_rules_and_keep_order(mg):
    """Paper-literal switch rule (A-3) and the caller's pull-list order."""
    g = gg.kronecker(15, 16, seed=3)
    comms, parts = _loopback_graphs(mg, g, 3, keep_order=True)
    _run_check(parts, g, gg.sources(g, 2), directions=("auto",), switch_rule=1)
    _run_check(parts, g, gg.sources(g, 1), directions=("auto",))
    _close(comms, parts)


def test_loopback_isolated_source_and_tiny(mg):
    """An isolated source (one level), a 2-vertex graph over 2 ranks, a path
    crossing every rank boundary (one remote ship per level)."""
    g = gg.from_edges(200, [(i, i + 1) for i in range(190)] + [(195, 196)])  # blocks of 64
    comms, parts = _loopback_graphs(mg, g, 4)
    _run_check(parts, g, [0, 100, 190, 199, 195], directions=("auto", "push", "pull"))
    _close(comms, parts)
    g = gg.from_edges(2, [(0, 1)])
    comms, parts = _loopback_graphs(mg, g, 1)
    _run_check(parts, g, [0, 1])
    _close(comms, parts)


def test_host_outputs_and_errors(mg):
    import paper_1501_05387_b200 as gr
    g = gg.rmat(10, 8, seed=1)
    comms, parts = _loopback_graphs(mg, g, 2)
    R, C, _ = g.numpy()
    ref, _ = oracle.bfs(R, C, 3)
    hd = [torch.empty(p.n_local, dtype=torch.int32, pin_memory=True) for p in parts]
    for p, d in zip(parts, hd):
        p.bfs(3, depth=d, want_pred=False)
    assert np.array_equal(torch.cat(hd).numpy(), ref)
    with pytest.raises(gr.GrError) as e:
        parts[0].bfs(g.n)
    assert e.value.status == 3
    parts[0].bfs(1)
    with pytest.raises(gr.GrError):  # rank 1 joins with another source
        parts[1].bfs(2)
    d = torch.empty(parts[0].n_local, dtype=torch.int32, device="cuda")
    assert gr.load().gr_bfs_async(parts[0].handle, 1, d.data_ptr(), None, None) == 1
    v0, v1, Rl, Cl, _ = mg.partition_csr(g.R, g.C, 2, 1)
    import ctypes
    h = ctypes.c_void_p()
    st = gr.load().gr_graph_create_partitioned(comms[0].handle, g.n, v0, v1, Cl.numel(), Rl.data_ptr(),
                                               Cl.data_ptr(), None, 1, None, ctypes.byref(h))
    assert st == 1 and "must own" in gr.gr_last_error()
    v0, v1, Rl, Cl, _ = mg.partition_csr(g.R, g.C, 2, 0)
    st = gr.load().gr_graph_create_partitioned(comms[0].handle, g.n, v0, v1, Cl.numel(), Rl.data_ptr(),
                                               Cl.data_ptr(), None, 0, None, ctypes.byref(h))
    assert st == 1 and "symmetric" in gr.gr_last_error()
    _close(comms, parts)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_world1_nccl_comm(mg):
    """A real rank: gr_comm_create over NCCL (unique id broadcast by
    torch.distributed), world size 1."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = mg.Comm.from_torch()
        g = gg.kronecker(16, 16, seed=4)
        v0, v1, Rl, Cl, _ = mg.partition_csr(g.R, g.C, 1, 0)
        part = mg.PartitionedGraph(comm, Rl.cuda(), Cl.cuda(), g.n)
        _run_check([part], g, gg.sources(g, 2))
        part.close()
        comm.close()
    finally:
        dist.destroy_process_group()


# ---- gr_sssp on a partitioned graph (psssp.cu) ------------------------------

def _loopback_weighted(mg, g, P):
    comms = mg.Comm.loopback(P)
    parts = []
    for r in range(P):
        v0, v1, Rl, Cl, Wl = mg.partition_csr(g.R, g.C, P, r, W=g.W)
        parts.append(mg.PartitionedGraph(comms[r], Rl.cuda(), Cl.cuda(), g.n, W_local=Wl.cuda()))
    return comms, parts


def _sssp_check(parts, g, srcs, deltas=(0,)):
    R, C, W = g.numpy()
    for s in srcs:
        ref, _ = oracle.sssp(R, C, W, s)
        for dl in deltas:
            outs = [p.sssp(s, delta=dl) for p in parts]
            dist = torch.cat([o[0] for o in outs]).cpu().numpy().view(np.uint32)
            pred = torch.cat([o[1] for o in outs]).cpu().numpy()
            bad = np.flatnonzero(dist != ref)
            assert bad.size == 0, (len(parts), s, dl, bad[:5], dist[bad[:5]], ref[bad[:5]])
            assert oracle.check_sssp(R, C, W, s, dist, pred) == [], (len(parts), s, dl)
            assert sum(p.run_stats()["reached"] for p in parts) == int((ref != oracle.UINT32_MAX).sum())


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_loopback_sssp_rmat(mg, P):
    """Near/far delta-stepping over P partitions (remote relaxations shipped
    as (vertex, dist, parent) records into the owners' inboxes), every delta
    regime: narrow bands, SPEC's ceil(mean w) = 33, one band (Bellman-Ford)."""
    g = gg.assign_weights(gg.rmat(13, 16, seed=6), seed=2)
    comms, parts = _loopback_weighted(mg, g, P)
    _sssp_check(parts, g, [0] + gg.sources(g, 2), deltas=(0, 1, 8, 33, 0xFFFFFFFF))
    _close(comms, parts)


@pytest.mark.parametrize("P", [2, 5])
def test_loopback_sssp_mesh_and_orkut(mg, P):
    """High-diameter mesh (hundreds of steps, many re-splits) and the
    orkut-like Chung-Lu shape, auto delta (A-10) and a wide band."""
    for g in (gg.make_config("c4_road", shrink=6, weights=True), gg.make_config("c3_orkut", shrink=8, weights=True)):
        comms, parts = _loopback_weighted(mg, g, P)
        _sssp_check(parts, g, gg.sources(g, 1), deltas=(0, 1024))
        _close(comms, parts)


def test_loopback_sssp_errors_and_tiny(mg):
    import paper_1501_05387_b200 as gr
    g = gg.rmat(10, 8, seed=1)  # no weights
    comms, parts = _loopback_graphs(mg, g, 2)
    for p in parts[:1]:
        with pytest.raises(gr.GrError) as e:
            p.sssp(0)
        assert e.value.status == 4
    _close(comms, parts)
    g = gg.assign_weights(gg.from_edges(200, [(i, i + 1) for i in range(190)] + [(195, 196)]), seed=3)
    comms, parts = _loopback_weighted(mg, g, 4)
    _sssp_check(parts, g, [0, 100, 199, 195], deltas=(0, 1, 0xFFFFFFFF))
    _close(comms, parts)


def test_world1_nccl_sssp(mg):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = mg.Comm.from_torch()
        g = gg.assign_weights(gg.kronecker(15, 16, seed=4), seed=5)
        v0, v1, Rl, Cl, Wl = mg.partition_csr(g.R, g.C, 1, 0, W=g.W)
        part = mg.PartitionedGraph(comm, Rl.cuda(), Cl.cuda(), g.n, W_local=Wl.cuda())
        _sssp_check([part], g, gg.sources(g, 2), deltas=(0, 64))
        part.close()
        comm.close()
    finally:
        dist.destroy_process_group()
