"""GPU tests of the 1D-partitioned BFS kernels (gr_part_bfs_*).

* loopback: P partitions in one process on one GPU, the exchange is a device
  copy -- exercises ownership, culling, bucketing and absorb of
  the CUDA kernels without a second GPU;
* world size 1 over a real torch.distributed NCCL group (the N>1 code path,
  degenerate exchange).
Depth is compared element-wise with the oracle; pred (global ids) by the
certificate.
"""
import os
import socket

import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def grd():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    from paper_1501_05387_b200 import dist
    return dist


def _loopback(grd, g, P, srcs, directions=("push", "pull", "auto"), ordered=False):
    parts = []
    deg_global = (g.R[1:] - g.R[:-1]).to(torch.int32).cuda()
    for r in range(P):
        v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, P, r)
        parts.append(grd.GpuPartition(Rl.cuda(), Cl.cuda(), g.n, P, r, symmetric=g.symmetric))
        if ordered:
            parts[-1].order_pull_lists(deg_global)
    grp = grd.LoopbackGroup(parts)
    R, C, _ = g.numpy()
    if not g.symmetric:
        directions = ("push",)
    for s, direction in [(s, d) for s in srcs for d in directions]:
        depths = [torch.empty(pt.n_local, dtype=torch.int32, device="cuda") for pt in parts]
        preds = [torch.empty(pt.n_local, dtype=torch.int32, device="cuda") for pt in parts]
        levels = grp.bfs(s, depths, preds, direction=direction)
        depth = torch.cat(depths).cpu().numpy()
        pred = torch.cat(preds).cpu().numpy()
        ref, _ = oracle.bfs(R, C, s)
        bad = np.flatnonzero(depth != ref)
        assert bad.size == 0, (P, s, bad[:5], depth[bad[:5]], ref[bad[:5]])
        assert oracle.check_bfs(R, C, s, depth, pred) == []
        assert levels == int(ref.max()) + 1
    for pt in parts:
        pt.close()


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_loopback_rmat(grd, P):
    g = gg.rmat(14, 16, seed=5)
    _loopback(grd, g, P, [0] + gg.sources(g, 2))


@pytest.mark.parametrize("P", [2, 5])
def test_loopback_directed_and_mesh(grd, P):
    _loopback(grd, gg.directed_random(30000, 200000, seed=3), P, gg.sources(gg.directed_random(30000, 200000, seed=3), 2))
    m = gg.make_config("c4_road", shrink=5)
    _loopback(grd, m, P, gg.sources(m, 1))


def test_loopback_kron_scale18(grd):
    g = gg.kronecker(18, 16, seed=1)
    _loopback(grd, g, 4, gg.sources(g, 2))


@pytest.mark.parametrize("P", [1, 3, 4])
def test_loopback_ordered_pull_lists(grd, P):
    """gr_part_order_pull_lists: pull lists sorted by global neighbour degree
    (a copy; push lists untouched) -- depths stay bit-exact, preds valid."""
    g = gg.kronecker(16, 16, seed=2)
    _loopback(grd, g, P, [0] + gg.sources(g, 2), ordered=True)


def test_order_pull_lists_errors(grd):
    import paper_1501_05387_b200 as gr
    g = gg.directed_random(2000, 10000, seed=4)
    v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, 2, 0)
    pt = grd.GpuPartition(Rl.cuda(), Cl.cuda(), g.n, 2, 0, symmetric=False)
    deg = (g.R[1:] - g.R[:-1]).to(torch.int32)
    with pytest.raises(gr.GrError):  # host degree array
        gr._check(gr.load().gr_part_order_pull_lists(pt.handle, deg.data_ptr()))
    pt.close()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_world1_nccl_group(grd):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = gg.rmat(13, 16, seed=9)
        v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, 1, 0)
        part = grd.GpuPartition(Rl.cuda(), Cl.cuda(), g.n, 1, 0)
        ex = grd.TorchDistExchange()
        dg = grd.global_degrees(part, ex)
        assert torch.equal(dg.cpu(), (g.R[1:] - g.R[:-1]).to(torch.int32))
        part.order_pull_lists(dg)
        R, C, _ = g.numpy()
        for s, direction in [(s, d) for s in gg.sources(g, 2) for d in ("push", "pull", "auto")]:
            depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
            pred = torch.empty(g.n, dtype=torch.int32, device="cuda")
            grd.bfs_partitioned(part, ex, s, depth, pred, direction=direction)
            ref, _ = oracle.bfs(R, C, s)
            assert np.array_equal(depth.cpu().numpy(), ref)
            assert oracle.check_bfs(R, C, s, depth.cpu().numpy(), pred.cpu().numpy()) == []
        part.close()
    finally:
        dist.destroy_process_group()


def test_part_errors(grd):
    import paper_1501_05387_b200 as gr
    g = gg.rmat(8, 4, seed=1)
    v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, 2, 1)
    import ctypes
    h = ctypes.c_void_p()
    Rc, Cc = Rl.cuda(), Cl.cuda()
    st = gr.load().gr_graph_create_part(g.n, 2, 0, v0, v1, Cc.numel(), Rc.data_ptr(), Cc.data_ptr(),
                                        4, 0, None, ctypes.byref(h))  # rank 0 does not own [v0, v1)
    assert st == 1 and "must own" in gr.gr_last_error()
    pt = grd.GpuPartition(Rc, Cc, g.n, 2, 1)
    # the single-GPU entry points must refuse a step-level partition handle
    # (its columns are global ids: depth/visited would be indexed out of range)
    dd = torch.empty(g.n, dtype=torch.int32, device="cuda")
    assert gr.load().gr_bfs(pt.handle, 0, dd.data_ptr(), None, None) == 1
    assert "partition" in gr.gr_last_error()
    assert gr.load().gr_sssp(pt.handle, 0, dd.data_ptr(), None, None) == 1
    d = torch.empty(pt.n_local, dtype=torch.int32)  # host memory: rejected
    with pytest.raises(gr.GrError):
        pt.begin(0, d, None)
    with pytest.raises(gr.GrError):
        pt.begin(g.n, d.cuda(), None)
