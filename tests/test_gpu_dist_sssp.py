"""GPU tests of the 1D-partitioned SSSP kernels (gr_part_sssp_*).

Loopback: P partitions in one process on one GPU, the exchange is a device
copy -- exercises relax / best-shipped culling / triple packing / absorb /
far re-split of the CUDA kernels without a second GPU. dist is compared
element by element with the oracle (binary-heap Dijkstra, bit-exact); pred
(global ids) by the tightness certificate (parity-unpinned by design, A-9).
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


def _parts(grd, g, P):
    parts = []
    for r in range(P):
        v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, P, r)
        Wl = grd.partition_weights(g.R, g.W, P, r)
        parts.append(grd.GpuPartition(Rl.cuda(), Cl.cuda(), g.n, P, r, symmetric=g.symmetric, W_local=Wl.cuda()))
    return parts


def _loopback_sssp(grd, g, P, srcs, deltas):
    parts = _parts(grd, g, P)
    grp = grd.LoopbackGroup(parts)
    R, C, W = g.numpy()
    for s in srcs:
        ref, _ = oracle.sssp(R, C, W, s)
        for delta in deltas:
            dists = [torch.empty(pt.n_local, dtype=torch.int32, device="cuda") for pt in parts]
            preds = [torch.empty(pt.n_local, dtype=torch.int32, device="cuda") for pt in parts]
            grp.sssp(s, dists, preds, delta=delta)
            dist = torch.cat(dists).cpu().numpy().view(np.uint32)
            pred = torch.cat(preds).cpu().numpy()
            bad = np.flatnonzero(dist != ref)
            assert bad.size == 0, (P, s, delta, bad[:5], dist[bad[:5]], ref[bad[:5]])
            assert oracle.check_sssp(R, C, W, s, dist, pred) == []
    for pt in parts:
        pt.close()


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_loopback_sssp_rmat(grd, P):
    g = gg.assign_weights(gg.rmat(13, 16, seed=5), seed=2)
    _loopback_sssp(grd, g, P, gg.sources(g, 2), deltas=[1, 8, 64, (1 << 32) - 1])


@pytest.mark.parametrize("P", [2, 5])
def test_loopback_sssp_directed_and_mesh(grd, P):
    d = gg.assign_weights(gg.directed_random(20000, 150000, seed=3), seed=2)
    _loopback_sssp(grd, d, P, gg.sources(d, 2), deltas=[3, 1024])
    m = gg.make_config("c4_road", shrink=6, weights=True)
    _loopback_sssp(grd, m, P, gg.sources(m, 1), deltas=[64, 2048])


def test_loopback_sssp_orkut_like(grd):
    g = gg.make_config("c3_orkut", shrink=6, weights=True)
    _loopback_sssp(grd, g, 4, gg.sources(g, 1), deltas=[3])


def test_loopback_sssp_tiny_and_isolated(grd):
    # a weighted path crossing all three 32-vertex blocks, a side edge, isolated
    # vertices (69 among them); sources: an end, a middle vertex, an isolated one
    g = gg.from_edges(70, [(0, 1), (1, 2), (2, 3), (3, 40), (40, 65), (65, 66), (10, 33), (2, 33)],
                      weights=[5, 1, 7, 2, 3, 1, 9, 20])
    for P in (1, 2, 3):
        _loopback_sssp(grd, g, P, [0, 40, 69], deltas=[1, 4, 100])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_world1_nccl_sssp(grd):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = gg.assign_weights(gg.rmat(12, 16, seed=9), seed=2)
        part = _parts(grd, g, 1)[0]
        ex = grd.TorchDistExchange()
        R, C, W = g.numpy()
        for s in gg.sources(g, 2):
            d = torch.empty(g.n, dtype=torch.int32, device="cuda")
            p = torch.empty(g.n, dtype=torch.int32, device="cuda")
            grd.sssp_partitioned(part, ex, s, d, p, delta=4)
            ref, _ = oracle.sssp(R, C, W, s)
            dd = d.cpu().numpy().view(np.uint32)
            assert np.array_equal(dd, ref)
            assert oracle.check_sssp(R, C, W, s, dd, p.cpu().numpy()) == []
        part.close()
    finally:
        dist.destroy_process_group()


def test_part_sssp_errors(grd):
    import ctypes
    import paper_1501_05387_b200 as gr
    g = gg.rmat(8, 4, seed=1)
    v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, 2, 0)
    part = grd.GpuPartition(Rl.cuda(), Cl.cuda(), g.n, 2, 0)  # no weights
    d = torch.empty(part.n_local, dtype=torch.int32, device="cuda")
    with pytest.raises(gr.GrError) as e:
        part.sssp_begin(0, d)
    assert e.value.status == 4  # GR_ERR_NO_WEIGHTS
    part.close()
    gw = gg.assign_weights(g, seed=2)
    part = _parts(grd, gw, 2)[0]
    with pytest.raises(gr.GrError):
        part.sssp_begin(g.n, d)  # source out of range
    with pytest.raises(gr.GrError):
        part.sssp_begin(0, torch.empty(part.n_local, dtype=torch.int32))  # host output
    part.sssp_begin(0, d)
    with pytest.raises(gr.GrError):
        part.sssp_resplit(0, 1, 0, 8, 8)  # threshold must grow
    part.close()
