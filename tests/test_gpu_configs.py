"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (same kernels, same default options).

Every config, C1-C5, element by element against the CPU oracle (BFS is
seconds per source, ~6 s on C5's 1.05B edges; Dijkstra on C3/C4 tens of
seconds, so one source), plus the oracle's O(m) certificate on the parents.
C5 is also run 1D-partitioned (the configuration it is defined on, SURVEY
§8(e)): 8 partitions in one process and a world-size-1 NCCL group.
"""
import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def gr():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1501_05387_b200 as m
    torch.cuda.set_device(0)
    return m


def _bfs_parity(gr, name, nsrc, dirs=("auto", "push")):
    g = gg.make_config(name, device="cuda")
    G = gr.Graph(g.R, g.C, g.W, symmetric=True)
    R, C, W = g.numpy()
    for s in gg.sources(g, nsrc):
        ref, _ = oracle.bfs(R, C, s, want_pred=False)
        for d in dirs:
            depth, pred = G.bfs(s, direction=d)
            got = depth.cpu().numpy()
            assert np.array_equal(got, ref), (name, s, d, int((got != ref).sum()))
            assert oracle.check_bfs(R, C, s, got, pred.cpu().numpy()) == []
    return g, G, (R, C, W)


def test_c2_kron21_bfs(gr):
    _bfs_parity(gr, "c2_kron21", 2)


def test_c3_orkut_bfs_sssp(gr):
    g, G, (R, C, W) = _bfs_parity(gr, "c3_orkut", 1)
    s = gg.sources(g, 1)[0]
    ref, _ = oracle.sssp(R, C, W, s, want_pred=False)
    dist, pred = G.sssp(s)
    got = gr.dist_to_u32(dist)
    assert np.array_equal(got, ref), int((got != ref).sum())
    assert oracle.check_sssp(R, C, W, s, got, pred.cpu().numpy()) == []


def test_c4_road_bfs_sssp(gr):
    g, G, (R, C, W) = _bfs_parity(gr, "c4_road", 1, dirs=("auto",))
    s = gg.sources(g, 1)[0]
    ref, _ = oracle.sssp(R, C, W, s, want_pred=False)
    dist, pred = G.sssp(s)
    got = gr.dist_to_u32(dist)
    assert np.array_equal(got, ref), int((got != ref).sum())


def test_c2_kron21_bfs_variants(gr):
    """The idempotent (atomic-free) discovery and the paper-literal switch
    rule (A-3, A-5, A-6) at C2's full size, bit-exact against the oracle."""
    g = gg.make_config("c2_kron21", device="cuda")
    G = gr.Graph(g.R, g.C, None, symmetric=True)
    R, C, _ = g.numpy()
    for s in gg.sources(g, 2):
        ref, _ = oracle.bfs(R, C, s, want_pred=False)
        for kw in (dict(idempotent=True), dict(switch_rule=1), dict(idempotent=True, direction="push"),
                   dict(direction="pull")):
            depth, pred = G.bfs(s, **kw)
            got = depth.cpu().numpy()
            assert np.array_equal(got, ref), (s, kw, int((got != ref).sum()))
            assert oracle.check_bfs(R, C, s, got, pred.cpu().numpy()) == [], (s, kw)
    G.close()


def test_c5_kron25_bfs(gr):
    """C5 (Kronecker scale 25, ~1.05B directed edges) single-GPU BFS, auto and
    push, element by element against the oracle's FIFO BFS (~6 s per source
    on one host core), plus the certificate on the parents; the run totals of
    gr_get_run_stats (reached, reached_edges) against the oracle's."""
    g = gg.make_config("c5_kron25", device="cuda")
    G = gr.Graph(g.R, g.C, None, symmetric=True)
    R, C, _ = g.numpy()
    for s in gg.sources(g, 2):
        ref, _ = oracle.bfs(R, C, s, want_pred=False)
        for d in ("auto", "push"):
            depth, pred = G.bfs(s, direction=d)
            got = depth.cpu().numpy()
            assert np.array_equal(got, ref), (s, d, int((got != ref).sum()))
            assert oracle.check_bfs(R, C, s, got, pred.cpu().numpy()) == [], (s, d)
            st = G.run_stats()
            assert st["reached"] == int((ref >= 0).sum())
            assert st["reached_edges"] == oracle.reached_edges(R, ref, -1)
    G.close()


def test_c5_kron25_bfs_partitioned(gr):
    """The 1D-partitioned BFS on the full C5 graph, in
    bench.py's configuration (collective gr_bfs on gr_graph_create_partitioned
    graphs, one persistent kernel per rank): a loopback group of 8 ranks (one
    launch hosts all of them) and a real world-size-1 rank over NCCL,
    bit-exact against the oracle."""
    import os
    import socket

    import torch.distributed as dist
    from paper_1501_05387_b200 import multigpu as mg
    g = gg.make_config("c5_kron25", device="cuda")
    R, C, _ = g.numpy()
    s = gg.sources(g, 1)[0]
    ref, _ = oracle.bfs(R, C, s, want_pred=False)
    P = 8
    comms = mg.Comm.loopback(P)
    parts = []
    for r in range(P):
        v0, v1, Rl, Cl, _ = mg.partition_csr(g.R, g.C, P, r)
        parts.append(mg.PartitionedGraph(comms[r], Rl, Cl, g.n))
        del Rl, Cl
    outs = [p.bfs(s) for p in parts]
    got = torch.cat([o[0] for o in outs]).cpu().numpy()
    assert np.array_equal(got, ref), int((got != ref).sum())
    assert oracle.check_bfs(R, C, s, got, torch.cat([o[1] for o in outs]).cpu().numpy()) == []
    for p in parts:
        p.close()
    for c in comms:
        c.close()
    del parts, outs
    torch.cuda.empty_cache()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
    sk.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = mg.Comm.from_torch()
        v0, v1, Rl, Cl, _ = mg.partition_csr(g.R, g.C, 1, 0)
        part = mg.PartitionedGraph(comm, Rl, Cl, g.n)
        del Rl, Cl
        depth, pred = part.bfs(s)
        got = depth.cpu().numpy()
        assert np.array_equal(got, ref), int((got != ref).sum())
        assert oracle.check_bfs(R, C, s, got, pred.cpu().numpy()) == []
        part.close()
        comm.close()
    finally:
        dist.destroy_process_group()


def test_c3_orkut_sssp_partitioned(gr):
    """gr_sssp on gr_graph_create_partitioned graphs (psssp.cu) on the full C3
    graph: a loopback group of 4 ranks against the oracle's Dijkstra."""
    from paper_1501_05387_b200 import multigpu as mg
    g = gg.make_config("c3_orkut", device="cuda")
    R, C, W = g.numpy()
    s = gg.sources(g, 1)[0]
    ref, _ = oracle.sssp(R, C, W, s, want_pred=False)
    P = 4
    comms = mg.Comm.loopback(P)
    parts = []
    for r in range(P):
        v0, v1, Rl, Cl, Wl = mg.partition_csr(g.R, g.C, P, r, W=g.W)
        parts.append(mg.PartitionedGraph(comms[r], Rl, Cl, g.n, W_local=Wl))
    outs = [p.sssp(s) for p in parts]
    got = torch.cat([o[0] for o in outs]).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, ref), int((got != ref).sum())
    assert oracle.check_sssp(R, C, W, s, got, torch.cat([o[1] for o in outs]).cpu().numpy()) == []
    for p in parts:
        p.close()
    for c in comms:
        c.close()


# ---- the paper's other primitives at full size --------

def test_c2_kron21_bc_cc_pagerank(gr):
    """BC of two sources (fp64, 1e-9 relative), CC (bit-exact labels and
    count) and PageRank (1e-9 relative after the full-sweep convergence
    check at tol 1e-12) on the full Kronecker scale-21 graph, in bench.py's
    launch configuration, against the C / numpy oracle."""
    g = gg.make_config("c2_kron21", device="cuda")
    G = gr.Graph(g.R, g.C, None, symmetric=True)
    R, C, _ = g.numpy()
    srcs = gg.sources(g, 2)
    bc = G.bc(srcs).cpu().numpy()
    ref = oracle.bc(R, C, srcs)
    nz = ref > 0
    assert np.array_equal(bc > 0, nz)
    assert np.max(np.abs(bc[nz] - ref[nz]) / ref[nz]) <= 1e-9
    comp, k = G.cc()
    cref, kref = oracle.cc(R, C)
    assert np.array_equal(comp.cpu().numpy(), cref) and k == kref
    x, it = G.pagerank(0.85, 1e-12, 1000)
    xref = oracle.pagerank(R, C, 0.85, tol=1e-15, max_iter=400)
    assert np.max(np.abs(x.cpu().numpy() - xref) / xref) <= 1e-9, it
    G.close()
