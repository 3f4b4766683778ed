"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

depth / dist must be bit-identical to the oracle (they are unique); pred is
checked by the certificate (any valid parent is correct).
"""
import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu

INF = oracle.UINT32_MAX
DIRS = ["push", "pull", "auto"]
DELTAS = [1, 8, 33, 64, 1024, 0xFFFFFFFF, 0]


@pytest.fixture(scope="module")
def gr():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1501_05387_b200 as m
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)
    return m


def _dev(g, gr):
    return gr.Graph(g.R.cuda(), g.C.cuda(), None if g.W is None else g.W.cuda(),
                    symmetric=g.symmetric)


def _check_bfs(gr, G, g, srcs, dirs=DIRS, **kw):
    R, C, _ = g.numpy()
    for s in srcs:
        ref, _ = oracle.bfs(R, C, s)
        for d in dirs:
            depth, pred = G.bfs(s, direction=d, **kw)
            got = depth.cpu().numpy()
            bad = np.flatnonzero(got != ref)
            assert bad.size == 0, "direction=%s src=%d: %d mismatches, first v=%d got %d want %d" % (
                d, s, bad.size, bad[0], got[bad[0]], ref[bad[0]])
            assert oracle.check_bfs(R, C, s, got, pred.cpu().numpy()) == []


def _check_sssp(gr, G, g, srcs, deltas=DELTAS):
    R, C, W = g.numpy()
    for s in srcs:
        ref, _ = oracle.sssp(R, C, W, s)
        for delta in deltas:
            dist, pred = G.sssp(s, delta=delta)
            got = gr.dist_to_u32(dist)
            bad = np.flatnonzero(got != ref)
            assert bad.size == 0, "delta=%d src=%d: %d mismatches, first v=%d got %d want %d" % (
                delta, s, bad.size, bad[0], got[bad[0]], ref[bad[0]])
            assert oracle.check_sssp(R, C, W, s, got, pred.cpu().numpy()) == []


# ------------------------------------------------------------------ small / closed form

def test_golden(gr, golden):
    ex = golden["bfs_g1"]
    g = gg.from_edges(ex["n"], [tuple(e) for e in ex["edges"]])
    G = _dev(g, gr)
    for d in DIRS:
        assert G.bfs(ex["src"], direction=d)[0].tolist() == ex["depth"]
    ex = golden["sssp_spec"]
    g = gg.from_edges(ex["n"], [tuple(e) for e in ex["edges"]], ex["weights"])
    G = _dev(g, gr)
    for delta in DELTAS:
        assert gr.dist_to_u32(G.sssp(ex["src"], delta=delta)[0]).tolist() == ex["dist"]


@pytest.mark.parametrize("maker", [
    lambda: gg.path(1000), lambda: gg.cycle(301), lambda: gg.grid(37, 53), lambda: gg.star(5000),
    lambda: gg.complete(70), lambda: gg.binary_tree(4095), lambda: gg.hypercube(10),
])
def test_closed_form_graphs(gr, maker):
    g = gg.assign_weights(maker(), seed=11)
    G = _dev(g, gr)
    srcs = [0, g.n // 2, g.n - 1]
    _check_bfs(gr, G, g, srcs)
    _check_sssp(gr, G, g, srcs[:2], deltas=[1, 64, 0])


@pytest.mark.parametrize("seed", range(6))
def test_random_graphs(gr, seed):
    makers = [lambda: gg.rmat(12, 16, seed=seed), lambda: gg.kronecker(13, 8, seed=seed),
              lambda: gg.erdos_renyi(50000, 120000, seed=seed),
              lambda: gg.directed_random(20000, 100000, seed=seed),
              lambda: gg.make_config("c3_orkut", shrink=4),
              lambda: gg.make_config("c4_road", shrink=4)]
    g = gg.assign_weights(makers[seed](), seed=seed + 1)
    G = _dev(g, gr)
    srcs = gg.sources(g, 3, seed=seed)
    _check_bfs(gr, G, g, srcs)
    _check_bfs(gr, G, g, srcs[:1], dirs=["auto"], switch_rule=1)
    _check_bfs(gr, G, g, srcs[:1], dirs=["push", "auto"], idempotent=True)
    _check_sssp(gr, G, g, srcs[:2])


def test_c1_rmat16_full(gr):
    g = gg.make_config("c1_rmat16")
    G = _dev(g, gr)
    _check_bfs(gr, G, g, [0] + gg.sources(g, 2))


# ------------------------------------------------------------------ edge cases

def test_single_vertex_and_empty(gr):
    g = gg.empty(1)
    g.W = g.C.clone()
    G = _dev(g, gr)
    assert G.bfs(0)[0].tolist() == [0]
    assert gr.dist_to_u32(G.sssp(0)[0]).tolist() == [0]
    g = gg.empty(100)
    g.W = g.C.clone()
    G = _dev(g, gr)
    d, p = G.bfs(7)
    assert d.cpu().numpy().tolist() == [0 if i == 7 else -1 for i in range(100)]
    assert p.cpu().numpy().tolist() == [7 if i == 7 else -1 for i in range(100)]


def test_isolated_source(gr):
    g = gg.assign_weights(gg.rmat(10, 8, seed=1), seed=2)
    iso = int(torch.nonzero(g.degrees() == 0)[0])
    G = _dev(g, gr)
    d, _ = G.bfs(iso)
    assert int((d >= 0).sum()) == 1 and int(d[iso]) == 0
    dist, _ = G.sssp(iso)
    assert (gr.dist_to_u32(dist) == INF).sum() == g.n - 1


def test_self_loops_multi_edges_zero_weights(gr):
    g = gg.from_edges(6, [(0, 0), (0, 1), (0, 1), (1, 2), (2, 3), (3, 3), (3, 4), (1, 4)],
                      [5, 9, 2, 0, 0, 1, 7, 30], dedupe=False, drop_self_loops=False)
    G = _dev(g, gr)
    _check_bfs(gr, G, g, [0, 3, 5])
    _check_sssp(gr, G, g, [0, 3], deltas=[1, 2, 0xFFFFFFFF])


def test_long_path_many_levels(gr):
    g = gg.assign_weights(gg.path(100_000), seed=3)
    G = _dev(g, gr)
    _check_bfs(gr, G, g, [0, 50_000], dirs=["auto"])
    _check_sssp(gr, G, g, [0], deltas=[0])


def test_star_hub_cta_path(gr):
    g = gg.assign_weights(gg.star(1 << 20), seed=4)
    G = _dev(g, gr)
    _check_bfs(gr, G, g, [0, 17])
    _check_sssp(gr, G, g, [0], deltas=[0])


def test_near_far_stranding_stress(gr):
    """Reading A-7: targets reachable in the same iteration through a heavy
    and a light edge; with a stamp that ignores the slice, dist goes wrong."""
    rng = np.random.default_rng(0)
    k = 3000
    edges, w = [], []
    # 0 -> a (w 1), 0 -> b (w 1); a -> t_i heavy, b -> t_i light
    for i in range(k):
        t = 3 + i
        edges += [(1, t), (2, t)]
        w += [int(rng.integers(40, 65)), int(rng.integers(1, 8))]
    edges += [(0, 1), (0, 2)]
    w += [1, 1]
    g = gg.from_edges(3 + k, edges, w)
    G = _dev(g, gr)
    for _ in range(5):
        _check_sssp(gr, G, g, [0], deltas=[4, 8, 16, 33])


def test_host_output_buffers(gr):
    g = gg.assign_weights(gg.rmat(11, 8, seed=5), seed=6)
    G = _dev(g, gr)
    R, C, W = g.numpy()
    s = gg.sources(g, 1)[0]
    depth = np.empty(g.n, np.int32)
    pred = np.empty(g.n, np.int32)
    G.bfs(s, depth, pred)
    assert np.array_equal(depth, oracle.bfs(R, C, s)[0])
    dist = np.empty(g.n, np.uint32)
    G.sssp(s, dist, None, want_pred=False)
    assert np.array_equal(dist, oracle.sssp(R, C, W, s)[0])


def test_host_input_arrays(gr):
    g = gg.assign_weights(gg.rmat(11, 8, seed=7), seed=8)
    R, C, W = g.numpy()
    G = gr.Graph(R, C, W, symmetric=True)
    s = gg.sources(g, 1)[0]
    assert np.array_equal(G.bfs(s)[0].cpu().numpy(), oracle.bfs(R, C, s)[0])


def test_errors(gr):
    g = gg.path(10)
    G = _dev(g, gr)
    with pytest.raises(gr.GrError) as e:
        G.bfs(10)
    assert e.value.status == 3
    with pytest.raises(gr.GrError) as e:
        G.sssp(0)
    assert e.value.status == 4  # no weights
    R = torch.tensor([0, 2, 1, 3], dtype=torch.int64)
    C = torch.tensor([1, 2, 0], dtype=torch.int32)
    with pytest.raises(gr.GrError) as e:
        gr.Graph(R.cuda(), C.cuda())
    assert e.value.status == 2 and "R[2]=1 < R[1]=2" in str(e.value)
    R = torch.tensor([0, 1, 2, 3], dtype=torch.int64)
    C = torch.tensor([1, 7, 0], dtype=torch.int32)
    with pytest.raises(gr.GrError) as e:
        gr.Graph(R.cuda(), C.cuda())
    assert e.value.status == 2 and "C[1]=7" in str(e.value)
    big = gg.from_edges(3, [(0, 1), (1, 2)], [1, 1])
    big.W = torch.full_like(big.C, 3_000_000_000 - (1 << 32))  # 3e9 as uint32 bits
    G = _dev(big, gr)
    with pytest.raises(gr.GrError) as e:
        G.sssp(0)
    assert e.value.status == 5


def test_run_stats_levels(gr):
    g = gg.make_config("c1_rmat16")
    G = _dev(g, gr)
    R, C, _ = g.numpy()
    ref, _ = oracle.bfs(R, C, 0)
    G.bfs(0, direction="push")
    st = G.run_stats()
    sizes = np.bincount(ref[ref >= 0])
    assert st["num_levels"] == len(sizes)
    # push, exactly-once claims: frontier sizes are the level sizes (deg>0 only)
    deg = np.diff(R)
    for rec in st["levels"]:
        L = rec["level"]
        want = int(((ref == L) & (deg > 0)).sum())
        assert rec["frontier"] == want
        assert rec["frontier_edges"] == int(deg[ref == L].sum())
    # run totals: vertices reached and the TEPS numerator (A-14)
    assert st["reached"] == int((ref >= 0).sum())
    assert st["reached_edges"] == oracle.reached_edges(R, ref, -1)
    gw = gg.assign_weights(gg.make_config("c1_rmat16"), seed=2)
    Gw = _dev(gw, gr)
    Rw, Cw, Ww = gw.numpy()
    s = gg.sources(gw, 1)[0]
    Gw.sssp(s)
    dref, _ = oracle.sssp(Rw, Cw, Ww, s)
    st = Gw.run_stats()
    assert st["reached"] == int((dref != oracle.UINT32_MAX).sum())
    assert st["reached_edges"] == oracle.reached_edges(Rw, dref, oracle.UINT32_MAX)
    # idempotent discovery (duplicates possible in the queue): totals stay exact
    G.bfs(s, direction="auto", idempotent=True)
    dref2, _ = oracle.bfs(R, C, s)
    st = G.run_stats()
    assert st["reached"] == int((dref2 >= 0).sum())
    assert st["reached_edges"] == oracle.reached_edges(R, dref2, -1)


@pytest.mark.parametrize("strategy", ["twc", "lb"])
def test_strategies_forced(gr, strategy):
    """Thread/warp/CTA and merge-path advances give the
    same depths on skewed (hub lists > CTA size), directed and mesh graphs."""
    for g in (gg.rmat(14, 16, seed=2), gg.star(200_000), gg.directed_random(40000, 300000, seed=4),
              gg.make_config("c4_road", shrink=4)):
        g = gg.assign_weights(g, seed=1)
        G = _dev(g, gr)
        srcs = gg.sources(g, 2)
        _check_bfs(gr, G, g, srcs, dirs=["push", "auto"], strategy=strategy)
        _check_bfs(gr, G, g, srcs[:1], dirs=["push"], strategy=strategy, idempotent=True)


def test_async_runs_match_oracle(gr):
    """gr_bfs_async / gr_sssp_async enqueue only; after gr_graph_sync the
    outputs of back-to-back runs equal the oracle's (include/gr.h)."""
    g = gg.assign_weights(gg.rmat(14, 16, seed=7), seed=8)
    R, C, W = g.numpy()
    G = _dev(g, gr)
    srcs = gg.sources(g, 3)
    outs = []
    for s in srcs:  # distinct output buffers, no host sync in between
        d = torch.empty(g.n, dtype=torch.int32, device="cuda")
        p = torch.empty(g.n, dtype=torch.int32, device="cuda")
        G.bfs(s, d, p, direction="auto", asynchronous=True)
        outs.append((s, d, p))
    dist = torch.empty(g.n, dtype=torch.int32, device="cuda")
    G.sssp(srcs[0], dist, None, want_pred=False, asynchronous=True)
    G.sync()
    for s, d, p in outs:
        ref, _ = oracle.bfs(R, C, s)
        got = d.cpu().numpy()
        assert np.array_equal(got, ref)
        assert oracle.check_bfs(R, C, s, got, p.cpu().numpy()) == []
    ref, _ = oracle.sssp(R, C, W, srcs[0])
    assert np.array_equal(gr.dist_to_u32(dist), ref)
    # host outputs are refused by the asynchronous entry points
    host = torch.empty(g.n, dtype=torch.int32)
    with pytest.raises(gr.GrError):
        G.bfs(srcs[0], host, None, want_pred=False, asynchronous=True)
    G.sync()  # nothing pending: OK
    G.close()


@pytest.mark.parametrize("env", [{}, {"GR_LB_CHUNKS": "16"}, {"GR_LB_CHUNKS": "0"},
                                 {"GR_PROBE_SKIP_PCT": "0"}, {"GR_SPLIT_ORDER": "0"},
                                 {"GR_CLAIM_CAS": "1"}])
def test_mid_size_variants(gr, env, monkeypatch):
    """Sizes where the grid-level machinery engages (dynamic merge-path pieces
    need >= 256 items per warp; long in-lists reach the warp scan of the pull
    step; pull -> push transitions rebuild the queue from the bitmap), under
    each tuning knob's alternative setting."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    graphs = [gg.kronecker(17, 16, seed=11), gg.make_config("c3_orkut", shrink=3),
              gg.directed_random(200_000, 2_000_000, seed=12)]
    for g in graphs:
        G = _dev(g, gr)
        _check_bfs(gr, G, g, gg.sources(g, 2), dirs=["push", "auto", "pull"])
        _check_bfs(gr, G, g, gg.sources(g, 1), dirs=["auto"], idempotent=True)
        G.close()


# ------------------------------------------------------------------ bounded-degree adjacency

def _bounded_directed(n, seed):
    """Directed graph with out-degrees 0..4 (the ELL record's capacity) and
    in-degrees unconstrained; weights 1..64."""
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 5, size=n)
    src = np.repeat(np.arange(n), deg)
    dst = rng.integers(0, n, size=src.size)
    w = rng.integers(1, 65, size=src.size)
    return gg.from_edges(n, list(zip(src.tolist(), dst.tolist())), w.tolist(), symmetrize=False)


@pytest.mark.parametrize("ell,cluster", [("1", "1"), ("1", "0"), ("0", "1")])
def test_bounded_degree_adjacency(gr, ell, cluster, monkeypatch):
    """Graphs whose out-degrees are all <= 4 get the 16-B / 32-B per-vertex
    adjacency records (gr_graph_info.bounded_degree); BFS in every direction
    and mode, and SSSP for several deltas, equal the oracle with the records
    and the narrow levels in one thread-block cluster (default), with the
    records on the grid kernel only (GR_ELL_CLUSTER=0), and without records
    (GR_ELL=0). The 2^18-vertex tree's frontiers outgrow the cluster (one
    entry per thread) and its delta=1 far piles outgrow its queues: both hand
    the traversal to the grid kernel mid-run."""
    monkeypatch.setenv("GR_ELL", ell)
    monkeypatch.setenv("GR_ELL_CLUSTER", cluster)
    graphs = [gg.assign_weights(gg.grid(61, 47), seed=3), gg.assign_weights(gg.path(3000), seed=4),
              gg.make_config("c4_road", shrink=3), _bounded_directed(60000, 5),
              gg.assign_weights(gg.binary_tree(20000), seed=6),
              gg.assign_weights(gg.binary_tree(1 << 18), seed=7)]
    for g in graphs:
        G = _dev(g, gr)
        info = G.info()
        assert info.bounded_degree == (1 if ell == "1" else 0), (g.n, info.max_degree)
        srcs = gg.sources(g, 2) + [0]
        _check_bfs(gr, G, g, srcs)
        _check_bfs(gr, G, g, srcs[:1], dirs=["push", "auto"], idempotent=True)
        _check_sssp(gr, G, g, srcs[:2], deltas=[1, 8, 64, 0xFFFFFFFF, 0])
        G.close()
    # max out-degree 5: no records
    g = gg.star(5)
    G = _dev(g, gr)
    assert G.info().bounded_degree == 0
    G.close()


@pytest.mark.parametrize("cluster", ["1", "0"])
def test_run_stats_bounded_degree(gr, cluster, monkeypatch):
    """Per-level records and run totals stay exact on the bounded-degree paths:
    levels run in the one-cluster kernel, in the grid kernel, and (the 2^18
    tree from its root: a 32K-vertex frontier) across the cluster -> grid
    handoff, whose records come from both kernels."""
    monkeypatch.setenv("GR_ELL_CLUSTER", cluster)
    for g, s in ((gg.make_config("c4_road", shrink=3), None), (gg.binary_tree(1 << 18), 0)):
        G = _dev(g, gr)
        assert G.info().bounded_degree == 1
        R, C, _ = g.numpy()
        src = gg.sources(g, 1)[0] if s is None else s
        ref, _ = oracle.bfs(R, C, src)
        G.bfs(src, direction="push")
        st = G.run_stats()
        sizes = np.bincount(ref[ref >= 0])
        assert st["num_levels"] == len(sizes)
        deg = np.diff(R)
        for rec in st["levels"]:
            L = rec["level"]
            assert rec["frontier"] == int(((ref == L) & (deg > 0)).sum()), L
            assert rec["frontier_edges"] == int(deg[ref == L].sum()), L
        assert st["reached"] == int((ref >= 0).sum())
        assert st["reached_edges"] == oracle.reached_edges(R, ref, -1)
        gw = gg.assign_weights(g, seed=9)
        Gw = _dev(gw, gr)
        Rw, Cw, Ww = gw.numpy()
        Gw.sssp(src)
        dref, _ = oracle.sssp(Rw, Cw, Ww, src)
        st = Gw.run_stats()
        assert st["reached"] == int((dref != oracle.UINT32_MAX).sum())
        assert st["reached_edges"] == oracle.reached_edges(Rw, dref, oracle.UINT32_MAX)
        G.close()
        Gw.close()
