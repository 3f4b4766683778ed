"""Pins for the CPU oracle (oracle/) against things other than itself.

Every check compares the oracle with a value fixed by the paper / SPEC worked
examples (tests/golden/, cited), a closed form, a textbook brute force, or a
library routine (scipy.sparse.csgraph) -- never with a retyped copy of the
oracle's own algorithm. The certificates (oracle.check_*) are pinned too: they
must reject plausible mistakes (dropped term, off-by-one, wrong parent).
"""
import itertools
import math

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse import csgraph

import graphgen as gg
import oracle

INF = oracle.UINT32_MAX


def _np(g):
    return g.numpy()


def _run_bfs(g, s):
    R, C, _ = _np(g)
    d, p = oracle.bfs(R, C, s)
    assert oracle.check_bfs(R, C, s, d, p) == []
    return d, p


def _run_sssp(g, s):
    R, C, W = _np(g)
    d, p = oracle.sssp(R, C, W, s)
    assert oracle.check_sssp(R, C, W, s, d, p) == []
    return d, p


# ---------------------------------------------------------------- golden (SPEC)

def test_golden_csr(golden):
    for key in ("csr_build", "csr_empty"):
        ex = golden[key]
        g = gg.from_edges(ex["n"], [tuple(e) for e in ex["edges"]], symmetrize=False) \
            if ex["edges"] else gg.empty(ex["n"])
        assert g.R.tolist() == ex["R"], ex["cite"]
        assert g.C.tolist() == ex["C"], ex["cite"]


def test_golden_bfs(golden):
    for key in ("bfs_g1", "bfs_single"):
        ex = golden[key]
        g = gg.from_edges(ex["n"], [tuple(e) for e in ex["edges"]]) if ex["edges"] else gg.empty(ex["n"])
        d, _ = _run_bfs(g, ex["src"])
        assert d.tolist() == ex["depth"], ex["cite"]


def test_golden_sssp(golden):
    for key in ("sssp_spec", "sssp_source_only"):
        ex = golden[key]
        if ex["edges"]:
            g = gg.from_edges(ex["n"], [tuple(e) for e in ex["edges"]], ex["weights"])
        else:
            g = gg.empty(ex["n"])
            g.W = g.C.clone()
        d, _ = _run_sssp(g, ex["src"])
        assert d.tolist() == ex["dist"], ex["cite"]


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("n,s", [(1, 0), (2, 1), (17, 0), (17, 9), (200, 57)])
def test_path(n, s):
    d, _ = _run_bfs(gg.path(n), s)
    assert d.tolist() == [abs(i - s) for i in range(n)]


def test_weighted_path_prefix_sums():
    n = 50
    w = [(7 * i * i + 3) % 64 + 1 for i in range(n - 1)]
    g = gg.from_edges(n, [(i, i + 1) for i in range(n - 1)], w)
    s = 13
    pre = [0] + list(itertools.accumulate(w))
    d, _ = _run_sssp(g, s)
    assert d.tolist() == [abs(pre[i] - pre[s]) for i in range(n)]


@pytest.mark.parametrize("n,s", [(3, 0), (101, 0), (101, 40), (64, 63)])
def test_cycle(n, s):
    d, _ = _run_bfs(gg.cycle(n), s)
    assert d.tolist() == [min(abs(i - s), n - abs(i - s)) for i in range(n)]


@pytest.mark.parametrize("r,c,s", [(13, 29, 0), (13, 29, 200), (1, 40, 5)])
def test_grid_manhattan(r, c, s):
    g = gg.grid(r, c)
    d, _ = _run_bfs(g, s)
    si, sj = divmod(s, c)
    assert d.tolist() == [abs(i - si) + abs(j - sj) for i in range(r) for j in range(c)]
    # constant weight 3 -> 3 * Manhattan
    g.W = torch_full_like(g.C, 3)
    dd, _ = _run_sssp(g, s)
    assert dd.tolist() == [3 * x for x in d.tolist()]


def torch_full_like(t, v):
    import torch
    return torch.full_like(t, v)


def test_complete_graph():
    n = 40
    d, _ = _run_bfs(gg.complete(n), 7)
    assert d.tolist() == [0 if i == 7 else 1 for i in range(n)]
    # w(i,j) = |i-j|: dist(0, j) = j (many tied paths exercise pred checks)
    e = [(i, j) for i in range(n) for j in range(i + 1, n)]
    g = gg.from_edges(n, e, [j - i for i, j in e])
    dd, _ = _run_sssp(g, 0)
    assert dd.tolist() == list(range(n))


def test_star():
    L = 30
    g = gg.star(L)
    d, _ = _run_bfs(g, 0)
    assert d.tolist() == [0] + [1] * L
    d, _ = _run_bfs(g, 5)
    assert d.tolist() == [1] + [0 if i == 5 else 2 for i in range(1, L + 1)]


def test_binary_tree():
    n = 1000
    d, _ = _run_bfs(gg.binary_tree(n), 0)
    assert d.tolist() == [int(math.floor(math.log2(i + 1))) for i in range(n)]


@pytest.mark.parametrize("dim,s", [(7, 0), (7, 77)])
def test_hypercube(dim, s):
    g = gg.hypercube(dim)
    d, _ = _run_bfs(g, s)
    assert d.tolist() == [bin(v ^ s).count("1") for v in range(1 << dim)]
    # w(u, u ^ 2^b) = b + 1  ->  dist = sum over differing bits of (b + 1)
    R, C, _ = _np(g)
    src = np.repeat(np.arange(g.n), np.diff(R))
    b = np.log2(src ^ C).astype(np.int64)
    g.W = torch_from(b + 1)
    dd, _ = _run_sssp(g, s)
    assert dd.tolist() == [sum(k + 1 for k in range(dim) if (v ^ s) >> k & 1) for v in range(1 << dim)]


def torch_from(a):
    import torch
    return torch.from_numpy(np.asarray(a, dtype=np.int32))


def test_disjoint_union_unreached():
    # path 0-1-2 plus a separate edge 3-4 and isolated 5
    g = gg.from_edges(6, [(0, 1), (1, 2), (3, 4)], [5, 6, 7])
    d, p = _run_bfs(g, 0)
    assert d.tolist() == [0, 1, 2, -1, -1, -1]
    assert p.tolist()[3:] == [-1, -1, -1] and p[0] == 0
    dd, _ = _run_sssp(g, 0)
    assert dd.tolist() == [0, 5, 11, INF, INF, INF]


def test_directed_follows_out_edges():
    g = gg.from_edges(3, [(0, 1), (1, 2)], symmetrize=False)
    assert _run_bfs(g, 0)[0].tolist() == [0, 1, 2]
    assert _run_bfs(g, 2)[0].tolist() == [-1, -1, 0]


def test_self_loops_and_multi_edges():
    # CSR that keeps a self-loop and two parallel copies of (0,1) with weights 9 and 2
    g = gg.from_edges(3, [(0, 0), (0, 1), (0, 1), (1, 2)], [1, 9, 2, 4],
                      dedupe=False, drop_self_loops=False)
    R, C, W = _np(g)
    assert (C == 0).any() and np.diff(R)[0] >= 3
    d, _ = _run_bfs(g, 0)
    assert d.tolist() == [0, 1, 2]
    dd, _ = _run_sssp(g, 0)
    assert dd.tolist() == [0, 2, 6]  # minimum parallel weight wins


def test_zero_weights():
    g = gg.from_edges(4, [(0, 1), (1, 2), (2, 3)], [0, 0, 5])
    dd, _ = _run_sssp(g, 0)
    assert dd.tolist() == [0, 0, 0, 5]


def test_unit_weights_equal_bfs():
    g = gg.erdos_renyi(3000, 9000, seed=5)
    g.W = torch_full_like(g.C, 1)
    for s in gg.sources(g, 3):
        d, _ = _run_bfs(g, s)
        dd, _ = _run_sssp(g, s)
        assert np.array_equal(np.where(d < 0, INF, d).astype(np.uint32), dd)


def test_errors():
    g = gg.path(4)
    R, C, _ = _np(g)
    with pytest.raises(ValueError):
        oracle.bfs(R, C, 4)
    with pytest.raises(ValueError):
        oracle.bfs(R, C, -1)
    # uint32 overflow of a distance is reported, not wrapped (A-19)
    big = gg.from_edges(3, [(0, 1), (1, 2)], [0, 0])
    Rb, Cb, _ = _np(big)
    W = np.array([3_000_000_000] * 4, dtype=np.uint32)
    with pytest.raises(OverflowError):
        oracle.sssp(Rb, Cb, W, 0)


# ---------------------------------------------------------------- brute force

def _floyd_warshall(n, R, C, W):
    D = [[None] * n for _ in range(n)]
    for i in range(n):
        D[i][i] = 0
    for u in range(n):
        for e in range(R[u], R[u + 1]):
            v = int(C[e]); w = int(W[e])
            if u != v and (D[u][v] is None or w < D[u][v]):
                D[u][v] = w
    for k in range(n):
        Dk = D[k]
        for i in range(n):
            dik = D[i][k]
            if dik is None:
                continue
            Di = D[i]
            for j in range(n):
                if Dk[j] is not None and (Di[j] is None or dik + Dk[j] < Di[j]):
                    Di[j] = dik + Dk[j]
    return D


def _all_simple_paths_min(n, adj, s):
    """n <= 8: enumerate every simple path from s (exponential, obviously right)."""
    best = [None] * n
    best[s] = 0

    def rec(u, cost, seen):
        for v, w in adj[u]:
            if v in seen:
                continue
            c = cost + w
            if best[v] is None or c < best[v]:
                best[v] = c
            rec(v, c, seen | {v})
    rec(s, 0, {s})
    return best


@pytest.mark.parametrize("seed", range(40))
def test_brute_force_small(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 40))
    mp = int(rng.integers(0, 3 * n))
    directed = bool(seed % 3 == 0)
    e = [(int(a), int(b)) for a, b in rng.integers(0, n, size=(mp, 2))]
    w = [int(x) for x in rng.integers(0 if seed % 5 == 0 else 1, 65, size=mp)]
    g = gg.from_edges(n, e, w, symmetrize=not directed) if e else gg.empty(n)
    if not e:
        g.W = g.C.clone()
    R, C, W = _np(g)
    D = _floyd_warshall(n, R, C, W)
    U = _floyd_warshall(n, R, C, np.ones_like(W))
    for s in range(min(n, 6)):
        dd, _ = _run_sssp(g, s)
        d, _ = _run_bfs(g, s)
        assert dd.tolist() == [INF if x is None else x for x in D[s]]
        assert d.tolist() == [-1 if x is None else x for x in U[s]]


@pytest.mark.parametrize("seed", range(25))
def test_brute_force_paths_tiny(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 8))
    mp = int(rng.integers(1, 2 * n + 2))
    e = [(int(a), int(b)) for a, b in rng.integers(0, n, size=(mp, 2))]
    w = [int(x) for x in rng.integers(1, 65, size=mp)]
    g = gg.from_edges(n, e, w, symmetrize=bool(seed % 2))
    R, C, W = _np(g)
    adj = [[(int(C[k]), int(W[k])) for k in range(R[u], R[u + 1])] for u in range(n)]
    s = int(rng.integers(0, n))
    best = _all_simple_paths_min(n, adj, s)
    dd, _ = _run_sssp(g, s)
    assert dd.tolist() == [INF if x is None else x for x in best]


# ---------------------------------------------------------------- library (scipy)

@pytest.mark.parametrize("maker", [
    lambda: gg.rmat(12, 16, seed=3),
    lambda: gg.kronecker(12, 16, seed=4),
    lambda: gg.erdos_renyi(20000, 40000, seed=6),
    lambda: gg.directed_random(5000, 30000, seed=7),
    lambda: gg.make_config("c4_road", shrink=5),
])
def test_scipy_crosscheck(maker):
    g = gg.assign_weights(maker(), seed=9)
    R, C, W = _np(g)
    n = g.n
    A = sp.csr_matrix((W.astype(np.float64), C, R), shape=(n, n))
    U = sp.csr_matrix((np.ones(C.size), C, R), shape=(n, n))
    for s in gg.sources(g, 3):
        d, _ = _run_bfs(g, s)
        ref = csgraph.shortest_path(U, method="D", directed=True, unweighted=True, indices=s)
        assert np.array_equal(np.where(np.isinf(ref), -1, ref).astype(np.int64), d.astype(np.int64))
        dd, _ = _run_sssp(g, s)
        refw = csgraph.dijkstra(A, directed=True, indices=s)
        assert np.array_equal(np.where(np.isinf(refw), INF, refw).astype(np.int64), dd.astype(np.int64))


# ---------------------------------------------------------------- certificates reject mistakes

def test_bfs_certificate_rejects_mistakes():
    g = gg.rmat(10, 8, seed=2)
    R, C, _ = _np(g)
    s = gg.sources(g, 1)[0]
    d, p = oracle.bfs(R, C, s)
    assert oracle.check_bfs(R, C, s, d, p) == []
    reached = np.flatnonzero(d > 0)
    rng = np.random.default_rng(0)
    v = int(rng.choice(reached))
    for bad_d in (d + (np.arange(d.size) == v), d - (np.arange(d.size) == v)):
        assert oracle.check_bfs(R, C, s, bad_d.astype(np.int32), p) != []
    unreached = np.flatnonzero(d < 0)
    if unreached.size:
        bd = d.copy(); bd[unreached[0]] = 3
        assert oracle.check_bfs(R, C, s, bd, p) != []
    bp = p.copy(); bp[v] = v  # self parent
    assert oracle.check_bfs(R, C, s, d, bp) != []
    bp = p.copy(); bp[s] = -1
    assert oracle.check_bfs(R, C, s, d, bp) != []
    # a parent at the same depth (exists in the graph, wrong level)
    same = [u for u in C[R[v]:R[v + 1]] if d[u] == d[v]]
    if same:
        bp = p.copy(); bp[v] = same[0]
        assert oracle.check_bfs(R, C, s, d, bp) != []


def test_sssp_certificate_rejects_mistakes():
    g = gg.assign_weights(gg.rmat(10, 8, seed=2), seed=3)
    R, C, W = _np(g)
    s = gg.sources(g, 1)[0]
    d, p = oracle.sssp(R, C, W, s)
    assert oracle.check_sssp(R, C, W, s, d, p) == []
    reached = np.flatnonzero((d != INF) & (np.arange(d.size) != s))
    v = int(reached[len(reached) // 2])
    for delta in (+1, -1):
        bd = d.astype(np.int64); bd[v] += delta
        assert oracle.check_sssp(R, C, W, s, bd.astype(np.uint32), p) != []
    bp = p.copy(); bp[v] = s if s != p[v] else int(C[R[v]])
    if bp[v] != p[v]:
        errs = oracle.check_sssp(R, C, W, s, d, bp)
        # either not an edge or not tight unless it is a genuinely tied parent
        nbr = C[R[bp[v]]:R[bp[v] + 1]]
        wts = W[R[bp[v]]:R[bp[v] + 1]]
        tied = any(int(x) == v and int(d[bp[v]]) + int(wt) == int(d[v]) for x, wt in zip(nbr, wts))
        assert (errs == []) == tied


# ---------------------------------------------------------------- TEPS arithmetic

def test_table3_teps_arithmetic():
    import json, os
    from paper_1501_05387_b200.metrics import teps
    with open(os.path.join(os.path.dirname(__file__), "golden", "table3_mteps.json")) as f:
        rows = json.load(f)["rows"]
    for r in rows:
        mteps = teps(r["edges_M"] * 1e6, r["ms"] * 1e-3) / 1e6
        assert abs(mteps - r["mteps"]) / r["mteps"] < 0.013, r


def test_metrics_aggregates():
    """Harmonic mean / median / Graph500 halving on values
    whose results are fixed by arithmetic: 1 edge per second per source at
    GTEPS 1, 2, 4 -> harmonic mean 3 / (1 + 1/2 + 1/4) = 12/7, median 2."""
    from paper_1501_05387_b200 import metrics
    edges = [1e9, 2e9, 4e9]
    ms = [1000.0, 1000.0, 1000.0]
    s = metrics.summarize(edges, ms)
    assert abs(s["harmonic_mean"] - 12.0 / 7.0) < 1e-12
    assert s["median"] == 2.0
    assert abs(s["aggregate"] - 7.0 / 3.0) < 1e-12
    assert abs(s["graph500_aggregate"] - 7.0 / 6.0) < 1e-12
    assert metrics.harmonic_mean([5.0]) == 5.0


# ---------------------------------------------------------------- reached_edges (TEPS numerator, A-14)

def test_reached_edges_closed_forms():
    """oracle.reached_edges = directed edges whose source is reached, checked
    against counts fixed by the graph's shape: path P_n from anywhere reaches
    all 2(n-1) directed edges; a disjoint union P_5 + K_4 reaches 8 edges from
    the path and 4*3 = 12 from the clique; a directed chain 0->1->...->n-1
    from vertex k reaches the n-1-k edges after it; an isolated source reaches
    no edge."""
    R, C, _ = gg.path(7).numpy()
    d, _ = oracle.bfs(R, C, 3)
    assert oracle.reached_edges(R, d, -1) == 12
    g = gg.from_edges(9, [(0, 1), (1, 2), (2, 3), (3, 4)] +
                      [(a, b) for a in range(5, 9) for b in range(a + 1, 9)])
    R, C, _ = g.numpy()
    assert oracle.reached_edges(R, oracle.bfs(R, C, 2)[0], -1) == 8
    assert oracle.reached_edges(R, oracle.bfs(R, C, 6)[0], -1) == 12
    n = 10
    g = gg.from_edges(n, [(i, i + 1) for i in range(n - 1)], symmetrize=False)
    R, C, _ = g.numpy()
    for k in (0, 4, 9):
        assert oracle.reached_edges(R, oracle.bfs(R, C, k)[0], -1) == n - 1 - k
    g = gg.from_edges(4, [(1, 2), (2, 3)])
    R, C, _ = g.numpy()
    assert oracle.reached_edges(R, oracle.bfs(R, C, 0)[0], -1) == 0
    # SSSP sentinel: unreached = UINT32_MAX
    gw = gg.assign_weights(gg.from_edges(6, [(0, 1), (1, 2), (3, 4)]), seed=1)
    R, C, W = gw.numpy()
    dist, _ = oracle.sssp(R, C, W, 0)
    assert oracle.reached_edges(R, dist, INF) == 4


def test_reached_edges_brute_force():
    """Against an explicit edge-list count on random small graphs: for every
    (u, v) in the edge list, count it iff u is reachable from s (reachability
    by scipy's breadth_first_order, a library routine)."""
    for seed in range(6):
        g = gg.directed_random(300, 900, seed=seed) if seed % 2 else gg.erdos_renyi(300, 400, seed=seed)
        R, C, _ = g.numpy()
        n = len(R) - 1
        A = sp.csr_matrix((np.ones(len(C)), C, R), shape=(n, n))
        for s in (0, 17, 150):
            order = csgraph.breadth_first_order(A, s, directed=True, return_predecessors=False)
            reach = np.zeros(n, bool)
            reach[order] = True
            src_of = np.repeat(np.arange(n), np.diff(R))
            want = int(reach[src_of].sum())
            assert oracle.reached_edges(R, oracle.bfs(R, C, s)[0], -1) == want
