"""Pins of the BC oracle (oracle.bc, Brandes 2001 Alg. 1) to things other
than itself (paper §5.3):

* SPEC worked examples: path a-b-c -> [0, 1, 0] and star K1,3
  centre -> 3 under the undirected halving convention;
* closed forms: path P_n vertex i -> i (n-1-i); star K1,k centre -> k(k-1)/2;
  complete K_n -> 0; odd cycle C_n -> (n-1)(n-3)/8 for every vertex;
* brute force: every shortest s-t path enumerated explicitly by DFS over the
  hop-distance DAG, bc[v] = sum over ordered pairs s != t of
  (#shortest s-t paths through v) / (#shortest s-t paths), on random small
  directed and undirected graphs (no Brandes recursion involved);
* single source on a tree: leaves have dependency 0.
"""
import itertools
import random

import numpy as np
import pytest

import graphgen as gg
import oracle


def _all(g):
    R, C, _ = g.numpy()
    return R, C, list(range(g.n))


def test_spec_examples():
    R, C, S = _all(gg.path(3))
    assert np.allclose(oracle.bc(R, C, S) / 2, [0, 1, 0])
    R, C, S = _all(gg.star(3))
    assert oracle.bc(R, C, S)[0] / 2 == pytest.approx(3.0)


@pytest.mark.parametrize("n", [2, 5, 9, 16])
def test_path_closed_form(n):
    R, C, S = _all(gg.path(n))
    i = np.arange(n)
    assert np.allclose(oracle.bc(R, C, S) / 2, i * (n - 1 - i))


@pytest.mark.parametrize("k", [1, 3, 10])
def test_star_closed_form(k):
    R, C, S = _all(gg.star(k))
    bc = oracle.bc(R, C, S) / 2
    assert bc[0] == pytest.approx(k * (k - 1) / 2)
    assert np.allclose(bc[1:], 0)


@pytest.mark.parametrize("n", [3, 6])
def test_complete_is_zero(n):
    R, C, S = _all(gg.complete(n))
    assert np.allclose(oracle.bc(R, C, S), 0)


@pytest.mark.parametrize("n", [5, 7, 11])
def test_odd_cycle_closed_form(n):
    R, C, S = _all(gg.cycle(n))
    assert np.allclose(oracle.bc(R, C, S) / 2, (n - 1) * (n - 3) / 8)


def test_tree_single_source_leaves_zero():
    g = gg.binary_tree(31)
    R, C, _ = g.numpy()
    bc = oracle.bc(R, C, [0])
    leaves = [v for v in range(31) if R[v + 1] - R[v] == 1 and v != 0]
    assert np.allclose(bc[leaves], 0)
    # heap tree from the root: delta(v) = size of the subtree below v (one path each)
    sub = np.zeros(31)
    for v in range(30, -1, -1):
        for c in (2 * v + 1, 2 * v + 2):
            if c < 31:
                sub[v] += 1 + sub[c]
    assert np.allclose(bc[1:], sub[1:])


def _brute_bc(n, adj):
    """Ordered-pair sum of path fractions by explicit enumeration."""
    def bfs(s):
        d = [-1] * n
        d[s] = 0
        q = [s]
        for v in q:
            for w in adj[v]:
                if d[w] < 0:
                    d[w] = d[v] + 1
                    q.append(w)
        return d

    bc = [0.0] * n
    for s in range(n):
        d = bfs(s)
        paths = {t: [] for t in range(n)}

        def dfs(v, path):
            paths[v].append(list(path))
            for w in adj[v]:
                if d[w] == d[v] + 1:
                    path.append(w)
                    dfs(w, path)
                    path.pop()
        dfs(s, [s])
        for t in range(n):
            if t == s or not paths[t]:
                continue
            tot = len(paths[t])
            for v in range(n):
                if v in (s, t):
                    continue
                bc[v] += sum(1 for p in paths[t] if v in p) / tot
    return np.array(bc)


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_random(seed):
    rnd = random.Random(seed)
    n = rnd.randint(2, 9)
    directed = seed % 2 == 1
    pairs = [(u, v) for u, v in itertools.permutations(range(n), 2) if rnd.random() < 0.35]
    g = gg.from_edges(n, pairs, symmetrize=not directed) if pairs else gg.empty(n)
    R, C, _ = g.numpy()
    adj = [list(C[R[v]:R[v + 1]]) for v in range(n)]
    assert np.allclose(oracle.bc(R, C, list(range(n))), _brute_bc(n, adj), rtol=1e-12, atol=1e-12)


def test_subset_of_sources_is_additive():
    g = gg.rmat(7, 4, seed=3)
    R, C, _ = g.numpy()
    a = oracle.bc(R, C, [1, 5])
    b = oracle.bc(R, C, [1]) + oracle.bc(R, C, [5])
    assert np.allclose(a, b)


def test_bad_source_raises():
    R, C, _ = gg.path(4).numpy()
    with pytest.raises(ValueError):
        oracle.bc(R, C, [4])
