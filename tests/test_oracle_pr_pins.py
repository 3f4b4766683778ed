"""Pins of the PageRank oracle (oracle.pagerank, Jacobi power iteration;
paper §5.5, reading A-23) to things other than itself:
* the fixed point as a linear system (I - d M^T) x = (1-d)/n 1 solved by a
  dense library solver (numpy.linalg.solve) on small graphs;
* closed forms: a regular graph (cycle, complete, hypercube) has x = 1/n; a
  star K1,k has centre c and leaves l solving c = (1-d)/n + d k l and
  l = (1-d)/n + d c / k (2x2 system by hand);
* invariants: with no dangling vertex the ranks sum to 1; an isolated vertex
  keeps (1-d)/n.
"""
import numpy as np
import pytest

import graphgen as gg
import oracle


def _dense_fixed_point(R, C, d):
    n = R.size - 1
    M = np.zeros((n, n))
    for u in range(n):
        deg = R[u + 1] - R[u]
        for v in C[R[u]:R[u + 1]]:
            M[v, u] += 1.0 / deg
    return np.linalg.solve(np.eye(n) - d * M, np.full(n, (1 - d) / n))


@pytest.mark.parametrize("name", ["rmat", "directed", "er"])
@pytest.mark.parametrize("d", [0.5, 0.85])
def test_linear_solve(name, d):
    g = {"rmat": lambda: gg.rmat(7, 4, seed=1), "directed": lambda: gg.directed_random(90, 400, seed=2),
         "er": lambda: gg.erdos_renyi(120, 200, seed=3)}[name]()
    R, C, _ = g.numpy()
    x = oracle.pagerank(R, C, d)
    ref = _dense_fixed_point(R, C, d)
    assert np.allclose(x, ref, rtol=1e-12, atol=0)


@pytest.mark.parametrize("g", [gg.cycle(17), gg.complete(9), gg.hypercube(6)])
def test_regular_uniform(g):
    R, C, _ = g.numpy()
    x = oracle.pagerank(R, C)
    assert np.allclose(x, 1.0 / g.n, rtol=1e-13)


@pytest.mark.parametrize("k", [1, 4, 30])
def test_star_closed_form(k):
    d, n = 0.85, k + 1
    R, C, _ = gg.star(k).numpy()
    x = oracle.pagerank(R, C, d)
    b = (1 - d) / n
    # c = b + d k l, l = b + d c / k  ->  c = b + d k b + d^2 c  ->  c = b (1 + d k) / (1 - d^2)
    c = b * (1 + d * k) / (1 - d * d)
    l = b + d * c / k
    assert x[0] == pytest.approx(c, rel=1e-13)
    assert np.allclose(x[1:], l, rtol=1e-13)
    assert x.sum() == pytest.approx(1.0, rel=1e-13)


def test_isolated_and_mass():
    g = gg.from_edges(6, [(0, 1), (1, 2), (2, 0), (3, 4)])  # vertex 5 isolated
    R, C, _ = g.numpy()
    x = oracle.pagerank(R, C)
    assert x[5] == pytest.approx(0.15 / 6, rel=1e-14)
    assert np.allclose(x[:3], x[0]) and np.allclose(x[3:5], x[3])
    assert x.sum() == pytest.approx(1.0 - 0.85 / 6, rel=1e-12)  # the isolated vertex's mass leaks
