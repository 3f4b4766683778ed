"""Pins of the connected-components oracle (oracle.cc: union-find, smallest
id per component; paper §5.4) to things other than itself:
closed forms (empty graph, path, grid, disjoint unions with known members),
brute force (transitive closure of the undirected adjacency matrix by
Boolean matrix powers on tiny graphs), and scipy.sparse.csgraph
(library special case: same partition, same count)."""
import random

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

import graphgen as gg
import oracle


def test_empty_graph_every_vertex_alone():
    R, C, _ = gg.empty(7).numpy()
    comp, k = oracle.cc(R, C)
    assert k == 7 and list(comp) == list(range(7))


def test_path_and_grid_one_component():
    for g in (gg.path(30), gg.grid(9, 13), gg.hypercube(5)):
        R, C, _ = g.numpy()
        comp, k = oracle.cc(R, C)
        assert k == 1 and not comp.any()


def test_disjoint_union_known_members():
    # components {0,5,9}, {1,2}, {3}, {4,6,7,8}: labels are the smallest ids
    g = gg.from_edges(10, [(9, 5), (5, 0), (2, 1), (8, 7), (7, 6), (6, 4)])
    R, C, _ = g.numpy()
    comp, k = oracle.cc(R, C)
    assert k == 4
    assert list(comp) == [0, 1, 1, 3, 4, 0, 4, 4, 4, 0]


def test_directed_edges_count_as_undirected():
    g = gg.from_edges(6, [(5, 0), (3, 4)], symmetrize=False)
    R, C, _ = g.numpy()
    comp, k = oracle.cc(R, C)
    assert k == 4 and list(comp) == [0, 1, 2, 3, 3, 0]


def _closure_labels(n, R, C):
    A = np.eye(n, dtype=bool)
    for u in range(n):
        for v in C[R[u]:R[u + 1]]:
            A[u, v] = A[v, u] = True
    reach = A.copy()
    while True:  # Boolean powers until the reachability matrix stops growing
        nxt = (reach.astype(np.int64) @ A.astype(np.int64)) > 0
        if (nxt == reach).all():
            break
        reach = nxt
    return np.array([np.flatnonzero(reach[v]).min() for v in range(n)], np.int32)


@pytest.mark.parametrize("seed", range(20))
def test_brute_force_closure(seed):
    rnd = random.Random(seed)
    n = rnd.randint(1, 14)
    pairs = [(rnd.randrange(n), rnd.randrange(n)) for _ in range(rnd.randint(0, 2 * n))]
    g = gg.from_edges(n, pairs, symmetrize=seed % 2 == 0) if pairs else gg.empty(n)
    R, C, _ = g.numpy()
    comp, k = oracle.cc(R, C)
    ref = _closure_labels(n, R, C)
    assert np.array_equal(comp, ref)
    assert k == len(set(ref.tolist()))


@pytest.mark.parametrize("name", ["rmat", "er", "directed", "mesh"])
def test_scipy_partition(name):
    g = {"rmat": lambda: gg.rmat(12, 4, seed=2), "er": lambda: gg.erdos_renyi(5000, 2600, seed=4),
         "directed": lambda: gg.directed_random(4000, 3000, seed=5),
         "mesh": lambda: gg.make_config("c4_road", shrink=8)}[name]()
    R, C, _ = g.numpy()
    comp, k = oracle.cc(R, C)
    n = R.size - 1
    A = sp.csr_matrix((np.ones(C.size), C, R), shape=(n, n))
    k2, lab = connected_components(A, directed=True, connection="weak")
    assert k == k2
    # same partition: the min-id label and scipy's label determine each other
    pairs = set(zip(comp.tolist(), lab.tolist()))
    assert len(pairs) == k
    assert all(comp[v] <= v for v in range(n))
