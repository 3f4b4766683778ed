"""Pins for readings of the paper's SSSP step structure (A-7, A-11).

Alg. 1 relaxes with atomicMin (UpdateLabel), records a
per-vertex output-queue id (SetPred) and removes redundant vertices
with it (RemoveRedundant); the priority queue splits the output
into near and far slices. The passage is garbled (the array name
differs and every copy passes as written). This test simulates the
bulk-synchronous near/far loop in plain Python with a RANDOM interleaving of
the two atomic halves of concurrent relaxations and checks against Dijkstra
(scipy):

  * stamp key = iteration only        -> wrong distances on some instances
    (an improvement into the far slice blocks a later improvement into the
    near slice of the same iteration: the vertex is stranded in far, then
    dropped as stale);
  * stamp key = 2*iteration + slice   -> always exact (the build's reading).

This pins the reading used by sssp.cu independently of the CUDA code.
"""
import random

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse import csgraph

INF = float("inf")


def nearfar_sim(n, adj, src, delta, slice_key, rng):
    dist = [INF] * n
    dist[src] = 0
    stamp = [-1] * n
    near, far = [src], []
    thr = delta
    it = 0
    while near or far:
        while near:
            it += 1
            # all relaxations of this bulk-synchronous step, in random order,
            # each split in two halves (atomicMin ; stamp exchange) that other
            # relaxations may interleave with
            ops = [(u, v, w) for u in near for (v, w) in adj[u]]
            du = {u: dist[u] for u in near}  # sources read at step start
            pending = []
            for (u, v, w) in ops:
                pending.append(("min", u, v, du[u] + w))
            rng.shuffle(pending)
            nxt = []
            staged = []
            while pending or staged:
                if staged and (not pending or rng.random() < 0.5):
                    v, nd = staged.pop(rng.randrange(len(staged)))
                    far_slice = nd >= thr
                    key = 2 * it + (1 if far_slice else 0) if slice_key else it
                    if stamp[v] != key:
                        stamp[v] = key
                        (far if far_slice else nxt).append(v)
                    continue
                _, u, v, nd = pending.pop()
                old = dist[v]
                if nd < old:               # atomicMin succeeded
                    dist[v] = nd
                    staged.append((v, nd))  # the stamp half runs later
            near = nxt
        # far re-split (A-11): drop stale, jump the threshold, split
        live = [v for v in far if dist[v] >= thr]
        far = []
        if not live:
            break
        thr = (min(dist[v] for v in live) // delta + 1) * delta
        it += 1
        seen = set()
        for v in live:
            if v in seen:
                continue
            seen.add(v)
            (near if dist[v] < thr else far).append(v)
    return dist


def random_graph(rng, n):
    m = rng.randint(n, 4 * n)
    edges = {}
    for _ in range(m):
        a, b = rng.randrange(n), rng.randrange(n)
        if a != b:
            w = rng.randint(1, 64)
            edges[(a, b)] = min(w, edges.get((a, b), 99))
            edges[(b, a)] = edges[(a, b)]
    adj = [[] for _ in range(n)]
    for (a, b), w in edges.items():
        adj[a].append((b, w))
    return adj, edges


def dijkstra(n, edges, src):
    if not edges:
        d = np.full(n, np.inf)
        d[src] = 0
        return d
    r = [a for a, b in edges]
    c = [b for a, b in edges]
    w = [float(x) for x in edges.values()]
    A = sp.csr_matrix((w, (r, c)), shape=(n, n))
    return csgraph.dijkstra(A, directed=True, indices=src)


def _run(slice_key, trials=400, seed=0):
    rng = random.Random(seed)
    wrong = 0
    for t in range(trials):
        n = rng.randint(5, 30)
        adj, edges = random_graph(rng, n)
        src = rng.randrange(n)
        delta = rng.choice([1, 4, 8, 16, 33, 64])
        got = nearfar_sim(n, adj, src, delta, slice_key, rng)
        ref = dijkstra(n, edges, src)
        if any((g != r) for g, r in zip(got, ref)):
            wrong += 1
    return wrong


def test_slice_keyed_stamp_is_exact():
    assert _run(slice_key=True) == 0


def test_iteration_only_stamp_strands_vertices():
    # the garbled literal reading loses distances on a visible fraction
    assert _run(slice_key=False) > 0


@pytest.mark.parametrize("delta", [1, 7, 64, 10 ** 9])
def test_delta_changes_work_not_results(delta):
    """S:342 'delta only affects work, never results' under the slice key."""
    rng = random.Random(delta)
    for _ in range(60):
        n = rng.randint(5, 25)
        adj, edges = random_graph(rng, n)
        src = rng.randrange(n)
        got = nearfar_sim(n, adj, src, delta, True, rng)
        ref = dijkstra(n, edges, src)
        assert all(g == r for g, r in zip(got, ref))
