"""The seeded input generators (graphgen/) -- shapes, determinism, contracts."""
import numpy as np
import torch

import graphgen as gg
import oracle


def _py_mix32(x):
    M = (1 << 32) - 1
    x &= M
    x ^= x >> 16
    x = (x * 0x45D9F3B) & M
    x ^= x >> 16
    x = (x * 0x45D9F3B) & M
    x ^= x >> 16
    return x


def test_rand32_matches_python_ints():
    idx = torch.tensor([0, 1, 2, 12345, (1 << 31) + 7, (1 << 40) + 3], dtype=torch.int64)
    got = gg.rand32(7, 3, idx).tolist()
    s1 = _py_mix32(7 * 0x9E3779B1 + 3 * 0x85EBCA77 + 0x165667B1)
    s2 = _py_mix32(s1 ^ 0xC2B2AE3D ^ (3 << 7))
    for i, v in zip(idx.tolist(), got):
        h = _py_mix32((i & 0xFFFFFFFF) ^ s1)
        h = _py_mix32(h ^ (((i >> 32) + s2) & 0xFFFFFFFF))
        assert v == h


def _check_csr(g, symmetric=True):
    R, C, W = g.numpy()
    assert R[0] == 0 and R[-1] == C.size and np.all(np.diff(R) >= 0)
    assert C.size == 0 or (C.min() >= 0 and C.max() < g.n)
    src = np.repeat(np.arange(g.n), np.diff(R))
    assert not np.any(src == C), "self-loop"
    key = src.astype(np.int64) * g.n + C
    assert np.all(np.diff(key) > 0), "neighbour lists sorted and deduplicated"
    if symmetric:
        rkey = np.sort(C.astype(np.int64) * g.n + src)
        assert np.array_equal(rkey, key), "symmetric"
    if W is not None:
        assert W.min() >= 1 and W.max() <= 64
        if symmetric:
            order = np.argsort(C.astype(np.int64) * g.n + src)
            assert np.array_equal(W[order], W), "w(u,v) == w(v,u)"


def test_configs_small_shapes_and_determinism():
    for name in gg.CONFIGS:
        shrink = {"c1_rmat16": 4, "c2_kron21": 8, "c3_orkut": 4, "c4_road": 5, "c5_kron25": 12}[name]
        g1 = gg.make_config(name, shrink=shrink)
        g2 = gg.make_config(name, shrink=shrink)
        _check_csr(g1)
        assert torch.equal(g1.R, g2.R) and torch.equal(g1.C, g2.C)
        if g1.W is not None:
            assert torch.equal(g1.W, g2.W)


def test_rmat16_shape_matches_calibration():
    # R-MAT s16 ef16 unpermuted -> ~1.82M directed edges,
    # vertex 0 is the max-degree hub (~9.7K), ~28.7% isolated.
    g = gg.make_config("c1_rmat16")
    d = g.degrees()
    assert 1.75e6 < g.m < 1.9e6
    assert int(d[0]) == int(d.max()) and 9000 < int(d[0]) < 10500
    assert 0.25 < float((d == 0).float().mean()) < 0.32


def test_kronecker_dedup_ratio():
    g = gg.kronecker(16, 16, seed=1)
    assert 1.65 < g.m / (g.n * 16) < 1.85   # ratio 1.815 at s18, lower at s16
    assert int(g.degrees()[0]) < int(g.degrees().max())  # permuted: 0 is not the hub


def test_mesh_connected_and_degree():
    g = gg.mesh(60, seed=1)
    _check_csr(g)
    assert int(g.degrees().max()) <= 4
    R, C, _ = g.numpy()
    d, _ = oracle.bfs(R, C, 0, want_pred=False)
    assert (d >= 0).all()


def test_weights_symmetric_uniform():
    g = gg.assign_weights(gg.erdos_renyi(4000, 200000, seed=3), seed=2)
    _check_csr(g)
    W = g.W.numpy()
    counts = np.bincount(W, minlength=65)[1:]
    assert counts.min() > 0.8 * counts.mean()


def test_directed_random_is_not_symmetric():
    g = gg.directed_random(500, 3000, seed=1)
    _check_csr(g, symmetric=False)
    R, C, _ = g.numpy()
    src = np.repeat(np.arange(g.n), np.diff(R))
    assert not np.array_equal(np.sort(C.astype(np.int64) * g.n + src), src.astype(np.int64) * g.n + C)


def test_sources_have_degree():
    g = gg.make_config("c1_rmat16", shrink=4)
    s = gg.sources(g, 16)
    assert len(set(s)) == 16
    assert all(int(g.degrees()[v]) > 0 for v in s)
