"""Pull-direction SSSP near iterations (the paper names
SSSP as a next user of pull; reading A-24): every vertex takes
the minimum over its in-edges from the near frontier, read from the weighted
transpose (u << 7 | w(u,v)). Element-by-element parity of dist with the
oracle's Dijkstra (bit-exact: integer weights), the certificate on pred, for
push-only, pull-only and the auto rule, on symmetric and directed graphs,
with symmetric and ASYMMETRIC weights (the transpose must carry w(u,v), not
w(v,u)), zero weights, and every delta regime."""
import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    import paper_1501_05387_b200 as gr
    return gr


def _graphs():
    a = gg.assign_weights(gg.rmat(13, 16, seed=2), seed=3)
    b = gg.assign_weights(gg.directed_random(20000, 150000, seed=4), seed=5)
    c = gg.rmat(12, 8, seed=6)  # symmetric structure, asymmetric weights in 0..127
    c.W = torch.randint(0, 128, (c.C.numel(),), generator=torch.Generator().manual_seed(7), dtype=torch.int32)
    d = gg.assign_weights(gg.make_config("c4_road", shrink=6), seed=8)
    return [a, b, c, d]


@pytest.mark.parametrize("direction", ["push", "pull", "auto"])
def test_sssp_pull_parity(gr, direction):
    for g in _graphs():
        R, C, W = g.numpy()
        G = gr.Graph(g.R.cuda(), g.C.cuda(), g.W.cuda(), symmetric=g.symmetric)
        assert G.info().packed_weights == 1
        for s in gg.sources(g, 2):
            ref, _ = oracle.sssp(R, C, W, s)
            for delta in (0, 1, 33, 0xFFFFFFFF):
                dist, pred = G.sssp(s, delta=delta, direction=direction)
                got = gr.dist_to_u32(dist)
                assert np.array_equal(got, ref), (direction, s, delta, int((got != ref).sum()))
                assert oracle.check_sssp(R, C, W, s, got, pred.cpu().numpy()) == [], (direction, s, delta)
        G.close()


def test_sssp_pull_is_used(gr):
    """Forced pull records pull steps (direction 5 in the per-level stats);
    the unpacked layout (weights > 127) falls back to push and stays exact."""
    g = gg.assign_weights(gg.rmat(12, 16, seed=9), seed=1)
    R, C, W = g.numpy()
    G = gr.Graph(g.R.cuda(), g.C.cuda(), g.W.cuda(), symmetric=True)
    s = gg.sources(g, 1)[0]
    G.sssp(s, direction="pull")
    assert 5 in [r["direction"] for r in G.run_stats()["levels"]]
    G.close()
    g.W = g.W * 1000  # too wide to pack
    R, C, W = g.numpy()
    G = gr.Graph(g.R.cuda(), g.C.cuda(), g.W.cuda(), symmetric=True)
    assert G.info().packed_weights == 0
    dist, pred = G.sssp(s, direction="pull")
    assert np.array_equal(gr.dist_to_u32(dist), oracle.sssp(R, C, W, s)[0])
    assert 5 not in [r["direction"] for r in G.run_stats()["levels"]]
    G.close()
