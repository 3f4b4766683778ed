"""GPU parity of betweenness centrality (gr_bc)
against the Brandes oracle, element by element, fp64 with relative
tolerance 1e-9: the GPU sums sigma and delta contributions in a
different order (atomics, warp reductions), so results agree to rounding,
not bit for bit. Graphs span several merge-path tiles and ragged tails;
edge cases: isolated / degree-0 sources, directed graphs, repeated sources.
"""
import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu
RTOL = 1e-9


@pytest.fixture(scope="module")
def gr():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    import paper_1501_05387_b200 as gr
    return gr


def _check(gr, g, srcs, symmetric=True, host=False, direction="auto"):
    R, C, _ = g.numpy()
    G = gr.Graph(g.R.cuda(), g.C.cuda(), None, symmetric=symmetric)
    if host:
        out = torch.empty(g.n, dtype=torch.float64, pin_memory=True)
        sig = np.empty(g.n, np.float64)
        G.bc(srcs, bc=out, sigma=sig, direction=direction)
        bc = out.numpy()
    else:
        sig_t = torch.empty(g.n, dtype=torch.float64, device="cuda")
        bc = G.bc(srcs, sigma=sig_t, direction=direction).cpu().numpy()
        sig = sig_t.cpu().numpy()
    ref = oracle.bc(R, C, srcs)
    scale = max(1.0, float(np.abs(ref).max()))
    err = np.abs(bc - ref) / np.maximum(np.abs(ref), 1e-300)
    bad = np.flatnonzero((err > RTOL) & (np.abs(bc - ref) > RTOL * scale * 1e-6))
    assert bad.size == 0, (bad[:5], bc[bad[:5]], ref[bad[:5]])
    # sigma of the last source: integral path counts, reached exactly where BFS reaches
    d, _ = oracle.bfs(R, C, srcs[-1])
    assert np.array_equal(sig > 0, d >= 0)
    assert np.allclose(sig, np.round(sig))
    G.close()
    return bc


def test_bc_closed_forms(gr):
    n = 40
    bc = _check(gr, gg.path(n), list(range(n)))
    i = np.arange(n)
    assert np.allclose(bc / 2, i * (n - 1 - i))
    bc = _check(gr, gg.star(50), list(range(51)))
    assert bc[0] / 2 == pytest.approx(50 * 49 / 2)


def test_bc_rmat(gr):
    g = gg.rmat(14, 16, seed=5)
    _check(gr, g, [0] + gg.sources(g, 6))


def test_bc_kron_scale18(gr):
    g = gg.kronecker(18, 16, seed=1)
    _check(gr, g, gg.sources(g, 3))


def test_bc_directed(gr):
    g = gg.directed_random(30000, 200000, seed=3)
    _check(gr, g, gg.sources(g, 4), symmetric=False)


def test_bc_mesh_and_grid(gr):
    _check(gr, gg.grid(37, 41), [0, 700, 1516])
    m = gg.make_config("c4_road", shrink=7)
    _check(gr, m, gg.sources(m, 1))


def test_bc_edge_cases(gr):
    g = gg.from_edges(70, [(0, 1), (1, 2), (2, 3), (3, 40), (40, 65), (65, 66), (10, 33), (2, 33)])
    _check(gr, g, [69, 0, 0, 40, 5], host=True)  # isolated first, repeated source
    e = gg.empty(10)
    R, C, _ = e.numpy()
    G = gr.Graph(e.R.cuda(), e.C.cuda(), None, symmetric=True)
    assert float(G.bc([3, 4]).abs().sum()) == 0.0
    assert float(G.bc([]).abs().sum()) == 0.0
    with pytest.raises(gr.GrError):
        G.bc([10])
    G.close()


@pytest.mark.parametrize("direction", ["push", "pull", "auto"])
def test_bc_pull_direction(gr, direction):
    """Pull (bottom-up) forward levels (P:832-834 names BC as a next user of
    pull; reading A-24): every level pulled, every level pushed, and the
    auto rule give the oracle's values on skewed, directed, mesh and
    multi-component graphs (hub in-lists > 32 edges take the warp path)."""
    for g, sym in ((gg.kronecker(13, 16, seed=3), True), (gg.rmat(12, 8, seed=4), True),
                   (gg.directed_random(3000, 20000, seed=5), False), (gg.grid(30, 40), True),
                   (gg.from_edges(50, [(i, i + 1) for i in range(20)] + [(30, 31), (31, 32)]), True)):
        srcs = gg.sources(g, 3)
        _check(gr, g, srcs, symmetric=sym, direction=direction)


def test_bc_pull_stats(gr):
    """The auto rule pulls the dense middle level of a Kronecker graph and
    reports each level's direction (gr_get_run_stats after gr_bc)."""
    g = gg.kronecker(15, 16, seed=6)
    G = gr.Graph(g.R.cuda(), g.C.cuda(), None, symmetric=True)
    s = gg.sources(g, 1)[0]
    G.bc([s], direction="auto")
    st = G.run_stats()
    dirs = [r["direction"] for r in st["levels"]]
    assert dirs[0] == 1 and 2 in dirs
    R, C, _ = g.numpy()
    d, _ = oracle.bfs(R, C, s)
    assert [r["frontier"] for r in st["levels"]] == [int((d == L).sum()) for L in range(len(dirs))]
