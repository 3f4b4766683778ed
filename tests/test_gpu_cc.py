"""GPU parity of connected components (gr_cc)
against the union-find oracle: labels (smallest id per component, reading
A-22) and the component count are integers, compared bit-exactly."""
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


def _check(gr, g, symmetric=True, host=False):
    R, C, _ = g.numpy()
    G = gr.Graph(g.R.cuda(), g.C.cuda(), None, symmetric=symmetric)
    out = torch.empty(g.n, dtype=torch.int32, pin_memory=True) if host else None
    comp, k = G.cc(out)
    ref, kref = oracle.cc(R, C)
    c = comp.cpu().numpy() if not host else comp.numpy()
    bad = np.flatnonzero(c != ref)
    assert bad.size == 0, (bad[:5], c[bad[:5]], ref[bad[:5]])
    assert k == kref
    G.close()


def test_cc_small_closed_forms(gr):
    _check(gr, gg.from_edges(10, [(9, 5), (5, 0), (2, 1), (8, 7), (7, 6), (6, 4)]))
    _check(gr, gg.empty(100))
    _check(gr, gg.path(5000))          # long chain: many hooking rounds
    _check(gr, gg.grid(61, 67), host=True)


@pytest.mark.parametrize("scale", [12, 16])
def test_cc_rmat(gr, scale):
    _check(gr, gg.rmat(scale, 8, seed=scale))


def test_cc_kron_and_er(gr):
    _check(gr, gg.kronecker(18, 16, seed=1))
    _check(gr, gg.erdos_renyi(200000, 110000, seed=4))   # many small components


def test_cc_directed_weak(gr):
    _check(gr, gg.directed_random(50000, 40000, seed=5), symmetric=False)


def test_cc_mesh(gr):
    _check(gr, gg.make_config("c4_road", shrink=5))
    _check(gr, gg.mesh(300, p_vertical=0.02, seed=3))  # rows joined rarely: few, long components
