"""Small traversals for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as gg, oracle
import paper_1501_05387_b200 as gr
torch.cuda.set_device(0)
for g in (gg.assign_weights(gg.rmat(9, 8, seed=1), seed=2), gg.assign_weights(gg.grid(20, 30), seed=3),
          gg.assign_weights(gg.directed_random(600, 3000, seed=4), seed=5)):
    G = gr.Graph(g.R.cuda(), g.C.cuda(), g.W.cuda(), symmetric=g.symmetric)
    R, C, W = g.numpy()
    for s in gg.sources(g, 2):
        for d in ("push", "pull", "auto"):
            for strat in ("auto", "twc", "lb"):
                depth, pred = G.bfs(s, direction=d, strategy=strat)
                assert np.array_equal(depth.cpu().numpy(), oracle.bfs(R, C, s)[0])
        dist, _ = G.sssp(s)
        assert np.array_equal(gr.dist_to_u32(dist), oracle.sssp(R, C, W, s)[0])
    # the paper's other primitives (BC, CC, PageRank)
    srcs = gg.sources(g, 2)
    bc = G.bc(srcs).cpu().numpy()
    assert np.allclose(bc, oracle.bc(R, C, srcs), rtol=1e-9, atol=1e-12)
    comp, k = G.cc()
    assert np.array_equal(comp.cpu().numpy(), oracle.cc(R, C)[0])
    x, _ = G.pagerank(0.85, 1e-12, 10000)
    assert np.allclose(x.cpu().numpy(), oracle.pagerank(R, C), rtol=1e-9, atol=0)
    G.close()
# partitioned BFS and SSSP (loopback group of 3 ranks, one launch: pbfs.cu / psssp.cu)
from paper_1501_05387_b200 import multigpu as mg
g = gg.assign_weights(gg.rmat(9, 8, seed=1), seed=2)
R, C, W = g.numpy()
comms = mg.Comm.loopback(3)
parts = []
for r in range(3):
    v0, v1, Rl, Cl, Wl = mg.partition_csr(g.R, g.C, 3, r, W=g.W)
    parts.append(mg.PartitionedGraph(comms[r], Rl.cuda(), Cl.cuda(), g.n, W_local=Wl.cuda()))
for s in gg.sources(g, 2):
    outs = [p.bfs(s) for p in parts]
    assert np.array_equal(torch.cat([o[0] for o in outs]).cpu().numpy(), oracle.bfs(R, C, s)[0])
    outs = [p.sssp(s, delta=8) for p in parts]
    assert np.array_equal(torch.cat([o[0] for o in outs]).cpu().numpy().view(np.uint32), oracle.sssp(R, C, W, s)[0])
for p in parts:
    p.close()
for c in comms:
    c.close()
print("sanitize workload ok")
