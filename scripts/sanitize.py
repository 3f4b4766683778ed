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
# partitioned BFS and SSSP (loopback, 3 partitions)
from paper_1501_05387_b200 import dist as grd
g = gg.assign_weights(gg.rmat(9, 8, seed=1), seed=2)
R, C, W = g.numpy()
parts = []
for r in range(3):
    v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, 3, r)
    parts.append(grd.GpuPartition(Rl.cuda(), Cl.cuda(), g.n, 3, r, W_local=grd.partition_weights(g.R, g.W, 3, r).cuda()))
grp = grd.LoopbackGroup(parts)
for s in gg.sources(g, 2):
    depths = [torch.empty(p.n_local, dtype=torch.int32, device="cuda") for p in parts]
    preds = [torch.empty(p.n_local, dtype=torch.int32, device="cuda") for p in parts]
    grp.bfs(s, depths, preds)
    assert np.array_equal(torch.cat(depths).cpu().numpy(), oracle.bfs(R, C, s)[0])
    grp.sssp(s, depths, preds, delta=8)
    assert np.array_equal(torch.cat(depths).cpu().numpy().view(np.uint32), oracle.sssp(R, C, W, s)[0])
for p in parts:
    p.close()
print("sanitize workload ok")
