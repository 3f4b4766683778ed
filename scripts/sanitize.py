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
    G.close()
print("sanitize workload ok")
