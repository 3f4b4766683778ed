"""Run a few traversals of one config (for ncu captures)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4_road")
ap.add_argument("--shrink", type=int, default=0)
ap.add_argument("--prim", default="bfs")
ap.add_argument("--direction", default="auto")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--delta", type=int, default=0)
a = ap.parse_args()
torch.cuda.set_device(0)
g = gg.make_config(a.config, device="cuda", shrink=a.shrink, weights=(a.prim == "sssp") or None)
G = gr.Graph(g.R, g.C, g.W, symmetric=True)
s = gg.sources(g, 1)[0]
for _ in range(a.reps):
    if a.prim == "bfs":
        G.bfs(s, direction=a.direction)
    else:
        G.sssp(s, delta=a.delta)
torch.cuda.synchronize()
print(G.run_stats()["num_levels"])
