"""Per-level time of one traversal bucketed by frontier size (run stats):
where a high-diameter traversal spends its time. Usage: level_hist.py [config] [bfs|sssp]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_road"
prim = sys.argv[2] if len(sys.argv) > 2 else "bfs"
torch.cuda.set_device(0)
g = gg.make_config(cfg, device="cuda", weights=(prim == "sssp") or None)
G = gr.Graph(g.R, g.C, g.W, symmetric=True)
s = gg.sources(g, 1)[0]
for rep in range(2):
    if prim == "bfs":
        G.bfs(s)
    else:
        G.sssp(s)
torch.cuda.synchronize()
st = G.run_stats()
rows = st["levels"]
print("%s %s src %d: %d levels, sum of level times %.2f ms, launches %d" % (
    cfg, prim, s, st["num_levels"], sum(r["ns"] for r in rows) / 1e6, gr.gr_kernel_launch_count()))
edges = [0, 1, 16, 128, 512, 1024, 2048, 4096, 8192, 16384, 1 << 40]
for lo, hi in zip(edges, edges[1:]):
    sel = [r for r in rows if lo <= r["frontier"] < hi]
    if not sel:
        continue
    ns = [r["ns"] for r in sel]
    print("  f in [%6d, %6d): %6d levels  total %8.2f ms  mean %6.2f us  dirs %s" % (
        lo, min(hi, 10 ** 9), len(sel), sum(ns) / 1e6, sum(ns) / len(ns) / 1e3, sorted(set(r["direction"] for r in sel))))
