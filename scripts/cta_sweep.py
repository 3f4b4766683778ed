"""Persistent-grid size sweep (GR_BFS_CTAS / GR_SSSP_CTAS): device time per
traversal on a high-diameter mesh (C4) and a scale-free graph (C2/C3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
torch.cuda.set_device(0)
for cfg, prims in [("c4_road", ["bfs", "sssp"]), ("c2_kron21", ["bfs"]), ("c3_orkut", ["sssp"])]:
    g = gg.make_config(cfg, device="cuda", weights=True if cfg != "c2_kron21" else None)
    G = gr.Graph(g.R, g.C, g.W, symmetric=True)
    s = gg.sources(g, 1)[0]
    d = torch.empty(g.n, dtype=torch.int32, device="cuda")
    p = torch.empty(g.n, dtype=torch.int32, device="cuda")
    for prim in prims:
        row = []
        for ctas in [0, 148, 74, 37, 16]:
            os.environ["GR_BFS_CTAS" if prim == "bfs" else "GR_SSSP_CTAS"] = str(ctas)
            best = 1e30
            for rep in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                if prim == "bfs":
                    G.bfs(s, d, p, asynchronous=True)
                else:
                    G.sssp(s, d, p, asynchronous=True)
                e1.record()
                G.sync()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            row.append("ctas=%s: %.3f ms" % (ctas or "all", best))
        os.environ.pop("GR_BFS_CTAS", None)
        os.environ.pop("GR_SSSP_CTAS", None)
        print(cfg, prim, " | ".join(row), flush=True)
    G.close()
    del g
    torch.cuda.empty_cache()
