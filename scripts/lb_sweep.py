"""Sweep of the auto strategy threshold T (reading A-4: thread/warp/CTA below
T, merge-path at or above): device time per traversal for each config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
Ts = [4096, 16384, 65536, 262144, 1 << 40]
jobs = [("c2_kron21", "bfs", "push"), ("c2_kron21", "bfs", "auto"), ("c3_orkut", "bfs", "auto"),
        ("c3_orkut", "sssp", None), ("c4_road", "bfs", "auto"), ("c4_road", "sssp", None),
        ("c5_kron25", "bfs", "auto")]
torch.cuda.set_device(0)
cache = {}
for cfg, prim, d in jobs:
    if cfg not in cache:
        cache.clear()
        torch.cuda.empty_cache()
        g = gg.make_config(cfg, device="cuda", weights=True if cfg in ("c3_orkut", "c4_road") else None)
        cache[cfg] = (g, gr.Graph(g.R, g.C, g.W, symmetric=True), gg.sources(g, 4))
    g, G, srcs = cache[cfg]
    srcs = srcs[:2] if cfg == "c4_road" else srcs
    out_d = torch.empty(g.n, dtype=torch.int32, device="cuda")
    out_p = torch.empty(g.n, dtype=torch.int32, device="cuda")
    env = "GR_LB_THRESHOLD" if prim == "bfs" else "GR_SSSP_LB_THRESHOLD"
    row = []
    for T in Ts:
        os.environ[env] = str(T)
        tot = 0.0
        for s in srcs:
            for rep in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                if prim == "bfs":
                    G.bfs(s, out_d, out_p, direction=d, asynchronous=True)
                else:
                    G.sssp(s, out_d, out_p, asynchronous=True)
                e1.record()
                G.sync()
                torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) * 1e3
        row.append(tot / len(srcs))
    os.environ.pop(env)
    print("%-10s %-4s %-5s " % (cfg, prim, d) + " ".join("T=%d: %.1f us" % (T if T < 1 << 40 else -1, t)
                                                     for T, t in zip(Ts, row)), flush=True)
