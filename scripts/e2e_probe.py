"""Per-call breakdown of the end-to-end (host-output) C-ABI call: where does
the time between the device-timed traversal and the host wall clock go?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_kron21"
direction = sys.argv[2] if len(sys.argv) > 2 else "auto"
torch.cuda.set_device(0)
g = gg.make_config(cfg, device="cuda")
G = gr.Graph(g.R, g.C, None, symmetric=True)
n = g.n
srcs = gg.sources(g, 12)
pin_d = torch.empty(n, dtype=torch.int32, pin_memory=True)
pin_p = torch.empty(n, dtype=torch.int32, pin_memory=True)
dd = torch.empty(n, dtype=torch.int32, device="cuda")
dp = torch.empty(n, dtype=torch.int32, device="cuda")
for s in srcs[:3]:
    G.bfs(s, pin_d, pin_p, direction=direction)
    G.bfs(s, dd, dp, direction=direction)
torch.cuda.synchronize()
for s in srcs:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.bfs(s, dd, dp, direction=direction)
    t1 = time.perf_counter()
    G.bfs(s, pin_d, pin_p, direction=direction)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    pin_d.copy_(dd, non_blocking=True); pin_p.copy_(dp, non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print("src %8d levels %2d  dev-out call %.3f ms  host-out call %.3f ms  torch d2h 2x%.1fMB %.3f ms"
          % (s, G.run_stats()["num_levels"], (t1 - t0) * 1e3, (t2 - t1) * 1e3, n * 4 / 1e6, (t4 - t3) * 1e3))
