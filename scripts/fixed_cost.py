"""Fixed per-call device cost of a BFS (launch + init + termination), with the
bench's timing (device sleep, L2 flush, events around the async call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def dev_ms(G, src, n, reps=10):
    depth = torch.empty(n, dtype=torch.int32, device="cuda")
    pred = torch.empty(n, dtype=torch.int32, device="cuda")
    G.bfs(src, depth, pred)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda._sleep(int(2e6) * (reps + 2))
    for e0, e1 in ev:
        flush.zero_()
        e0.record()
        G.bfs(src, depth, pred, asynchronous=True)
        e1.record()
    G.sync()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2] * 1e3


g = gg.path(2)
G = gr.Graph(g.R.cuda(), g.C.cuda(), None, symmetric=True)
print("path(2) BFS: %.1f us per call (levels %d)" % (dev_ms(G, 0, 2), G.run_stats()["num_levels"]))
g = gg.make_config("c2_kron21", device="cuda")
G = gr.Graph(g.R, g.C, None, symmetric=True)
deg = (g.R[1:] - g.R[:-1]).cpu()
iso = int(torch.nonzero(deg == 0)[0])
print("c2 isolated source: %.1f us per call (levels %d)" % (dev_ms(G, iso, g.n), G.run_stats()["num_levels"]))
s = gg.sources(g, 1)[0]
print("c2 source %d: %.1f us per call" % (s, dev_ms(G, s, g.n)))
