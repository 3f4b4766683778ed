"""Per-level internal timeline of block 0 / thread 0 (GR_TRACE build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_road"
shrink = int(sys.argv[2]) if len(sys.argv) > 2 else 2
gr.load(os.path.join(os.path.dirname(gr.LIB_PATH), "libgr_b200_trace.so"))
torch.cuda.set_device(0)
tr = torch.zeros(256 * 16, dtype=torch.int64, device="cuda")
gr._lib.gr_debug_trace_set.argtypes = [ctypes.c_void_p]
g = gg.make_config(cfg, device="cuda", shrink=shrink)
G = gr.Graph(g.R, g.C, None, symmetric=True)
s = gg.sources(g, 1)[0]
G.bfs(s)
assert gr._lib.gr_debug_trace_set(tr.data_ptr()) == 0
G.bfs(s)
torch.cuda.synchronize()
t = tr.view(256, 16).cpu().numpy()
st = G.run_stats()["levels"]
for L in [x for x in list(range(0, 12)) + list(range(100, 106)) if x + 1 < len(st)]:
    row = t[L]
    base = row[0]
    if base == 0:
        continue
    d = ["%6.2f" % ((x - base) / 1e3) if x else "   -  " for x in row[:10]]
    print("L%-4d f=%-6d %s   next-start %+.2f" % (L, st[L]["frontier"], " ".join(d), (t[L + 1][0] - base) / 1e3))
