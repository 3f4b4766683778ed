"""Per-level internal timeline of block 0 / thread 0 on a high-diameter graph
(GR_TRACE build; stamps of bfs.cu / frontier.cuh): which part of a level's
dependent chain the time goes to. Usage: trace_c4.py [config] [shrink] [L0]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_road"
shrink = int(sys.argv[2]) if len(sys.argv) > 2 else 0
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
print("info bounded_degree=%d  levels=%d" % (G.info().bounded_degree, len(st)))
print("stamps relative to level start (us): 0 start, 1 list loaded, 2 claims back, 4 slots done, "
      "5 expand done, 6 flush done, 7 pre-barrier, 8 post-barrier, 9 small-mode pre-expand")
rows = []
for L in range(0, 255):
    row = t[L]
    base = row[0]
    if base == 0 or t[L + 1][0] == 0:
        continue
    d = ["%6.2f" % ((x - base) / 1e3) if x else "   -  " for x in row[:10]]
    rows.append((L, st[L]["frontier"], st[L]["direction"], (t[L + 1][0] - base) / 1e3, d))
for L, f, dr, nxt, d in rows[:8] + rows[-40:]:
    print("L%-4d dir %d f=%-6d %s   next-start %+.2f" % (L, dr, f, " ".join(d), nxt))
