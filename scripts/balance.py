"""Per-level load balance of the grid levels (GR_TRACE build): for every CTA,
when its first and its last warp finished the step's work, relative to the
step start (block 0). Usage: python scripts/balance.py [config] [direction]."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_kron21"
direction = sys.argv[2] if len(sys.argv) > 2 else "push"
gr.load(os.path.join(os.path.dirname(gr.LIB_PATH), "libgr_b200_trace.so"))
torch.cuda.set_device(0)
tr = torch.zeros(256 * 16, dtype=torch.int64, device="cuda")
bal = torch.zeros(64 * 1024 * 2, dtype=torch.int64, device="cuda")
for f in ("gr_debug_trace_set", "gr_debug_balance_set"):
    getattr(gr._lib, f).argtypes = [ctypes.c_void_p]
g = gg.make_config(cfg, device="cuda")
G = gr.Graph(g.R, g.C, None, symmetric=True)
for s in gg.sources(g, 2):
    G.bfs(s, direction=direction)
    assert gr._lib.gr_debug_trace_set(tr.data_ptr()) == 0
    assert gr._lib.gr_debug_balance_set(bal.data_ptr()) == 0
    tr.zero_(); bal.zero_()
    G.bfs(s, direction=direction)
    torch.cuda.synchronize()
    t = tr.view(256, 16).cpu().numpy()
    st = G.run_stats()["levels"]
    nb = torch.cuda.get_device_properties(0).multi_processor_count * int(os.environ.get("GR_CTAS_PER_SM", "2"))
    b = bal[: 64 * nb * 2].view(64, nb, 2).cpu().numpy()
    print("src %d %s, %d CTAs" % (s, direction, nb))
    for L in range(min(len(st), 64)):
        row = b[L, :nb]
        if row[:, 1].min() == 0 or t[L][0] == 0:
            continue
        t0 = t[L][0]
        last = (row[:, 1] - t0) / 1e3
        first = (row[:, 0] - t0) / 1e3
        print("  L%-3d dir %d mf %11d  level %7.1f us | CTA last-warp done: min %7.1f med %7.1f max %7.1f | "
              "in-CTA spread mean %6.1f us" % (L, st[L]["direction"], st[L]["frontier_edges"], st[L]["ns"] / 1e3,
                                               last.min(), np.median(last), last.max(), (last - first).mean()))
