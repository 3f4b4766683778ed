"""Debug: which (src, delta) of test_random_graphs[4] overflows, with per-step stats."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
torch.cuda.set_device(0)
g = gg.assign_weights(gg.make_config("c3_orkut", shrink=4), seed=5)
G = gr.Graph(g.R.cuda(), g.C.cuda(), g.W.cuda(), symmetric=True)
srcs = gg.sources(g, 3, seed=4)
for s in srcs[:2]:
    for delta in [1, 8, 33, 64, 1024, 0xFFFFFFFF, 0]:
        try:
            G.sssp(s, delta=delta)
            print("ok", s, delta, flush=True)
        except gr.GrError as e:
            import ctypes
            gr._lib.gr_debug_overflow.restype = ctypes.c_ulonglong
            gr._lib.gr_debug_overflow.argtypes = [ctypes.c_void_p]
            ov = gr._lib.gr_debug_overflow(G.handle)
            print("FAIL", s, delta, e, "overflow word: tag %d count %d (n %d m %d)" % (ov & 255, ov >> 8, g.n, g.R[-1].item()), flush=True)
            st = G.run_stats()["levels"]
            for r in st[:80]:
                print("   ", r)
