"""Per-level times of push-only BFS under strategy / env variants (experiment)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_kron21"
torch.cuda.set_device(0)
g = gg.make_config(cfg, device="cuda")
G = gr.Graph(g.R, g.C, None, symmetric=True)
srcs = gg.sources(g, 3)
variants = [("default", {}, "auto"), ("lb", {}, "lb"), ("twc", {}, "twc"),
            ("probe-always", {"GR_PROBE_SKIP_PCT": "101"}, "auto"),
            ("probe-never", {"GR_PROBE_SKIP_PCT": "0"}, "auto"),
            ("chunks8", {"GR_LB_CHUNKS": "8"}, "auto"), ("static", {"GR_LB_CHUNKS": "0"}, "auto"),
            ("idem", {}, "auto")]
for s in srcs:
    for name, env, strat in variants:
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        for _ in range(3):
            G.bfs(s, direction="push", strategy=strat, idempotent=(name == "idem"))
        torch.cuda.synchronize()
        st = G.run_stats()
        for k, v in old.items():
            if v is None: os.environ.pop(k)
            else: os.environ[k] = v
        lv = st["levels"]
        print("src %8d %-13s total %7.1f us | " % (s, name, sum(r["ns"] for r in lv) / 1e3) +
              " ".join("L%d f=%d mf=%d %.1f" % (r["level"], r["frontier"], r["frontier_edges"], r["ns"] / 1e3)
                       for r in lv if r["ns"] > 20e3))
