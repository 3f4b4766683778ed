"""ablation of the hot path's variants on B200, the analog of
the paper's Fig. exp_optimization and its DO speedup claim
(1.52x scale-free, 1.28x small-degree large-diameter):

  BFS   load balancing: merge-path over edges (lb) vs thread/warp/CTA (twc) vs
        auto; idempotent discovery on/off; direction: push only vs
        direction-optimizing (Beamer rule) vs the paper's literal rule
        "unvisited < frontier" (switch_rule=1)
  BC    forward levels push only vs pull only vs auto (reading A-24)
  SSSP  near iterations push only vs pull only vs auto (A-24)

Times are device times of the whole traversal (CUDA events), mean over the
sources, with L2 flushed (a 256 MiB write) before every timed run, as in
bench.py. Writes markdown tables to stdout and JSON to --out.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import graphgen as gg
import paper_1501_05387_b200 as gr

BFS_VARIANTS = [
    ("push lb", dict(direction="push", strategy="lb")),
    ("push twc", dict(direction="push", strategy="twc")),
    ("push auto", dict(direction="push", strategy="auto")),
    ("push auto idempotent", dict(direction="push", strategy="auto", idempotent=True)),
    ("DO Beamer", dict(direction="auto", strategy="auto")),
    ("DO paper-literal", dict(direction="auto", strategy="auto", switch_rule=1)),
    ("DO Beamer idempotent", dict(direction="auto", strategy="auto", idempotent=True)),
]
DIRS = [("push", "push"), ("pull", "pull"), ("auto", "auto")]

_flush = None


def timed(fn):
    global _flush
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def run_bfs(cfg, nsrc, reps):
    g = gg.make_config(cfg, device="cuda", weights=False)
    G = gr.Graph(g.R, g.C, None, symmetric=True)
    srcs = gg.sources(g, nsrc)
    rows = []
    for name, kw in BFS_VARIANTS:
        ms, edges, insp, levels = 0.0, 0, 0, 0
        for s in srcs:
            G.bfs(s, **kw)  # warm
            for _ in range(reps):
                ms += timed(lambda: G.bfs(s, **kw))
                st = G.run_stats()
                insp += sum(r["inspected_edges"] for r in st["levels"])
                levels += st["num_levels"]
                edges += st["reached_edges"]
        k = len(srcs) * reps
        rows.append(dict(variant=name, ms=ms / k, gteps=edges / (ms * 1e-3) / 1e9,
                         inspected_edges=insp / k, levels=levels / k))
    G.close()
    return dict(config=cfg, prim="bfs", n=g.n, m=g.m, rows=rows)


def run_dir(cfg, prim, nsrc, reps):
    g = gg.make_config(cfg, device="cuda", weights=True if prim == "sssp" else None)
    G = gr.Graph(g.R, g.C, g.W if prim == "sssp" else None, symmetric=True)
    srcs = gg.sources(g, nsrc)
    rows = []
    for name, d in DIRS:
        ms, edges, npull, steps = 0.0, 0, 0, 0
        for s in srcs:
            def one():
                if prim == "sssp":
                    G.sssp(s, direction=d)
                else:
                    G.bc([s], direction=d)
            one()
            for _ in range(reps):
                ms += timed(one)
                st = G.run_stats()
                npull += sum(1 for r in st["levels"] if r["direction"] in (2, 5))
                steps += st["num_levels"]
                if prim == "sssp":
                    edges += st["reached_edges"]
                else:
                    G.bfs(s)
                    edges += 2 * G.run_stats()["reached_edges"]  # BC TEPS = 2 m_reached / t
        k = len(srcs) * reps
        rows.append(dict(variant="%s %s" % (prim, name), ms=ms / k, gteps=edges / (ms * 1e-3) / 1e9,
                         pull_steps=npull / k, steps=steps / k))
    G.close()
    return dict(config=cfg, prim=prim, n=g.n, m=g.m, rows=rows)


def run_ell(cfg, nsrc):
    """Bounded-degree graphs: CSR-only grid kernel vs the
    ELL records on the grid kernel vs ELL + the one-cluster narrow levels."""
    g = gg.make_config(cfg, device="cuda", weights=True)
    srcs = gg.sources(g, nsrc)
    rows = []
    for name, ell, cl in (("CSR, grid kernel", "0", "0"), ("ELL records, grid kernel", "1", "0"),
                          ("ELL records, cluster mode", "1", "1")):
        os.environ["GR_ELL"] = ell
        os.environ["GR_ELL_CLUSTER"] = cl
        G = gr.Graph(g.R, g.C, g.W, symmetric=True)
        for prim in ("bfs", "sssp"):
            ms, edges, steps = 0.0, 0, 0
            for s in srcs:
                one = (lambda: G.bfs(s)) if prim == "bfs" else (lambda: G.sssp(s))
                one()
                ms += timed(one)
                st = G.run_stats()
                steps += st["num_levels"]
                edges += st["reached_edges"]
            k = len(srcs)
            rows.append(dict(variant="%s %s" % (prim, name), ms=ms / k, gteps=edges / (ms * 1e-3) / 1e9,
                             steps=steps / k, us_per_step=ms * 1e3 / steps))
        G.close()
    os.environ.pop("GR_ELL", None)
    os.environ.pop("GR_ELL_CLUSTER", None)
    return dict(config=cfg, prim="ell", n=g.n, m=g.m, rows=rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2_kron21,c3_orkut,c4_road")
    ap.add_argument("--nsrc", type=int, default=4)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    res = []
    for cfg in a.configs.split(","):
        nsrc = 2 if cfg == "c4_road" else a.nsrc
        reps = 1 if cfg == "c4_road" else a.reps
        r = run_bfs(cfg, nsrc, reps)
        res.append(r)
        print("\n### %s BFS (n=%d, m=%d)\n" % (cfg, r["n"], r["m"]))
        print("| variant | ms / BFS | GTEPS | edges inspected / BFS | levels |")
        print("|---|---|---|---|---|")
        for row in r["rows"]:
            print("| %s | %.3f | %.1f | %.3g | %.1f |" % (row["variant"], row["ms"], row["gteps"],
                                                         row["inspected_edges"], row["levels"]))
        by = {row["variant"]: row for row in r["rows"]}
        print("\nDO speedup over push-only (auto strategy): %.2fx (Beamer), %.2fx (paper-literal)"
              % (by["push auto"]["ms"] / by["DO Beamer"]["ms"], by["push auto"]["ms"] / by["DO paper-literal"]["ms"]))
        prims = ["bc"] if cfg != "c4_road" else []
        if cfg in ("c3_orkut", "c4_road"):
            prims.append("sssp")
        for prim in prims:
            r = run_dir(cfg, prim, 2 if prim == "bc" or cfg == "c4_road" else nsrc, 1)
            res.append(r)
            print("\n### %s %s (direction of the frontier steps)\n" % (cfg, prim.upper()))
            print("| variant | ms | GTEPS | pull steps | steps |")
            print("|---|---|---|---|---|")
            for row in r["rows"]:
                print("| %s | %.3f | %.1f | %.1f | %.1f |" % (row["variant"], row["ms"], row["gteps"],
                                                           row["pull_steps"], row["steps"]))
        if cfg == "c4_road":
            r = run_ell(cfg, 2)
            res.append(r)
            print("\n### %s bounded-degree paths (records, cluster mode)\n" % cfg)
            print("| variant | ms | GTEPS | steps | us / step |")
            print("|---|---|---|---|---|")
            for row in r["rows"]:
                print("| %s | %.2f | %.3f | %.0f | %.2f |" % (row["variant"], row["ms"], row["gteps"], row["steps"],
                                                          row["us_per_step"]))
        sys.stdout.flush()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
