"""Per-level profile of one traversal (device %globaltimer per step)."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
import paper_1501_05387_b200 as gr

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_kron21")
ap.add_argument("--prim", default="bfs")
ap.add_argument("--directions", default="auto,push")
ap.add_argument("--nsrc", type=int, default=2)
ap.add_argument("--delta", type=int, default=0)
ap.add_argument("--maxrows", type=int, default=40)
ap.add_argument("--idempotent", type=int, default=0)
a = ap.parse_args()
torch.cuda.set_device(0)
g = gg.make_config(a.config, device="cuda", weights=(a.prim == "sssp") or None)
SRCS = gg.sources(g, a.nsrc)
if os.environ.get("NBRSORT"):  # experiment: each list ordered by neighbour degree, descending
    deg = g.R[1:] - g.R[:-1]
    src_e = torch.repeat_interleave(torch.arange(g.n, device="cuda"), deg)
    key = src_e * (int(deg.max()) + 1) + (int(deg.max()) - deg[g.C.long()])
    order = torch.argsort(key, stable=True)
    g = gg.Graph(g.n, g.R, g.C[order].contiguous(), None if g.W is None else g.W[order].contiguous(), True, g.meta)
    print("neighbour lists sorted by degree")
if os.environ.get("RELABEL"):  # experiment: degree-descending vertex order
    deg = g.R[1:] - g.R[:-1]
    new2old = torch.argsort(-deg * g.n - torch.arange(g.n, device="cuda"), stable=True)
    new2old = torch.sort(-deg, stable=True).indices
    old2new = torch.empty_like(new2old)
    old2new[new2old] = torch.arange(g.n, device="cuda")
    src_e = torch.repeat_interleave(torch.arange(g.n, device="cuda"), deg)
    key = old2new[src_e] * g.n + old2new[g.C.long()]
    order = torch.argsort(key)
    key = key[order]
    C2 = (key % g.n).to(torch.int32)
    R2 = torch.zeros(g.n + 1, dtype=torch.int64, device="cuda")
    R2[1:] = torch.cumsum(deg[new2old], 0)
    W2 = None if g.W is None else g.W[order]
    g = gg.Graph(g.n, R2, C2, W2, True, g.meta)
    SRCS = [int(old2new[s]) for s in SRCS]
    print("relabelled by degree")
G = gr.Graph(g.R, g.C, g.W, symmetric=True)
for s in SRCS:
    for d in a.directions.split(","):
        for rep in range(3):
            if a.prim == "bfs":
                G.bfs(s, direction=d, idempotent=bool(a.idempotent))
            else:
                G.sssp(s, delta=a.delta, direction=os.environ.get("SSSP_DIR", "auto"))
        torch.cuda.synchronize()
        st = G.run_stats()
        tot = sum(r["ns"] for r in st["levels"])
        print("src %d %s %s: levels %d total %.1f us delta %d" % (s, a.prim, d, st["num_levels"], tot / 1e3, st["delta"]))
        rows = st["levels"]
        if len(rows) > a.maxrows:
            rows = rows[: a.maxrows // 2] + rows[-a.maxrows // 2:]
        for r in rows:
            print("  L%-5d dir %d f %9d mf %11d disc %9d insp %11d aux %10d  %8.1f us" % (
                r["level"], r["direction"], r["frontier"], r["frontier_edges"], r["discovered"],
                r["inspected_edges"], r["aux"], r["ns"] / 1e3))
        if a.prim == "sssp":
            break
# summary by frontier-size bucket (last run)
import collections
b = collections.defaultdict(lambda: [0, 0.0])
for r in st["levels"]:
    k = (r["direction"], 1 << max(0, int(r["frontier"]).bit_length() - 1))
    b[k][0] += 1
    b[k][1] += r["ns"] / 1e3
print("dir  f>=      levels   total_us   us/level")
for k in sorted(b):
    print("%d %9d %8d %10.1f %8.2f" % (k[0], k[1], b[k][0], b[k][1], b[k][1] / b[k][0]))
