#!/usr/bin/env python
"""Benchmark: BFS GTEPS on the BASELINE.json configs (default: config 2,
direction-optimizing push-pull BFS on a kron_g500-logn21-shaped Kronecker
graph), plus the roofline of the dominant kernel, a CPU-oracle baseline and an
end-to-end number through the C ABI with host output buffers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_kron21]
                    [--prim bfs|sssp] [--direction auto|push|pull]
                    [--impl ours|reference] [--no-cpu-baseline]

One "step" = one full traversal (every level of the hot path)
from one seeded source, inputs resident in HBM. K steps cycle through K
seeded sources (degree >= 1). L2 is flushed (a 256 MiB write) between
timed steps, outside each step's CUDA-event bracket.
Multi-GPU (torchrun, N>1): sources are independent problems, sharded across
ranks (weak scaling; each rank owns the whole graph), no collective on the
data path; value = edges traversed by all ranks / max-over-ranks time.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# the image sets NCCL_DEBUG=VERSION, which prints a banner on STDOUT and breaks
# the one-JSON-line contract; keep NCCL to warnings (on stderr) unless asked
os.environ["NCCL_DEBUG"] = os.environ.get("GR_NCCL_DEBUG", "WARN")
# Anything native libraries print on fd 1 goes to stderr; the JSON line is
# written to a saved duplicate of the real stdout.
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(obj):
    os.write(_JSON_FD, (json.dumps(obj) + "\n").encode())
sys.path.insert(0, ROOT)

METRIC = "BFS/SSSP GTEPS at 1/2/4/8 B200; achieved HBM GB/s as fraction of roofline"
CONFIG_DESC = {
    "c1_rmat16": "R-MAT scale 16, edge factor 16, unpermuted, BFS from vertex 0",
    "c2_kron21": "Kronecker (Graph500 A,B,C=.57,.19,.19) scale 21, edge factor 48, permuted, "
                 "symmetrised (kron_g500-logn21 shape)",
    "c3_orkut": "Chung-Lu n=3,072,441, ~234M directed edges, weights U{1..64} (soc-orkut shape)",
    "c4_road": "row-connected mesh 4899^2, p_vertical=0.2, weights U{1..64} (road_usa shape)",
    "c5_kron25": "Graph500 Kronecker scale 25, edge factor 16, permuted, symmetrised",
}
PAPER_CONTEXT = {  # Table 3, K40c, real datasets: context only
    ("c2_kron21", "bfs"): "Gunrock BFS kron_g500-logn21 on K40c: 19.15 ms, 9.51 GTEPS (P:1146-1147)",
    ("c3_orkut", "bfs"): "Gunrock BFS soc-orkut on K40c: 47.23 ms, 4.50 GTEPS (P:1140-1141)",
    ("c3_orkut", "sssp"): "Gunrock SSSP soc-orkut on K40c: 1088 ms, 0.1955 GTEPS (P:1152-1153)",
    ("c4_road", "bfs"): "Gunrock BFS roadnet_CA (11x fewer edges) on K40c: 0.178 GTEPS (P:1150-1151)",
    ("c4_road", "sssp"): "Gunrock SSSP roadnet_CA on K40c: 0.0249 GTEPS (P:1162-1163)",
    ("c2_kron21", "bc"): "Gunrock BC kron_g500-logn21 on K40c: 716.1 ms, 0.5085 GTEPS as 2|E|/t (P:1164-1171)",
    ("c3_orkut", "bc"): "Gunrock BC soc-orkut on K40c: 721.2 ms, 0.5898 GTEPS as 2|E|/t (P:1164-1165)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2_kron21", choices=sorted(CONFIG_DESC))
    ap.add_argument("--prim", default="bfs", choices=["bfs", "sssp", "bc", "cc", "pr"])
    ap.add_argument("--direction", default="auto", choices=["auto", "push", "pull"])
    ap.add_argument("--delta", type=int, default=0)
    ap.add_argument("--sssp-direction", default="auto", choices=["auto", "push", "pull"],
                    help="SSSP near iterations: push, pull over in-edges, or the auto rule (A-24)")
    ap.add_argument("--bc-direction", default="auto", choices=["auto", "push", "pull"],
                    help="BC forward levels: push, pull, or the auto rule (A-24)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    ap.add_argument("--keep-order", action="store_true",
                    help="partitioned BFS: keep the caller's pull-list order (GR_KEEP_ORDER)")
    ap.add_argument("--partitioned", action="store_true",
                    help="1D-partitioned BFS / SSSP over all ranks; default graph c5_kron25 (BFS) / "
                         "c3_orkut (SSSP). The default for --gpus N > 1 (BASELINE config 5)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas of the single-GPU run (sources sharded) instead "
                         "of the 1D-partitioned config-5 run")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0")) or a.gpus
    if world > 1 and not a.replicas and a.prim in ("bfs", "sssp"):
        a.partitioned = True
    if a.partitioned and a.config == "c2_kron21" and "--config" not in sys.argv:
        a.config = "c3_orkut" if a.prim == "sssp" else "c5_kron25"
    return a


# ----------------------------------------------------------------- clocks sampler

class Clocks:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, val in zip(names, p[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- byte model

def algorithmic_bytes(stats, n, prim, packed=False):
    """SURVEY §8(d) algorithmic HBM bytes of one traversal from its per-level
    records (4-byte words; bitmap probes are L2 traffic and not counted):
      push level  12 f + 4 m_f + 12 d
      pull level  n/8 + 8 u + 4 e_insp + 8 d + n/8
      SSSP relax  16 f + 8 e + 12 r ;  far re-split 8 |far|
      per run     8 n (depth/pred init) [+ 12 n for SSSP (dist/pred + stamp)]
    """
    B = 8 * n if prim == "bfs" else 12 * n
    for r in stats["levels"]:
        f, mf, d, ins = r["frontier"], r["frontier_edges"], r["discovered"], r["inspected_edges"]
        if r["direction"] == 1:
            B += 12 * f + 4 * mf + 12 * d
        elif r["direction"] == 2:
            B += n / 8 + 8 * r["aux"] + 4 * ins + 8 * d + n / 8
        elif r["direction"] == 3:  # C + W = 8 B per edge, or the packed (C << 7) | W word: 4 B
            B += 16 * f + (4 if packed else 8) * mf + 12 * d
        elif r["direction"] == 5:  # pull relax: frontier bitmap, every in-list, dist of frontier in-edges
            m_all = stats.get("m", 0)
            B += 4 * f + n / 8 + 16 * n + 4 * m_all + 8 * mf + 12 * d
        else:
            B += 8 * f
    return B


def load_traffic(workload):
    """DRAM bytes per launch of the dominant kernel for this workload, from the
    committed `ncu --set full` capture summary (profiles/ncu_traffic.json:
    dram__bytes_read.sum + dram__bytes_write.sum of one launch), or None."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            rec = json.load(f).get(workload)
    except (OSError, ValueError):
        return None, None, None
    if not rec:
        return None, None, None
    return rec.get("bytes_per_launch"), rec.get("source"), rec.get("warp_efficiency")


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy, burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The CPU oracle as it stands, timed on this box's host cores (rank 0)."""
    import numpy as np
    import torch

    import graphgen as gg
    import oracle
    if rank != 0:
        return
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g = gg.make_config(args.config, device=dev)
    R, C, W = g.numpy()
    srcs = [0] if args.config == "c1_rmat16" else gg.sources(g, args.warmup + args.steps)
    srcs = (srcs * (args.warmup + args.steps))[: args.warmup + args.steps]
    edges, secs = 0, 0.0
    for i, s in enumerate(srcs):
        t0 = time.perf_counter()
        mult = 1
        if args.prim == "bfs":
            x, _ = oracle.bfs(R, C, s, want_pred=True)
            unreached = -1
        elif args.prim == "bc":
            oracle.bc(R, C, [s])
            dt = time.perf_counter() - t0
            x, _ = oracle.bfs(R, C, s, want_pred=False)  # untimed: reached edges
            unreached, mult = -1, 2                         # BC TEPS = 2 m_reached / t
        else:
            x, _ = oracle.sssp(R, C, W, s, want_pred=True)
            unreached = oracle.UINT32_MAX
        if args.prim != "bc":
            dt = time.perf_counter() - t0
        if i >= args.warmup:
            edges += mult * oracle.reached_edges(R, x, unreached)
            secs += dt
    value = edges / secs / 1e9
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": {"bfs": "int32", "sssp": "u32", "bc": "f64"}[args.prim], "data": "synthetic",
           "config": {"workload": "%s %s" % (args.config, args.prim), "graph": CONFIG_DESC[args.config],
                      "n": g.n, "m": g.m},
           "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                            "sample": "%d %s traversals of %s (one per step), single-threaded C oracle"
                                      % (args.steps, args.prim, args.config)},
           "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


# ----------------------------------------------------------------- partitioned (multi-GPU) arm

NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction per GPU (900 nominal)


def partitioned_bytes(levels, n, nonisolated):
    """SURVEY §8(d) algorithmic HBM bytes of one partitioned BFS, summed over
    all ranks, from the global per-level records (the single-GPU model; u of
    a pull level = non-isolated vertices not yet discovered)."""
    B = 8 * n
    found = 1
    for r in levels:
        f, mf, d, ins = r["frontier"], r["frontier_edges"], r["discovered"], r["inspected_edges"]
        if r["direction"] == 1:
            B += 12 * f + 4 * mf + 12 * d
        else:
            B += n / 8 + 8 * max(0, nonisolated - found) + 4 * ins + 8 * d + n / 8
        found += d
    return B


def run_partitioned(args, rank, world, dev):
    """BASELINE config 5: BFS (or, --prim sssp, delta-stepping SSSP: SURVEY
    §8(f) f2) over a 1D vertex partition of one graph across all ranks
     through the library's own group (gr_comm_create:
    NCCL communicator bootstrapped from a torch.distributed broadcast of the
    unique id) and collective gr_bfs / gr_sssp on gr_graph_create_partitioned
    graphs: one persistent kernel per rank runs every level, exchange
    included (peer-memory stores over NVLink). Strong scaling: the graph is
    fixed, each rank owns n/P vertices. Each timed step = one full traversal;
    time = max over ranks of the CUDA-event span of the call. E(P) =
    GTEPS(P) / (P * GTEPS(1)), GTEPS(1) = rank 0's single-GPU kernel (gr_bfs /
    gr_sssp on the whole graph) on the same sources, measured in this run."""
    import torch
    import torch.distributed as dist

    import graphgen as gg
    import paper_1501_05387_b200 as gr
    from paper_1501_05387_b200 import metrics
    from paper_1501_05387_b200 import multigpu as mg
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    sssp = args.prim == "sssp"
    g = gg.make_config(args.config, device=dev, weights=True if sssp else None)
    n, m = g.n, g.m
    srcs = gg.sources(g, args.warmup + args.steps)
    nonisolated = int((g.R[1:] > g.R[:-1]).sum())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # single-GPU reference for E(P): rank 0, whole graph, same sources
    single = None
    if rank == 0 and not args.no_extras:
        G = gr.Graph(g.R, g.C, g.W if sssp else None, symmetric=True)
        d1 = torch.empty(n, dtype=torch.int32, device=dev)

        def one(s):
            if sssp:
                G.sssp(s, d1, None, delta=args.delta)
            else:
                G.bfs(s, d1, None)
        for s in srcs[: args.warmup]:
            one(s)
        e1s, ms1 = 0, 0.0
        for s in srcs[args.warmup:]:
            flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            one(s)
            a1.record()
            torch.cuda.synchronize()
            ms1 += a0.elapsed_time(a1)
            e1s += G.run_stats()["reached_edges"]
        single = metrics.gteps(e1s, ms1 * 1e-3)
        G.close()
        del d1
    v0, v1, Rl, Cl, Wl = mg.partition_csr(g.R, g.C, world, rank, W=g.W if sssp else None)
    del g
    torch.cuda.empty_cache()
    comm = mg.Comm.from_torch(dev.index)
    part = mg.PartitionedGraph(comm, Rl, Cl, n, W_local=Wl, keep_order=args.keep_order)
    del Rl, Cl, Wl

    def run(s, d, p):
        if sssp:
            return part.sssp(s, d, p, delta=args.delta)
        return part.bfs(s, d, p)
    torch.cuda.empty_cache()
    depth = torch.empty(v1 - v0, dtype=torch.int32, device=dev)
    pred = torch.empty(v1 - v0, dtype=torch.int32, device=dev)
    for s in srcs[: args.warmup]:
        run(s, depth, pred)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = gr.gr_kernel_launch_count()
    ms, edges, recs = [], [], []
    with Clocks(dev.index) as clk:
        for s in srcs[args.warmup:]:
            flush.zero_()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(s, depth, pred)
            e1.record()
            torch.cuda.synchronize()
            st = part.run_stats()
            t_all, e_all = metrics.reduce_over_ranks(e0.elapsed_time(e1), st["reached_edges"], *reducers(dev))
            ms.append(t_all)
            edges.append(e_all)
            recs.append(st)
    launches = gr.gr_kernel_launch_count() - launches0
    # end to end through the C ABI: host (pinned) outputs, host wall clock, max over ranks
    pin_d = torch.empty(v1 - v0, dtype=torch.int32, pin_memory=True)
    pin_p = torch.empty(v1 - v0, dtype=torch.int32, pin_memory=True)
    run(srcs[0], pin_d, pin_p)
    e2e = []
    for s in srcs[args.warmup:]:
        dist.barrier()
        t0 = time.perf_counter()
        run(s, pin_d, pin_p)
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e.append(float(t[0]))
    dist.barrier()
    if rank == 0:
        summ = metrics.summarize(edges, ms)
        value = summ["aggregate"]
        peak, peak_src = load_peaks()
        byts = [algorithmic_bytes(r, n, "sssp") if sssp else partitioned_bytes(r["levels"], n, nonisolated)
                for r in recs]
        xbytes = [sum(l["aux"] for l in r["levels"]) for r in recs]
        tot_s = sum(ms) * 1e-3
        per_gpu = sum(byts) / world / tot_s / 1e9
        nv = sum(xbytes) / world / tot_s / 1e9
        lv = recs[-1]["levels"]
        out = {"metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": sum(ms) / len(ms), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "u32" if sssp else "int32",
               "data": "synthetic",
               "config": {"workload": ("%s sssp 1D-partitioned near/far delta-stepping (delta %d), fused exchange "
                                       "over peer memory (gr_comm + gr_graph_create_partitioned + collective "
                                       "gr_sssp)" % (args.config, recs[-1]["delta"])) if sssp else
                                      ("%s bfs 1D-partitioned direction-optimizing, fused exchange over peer "
                                       "memory (gr_comm + gr_graph_create_partitioned + collective gr_bfs)"
                                       % args.config),
                          "graph": CONFIG_DESC[args.config], "n": n, "m": m,
                          "sources": "%d seeded sources with degree>=1 (S:519)" % args.steps,
                          "parallelism": "1D vertex partition over %d rank(s), one persistent kernel per rank" % world,
                          "l2": "flushed (256 MiB write) between timed steps"},
               "throughput": summ,
               "roofline": {"bound": "hbm", "kernel": "psssp_kernel" if sssp else "pbfs_kernel",
                            "achieved": per_gpu, "peak": peak,
                            "unit": "GB/s", "frac": per_gpu / peak, "traffic": None, "peak_source": peak_src,
                            "bytes_per_launch": sum(byts) / len(byts) / world,
                            "model": "SURVEY 8(d) algorithmic bytes of the global per-level records / P "
                                     + ("(relax 16f+8e+12r; re-split 8|far|; +12n init)" if sssp else
                                        "(push 12f+4m_f+12d; pull n/4+8u+4e_insp+8d; +8n init)")},
               "exchange": {"bytes_per_step": sum(xbytes) / len(xbytes),
                            "bytes_per_level": [l["aux"] for l in lv],
                            "level_us": [round(l["ns"] / 1e3, 1) for l in lv],
                            "level_direction": [l["direction"] for l in lv],
                            "achieved_gbs_per_gpu": nv, "peak_gbs": NVLINK_PEER_GBS,
                            "frac": nv / NVLINK_PEER_GBS,
                            "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)"},
               "gpu_launches": launches, "levels_per_step": statistics.mean(r["num_levels"] for r in recs),
               "clocks": clk.summary(),
               "e2e": {"value": sum(edges) / sum(e2e) / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 8 * n,
                       "what": "collective gr_bfs through the C ABI writing host (pinned) depth+pred of each "
                               "rank's block; host wall clock, max over ranks"}}
        if single is not None:
            out["single_gpu_gteps"] = single
            out["efficiency"] = {"E": value / (world * single),
                                 "what": "GTEPS(P) / (P x GTEPS(1)), GTEPS(1) = single-GPU gr_bfs on the "
                                         "whole graph, same sources, this run"}
        emit(out)
    part.close()
    comm.close()
    dist.destroy_process_group()


def run_bc(args, rank, world, dev):
    """Betweenness centrality: one step = the Brandes
    forward + backward passes of one source (gr_bc, synchronous: one host
    read per level, so the events include those bubbles). TEPS = 2 m_reached
    / t (the paper's BC convention, both passes traverse the edges).
    Replicas: sources sharded over the ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import graphgen as gg
    import paper_1501_05387_b200 as gr
    g = gg.make_config(args.config, device=dev)
    G = gr.Graph(g.R, g.C, None, symmetric=True)
    deg = g.R[1:] - g.R[:-1]
    n, m = g.n, g.m
    srcs = gg.sources(g, args.warmup + args.steps * world)
    mine = srcs[args.warmup + rank * args.steps: args.warmup + (rank + 1) * args.steps]
    bcv = torch.empty(n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for s in srcs[: args.warmup]:
        G.bc([s], bc=bcv, direction=args.bc_direction)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = gr.gr_kernel_launch_count()
    ms = []
    with Clocks(local_index(dev)) as clk:
        for s in mine:
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            G.bc([s], bc=bcv, direction=args.bc_direction)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
    launches = gr.gr_kernel_launch_count() - l0
    # untimed: reached edges / vertices of each source (BFS depth) for TEPS and the byte model
    depth = torch.empty(n, dtype=torch.int32, device=dev)
    edges, byts = 0, []
    for s in mine:
        G.bfs(s, depth, None)
        r = depth >= 0
        mr, nr, q = int(deg[r].sum()), int(r.sum()), int((r & (deg > 0)).sum())
        edges += 2 * mr
        # init 20n + fwd (20 Q + 4 m_r + 24 n_r) + bwd (20 Q + 4 m_r + 8 Q) + accumulate 24 n
        byts.append(20 * n + 20 * q + 4 * mr + 24 * nr + 28 * q + 4 * mr + 24 * n)
    tot = sum(ms)
    if world > 1:
        t = torch.tensor([tot, float(edges)], dtype=torch.float64, device=dev)
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:])
        tot_all, edges_all = float(tm[0]), float(t[1])
    else:
        tot_all, edges_all = tot, float(edges)
    peak, peak_src = load_peaks()
    achieved = sum(byts) / (tot * 1e-3) / 1e9
    workload = "%s bc (Brandes, one source per step)" % args.config
    out = {"metric": METRIC, "value": edges_all / (tot_all * 1e-3) / 1e9, "unit": "GTEPS", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_all / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": workload, "graph": CONFIG_DESC[args.config], "n": n, "m": m,
                      "sources": "%d seeded sources with degree>=1 per rank (S:519)" % args.steps,
                      "teps": "2 m_reached / t (paper's BC convention, P:1164-1171)",
                      "l2": "flushed (256 MiB write) between timed steps",
                      "parallelism": "replicas: sources sharded over %d rank(s)" % world},
           "roofline": {"bound": "hbm", "kernel": "bc_fwd_kernel+bc_bwd_kernel", "achieved": achieved,
                        "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                        "peak_source": peak_src,
                        "model": "init 20n + fwd 20Q+4m_r+24n_r + bwd 28Q+4m_r + accumulate 24n "
                                 "(Q = reached vertices with out-degree > 0)"},
           "gpu_launches": launches, "paper_context": PAPER_CONTEXT.get((args.config, "bc"))}
    if rank == 0:
        out["clocks"] = clk.summary()
    # end to end: host (pinned) output buffer through the C ABI
    pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    G.bc(mine[:1], bc=pin, direction=args.bc_direction)
    e2e_s = 0.0
    for s in mine:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.bc([s], bc=pin, direction=args.bc_direction)
        e2e_s += time.perf_counter() - t0
    out["e2e"] = {"value": edges / e2e_s / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": 4,
                  "d2h_bytes_per_step": 8 * n,
                  "what": "gr_bc through the C ABI writing a host (pinned) bc array; host wall clock per call"}
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        R, C, _ = g.numpy()
        ce, cs, cnt = 0, 0.0, 0
        for s in mine:
            t0 = time.perf_counter()
            oracle.bc(R, C, [s])
            cs += time.perf_counter() - t0
            d, _ = oracle.bfs(R, C, s)
            ce += 2 * oracle.reached_edges(R, d, -1)
            cnt += 1
            if cs > args.cpu_sample_s:
                break
        out["cpu_baseline"] = {"value": ce / cs / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                               "sample": "%d of the timed sources, full Brandes single-source passes of %s, "
                                         "single-threaded C oracle (%d host cores available)"
                                         % (cnt, args.config, os.cpu_count())}
    if rank == 0:
        emit(out)
    G.close()
    if world > 1:
        dist.destroy_process_group()


def run_whole_graph(args, rank, world, dev):
    """Connected components / PageRank: one step = one full
    run over the whole graph (gr_cc / gr_pagerank, synchronous: the events
    include the host reads between passes). GTEPS = m / t for CC and
    m x iterations / t for PageRank (the paper normalises PageRank to one
    iteration, Table 3 caption P:1190-1191). Replicas: every rank runs the
    same whole-graph problem (no data-path collective)."""
    import torch
    import torch.distributed as dist

    import graphgen as gg
    import paper_1501_05387_b200 as gr
    g = gg.make_config(args.config, device=dev)
    G = gr.Graph(g.R, g.C, None, symmetric=True)
    n, m = g.n, g.m
    comp = torch.empty(n, dtype=torch.int32, device=dev)
    rank_v = torch.empty(n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        if args.prim == "cc":
            return 1, G.cc(comp)[1]
        _, it = G.pagerank(0.85, 1e-6, 1000, rank=rank_v)
        return it, None

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = gr.gr_kernel_launch_count()
    ms, iters = [], []
    with Clocks(local_index(dev)) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            it, k = step()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            iters.append(it)
    launches = gr.gr_kernel_launch_count() - l0
    tot = sum(ms)
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_all = float(t[0])
    else:
        tot_all = tot
    edges = float(m) * sum(iters) * world
    peak, peak_src = load_peaks()
    if args.prim == "cc":
        passes = G.run_stats()["num_levels"]
        byts = 2 * (8 * n + 4 * m) + (passes + 1) * 8 * n  # lower bound: two CSR passes + jumps + init
        model = "lower bound: 2 CSR hooking passes (8n + 4m each) + (passes + 1) x 8n (init, pointer jumping)"
    else:
        byts = sum(iters) / len(iters) * (40 * n + 4 * m) + 36 * n
        model = "upper bound per iteration with a full frontier: 40n + 4m (queue, acc, rank, in-list stream); init 36n"
    achieved = byts / (tot / len(ms) * 1e-3) / 1e9
    workload = "%s %s" % (args.config, {"cc": "cc (hooking + pointer jumping)",
                                        "pr": "pagerank (d=0.85, tol=1e-6 per vertex)"}[args.prim])
    out = {"metric": METRIC, "value": edges / (tot_all * 1e-3) / 1e9, "unit": "GTEPS", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_all / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "int32" if args.prim == "cc" else "f64", "data": "synthetic",
           "config": {"workload": workload, "graph": CONFIG_DESC[args.config], "n": n, "m": m,
                      "teps": "m / t" if args.prim == "cc" else "m x iterations / t",
                      "l2": "flushed (256 MiB write) between timed steps",
                      "parallelism": "replicas: the whole graph on each of %d rank(s)" % world},
           "roofline": {"bound": "hbm", "kernel": "cc_hook_*+cc_jump" if args.prim == "cc" else
                        "pr_advance+pr_filter", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": None, "peak_source": peak_src, "model": model},
           "gpu_launches": launches}
    if args.prim == "pr":
        out["iterations_per_step"] = sum(iters) / len(iters)
        out["ms_per_iteration"] = tot_all / sum(iters)
    if rank == 0:
        out["clocks"] = clk.summary()
    # end to end: host (pinned) outputs through the C ABI
    pin_c = torch.empty(n, dtype=torch.int32, pin_memory=True)
    pin_r = torch.empty(n, dtype=torch.float64, pin_memory=True)
    e2e_s, e2e_it = 0.0, 0
    for _ in range(max(1, min(args.steps, 4))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if args.prim == "cc":
            G.cc(pin_c)
            e2e_it += 1
        else:
            e2e_it += G.pagerank(0.85, 1e-6, 1000, rank=pin_r)[1]
        e2e_s += time.perf_counter() - t0
    out["e2e"] = {"value": m * e2e_it / e2e_s / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": n * (4 if args.prim == "cc" else 8),
                  "what": "gr_cc / gr_pagerank through the C ABI writing host (pinned) outputs"}
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        R, C, _ = g.numpy()
        t0 = time.perf_counter()
        if args.prim == "cc":
            oracle.cc(R, C)
            it = 1
            what = "one full union-find CC of %s, single-threaded C oracle" % args.config
        else:
            oracle.pagerank(R, C, 0.85, tol=1e-6, max_iter=5)
            it = 5
            what = "5 Jacobi iterations of the numpy oracle on %s" % args.config
        cs = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": m * it / cs / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                               "sample": what}
    if rank == 0:
        emit(out)
    G.close()
    if world > 1:
        dist.destroy_process_group()


def reducers(dev):
    """(max, sum) of a float over the torch.distributed group (NCCL on GPUs)."""
    import torch
    import torch.distributed as dist

    def mx(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def sm(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t[0])
    return mx, sm


def cpu_model():
    """lscpu model name of this host (the CPU baseline's hardware)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def local_index(dev):
    return dev.index if dev.index is not None else 0


# ----------------------------------------------------------------- our arm

def spawn(args):
    """`bench.py --gpus N` outside torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous);
    rank 0's JSON line goes to this process's stdout."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, stdout=_JSON_FD, stderr=2)
    sys.exit(r.returncode)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "--gpus" in " ".join(sys.argv) and args.gpus != world:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import graphgen as gg
    import paper_1501_05387_b200 as gr
    from paper_1501_05387_b200 import metrics
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    dev = torch.device("cuda", local)
    if args.partitioned:
        return run_partitioned(args, rank, world, dev)
    if args.prim == "bc":
        return run_bc(args, rank, world, dev)
    if args.prim in ("cc", "pr"):
        return run_whole_graph(args, rank, world, dev)
    want_w = args.prim == "sssp"
    g = gg.make_config(args.config, device=dev, weights=want_w or None)
    G = gr.Graph(g.R, g.C, g.W if want_w else None, symmetric=True)
    deg = (g.R[1:] - g.R[:-1])
    n, m = g.n, g.m
    nsrc = args.warmup + args.steps * world
    if args.config == "c1_rmat16":
        all_srcs = [0] * nsrc
    else:
        all_srcs = gg.sources(g, nsrc)
    warm_srcs = all_srcs[: args.warmup]
    my_srcs = all_srcs[args.warmup + rank * args.steps: args.warmup + (rank + 1) * args.steps]

    depth = torch.empty(n, dtype=torch.int32, device=dev)
    pred = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(s, direction=args.direction, asynchronous=False):
        if args.prim == "bfs":
            G.bfs(s, depth, pred, direction=direction, asynchronous=asynchronous)
        else:
            G.sssp(s, depth, pred, delta=args.delta, direction=args.sssp_direction, asynchronous=asynchronous)

    for s in warm_srcs:
        step(s)
    torch.cuda.synchronize()

    def timed(srcs, direction):
        """Device time of each traversal: the runs are only enqueued (gr_*_async),
        so the events bracket the GPU work of one call and nothing of the host.
        A device-side sleep first lets the host enqueue every step before the
        GPU reaches the first event (no host latency inside any bracket)."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in srcs]
        torch.cuda._sleep(int(2e6) * (len(srcs) + 2))
        l0 = gr.gr_kernel_launch_count()
        for (e0, e1), s in zip(ev, srcs):
            flush.zero_()
            e0.record(stream)
            step(s, direction, asynchronous=True)
            e1.record(stream)
        G.sync()
        torch.cuda.synchronize()
        timed.launches = gr.gr_kernel_launch_count() - l0
        ms = [a.elapsed_time(b) for a, b in ev]
        # reached edges (gr_run_stats.reached_edges, A-14) and level stats:
        # untimed re-runs (depth is deterministic)
        edges, recs = [], []
        for s in srcs:
            step(s, direction)
            recs.append(G.run_stats())
            edges.append(recs[-1]["reached_edges"])
        return edges, ms, recs

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        edges, ms, recs = timed(my_srcs, args.direction)
    launches = timed.launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tot_ms = sum(ms)
    summ = metrics.summarize(edges, ms)
    edges = sum(edges)
    if world > 1:
        tot_ms_all, edges_all = metrics.reduce_over_ranks(tot_ms, edges, *reducers(dev))
    else:
        tot_ms_all, edges_all = tot_ms, float(edges)
    value = metrics.gteps(edges_all, tot_ms_all * 1e-3)

    peak, peak_src = load_peaks()
    packed = bool(G.info().packed_weights) if args.prim == "sssp" else False
    for r in recs:
        r["m"] = m
    byts = [algorithmic_bytes(r, n, args.prim, packed) for r in recs]
    kname = "bfs_kernel" if args.prim == "bfs" else "sssp_kernel"
    if G.info().bounded_degree:  # narrow levels in one cluster; the grid kernel resumes only if they outgrow it
        kname = ("bfs" if args.prim == "bfs" else "sssp") + "_ell_cluster_kernel (+ init, + resumed grid kernel)"
    achieved = sum(byts) / (tot_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                "bytes_per_launch": sum(byts) / len(byts),
                "model": ("SURVEY 8(d) algorithmic bytes from per-level run stats (relax 16f+%de+12r; "
                          "re-split 8|far|; +12n init); one launch per traversal" % (4 if packed else 8))
                         if args.prim == "sssp" else
                         "SURVEY 8(d) algorithmic bytes from per-level run stats (push 12f+4m_f+12d; "
                         "pull n/4+8u+4e_insp+8d; +8n init); one launch per traversal"}

    workload = "%s %s direction=%s" % (args.config, args.prim, args.direction)
    roofline["traffic"], tsrc, weff = load_traffic(workload)
    if tsrc:
        roofline["traffic_source"] = tsrc
    if weff is not None:
        # the paper's Table 4 analog (warp execution efficiency):
        # active threads per executed warp instruction / 32, from the same capture
        roofline["warp_efficiency"] = weff
        roofline["warp_efficiency_paper"] = "BFS 96.72-97.97%, SSSP 82.56-85.15% on K40c (P:1326-1334)"
    out = {"metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": tot_ms_all / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None,
           "dtype": "int32" if args.prim == "bfs" else "u32", "data": "synthetic",
           "config": {"workload": workload,
                      "graph": CONFIG_DESC[args.config], "n": n, "m": m,
                      "sources": "%d seeded sources with degree>=1 per rank (S:519)" % args.steps,
                      "l2": "flushed (256 MiB write) between timed steps",
                      "parallelism": "replicas: sources sharded over %d rank(s)" % world},
           "roofline": roofline, "gpu_launches": launches,
           "throughput": summ if world == 1 else None}
    if rank == 0:
        out["clocks"] = clk.summary()
        out["paper_context"] = PAPER_CONTEXT.get((args.config, args.prim))
        out["levels_per_step"] = statistics.mean(r["num_levels"] for r in recs)
        if args.prim == "sssp":
            # work inflation the paper's SSSP MTEPS hides: edges
            # relaxed per reached edge, and near iterations / re-splits per run
            relaxed = [sum(l["frontier_edges"] for l in r["levels"] if l["direction"] in (3, 5)) for r in recs]
            out["sssp_work"] = {"relaxations_per_edge": sum(relaxed) / max(1, sum(r["reached_edges"] for r in recs)),
                                "near_iterations": statistics.mean(sum(1 for l in r["levels"] if l["direction"] in (3, 5))
                                                                   for r in recs),
                                "resplits": statistics.mean(sum(1 for l in r["levels"] if l["direction"] == 4)
                                                            for r in recs),
                                "pull_iterations": statistics.mean(sum(1 for l in r["levels"] if l["direction"] == 5)
                                                                   for r in recs),
                                "delta": recs[-1]["delta"]}

    if rank == 0 and not args.no_extras and args.prim == "bfs" and args.direction == "auto":
        # the push-only roofline row of the north star (same sources)
        pe, pms, precs = timed(my_srcs, "push")
        pb = [algorithmic_bytes(r, n, "bfs") for r in precs]
        pach = sum(pb) / (sum(pms) * 1e-3) / 1e9
        out["push_only"] = {"value": metrics.gteps(sum(pe), sum(pms) * 1e-3), "unit": "GTEPS",
                            "ms_per_step": sum(pms) / len(pms), "achieved_gbs": pach,
                            "frac": pach / peak}
        # north-star reading of the bar: "bytes touched per traversed edge x
        # TEPS / peak" with the push-only byte model (SURVEY 8(d) M-1 F_edge,
        # "push-equivalent"): credits the edges direction optimisation skips
        roofline["push_equivalent"] = {
            "achieved": sum(pb) / (tot_ms * 1e-3) / 1e9, "frac": sum(pb) / (tot_ms * 1e-3) / 1e9 / peak,
            "what": "F_edge (SURVEY 8(d) M-1): push-only model bytes of the same sources / push-pull time / peak"}

    # ---- end to end through the C ABI with host buffers (rank 0 measures; all ranks run)
    pin_d = torch.empty(n, dtype=torch.int32, pin_memory=True)
    pin_p = torch.empty(n, dtype=torch.int32, pin_memory=True)
    for s in warm_srcs:  # untimed: the first host-output call allocates the staging buffers
        if args.prim == "bfs":
            G.bfs(s, pin_d, pin_p, direction=args.direction)
        else:
            G.sssp(s, pin_d, pin_p, delta=args.delta, direction=args.sssp_direction)
    e2e_edges, e2e_s, per_call = 0, 0.0, []
    for s in my_srcs:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if args.prim == "bfs":
            G.bfs(s, pin_d, pin_p, direction=args.direction)
        else:
            G.sssp(s, pin_d, pin_p, delta=args.delta, direction=args.sssp_direction)
        per_call.append(time.perf_counter() - t0)
        e2e_s += per_call[-1]
        e2e_edges += G.run_stats()["reached_edges"]
    out["e2e"] = {"value": e2e_edges / e2e_s / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 8 * n,
                  "what": "gr_bfs/gr_sssp through the C ABI writing host (pinned) depth+pred; "
                          "host wall clock per call; graph resident (created once, P:1089-1090: the "
                          "paper's runtimes ignore transfer time); the source id is a call argument",
                  "per_call_ms": [round(x * 1e3, 3) for x in per_call]}
    if rank == 0 and not args.no_extras:
        # cold end to end, once (context): gr_graph_create from pinned host CSR
        # (copy, validation, degree-ordered pull lists, pull head) + one traversal
        # with host outputs + destroy
        Rh, Ch = g.R.cpu().pin_memory(), g.C.cpu().pin_memory()
        Wh = g.W.cpu().pin_memory() if want_w else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Gc = gr.Graph(Rh, Ch, Wh, symmetric=True)
        t1 = time.perf_counter()
        if args.prim == "bfs":
            Gc.bfs(my_srcs[0], pin_d, pin_p, direction=args.direction)
        else:
            Gc.sssp(my_srcs[0], pin_d, pin_p, delta=args.delta)
        t2 = time.perf_counter()
        ce = Gc.run_stats()["reached_edges"]
        Gc.close()
        out["e2e"]["cold"] = {"value": ce / (t2 - t0) / 1e9, "unit": "GTEPS", "create_ms": (t1 - t0) * 1e3,
                              "traversal_ms": (t2 - t1) * 1e3,
                              "h2d_bytes": int(Rh.numel() * 8 + Ch.numel() * 4 + (Wh.numel() * 4 if want_w else 0)),
                              "d2h_bytes": 8 * n,
                              "what": "one traversal including gr_graph_create from pinned host CSR"}
        del Rh, Ch, Wh

    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        R, C, W = g.numpy()
        ce, cs, cnt = 0, 0.0, 0
        for s in my_srcs:
            t0 = time.perf_counter()
            if args.prim == "bfs":
                x, _ = oracle.bfs(R, C, s)
                un = -1
            else:
                x, _ = oracle.sssp(R, C, W, s)
                un = oracle.UINT32_MAX
            cs += time.perf_counter() - t0
            ce += oracle.reached_edges(R, x, un)
            cnt += 1
            if cs > args.cpu_sample_s:
                break
        out["cpu_baseline"] = {"value": ce / cs / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                               "sample": "%d of the timed sources, full %s traversals of %s, "
                                         "single-threaded C oracle (%d host cores available)"
                                         % (cnt, args.prim, args.config, os.cpu_count()),
                               "cpu_model": cpu_model()}
    if rank == 0:
        emit(out)
    G.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
