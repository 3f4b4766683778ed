#!/usr/bin/env python
"""Where does the host-driven partitioned level loop spend its time?

Runs dist.bfs_partitioned (or sssp_partitioned) at world size 1 over NCCL on
one GPU and wraps every partition / exchange call with a host timer, once
without synchronisation (the real loop: host issue cost + blocking reads) and
once with a device synchronisation after each call (device-side attribution).

    python scripts/part_host_profile.py [--config c5_kron25] [--prim bfs|sssp] [--runs 3]
"""
import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

import graphgen as gg
from paper_1501_05387_b200 import dist as grd


def wrap(obj, names, acc, sync):
    for name in names:
        f = getattr(obj, name, None)
        if f is None:
            continue

        def make(f, name):
            def g(*a, **k):
                t0 = time.perf_counter()
                r = f(*a, **k)
                if sync:
                    torch.cuda.synchronize()
                acc[name][0] += 1
                acc[name][1] += time.perf_counter() - t0
                return r
            return g
        setattr(obj, name, make(f, name))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5_kron25")
    ap.add_argument("--prim", default="bfs", choices=["bfs", "sssp"])
    ap.add_argument("--runs", type=int, default=3)
    a = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    sssp = a.prim == "sssp"
    g = gg.make_config(a.config, device=dev, weights=True if sssp else None)
    srcs = gg.sources(g, a.runs + 1)
    _, _, Rl, Cl = grd.partition_csr(g.R, g.C, 1, 0)
    Wl = grd.partition_weights(g.R, g.W, 1, 0) if sssp else None
    delta = 3 if sssp else 0
    part = grd.GpuPartition(Rl, Cl, g.n, 1, 0, device=0, W_local=Wl)
    ex = grd.TorchDistExchange()
    if not sssp:
        part.order_pull_lists(grd.global_degrees(part, ex))
    del g
    depth = torch.empty(part.n_local, dtype=torch.int32, device=dev)
    pred = torch.empty(part.n_local, dtype=torch.int32, device=dev)

    def run(s):
        if sssp:
            return grd.sssp_partitioned(part, ex, s, depth, pred, delta=delta)
        return grd.bfs_partitioned(part, ex, s, depth, pred)

    run(srcs[0])
    torch.cuda.synchronize()
    pnames = ["begin", "expand", "absorb", "frontier_dev", "shard", "pull", "sssp_begin", "sssp_relax",
              "sssp_absorb", "sssp_counts_dev", "sssp_far_min", "sssp_resplit", "sssp_end"]
    enames = ["counts", "pairs", "allreduce_sum", "allreduce_min", "allgather"]
    for sync in (False, True):
        acc = collections.defaultdict(lambda: [0, 0.0])
        wrap(part, pnames, acc, sync)
        wrap(ex, enames, acc, sync)
        tot = 0.0
        for s in srcs[1:]:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run(s)
            torch.cuda.synchronize()
            tot += time.perf_counter() - t0
        for n in pnames:
            if n in part.__dict__:
                del part.__dict__[n]
        for n in enames:
            if n in ex.__dict__:
                del ex.__dict__[n]
        print("== %s %s, %s: %.3f ms per run (host wall clock)" %
              (a.config, a.prim, "sync after each call" if sync else "as issued", 1e3 * tot / a.runs))
        covered = 0.0
        for k, (c, t) in sorted(acc.items(), key=lambda x: -x[1][1]):
            covered += t
            print("  %-16s %5d calls  %8.1f us per run  %6.1f us per call" %
                  (k, c // a.runs, 1e6 * t / a.runs, 1e6 * t / max(c, 1)))
        print("  %-16s %8.1f us per run" % ("(rest: python)", 1e6 * (tot - covered) / a.runs))
    part.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
