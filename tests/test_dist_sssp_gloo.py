"""Multi-process (world size 2, gloo, CPU) test of the partitioned-SSSP step
driver (paper_1501_05387_b200/dist.py: sssp_partitioned): triple routing
through all_to_all_single, the all-reduced near count, the all-reduced
MINIMUM far distance and the band jump of the re-split (reading A-11).

The per-rank partition here is a plain-Python TEST DOUBLE of the CUDA
kernels (same contract as gr_part_sssp_*: iteration+slice stamp (A-7),
best-shipped culling, one bucket entry per vertex per step). It is test code,
not a product fallback: the product path is GpuPartition (C ABI, CUDA only).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen as gg
import oracle
from paper_1501_05387_b200 import dist as grd

INF = (1 << 32) - 1


class SsspPartitionDouble:
    def __init__(self, R_local, C_local, W_local, n_global, nparts, rank):
        self.R, self.C, self.W = R_local.numpy(), C_local.numpy(), W_local.numpy().astype(np.int64)
        self.n_global, self.nparts, self.rank = n_global, nparts, rank
        self.v_begin, self.v_end = grd.owned_range(n_global, nparts, rank)
        self.n_local = self.v_end - self.v_begin
        self.block = grd.block_size(n_global, nparts)
        self.send_triples = torch.zeros(3 * nparts * self.block, dtype=torch.int32)
        self.recv_triples = torch.zeros(3 * nparts * self.block, dtype=torch.int32)
        self.send_counts = torch.zeros(nparts, dtype=torch.int64)

    def sssp_begin(self, src, dist_out, pred_out):
        self.out = (dist_out, pred_out)
        self.d = [INF] * self.n_local
        self.p = [-1] * self.n_local
        self.stamp = [-1] * self.n_local
        self.best = {}
        self.sstamp = {}
        self.near = {0: []}
        self.far = {0: [], 1: []}
        if self.v_begin <= src < self.v_end:
            s = src - self.v_begin
            self.d[s], self.p[s] = 0, src
            if self.R[s + 1] > self.R[s]:
                self.near[0] = [s]

    def _owned(self, lv, nd, parent, thr, it, step, fp):
        if nd >= self.d[lv]:
            return
        self.d[lv], self.p[lv] = nd, parent
        far = nd >= thr
        key = 2 * it + (1 if far else 0)
        if self.stamp[lv] == key:
            return
        self.stamp[lv] = key
        if far:
            self.far[fp].append(lv)
        elif self.R[lv + 1] > self.R[lv]:
            self.near.setdefault(step + 1, []).append(lv)

    def sssp_relax(self, step, it, fp, thr):
        self.send_counts.zero_()
        self.near.setdefault(step + 1, [])
        for u in self.near.get(step, []):
            for e in range(self.R[u], self.R[u + 1]):
                v = int(self.C[e])
                nd = self.d[u] + int(self.W[e])
                lv = v - self.v_begin
                if 0 <= lv < self.n_local:
                    self._owned(lv, nd, self.v_begin + u, thr, it, step, fp)
                elif nd < self.best.get(v, (INF, 0))[0]:
                    self.best[v] = (nd, self.v_begin + u)
                    if self.sstamp.get(v) != step:
                        self.sstamp[v] = step
                        q = v // self.block
                        k = int(self.send_counts[q])
                        self.send_triples[3 * (q * self.block + k)] = v
                        self.send_counts[q] += 1
        for q in range(self.nparts):  # pack: final best values
            for k in range(int(self.send_counts[q])):
                i = 3 * (q * self.block + k)
                v = int(self.send_triples[i])
                self.send_triples[i + 1] = int(np.int32(np.uint32(self.best[v][0])))
                self.send_triples[i + 2] = self.best[v][1]

    def sssp_absorb(self, step, it, fp, thr, triples, nrecv):
        self.near.setdefault(step + 1, [])
        for j in range(nrecv):
            v, nd, parent = (int(x) for x in triples[3 * j: 3 * j + 3])
            lv = v - self.v_begin
            assert 0 <= lv < self.n_local, "misrouted triple"
            self._owned(lv, nd & 0xFFFFFFFF, parent, thr, it, step, fp)

    def sssp_counts(self, step, fp):
        return len(self.near.get(step, [])), len(self.far[fp])

    def sssp_far_min(self, step, fp, thr):
        live = [self.d[v] for v in self.far[fp] if self.d[v] >= thr]
        return min(live) if live else grd.NO_FAR

    def sssp_resplit(self, step, it, fp, thr_old, thr):
        nxt = self.near.setdefault(step + 1, [])
        self.far[fp ^ 1] = []
        for v in self.far[fp]:
            d = self.d[v]
            if d < thr_old:
                continue  # stale (A-11)
            nearb = d < thr
            key = 2 * it + (0 if nearb else 1)
            if self.stamp[v] == key:
                continue
            self.stamp[v] = key
            if nearb:
                if self.R[v + 1] > self.R[v]:
                    nxt.append(v)
            else:
                self.far[fp ^ 1].append(v)
        self.far[fp] = []

    def sssp_end(self):
        dist_out, pred_out = self.out
        dist_out.copy_(torch.tensor(np.array(self.d, np.uint32).view(np.int32)))
        if pred_out is not None:
            pred_out.copy_(torch.tensor(self.p, dtype=torch.int32))


def _graph(name):
    if name == "rmat":
        return gg.assign_weights(gg.rmat(9, 8, seed=4), seed=2)
    if name == "directed":
        return gg.assign_weights(gg.directed_random(500, 3000, seed=2), seed=2)
    return gg.assign_weights(gg.grid(13, 17), seed=2)


def _worker(rank, world, port, graph_name, srcs, deltas, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(graph_name)
        v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, world, rank)
        Wl = grd.partition_weights(g.R, g.W, world, rank)
        part = SsspPartitionDouble(Rl, Cl, Wl, g.n, world, rank)
        ex = grd.TorchDistExchange()
        res = []
        for s in srcs:
            for delta in deltas:
                d = torch.empty(v1 - v0, dtype=torch.int32)
                p = torch.empty(v1 - v0, dtype=torch.int32)
                steps = grd.sssp_partitioned(part, ex, s, d, p, delta=delta)
                res.append((d.numpy().copy(), p.numpy().copy(), steps))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("graph_name", ["rmat", "directed", "grid"])
def test_partitioned_sssp_world2_gloo(graph_name):
    g = _graph(graph_name)
    srcs = gg.sources(g, 2)
    deltas = [1, 16, INF]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), graph_name, srcs, deltas, out), nprocs=2, join=True)
    R, C, W = g.numpy()
    for k in range(len(out[0])):
        s = srcs[k // len(deltas)]
        d = np.concatenate([out[r][k][0] for r in range(2)]).view(np.uint32)
        p = np.concatenate([out[r][k][1] for r in range(2)])
        ref, _ = oracle.sssp(R, C, W, s)
        assert np.array_equal(d, ref), (graph_name, s, deltas[k % len(deltas)])
        assert oracle.check_sssp(R, C, W, s, d, p) == []
        assert out[0][k][2] == out[1][k][2]  # every rank ran the same steps


def test_next_threshold_band_jump():
    # A-11: the threshold moves to the end of the band holding the minimum
    assert grd.next_threshold(0, 4) == 4
    assert grd.next_threshold(3, 4) == 4
    assert grd.next_threshold(4, 4) == 8
    assert grd.next_threshold(17, 8) == 24
    assert grd.next_threshold(5, INF) == INF
