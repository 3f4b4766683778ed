"""Multi-process (world size 2, gloo, CPU) test of the partitioned-BFS level
driver (paper_1501_05387_b200/dist.py): 1D ownership, bucket routing through
all_to_all_single, absorb, all-reduced termination.

The per-rank partition here is a plain-Python TEST DOUBLE of the CUDA
partition kernels (same contract as gr_part_bfs_*: local claims, an
"already sent" bitmap, (vertex, parent) buckets per owner). It is test code,
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


class PartitionDouble:
    def __init__(self, R_local, C_local, n_global, nparts, rank):
        self.R = R_local.numpy()
        self.C = C_local.numpy()
        self.n_global, self.nparts, self.rank = n_global, nparts, rank
        self.v_begin, self.v_end = grd.owned_range(n_global, nparts, rank)
        self.n_local = self.v_end - self.v_begin
        self.block = grd.block_size(n_global, nparts)
        self.send_pairs = torch.zeros(2 * nparts * self.block, dtype=torch.int32)
        self.send_counts = torch.zeros(nparts, dtype=torch.int64)
        self.recv_pairs = torch.zeros(2 * n_global, dtype=torch.int32)
        self.global_buf = torch.zeros(nparts * self.block // 32, dtype=torch.int32)
        deg = np.diff(self.R)
        self.nonisolated_local = int((deg > 0).sum())
        self.m_local = int(self.C.size)

    def degree(self, v):
        return int(self.R[v - self.v_begin + 1] - self.R[v - self.v_begin]) if self.v_begin <= v < self.v_end else 0

    def shard(self, level):
        bits = np.zeros(self.block // 32, np.uint32)
        for v in self.queues.get(level, []):
            bits[v >> 5] |= np.uint32(1 << (v & 31))
        return torch.from_numpy(bits.view(np.int32))

    def pull(self, level, global_bits):
        g = global_bits.numpy().view(np.uint32)
        nxt = self.queues.setdefault(level + 1, [])
        for v in range(self.n_local):
            if self.visited[v]:
                continue
            for e in range(self.R[v], self.R[v + 1]):
                u = int(self.C[e])
                if (g[u >> 5] >> (u & 31)) & 1:
                    self.visited[v] = True
                    self.depth[v] = level + 1
                    self.pred[v] = u
                    nxt.append(v)
                    break

    def begin(self, src, depth, pred):
        self.depth, self.pred = depth, pred
        depth.fill_(-1)
        pred.fill_(-1)
        self.visited = np.zeros(self.n_local, bool)
        self.sent = np.zeros(self.n_global, bool)
        self.sent[src] = True
        self.queues = {0: []}
        if self.v_begin <= src < self.v_end:
            s = src - self.v_begin
            depth[s] = 0
            pred[s] = src
            self.visited[s] = True
            if self.R[s + 1] > self.R[s]:
                self.queues[0] = [s]

    def expand(self, level):
        nxt = self.queues.setdefault(level + 1, [])
        self.send_counts.zero_()
        for u in self.queues[level]:
            for e in range(self.R[u], self.R[u + 1]):
                w = int(self.C[e])
                lw = w - self.v_begin
                if 0 <= lw < self.n_local:
                    if not self.visited[lw]:
                        self.visited[lw] = True
                        self.depth[lw] = level + 1
                        self.pred[lw] = self.v_begin + u
                        if self.R[lw + 1] > self.R[lw]:
                            nxt.append(lw)
                elif not self.sent[w]:
                    self.sent[w] = True
                    q = w // self.block
                    k = int(self.send_counts[q])
                    self.send_pairs[2 * (q * self.block + k)] = w
                    self.send_pairs[2 * (q * self.block + k) + 1] = self.v_begin + u
                    self.send_counts[q] += 1

    def absorb(self, level, pairs, n):
        nxt = self.queues.setdefault(level + 1, [])
        for j in range(n):
            w, parent = int(pairs[2 * j]), int(pairs[2 * j + 1])
            lw = w - self.v_begin
            assert 0 <= lw < self.n_local, "misrouted pair"
            if not self.visited[lw]:
                self.visited[lw] = True
                self.depth[lw] = level + 1
                self.pred[lw] = parent
                if self.R[lw + 1] > self.R[lw]:
                    nxt.append(lw)

    def frontier(self, level):
        q = self.queues.get(level, [])
        return len(q), int(sum(self.R[u + 1] - self.R[u] for u in q))


def _worker(rank, world, port, graph_name, srcs, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(graph_name)
        v0, v1, Rl, Cl = grd.partition_csr(g.R, g.C, world, rank)
        part = PartitionDouble(Rl, Cl, g.n, world, rank)
        part.symmetric = g.symmetric
        ex = grd.TorchDistExchange()
        res = []
        for s in srcs:
            for direction in ("push", "pull", "auto"):
                if direction == "pull" and graph_name == "directed":
                    continue  # pull reads out-lists as in-lists: symmetric graphs only
                depth = torch.empty(v1 - v0, dtype=torch.int32)
                pred = torch.empty(v1 - v0, dtype=torch.int32)
                levels = grd.bfs_partitioned(part, ex, s, depth, pred, direction=direction)
                res.append((depth, pred, levels))
        out[rank] = [(d.numpy().copy(), p.numpy().copy(), L) for d, p, L in res]
    finally:
        dist.destroy_process_group()


def _graph(name):
    if name == "rmat":
        return gg.rmat(10, 8, seed=4)
    if name == "directed":
        return gg.directed_random(700, 4000, seed=2)
    return gg.grid(17, 23)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("graph_name", ["rmat", "directed", "grid"])
def test_partitioned_bfs_world2_gloo(graph_name):
    g = _graph(graph_name)
    srcs = gg.sources(g, 3)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), graph_name, srcs, out), nprocs=2, join=True)
    R, C, _ = g.numpy()
    per_src = 2 if graph_name == "directed" else 3
    for k in range(len(out[0])):
        s = srcs[k // per_src]
        depth = np.concatenate([out[r][k][0] for r in range(2)])
        pred = np.concatenate([out[r][k][1] for r in range(2)])
        ref, _ = oracle.bfs(R, C, s)
        assert np.array_equal(depth, ref)
        assert oracle.check_bfs(R, C, s, depth, pred) == []
        levels = {out[r][k][2] for r in range(2)}
        assert levels == {int(ref.max()) + 1}


def test_owned_ranges_cover_exactly():
    for n in (1, 7, 64, 1000, 33_554_432):
        for P in (1, 2, 3, 8):
            ranges = [grd.owned_range(n, P, r) for r in range(P)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
            B = grd.block_size(n, P)
            assert all(v // B == r for r, (a, b) in enumerate(ranges) for v in (a, b - 1) if b > a)


def test_partition_csr_rows_and_global_columns():
    g = gg.rmat(9, 8, seed=1)
    parts = [grd.partition_csr(g.R, g.C, 3, r) for r in range(3)]
    assert torch.equal(torch.cat([p[3] for p in parts]), g.C)
    for v0, v1, Rl, Cl in parts:
        assert int(Rl[0]) == 0 and int(Rl[-1]) == Cl.numel()
        assert torch.equal(Rl, g.R[v0:v1 + 1] - g.R[v0])
