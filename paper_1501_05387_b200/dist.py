"""Multi-GPU BFS over a 1D vertex partition.

One process per GPU. Rank q owns vertices [q*B, min(n, (q+1)*B)), B =
ceil(n/P), and the out-edges of those vertices with global column ids. Per
level (the paper's bulk-synchronous step, extended with an
exchange; multi-GPU itself is the paper's future work):

  1. expand   -- CUDA kernel (gr_part_bfs_expand): local push advance; owned
                 targets claimed locally, remote targets culled by an
                 "already sent" bitmap and bucketed per owner;
  2. exchange -- all-to-all of the bucket sizes, then of the (vertex, parent)
                 pairs: torch.distributed (NCCL over NVLink on GPUs, gloo in
                 the CPU tests) -- plumbing only, no arithmetic of the method;
  3. absorb   -- CUDA kernel (gr_part_bfs_absorb): the owner claims the
                 received vertices;
  4. frontier -- local next-frontier size, all-reduced; stop at 0.

The level driver (`bfs_partitioned`) is written against two small
interfaces -- a partition backend (the C ABI on a GPU) and an exchange -- so
its routing / termination logic is exercised on CPU with gloo at world size 2
(tests/test_dist_gloo.py) and on one GPU with several partitions
(`LoopbackExchange`, tests/test_gpu_dist.py).
"""
from __future__ import annotations

import ctypes
from typing import List, Sequence

import torch

from . import GrError, _check, _ptr, load

GR_VALIDATE = 4


def block_size(n: int, nparts: int) -> int:
    return (n + nparts - 1) // nparts


def owned_range(n: int, nparts: int, rank: int):
    """The 1D block of `rank`: [v_begin, v_end)."""
    b = block_size(n, nparts)
    return min(n, rank * b), min(n, (rank + 1) * b)  # empty when nparts > n (unsupported by the C ABI)


def partition_csr(R: torch.Tensor, C: torch.Tensor, nparts: int, rank: int):
    """Rows of the owned block with global column ids (host logic, any device)."""
    n = R.numel() - 1
    v0, v1 = owned_range(n, nparts, rank)
    e0, e1 = int(R[v0]), int(R[v1])
    return v0, v1, (R[v0:v1 + 1] - e0).contiguous(), C[e0:e1].contiguous()


class _CudaArray:
    """Wraps a raw device pointer for torch.as_tensor (no copy)."""

    def __init__(self, ptr, n, typestr, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


class GpuPartition:
    """The partition of this rank on one GPU (C ABI gr_graph_create_part)."""

    def __init__(self, R_local, C_local, n_global: int, nparts: int, rank: int, device: int = None,
                 stream=None, validate: bool = True):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.n_global, self.nparts, self.rank = n_global, nparts, rank
        self.v_begin, self.v_end = owned_range(n_global, nparts, rank)
        self.n_local = self.v_end - self.v_begin
        assert R_local.numel() == self.n_local + 1
        h = ctypes.c_void_p()
        rp, rk = _ptr(R_local)
        cp, ck = _ptr(C_local)
        _check(load().gr_graph_create_part(n_global, nparts, rank, self.v_begin, self.v_end,
                                           int(C_local.numel()), rp, cp,
                                           GR_VALIDATE if validate else 0, device,
                                           ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self.handle = h
        sp, sc, rv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        blk = ctypes.c_int64()
        _check(load().gr_part_buffers(h, ctypes.byref(sp), ctypes.byref(sc), ctypes.byref(rv),
                                      ctypes.byref(blk)))
        self.block = blk.value
        dev = torch.device("cuda", device)
        self.send_pairs = torch.as_tensor(_CudaArray(sp.value, 2 * nparts * self.block, "<i4", device), device=dev)
        self.send_counts = torch.as_tensor(_CudaArray(sc.value, nparts, "<i8", device), device=dev)
        self.recv_pairs = torch.as_tensor(_CudaArray(rv.value, 2 * n_global, "<i4", device), device=dev)

    def close(self):
        if getattr(self, "handle", None) is not None:
            load().gr_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def begin(self, src: int, depth: torch.Tensor, pred: torch.Tensor):
        _check(load().gr_part_bfs_begin(self.handle, int(src), depth.data_ptr(),
                                        pred.data_ptr() if pred is not None else None))

    def expand(self, level: int):
        _check(load().gr_part_bfs_expand(self.handle, level))

    def absorb(self, level: int, pairs: torch.Tensor, nrecv: int):
        if nrecv:
            _check(load().gr_part_bfs_absorb(self.handle, level, pairs.data_ptr(), int(nrecv)))

    def frontier(self, level: int):
        f, mf = ctypes.c_int64(), ctypes.c_int64()
        _check(load().gr_part_bfs_frontier(self.handle, level, ctypes.byref(f), ctypes.byref(mf)))
        return f.value, mf.value


class TorchDistExchange:
    """Exchange over a torch.distributed process group (NCCL or gloo)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.device = device

    def counts(self, send_counts: torch.Tensor) -> torch.Tensor:
        recv = torch.empty_like(send_counts)
        self.dist.all_to_all_single(recv, send_counts, group=self.group)
        return recv

    def pairs(self, send_flat: torch.Tensor, out: torch.Tensor, in_splits: List[int],
              out_splits: List[int]) -> torch.Tensor:
        self.dist.all_to_all_single(out, send_flat, output_split_sizes=out_splits,
                                    input_split_sizes=in_splits, group=self.group)
        return out

    def allreduce_sum(self, x: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(x, group=self.group)
        return x


def _gather_buckets(part, send_counts_host: Sequence[int]):
    """Concatenate the used part of every peer bucket (pairs, flat int32)."""
    B = part.block
    pieces = [part.send_pairs[2 * q * B: 2 * q * B + 2 * int(c)] for q, c in enumerate(send_counts_host)]
    return torch.cat(pieces) if pieces else part.send_pairs[:0]


def bfs_partitioned(part, exchange, src: int, depth: torch.Tensor, pred: torch.Tensor = None,
                    max_levels: int = 1 << 30):
    """Runs one BFS over the partition of this rank. Returns the number of levels."""
    dev = depth.device
    part.begin(src, depth, pred)
    f, _ = part.frontier(0)
    tot = exchange.allreduce_sum(torch.tensor([f], dtype=torch.int64, device=dev))
    level = 0
    while int(tot[0]) > 0 and level < max_levels:
        part.expand(level)
        sc = part.send_counts.clone() if part.send_counts.device == dev else part.send_counts.to(dev)
        rc = exchange.counts(sc)
        sc_h = sc.tolist()
        rc_h = rc.tolist()
        send_flat = _gather_buckets(part, sc_h)
        nrecv = int(sum(rc_h))
        out = part.recv_pairs[: 2 * nrecv]
        exchange.pairs(send_flat, out, [2 * c for c in sc_h], [2 * c for c in rc_h])
        part.absorb(level, out, nrecv)
        level += 1
        f, _ = part.frontier(level)
        tot = exchange.allreduce_sum(torch.tensor([f], dtype=torch.int64, device=dev))
    return level


class LoopbackGroup:
    """P partitions in ONE process (one GPU): the exchange is a device copy.
    Tests the partition kernels' routing without a second GPU."""

    def __init__(self, parts):
        self.parts = parts

    def bfs(self, src: int, depths, preds):
        P = len(self.parts)
        dev = depths[0].device
        for q, pt in enumerate(self.parts):
            pt.begin(src, depths[q], preds[q] if preds else None)
        level = 0
        tot = sum(pt.frontier(0)[0] for pt in self.parts)
        while tot > 0:
            for pt in self.parts:
                pt.expand(level)
            counts = [pt.send_counts.tolist() for pt in self.parts]  # counts[src_rank][dst_rank]
            for dst in range(P):
                pieces = []
                for s in range(P):
                    c = counts[s][dst]
                    B = self.parts[s].block
                    pieces.append(self.parts[s].send_pairs[2 * dst * B: 2 * dst * B + 2 * c])
                flat = torch.cat(pieces)
                n = flat.numel() // 2
                self.parts[dst].recv_pairs[: flat.numel()].copy_(flat)
                self.parts[dst].absorb(level, self.parts[dst].recv_pairs, n)
            level += 1
            tot = sum(pt.frontier(level)[0] for pt in self.parts)
        return level
