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

GR_SYMMETRIC = 1
GR_VALIDATE = 4
NO_FAR = (1 << 63) - 1   # "no live far entry" (int64 max: all-reducible as int64)


def block_size(n: int, nparts: int) -> int:
    """Vertices per partition, a multiple of 32 (bitmap shards concatenate)."""
    return 32 * ((n + 32 * nparts - 1) // (32 * nparts))


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


def partition_weights(R: torch.Tensor, W: torch.Tensor, nparts: int, rank: int):
    """Weights of the owned block's rows (aligned with partition_csr's C)."""
    n = R.numel() - 1
    v0, v1 = owned_range(n, nparts, rank)
    return W[int(R[v0]):int(R[v1])].contiguous()


class _CudaArray:
    """Wraps a raw device pointer for torch.as_tensor (no copy)."""

    def __init__(self, ptr, n, typestr, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


class GpuPartition:
    """The partition of this rank on one GPU (C ABI gr_graph_create_part)."""

    def __init__(self, R_local, C_local, n_global: int, nparts: int, rank: int, device: int = None,
                 stream=None, validate: bool = True, symmetric: bool = True, W_local=None):
        self.symmetric = symmetric
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
        if W_local is None:
            _check(load().gr_graph_create_part(n_global, nparts, rank, self.v_begin, self.v_end,
                                               int(C_local.numel()), rp, cp,
                                               (GR_VALIDATE if validate else 0) | (GR_SYMMETRIC if symmetric else 0), device,
                                               ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        else:
            wp, wk = _ptr(W_local)
            _check(load().gr_graph_create_part_w(n_global, nparts, rank, self.v_begin, self.v_end,
                                                 int(C_local.numel()), rp, cp, wp,
                                                 (GR_VALIDATE if validate else 0) | (GR_SYMMETRIC if symmetric else 0), device,
                                                 ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self.weighted = W_local is not None
        self._ps = None
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
        # dense levels: this rank's frontier-bitmap shard and the gathered global bitmap
        self.shard_buf = torch.zeros(self.block // 32, dtype=torch.int32, device=dev)
        self.global_buf = torch.zeros(nparts * self.block // 32, dtype=torch.int32, device=dev)
        deg = R_local[1:] - R_local[:-1]
        self.nonisolated_local = int((deg > 0).sum())
        self.m_local = int(C_local.numel())
        self._deg = deg

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

    def order_pull_lists(self, deg_global: torch.Tensor):
        """Pull lists ordered by global neighbour degree (gr_part_order_pull_lists);
        deg_global: device int32[n_global]."""
        assert deg_global.dtype == torch.int32 and deg_global.numel() == self.n_global and deg_global.is_cuda
        _check(load().gr_part_order_pull_lists(self.handle, deg_global.data_ptr()))

    def frontier_dev(self, level: int) -> torch.Tensor:
        """{f, m_f, overflow} of level `level` as a DEVICE int64[3] tensor,
        written on the partition's stream without a host synchronisation
        (gr_part_bfs_frontier_async); the caller all-reduces it."""
        if getattr(self, "_fbuf", None) is None:
            self._fbuf = torch.zeros(3, dtype=torch.int64, device=torch.device("cuda", self.device))
        _check(load().gr_part_bfs_frontier_async(self.handle, level, self._fbuf.data_ptr()))
        return self._fbuf

    def degree(self, v_global: int) -> int:
        """Out-degree of an owned vertex (0 if not owned)."""
        if self.v_begin <= v_global < self.v_end:
            return int(self._deg[v_global - self.v_begin])
        return 0

    def shard(self, level: int) -> torch.Tensor:
        _check(load().gr_part_bfs_shard(self.handle, level, self.shard_buf.data_ptr()))
        return self.shard_buf

    def pull(self, level: int, global_bits: torch.Tensor):
        _check(load().gr_part_bfs_pull(self.handle, level, global_bits.data_ptr()))

    # ---- partitioned SSSP (gr_part_sssp_*) -----------------
    def sssp_begin(self, src: int, dist: torch.Tensor, pred: torch.Tensor = None):
        """dist: int32 device tensor holding uint32 bits [n_local]; pred int32 or None."""
        _check(load().gr_part_sssp_begin(self.handle, int(src), dist.data_ptr(),
                                         pred.data_ptr() if pred is not None else None))
        if self._ps is None:
            st, sc, rv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
            blk = ctypes.c_int64()
            _check(load().gr_part_sssp_buffers(self.handle, ctypes.byref(st), ctypes.byref(sc),
                                               ctypes.byref(rv), ctypes.byref(blk)))
            dev = torch.device("cuda", self.device)
            P, B = self.nparts, blk.value
            self._ps = (torch.as_tensor(_CudaArray(st.value, 3 * P * B, "<i4", self.device), device=dev),
                        torch.as_tensor(_CudaArray(rv.value, 3 * P * B, "<i4", self.device), device=dev))
        self.send_triples, self.recv_triples = self._ps

    def sssp_relax(self, step: int, it: int, fp: int, thr: int):
        _check(load().gr_part_sssp_relax(self.handle, step, it, fp, thr))

    def sssp_absorb(self, step: int, it: int, fp: int, thr: int, triples: torch.Tensor, nrecv: int):
        if nrecv:
            _check(load().gr_part_sssp_absorb(self.handle, step, it, fp, thr, triples.data_ptr(), int(nrecv)))

    def sssp_counts(self, step: int, fp: int):
        f, fc = ctypes.c_int64(), ctypes.c_int64()
        _check(load().gr_part_sssp_counts(self.handle, step, fp, ctypes.byref(f), ctypes.byref(fc)))
        return f.value, fc.value

    def sssp_counts_dev(self, step: int, fp: int) -> torch.Tensor:
        """{near, far, overflow} as a DEVICE int64[3] tensor, no host sync
        (gr_part_sssp_counts_async); the caller all-reduces it."""
        if getattr(self, "_cbuf", None) is None:
            self._cbuf = torch.zeros(3, dtype=torch.int64, device=torch.device("cuda", self.device))
        _check(load().gr_part_sssp_counts_async(self.handle, step, fp, self._cbuf.data_ptr()))
        return self._cbuf

    def sssp_far_min(self, step: int, fp: int, thr: int) -> int:
        mn = ctypes.c_uint64()
        _check(load().gr_part_sssp_far_min(self.handle, step, fp, thr, ctypes.byref(mn)))
        return mn.value if mn.value != (1 << 64) - 1 else NO_FAR

    def sssp_resplit(self, step: int, it: int, fp: int, thr_old: int, thr: int):
        _check(load().gr_part_sssp_resplit(self.handle, step, it, fp, thr_old, thr))

    def sssp_end(self):
        _check(load().gr_part_sssp_end(self.handle))


def global_degrees(part, exchange) -> torch.Tensor:
    """int32[n_global] out-degree of every global vertex on this rank's device:
    the all-gather of every rank's local degrees (blocks are padded to
    `block`, the padding sliced off)."""
    dev = torch.device("cuda", part.device) if isinstance(part.device, int) else part.device
    loc = torch.zeros(part.block, dtype=torch.int32, device=dev)
    loc[: part.n_local] = part._deg.to(device=dev, dtype=torch.int32)
    out = torch.empty(part.nparts * part.block, dtype=torch.int32, device=dev)
    exchange.allgather(loc, out)
    return out[: part.n_global].contiguous()


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

    def allreduce_min(self, x: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(x, op=self.dist.ReduceOp.MIN, group=self.group)
        return x

    def allgather(self, shard: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        try:
            self.dist.all_gather_into_tensor(out, shard, group=self.group)
        except (RuntimeError, NotImplementedError):  # backends without the fused variant
            parts = list(out.chunk(self.dist.get_world_size(self.group)))
            self.dist.all_gather(parts, shard, group=self.group)
        return out


def _gather_buckets(part, send_counts_host: Sequence[int]):
    """Concatenate the used part of every peer bucket (pairs, flat int32)."""
    B = part.block
    pieces = [part.send_pairs[2 * q * B: 2 * q * B + 2 * int(c)] for q, c in enumerate(send_counts_host)]
    return torch.cat(pieces) if pieces else part.send_pairs[:0]


def decide_direction(direction: str, cur: str, f: int, mf: int, u: int, m_u: int, prev_f: int,
                     n: int, nonisolated: int, alpha: float = 14.0, beta: float = 24.0) -> str:
    """Beamer's rule on GLOBAL counters (reading A-3; same rule as the
    single-GPU kernel): push->pull when m_f > m_u/alpha and m_f >= n/32,
    pull->push when f < nonisolated/beta and the frontier shrinks."""
    if direction in ("push", "pull"):
        return direction
    if cur == "push":
        return "pull" if (mf > m_u / alpha and mf >= (n + 31) // 32) else "push"
    return "push" if (f < nonisolated / beta and f < prev_f) else "pull"


def _global_frontier(part, exchange, level: int, dev):
    """Global (f, m_f) of `level`: the local counters are summed over ranks on
    the device and read with ONE host synchronisation (the partition's
    frontier_dev when it has one; otherwise its host frontier())."""
    fd = getattr(part, "frontier_dev", None)
    if fd is not None:
        loc = fd(level).clone()
    else:
        lf, lmf = part.frontier(level)
        loc = torch.tensor([lf, lmf, 0], dtype=torch.int64, device=dev)
    f, mf, ov = exchange.allreduce_sum(loc).tolist()
    if ov:
        raise GrError(5, "overflow on some rank (local frontier queue overflow or a received "
                         "vertex the rank does not own)")  # 5 = GR_ERR_OVERFLOW
    return f, mf


def bfs_partitioned(part, exchange, src: int, depth: torch.Tensor, pred: torch.Tensor = None,
                    direction: str = "auto", max_levels: int = 1 << 30, trace: list = None):
    """Runs one BFS over the partition of this rank (all ranks call it with the
    same arguments). Sparse levels push + all-to-all; dense levels all-gather
    the frontier bitmap and pull. Returns the number of levels."""
    dev = depth.device
    part.begin(src, depth, pred)
    dsrc = part.degree(src)
    f, mf = part.frontier(0)
    init = torch.tensor([f, mf, part.nonisolated_local - (1 if dsrc > 0 else 0), part.m_local - dsrc,
                         part.nonisolated_local], dtype=torch.int64, device=dev)
    init = exchange.allreduce_sum(init).tolist()
    f, mf, u, m_u, nonisolated = init
    n = part.n_global
    level, cur, prev_f = 0, "push", 0
    if not getattr(part, "symmetric", True):
        direction = "push"  # pull reads out-lists as in-lists: symmetric graphs only
    while f > 0 and level < max_levels:
        cur = decide_direction(direction, cur, f, mf, u, m_u, prev_f, n, nonisolated)
        if trace is not None:
            trace.append((level, cur, f, mf))
        if cur == "push":
            part.expand(level)
            sc = part.send_counts.clone() if part.send_counts.device == dev else part.send_counts.to(dev)
            rc = exchange.counts(sc)
            both = torch.cat([sc, rc]).tolist()  # one host read for both count vectors
            sc_h, rc_h = both[: len(both) // 2], both[len(both) // 2:]
            send_flat = _gather_buckets(part, sc_h)
            nrecv = int(sum(rc_h))
            out = part.recv_pairs[: 2 * nrecv]
            exchange.pairs(send_flat, out, [2 * c for c in sc_h], [2 * c for c in rc_h])
            part.absorb(level, out, nrecv)
        else:
            shard = part.shard(level)
            exchange.allgather(shard, part.global_buf)
            part.pull(level, part.global_buf)
        level += 1
        prev_f = f
        f, mf = _global_frontier(part, exchange, level, dev)
        u -= f  # symmetric graphs: every discovered vertex has out-degree > 0
        m_u -= mf
    return level


def next_threshold(mn: int, delta: int) -> int:
    """Band jump of the far re-split (reading A-11): the threshold
    moves to the end of the delta-band holding the minimum far distance."""
    return (mn // delta + 1) * delta


def _global_near(part, exchange, step: int, fp: int, dev) -> int:
    """Global near-queue size of `step`: local counters summed over ranks on
    the device, one host read (sssp_counts_dev when the partition has it)."""
    cd = getattr(part, "sssp_counts_dev", None)
    if cd is not None:
        loc = cd(step, fp).clone()
    else:
        loc = torch.tensor([part.sssp_counts(step, fp)[0], 0, 0], dtype=torch.int64, device=dev)
    near, _, ov = exchange.allreduce_sum(loc).tolist()
    if ov:
        raise GrError(5, "overflow on some rank (a near/far queue exceeded its capacity or a received "
                         "vertex the rank does not own)")  # 5 = GR_ERR_OVERFLOW
    return near


def sssp_partitioned(part, exchange, src: int, dist: torch.Tensor, pred: torch.Tensor = None,
                     delta: int = 1, trace: list = None):
    """Near/far delta-stepping SSSP (Alg. 1) over the 1D
    partition of this rank; every rank calls it with the same arguments.
    Near iterations relax + all-to-all the (vertex, dist, parent) triples +
    absorb; when the near queues are empty on every rank, the far piles are
    re-split at the all-reduced minimum (A-11). Returns the number of steps."""
    if delta < 1:
        raise ValueError("delta must be >= 1")
    dev = dist.device
    part.sssp_begin(src, dist, pred)
    k, it, fp, thr = 0, 0, 0, int(delta)
    f = _global_near(part, exchange, 0, fp, dev)
    while True:
        if f > 0:
            it += 1
            if trace is not None:
                trace.append(("near", k, it, thr, f))
            part.sssp_relax(k, it, fp, thr)
            sc = part.send_counts.clone() if part.send_counts.device == dev else part.send_counts.to(dev)
            rc = exchange.counts(sc)
            both = torch.cat([sc, rc]).tolist()  # one host read for both count vectors
            sc_h, rc_h = both[: len(both) // 2], both[len(both) // 2:]
            B = part.block
            send_flat = torch.cat([part.send_triples[3 * q * B: 3 * q * B + 3 * int(c)]
                                   for q, c in enumerate(sc_h)])
            nrecv = int(sum(rc_h))
            out = part.recv_triples[: 3 * nrecv]
            exchange.pairs(send_flat, out, [3 * c for c in sc_h], [3 * c for c in rc_h])
            part.sssp_absorb(k, it, fp, thr, out, nrecv)
        else:
            mn = part.sssp_far_min(k, fp, thr)
            mn = int(exchange.allreduce_min(torch.tensor([mn], dtype=torch.int64, device=dev)).item())
            if mn == NO_FAR:
                break
            thr_old, thr = thr, next_threshold(mn, int(delta))
            it += 1
            if trace is not None:
                trace.append(("resplit", k, it, thr, mn))
            part.sssp_resplit(k, it, fp, thr_old, thr)
            fp ^= 1
        k += 1
        f = _global_near(part, exchange, k, fp, dev)
    part.sssp_end()
    return k


class LoopbackGroup:
    """P partitions in ONE process (one GPU): the exchange is a device copy.
    Tests the partition kernels' routing without a second GPU."""

    def __init__(self, parts):
        self.parts = parts

    def bfs(self, src: int, depths, preds, direction: str = "auto"):
        P = len(self.parts)
        for q, pt in enumerate(self.parts):
            pt.begin(src, depths[q], preds[q] if preds else None)
        dsrc = sum(pt.degree(src) for pt in self.parts)
        f = sum(pt.frontier(0)[0] for pt in self.parts)
        mf = sum(pt.frontier(0)[1] for pt in self.parts)
        nonisolated = sum(pt.nonisolated_local for pt in self.parts)
        u = nonisolated - (1 if dsrc > 0 else 0)
        m_u = sum(pt.m_local for pt in self.parts) - dsrc
        n = self.parts[0].n_global
        level, cur, prev_f = 0, "push", 0
        self.dirs = []
        if not all(getattr(pt, "symmetric", True) for pt in self.parts):
            direction = "push"
        while f > 0:
            cur = decide_direction(direction, cur, f, mf, u, m_u, prev_f, n, nonisolated)
            self.dirs.append(cur)
            if cur == "push":
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
                    self.parts[dst].recv_pairs[: flat.numel()].copy_(flat)
                    self.parts[dst].absorb(level, self.parts[dst].recv_pairs, flat.numel() // 2)
            else:
                gathered = torch.cat([pt.shard(level).clone() for pt in self.parts])
                for pt in self.parts:
                    pt.pull(level, gathered)
            level += 1
            prev_f = f
            f = sum(pt.frontier(level)[0] for pt in self.parts)
            mf = sum(pt.frontier(level)[1] for pt in self.parts)
            u -= f
            m_u -= mf
        return level

    def sssp(self, src: int, dists, preds, delta: int = 1):
        """Partitioned SSSP of all partitions in this process (device-copy exchange)."""
        P = len(self.parts)
        for q, pt in enumerate(self.parts):
            pt.sssp_begin(src, dists[q], preds[q] if preds else None)
        k, it, fp, thr = 0, 0, 0, int(delta)
        f = sum(pt.sssp_counts(0, fp)[0] for pt in self.parts)
        while True:
            if f > 0:
                it += 1
                for pt in self.parts:
                    pt.sssp_relax(k, it, fp, thr)
                counts = [pt.send_counts.tolist() for pt in self.parts]
                for dst in range(P):
                    pieces = [self.parts[s].send_triples[3 * dst * self.parts[s].block:
                                                         3 * dst * self.parts[s].block + 3 * counts[s][dst]]
                              for s in range(P)]
                    flat = torch.cat(pieces)
                    self.parts[dst].recv_triples[: flat.numel()].copy_(flat)
                    self.parts[dst].sssp_absorb(k, it, fp, thr, self.parts[dst].recv_triples, flat.numel() // 3)
            else:
                mn = min(pt.sssp_far_min(k, fp, thr) for pt in self.parts)
                if mn == NO_FAR:
                    break
                thr_old, thr = thr, next_threshold(mn, int(delta))
                it += 1
                for pt in self.parts:
                    pt.sssp_resplit(k, it, fp, thr_old, thr)
                fp ^= 1
            k += 1
            f = sum(pt.sssp_counts(k, fp)[0] for pt in self.parts)
        for pt in self.parts:
            pt.sssp_end()
        return k
