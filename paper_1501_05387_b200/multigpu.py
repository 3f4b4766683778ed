"""Multi-GPU group and partitioned graph of the C ABI (include/gr.h, SURVEY
§8(b)): argument marshalling only.

    comm = Comm.from_torch()             # one process per GPU, torch.distributed up
    g = PartitionedGraph(comm, R_local, C_local, n_global)
    depth, pred = g.bfs(src)             # collective: every rank calls it

The library owns the NCCL communicator (torch.distributed only broadcasts the
128-byte ncclUniqueId) and runs every level of the partitioned BFS, exchange
included, inside one persistent kernel per rank (csrc/pbfs.cu). Comm.loopback(P)
gives P virtual ranks in this process on one GPU (one launch hosts them all),
which is how the multi-rank path is tested with a single GPU.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional

from . import (DIRECTION, GR_SYMMETRIC, GR_VALIDATE, _check, _ptr, gr_bfs_opts, gr_get_run_stats, gr_sssp_opts,
               load)

GR_KEEP_ORDER = 8


def block_size(n: int, nranks: int) -> int:
    """Vertices per rank, a multiple of 32 (include/gr.h)."""
    return 32 * ((n + 32 * nranks - 1) // (32 * nranks))


def owned_range(n: int, nranks: int, rank: int):
    b = block_size(n, nranks)
    return min(n, rank * b), min(n, (rank + 1) * b)


def partition_csr(R, C, nranks: int, rank: int, W=None):
    """Rows of rank's block with global column ids (and their weights)."""
    n = R.numel() - 1
    v0, v1 = owned_range(n, nranks, rank)
    e0, e1 = int(R[v0]), int(R[v1])
    Wl = None if W is None else W[e0:e1].contiguous()
    return v0, v1, (R[v0:v1 + 1] - e0).contiguous(), C[e0:e1].contiguous(), Wl


def _nccl_unique_id() -> bytes:
    uid = ctypes.create_string_buffer(128)
    _check(load().gr_comm_get_unique_id(uid))
    return uid.raw


def broadcast_unique_id(make_id, group=None) -> bytes:
    """Bootstrap of a gr_comm (the only job torch.distributed has here):
    rank 0 calls make_id() for the 128-byte ncclUniqueId, every rank gets it."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise ValueError("unique id must be 128 bytes")
    return bytes(uid)


class Comm:
    """gr_comm: one (real or loopback) rank of a multi-GPU group."""

    def __init__(self, handle, rank: int, nranks: int, device: int, loopback: bool):
        self.handle, self.rank, self.nranks, self.device, self.loopback = handle, rank, nranks, device, loopback

    @classmethod
    def from_torch(cls, device: Optional[int] = None, group=None) -> "Comm":
        """Every rank of an initialised torch.distributed group calls this."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        uid = broadcast_unique_id(_nccl_unique_id, group)
        buf = ctypes.create_string_buffer(uid, 128)
        h = ctypes.c_void_p()
        _check(load().gr_comm_create(rank, world, buf, int(device), ctypes.byref(h)))
        return cls(h, rank, world, int(device), False)

    @classmethod
    def loopback(cls, nranks: int, device: Optional[int] = None) -> List["Comm"]:
        import torch
        if device is None:
            device = torch.cuda.current_device()
        arr = (ctypes.c_void_p * nranks)()
        _check(load().gr_comm_create_loopback(nranks, int(device), arr))
        return [cls(ctypes.c_void_p(arr[r]), r, nranks, int(device), True) for r in range(nranks)]

    def close(self):
        if getattr(self, "handle", None) is not None:
            _check(load().gr_comm_destroy(self.handle))
            self.handle = None


class PartitionedGraph:
    """This rank's block of a symmetric graph (gr_graph_create_partitioned)."""

    def __init__(self, comm: Comm, R_local, C_local, n_global: int, W_local=None, *, stream=None,
                 validate: bool = True, keep_order: bool = False):
        import torch
        self.comm = comm
        self.n_global = int(n_global)
        self.v_begin, self.v_end = owned_range(self.n_global, comm.nranks, comm.rank)
        self.n_local = self.v_end - self.v_begin
        if stream is None:
            stream = torch.cuda.current_stream(comm.device)
        self.stream = stream
        rp, rk = _ptr(R_local)
        cp, ck = _ptr(C_local)
        wp, wk = _ptr(W_local)
        flags = GR_SYMMETRIC | (GR_VALIDATE if validate else 0) | (GR_KEEP_ORDER if keep_order else 0)
        h = ctypes.c_void_p()
        _check(load().gr_graph_create_partitioned(comm.handle, self.n_global, self.v_begin, self.v_end,
                                                  int(C_local.shape[0]), rp, cp, wp, flags,
                                                  ctypes.c_void_p(stream.cuda_stream), ctypes.byref(h)))
        self.handle = h
        self._keep = (rk, ck, wk)

    def bfs(self, src: int, depth=None, pred=None, *, want_pred: bool = True, direction="auto",
            switch_rule: int = 0, alpha: float = 0.0, beta: float = 0.0):
        """Collective BFS from GLOBAL src; outputs cover the owned block."""
        import torch
        dev = torch.device("cuda", self.comm.device)
        if depth is None:
            depth = torch.empty(self.n_local, dtype=torch.int32, device=dev)
        if pred is None and want_pred:
            pred = torch.empty(self.n_local, dtype=torch.int32, device=dev)
        o = gr_bfs_opts(DIRECTION.get(direction, direction), 0, 0, int(switch_rule), float(alpha), float(beta), 0)
        dp, _ = _ptr(depth)
        pp, _ = _ptr(pred)
        _check(load().gr_bfs(self.handle, int(src), dp, pp, ctypes.byref(o)))
        return depth, pred

    def sssp(self, src: int, dist=None, pred=None, *, want_pred: bool = True, delta: int = 0):
        """Collective SSSP from GLOBAL src (int32 tensor holding uint32 dist bits);
        outputs cover the owned block; delta 0 = auto (reading A-10)."""
        import torch
        dev = torch.device("cuda", self.comm.device)
        if dist is None:
            dist = torch.empty(self.n_local, dtype=torch.int32, device=dev)
        if pred is None and want_pred:
            pred = torch.empty(self.n_local, dtype=torch.int32, device=dev)
        o = gr_sssp_opts(int(delta) & 0xFFFFFFFF, 0, 1, 0.0)
        dp, _ = _ptr(dist)
        pp, _ = _ptr(pred)
        _check(load().gr_sssp(self.handle, int(src), dp, pp, ctypes.byref(o)))
        return dist, pred

    def run_stats(self):
        st = gr_get_run_stats(self.handle)
        recs = [st.levels[i] for i in range(st.num_records)]
        return dict(num_levels=st.num_levels, reached=st.reached, reached_edges=st.reached_edges,
                    kernel_launches=st.kernel_launches, delta=st.delta,
                    levels=[dict(level=r.level, direction=r.direction, frontier=r.frontier,
                                 frontier_edges=r.frontier_edges, discovered=r.discovered,
                                 inspected_edges=r.inspected_edges, aux=r.aux, ns=r.ns) for r in recs])

    def close(self):
        if getattr(self, "handle", None) is not None:
            _check(load().gr_graph_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
