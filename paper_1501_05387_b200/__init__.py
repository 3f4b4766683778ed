"""Python binding of the B200 frontier library (include/gr.h).

Argument marshalling only: every step of BFS / SSSP runs in the CUDA kernels
of libgr_b200.so. There is NO CPU fallback: if the library cannot be loaded
(not built, no driver, no GPU) every entry point raises GrError.

Low-level functions carry the C names (gr_graph_create, gr_bfs, gr_sssp, ...)
and take raw pointers; `Graph` is a convenience wrapper that accepts torch
tensors (device or host) or numpy arrays and returns torch tensors.
PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("GR_LIB", "libgr_b200.so"))  # GR_LIB: tuning builds

GR_OK = 0
GR_SYMMETRIC = 1
GR_VALIDATE = 4
STATUS = {0: "GR_OK", 1: "GR_ERR_INVALID_ARGUMENT", 2: "GR_ERR_INVALID_GRAPH",
          3: "GR_ERR_OUT_OF_RANGE", 4: "GR_ERR_NO_WEIGHTS", 5: "GR_ERR_OVERFLOW",
          6: "GR_ERR_OUT_OF_MEMORY", 7: "GR_ERR_CUDA", 8: "GR_ERR_NCCL"}
DIRECTION = {"auto": 0, "push": 1, "pull": 2}
STRATEGY = {"auto": 0, "twc": 1, "lb": 2}
UINT32_MAX = 0xFFFFFFFF


class GrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class gr_bfs_opts(ctypes.Structure):
    _fields_ = [("direction", ctypes.c_int32), ("strategy", ctypes.c_int32),
                ("idempotent", ctypes.c_int32), ("switch_rule", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("lb_threshold", ctypes.c_int64)]


class gr_sssp_opts(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_uint32), ("strategy", ctypes.c_int32), ("direction", ctypes.c_int32),
                ("alpha", ctypes.c_double)]


class gr_bc_opts(ctypes.Structure):
    _fields_ = [("direction", ctypes.c_int32), ("alpha", ctypes.c_double)]


class gr_graph_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("max_degree", ctypes.c_int64),
                ("nonisolated", ctypes.c_int64), ("symmetric", ctypes.c_int32),
                ("has_weights", ctypes.c_int32), ("max_weight", ctypes.c_uint32),
                ("device", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
                ("packed_weights", ctypes.c_int32), ("bounded_degree", ctypes.c_int32)]


class gr_level_stats(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("direction", ctypes.c_int32),
                ("frontier", ctypes.c_int64), ("frontier_edges", ctypes.c_int64),
                ("discovered", ctypes.c_int64), ("inspected_edges", ctypes.c_int64),
                ("aux", ctypes.c_int64), ("ns", ctypes.c_int64)]


class gr_run_stats(ctypes.Structure):
    _fields_ = [("num_levels", ctypes.c_int32), ("num_records", ctypes.c_int32),
                ("levels", ctypes.POINTER(gr_level_stats)), ("reached", ctypes.c_int64),
                ("delta", ctypes.c_uint32), ("kernel_launches", ctypes.c_int32),
                ("reached_edges", ctypes.c_int64)]


_lib = None
EXPORTS = ["gr_graph_create", "gr_graph_destroy", "gr_graph_set_stream", "gr_graph_info_get",
           "gr_bfs", "gr_sssp", "gr_bfs_async", "gr_sssp_async", "gr_graph_sync",
           "gr_get_run_stats", "gr_last_error", "gr_kernel_launch_count",
           "gr_version", "gr_bc", "gr_bc_ex", "gr_cc", "gr_pagerank",
           "gr_comm_get_unique_id", "gr_comm_create", "gr_comm_create_loopback", "gr_comm_destroy",
           "gr_comm_info", "gr_graph_create_partitioned"]


def load(path: str = LIB_PATH):
    """Load libgr_b200.so (raises GrError if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GrError(7, "CUDA library %s is not built (run __graft_entry__.build())" % path)
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:
        raise GrError(7, "cannot load %s: %s" % (path, e))
    p = ctypes.c_void_p
    P = ctypes.POINTER
    lib.gr_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, p, p, p, ctypes.c_uint32,
                                    ctypes.c_int, p, P(p)]
    lib.gr_graph_destroy.argtypes = [p]
    lib.gr_graph_set_stream.argtypes = [p, p]
    lib.gr_graph_info_get.argtypes = [p, P(gr_graph_info)]
    lib.gr_bfs.argtypes = [p, ctypes.c_int32, p, p, P(gr_bfs_opts)]
    lib.gr_sssp.argtypes = [p, ctypes.c_int32, p, p, P(gr_sssp_opts)]
    lib.gr_bfs_async.argtypes = [p, ctypes.c_int32, p, p, P(gr_bfs_opts)]
    lib.gr_sssp_async.argtypes = [p, ctypes.c_int32, p, p, P(gr_sssp_opts)]
    lib.gr_graph_sync.argtypes = [p]
    lib.gr_get_run_stats.argtypes = [p, P(gr_run_stats)]
    lib.gr_last_error.restype = ctypes.c_char_p
    lib.gr_kernel_launch_count.restype = ctypes.c_uint64
    lib.gr_version.restype = ctypes.c_char_p
    i64, i32 = ctypes.c_int64, ctypes.c_int32
    lib.gr_bc.argtypes = [p, p, i64, p, p]
    lib.gr_bc_ex.argtypes = [p, p, i64, p, p, P(gr_bc_opts)]
    lib.gr_cc.argtypes = [p, p, P(i64)]
    lib.gr_pagerank.argtypes = [p, ctypes.c_double, ctypes.c_double, i32, p, P(i32)]
    lib.gr_comm_get_unique_id.argtypes = [p]
    lib.gr_comm_create.argtypes = [ctypes.c_int, ctypes.c_int, p, ctypes.c_int, P(p)]
    lib.gr_comm_create_loopback.argtypes = [ctypes.c_int, ctypes.c_int, p]
    lib.gr_comm_destroy.argtypes = [p]
    lib.gr_comm_info.argtypes = [p, P(i32), P(i32), P(i32)]
    lib.gr_graph_create_partitioned.argtypes = [p, i64, i64, i64, i64, p, p, p, ctypes.c_uint32, p, P(p)]
    for f in ("gr_graph_create", "gr_graph_destroy", "gr_graph_set_stream", "gr_graph_info_get",
              "gr_bfs", "gr_sssp", "gr_bfs_async", "gr_sssp_async", "gr_graph_sync",
              "gr_get_run_stats", "gr_bc", "gr_bc_ex", "gr_cc", "gr_pagerank",
              "gr_comm_get_unique_id", "gr_comm_create", "gr_comm_create_loopback", "gr_comm_destroy",
              "gr_comm_info", "gr_graph_create_partitioned"):
        getattr(lib, f).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status):
    if status != GR_OK:
        raise GrError(status, load().gr_last_error().decode(errors="replace"))


# ----------------------------------------------------------------- C-named API

def gr_graph_create(n, m, row_offsets, col_indices, weights, flags, device, stream):
    h = ctypes.c_void_p()
    _check(load().gr_graph_create(n, m, row_offsets, col_indices, weights, flags, device,
                                  stream, ctypes.byref(h)))
    return h


def gr_graph_destroy(h):
    _check(load().gr_graph_destroy(h))


def gr_bfs(h, src, depth_ptr, pred_ptr, opts: Optional[gr_bfs_opts] = None):
    _check(load().gr_bfs(h, int(src), depth_ptr, pred_ptr,
                         ctypes.byref(opts) if opts is not None else None))


def gr_sssp(h, src, dist_ptr, pred_ptr, opts: Optional[gr_sssp_opts] = None):
    _check(load().gr_sssp(h, int(src), dist_ptr, pred_ptr,
                          ctypes.byref(opts) if opts is not None else None))


def gr_bfs_async(h, src, depth_ptr, pred_ptr, opts: Optional[gr_bfs_opts] = None):
    _check(load().gr_bfs_async(h, int(src), depth_ptr, pred_ptr,
                               ctypes.byref(opts) if opts is not None else None))


def gr_sssp_async(h, src, dist_ptr, pred_ptr, opts: Optional[gr_sssp_opts] = None):
    _check(load().gr_sssp_async(h, int(src), dist_ptr, pred_ptr,
                                ctypes.byref(opts) if opts is not None else None))


def gr_graph_sync(h):
    _check(load().gr_graph_sync(h))


def gr_get_run_stats(h):
    st = gr_run_stats()
    _check(load().gr_get_run_stats(h, ctypes.byref(st)))
    return st


def gr_graph_info_get(h):
    info = gr_graph_info()
    _check(load().gr_graph_info_get(h, ctypes.byref(info)))
    return info


def gr_kernel_launch_count() -> int:
    return int(load().gr_kernel_launch_count())


def gr_version() -> str:
    return load().gr_version().decode()


def gr_last_error() -> str:
    return load().gr_last_error().decode(errors="replace")


# ----------------------------------------------------------------- convenience

def _ptr(x):
    """(pointer, keepalive) for a torch tensor / numpy array / None."""
    if x is None:
        return None, None
    import numpy as np
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x)
        return x.ctypes.data, x
    assert x.is_contiguous(), "tensor must be contiguous"
    return x.data_ptr(), x


class Graph:
    """A graph resident on one GPU. R int64[n+1], C int32[m], W uint32/int32[m].

    Inputs may be torch tensors (host or device) or numpy arrays.
    """

    def __init__(self, R, C, W=None, *, symmetric: bool = True, validate: bool = True,
                 device: Optional[int] = None, stream=None):
        import torch
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        n = int(R.shape[0]) - 1
        m = int(C.shape[0])
        rp, rk = _ptr(R)
        cp, ck = _ptr(C)
        wp, wk = _ptr(W)
        flags = (GR_SYMMETRIC if symmetric else 0) | (GR_VALIDATE if validate else 0)
        self.n, self.m = n, m
        self.handle = gr_graph_create(n, m, rp, cp, wp, flags, self.device,
                                      ctypes.c_void_p(stream.cuda_stream))
        self._keep = (rk, ck, wk)

    def close(self):
        if getattr(self, "handle", None) is not None:
            gr_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> gr_graph_info:
        return gr_graph_info_get(self.handle)

    def bfs(self, src: int, depth=None, pred=None, *, want_pred: bool = True,
            direction="auto", strategy="auto", idempotent: bool = False,
            switch_rule: int = 0, alpha: float = 0.0, beta: float = 0.0, lb_threshold: int = 0,
            asynchronous: bool = False):
        """BFS from src. asynchronous=True enqueues only (device outputs; see sync())."""
        import torch
        dev = torch.device("cuda", self.device)
        if depth is None:
            depth = torch.empty(self.n, dtype=torch.int32, device=dev)
        if pred is None and want_pred:
            pred = torch.empty(self.n, dtype=torch.int32, device=dev)
        o = gr_bfs_opts(DIRECTION.get(direction, direction), STRATEGY.get(strategy, strategy),
                        int(idempotent), int(switch_rule), float(alpha), float(beta),
                        int(lb_threshold))
        dp, _ = _ptr(depth)
        pp, _ = _ptr(pred)
        (gr_bfs_async if asynchronous else gr_bfs)(self.handle, src, dp, pp, o)
        return depth, pred

    def sssp(self, src: int, dist=None, pred=None, *, want_pred: bool = True,
             delta: int = 0, strategy="auto", direction="auto", alpha: float = 0.0,
             asynchronous: bool = False):
        import torch
        dev = torch.device("cuda", self.device)
        if dist is None:
            dist = torch.empty(self.n, dtype=torch.int32, device=dev)  # uint32 bits
        if pred is None and want_pred:
            pred = torch.empty(self.n, dtype=torch.int32, device=dev)
        o = gr_sssp_opts(int(delta) & 0xFFFFFFFF, STRATEGY.get(strategy, strategy),
                         DIRECTION.get(direction, direction), float(alpha))
        dp, _ = _ptr(dist)
        pp, _ = _ptr(pred)
        (gr_sssp_async if asynchronous else gr_sssp)(self.handle, src, dp, pp, o)
        return dist, pred

    def bc(self, sources, bc=None, sigma=None, direction="auto", alpha: float = 0.0):
        """Betweenness centrality (Brandes): bc[v] = sum over the
        given sources s of the dependency delta_s(v) (fp64; no halving -- for
        a symmetric graph over all sources Brandes's value is bc / 2)."""
        import numpy as np
        import torch
        src = np.ascontiguousarray(np.asarray(list(sources), dtype=np.int32))
        if bc is None:
            bc = torch.empty(self.n, dtype=torch.float64, device=torch.device("cuda", self.device))
        bp, _ = _ptr(bc)
        sp, _ = _ptr(sigma)
        o = gr_bc_opts(DIRECTION.get(direction, direction), float(alpha))
        _check(load().gr_bc_ex(self.handle, src.ctypes.data_as(ctypes.c_void_p), int(src.size), bp, sp,
                               ctypes.byref(o)))
        return bc

    def cc(self, comp=None):
        """Connected components: (comp, count), comp[v] = the
        smallest vertex id of v's (weak) component."""
        import torch
        if comp is None:
            comp = torch.empty(self.n, dtype=torch.int32, device=torch.device("cuda", self.device))
        cp, _ = _ptr(comp)
        k = ctypes.c_int64()
        _check(load().gr_cc(self.handle, cp, ctypes.byref(k)))
        return comp, k.value

    def pagerank(self, damping: float = 0.85, tol: float = 1e-10, max_iter: int = 1000, rank=None):
        """PageRank (reading A-23): (rank float64[n], iterations)."""
        import torch
        if rank is None:
            rank = torch.empty(self.n, dtype=torch.float64, device=torch.device("cuda", self.device))
        rp, _ = _ptr(rank)
        it = ctypes.c_int32()
        _check(load().gr_pagerank(self.handle, float(damping), float(tol), int(max_iter), rp, ctypes.byref(it)))
        return rank, it.value

    def sync(self):
        """Wait for the asynchronous runs of this graph; raises on a queue overflow."""
        gr_graph_sync(self.handle)

    def run_stats(self):
        st = gr_get_run_stats(self.handle)
        recs = [st.levels[i] for i in range(st.num_records)]
        return dict(num_levels=st.num_levels, delta=st.delta, kernel_launches=st.kernel_launches,
                    reached=st.reached, reached_edges=st.reached_edges,
                    levels=[dict(level=r.level, direction=r.direction, frontier=r.frontier,
                                 frontier_edges=r.frontier_edges, discovered=r.discovered,
                                 inspected_edges=r.inspected_edges, aux=r.aux, ns=r.ns)
                            for r in recs])


def dist_to_u32(t):
    """View an int32 tensor holding uint32 distances as int64 values in [0, 2^32)."""
    return t.to("cpu").numpy().view("uint32")
