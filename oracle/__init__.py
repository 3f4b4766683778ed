"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package. It shares no code with the
CUDA path (paper_1501_05387_b200/) and never imports it.

Contents
--------
* bfs(R, C, src)        -> (depth int32[n], pred int32[n])  FIFO-queue BFS (oracle.c)
* sssp(R, C, W, src)    -> (dist uint32[n], pred int32[n])  binary-heap Dijkstra (oracle.c)
* bc(R, C, sources)     -> float64[n]  Brandes 2001 Algorithm 1 (oracle.c)
* cc(R, C)              -> (comp int32[n], count)  union-find, min id per component
* pagerank(R, C, d)     -> float64[n]  Jacobi power iteration in numpy (reading A-23)
* check_bfs / check_sssp -- O(m) certificates: they decide
  exactness of depth / dist without any reference output, and validate any
  predecessor array (pred is "any valid parent": parity-unpinned by design,
  pinned only by these invariants).
* reached_edges(R, depth) -- the TEPS numerator m_reached (reading A-14).

Pins: tests/test_oracle_pins.py checks this oracle against values printed in
SPEC.md's worked examples, closed forms, brute force on tiny graphs and scipy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

UINT32_MAX = 0xFFFFFFFF


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no vectorisation tricks needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        p = ctypes.c_void_p
        lib.oracle_bfs.argtypes = [ctypes.c_int64, p, p, ctypes.c_int32, p, p]
        lib.oracle_bfs.restype = ctypes.c_int
        lib.oracle_sssp.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int32, p, p]
        lib.oracle_sssp.restype = ctypes.c_int
        lib.oracle_bc.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int64, p]
        lib.oracle_bc.restype = ctypes.c_int
        lib.oracle_cc.argtypes = [ctypes.c_int64, p, p, p, p]
        lib.oracle_cc.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _as(a, dt):
    return np.ascontiguousarray(np.asarray(a), dtype=dt)


def bfs(R, C, src: int, want_pred: bool = True):
    R = _as(R, np.int64)
    C = _as(C, np.int32)
    n = R.size - 1
    depth = np.empty(n, np.int32)
    pred = np.empty(n, np.int32) if want_pred else None
    rc = _load().oracle_bfs(n, _ptr(R), _ptr(C), int(src), _ptr(depth), _ptr(pred))
    if rc != 0:
        raise ValueError("oracle_bfs failed with code %d" % rc)
    return depth, pred


def sssp(R, C, W, src: int, want_pred: bool = True):
    R = _as(R, np.int64)
    C = _as(C, np.int32)
    W = _as(W, np.uint32)
    n = R.size - 1
    dist = np.empty(n, np.uint32)
    pred = np.empty(n, np.int32) if want_pred else None
    rc = _load().oracle_sssp(n, _ptr(R), _ptr(C), _ptr(W), int(src), _ptr(dist), _ptr(pred))
    if rc == 3:
        raise OverflowError("a shortest distance does not fit in uint32")
    if rc != 0:
        raise ValueError("oracle_sssp failed with code %d" % rc)
    return dist, pred


def bc(R, C, sources):
    """Sum over `sources` of Brandes's dependency delta_s(v) (no halving)."""
    R = _as(R, np.int64)
    C = _as(C, np.int32)
    S = _as(list(sources), np.int32)
    n = R.size - 1
    out = np.empty(n, np.float64)
    rc = _load().oracle_bc(n, _ptr(R), _ptr(C), _ptr(S), int(S.size), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_bc failed with code %d" % rc)
    return out


def cc(R, C):
    """(comp, count): comp[v] = smallest vertex id of v's weakly connected component."""
    R = _as(R, np.int64)
    C = _as(C, np.int32)
    n = R.size - 1
    comp = np.empty(n, np.int32)
    k = np.zeros(1, np.int64)
    rc = _load().oracle_cc(n, _ptr(R), _ptr(C), _ptr(comp), _ptr(k))
    if rc != 0:
        raise ValueError("oracle_cc failed with code %d" % rc)
    return comp, int(k[0])


def pagerank(R, C, damping: float = 0.85, tol: float = 1e-15, max_iter: int = 100000):
    """PR(v) = (1-d)/n + d * sum over edges (u,v) of PR(u)/outdeg(u), start 1/n,
    no dangling redistribution (paper §5.5; reading A-23).
    Plain Jacobi power iteration in fp64 until max |PR_new - PR| <= tol * max PR."""
    R = _as(R, np.int64)
    C = _as(C, np.int64)
    n = R.size - 1
    outdeg = np.diff(R)
    src = np.repeat(np.arange(n), outdeg)
    x = np.full(n, 1.0 / n)
    for _ in range(max_iter):
        share = np.zeros(n)
        nz = outdeg > 0
        share[nz] = x[nz] / outdeg[nz]
        y = (1.0 - damping) / n + damping * np.bincount(C, weights=share[src], minlength=n)
        done = np.abs(y - x).max() <= tol * y.max()
        x = y
        if done:
            break
    return x


# ---------------------------------------------------------------------------
# O(m) certificates. Each returns a list of violated
# conditions (empty list == certificate holds).
# ---------------------------------------------------------------------------

def _edge_src(R):
    return np.repeat(np.arange(R.size - 1, dtype=np.int64), np.diff(R))


def check_bfs(R, C, src: int, depth, pred=None):
    """BFS certificate. (i) depth[src]=0 and only src has depth 0;
    (ii) every edge (u,v) with depth[u]>=0 has 0 <= depth[v] <= depth[u]+1;
    (iii) every reached v != src has (pred[v], v) in E with
          depth[pred[v]] = depth[v]-1, and pred[src] = src;
    (iv) depth = -1 <=> pred = -1.
    (ii) gives depth <= true distance, (iii) gives a walk of exactly depth[v]
    edges, so together they certify exact hop distances."""
    R = _as(R, np.int64); C = _as(C, np.int64); depth = _as(depth, np.int64)
    n = R.size - 1
    errs = []
    if depth[src] != 0:
        errs.append("depth[src] != 0")
    if np.count_nonzero(depth == 0) != 1:
        errs.append("more than one vertex with depth 0")
    if np.any(depth < -1):
        errs.append("depth < -1")
    s = _edge_src(R)
    du = depth[s]
    dv = depth[C]
    live = du >= 0
    bad = live & ((dv < 0) | (dv > du + 1))
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        errs.append("edge (%d,%d): depth %d -> %d violates depth[v] <= depth[u]+1"
                    % (s[i], C[i], du[i], dv[i]))
    if pred is not None:
        pred = _as(pred, np.int64)
        if pred[src] != src:
            errs.append("pred[src] != src")
        if np.any((depth == -1) != (pred == -1)):
            errs.append("depth == -1 and pred == -1 disagree")
        reached = np.flatnonzero((depth > 0))
        p = pred[reached]
        if np.any((p < 0) | (p >= n)):
            errs.append("pred out of range")
        else:
            if np.any(depth[p] != depth[reached] - 1):
                errs.append("depth[pred[v]] != depth[v]-1")
            # (pred[v], v) must be an edge: look it up in the sorted-or-not list
            if not _edges_exist(R, C, p, reached):
                errs.append("(pred[v], v) is not an edge")
    return errs


def _edges_exist(R, C, us, vs):
    """Vectorised membership test of edges (us[i], vs[i]) in the CSR."""
    if us.size == 0:
        return True
    n = R.size - 1
    key_all = _edge_src(R) * n + C
    key_all = np.sort(key_all)
    key = us.astype(np.int64) * n + vs.astype(np.int64)
    pos = np.searchsorted(key_all, key)
    pos = np.minimum(pos, key_all.size - 1)
    return bool(np.all(key_all[pos] == key))


def check_sssp(R, C, W, src: int, dist, pred=None):
    """SSSP certificate. (i) dist[src]=0; (ii) dist[v] <= dist[u]+w for every
    edge with dist[u] finite (feasibility); (iii) every reached v != src has an
    in-edge with dist[u]+w = dist[v] (tightness); pred, if given, must be such
    a tight in-neighbour. (i)-(iii) imply exact distances when every cycle of
    tight edges has positive weight (w >= 1); zero weights are covered by the
    BFS cross-check (iv): dist finite <=> reachable (reading A-17)."""
    R = _as(R, np.int64); C = _as(C, np.int64); W = _as(W, np.int64)
    dist = _as(dist, np.int64)
    INF = UINT32_MAX
    n = R.size - 1
    errs = []
    if dist[src] != 0:
        errs.append("dist[src] != 0")
    s = _edge_src(R)
    du = dist[s]
    dv = dist[C]
    live = du != INF
    if np.any(live & (dv > du + W)):
        i = int(np.flatnonzero(live & (dv > du + W))[0])
        errs.append("edge (%d,%d) w=%d not relaxed: %d > %d + %d"
                    % (s[i], C[i], W[i], dv[i], du[i], W[i]))
    tight = live & (dv == du + W)
    has_tight = np.zeros(n, bool)
    has_tight[C[tight]] = True
    reached = (dist != INF)
    need = reached.copy()
    need[src] = False
    if np.any(need & ~has_tight):
        v = int(np.flatnonzero(need & ~has_tight)[0])
        errs.append("vertex %d (dist %d) has no tight in-edge" % (v, dist[v]))
    depth, _ = bfs(R, C, src, want_pred=False)
    if np.any((depth >= 0) != reached):
        errs.append("finite dist disagrees with reachability")
    if pred is not None:
        pred = _as(pred, np.int64)
        if pred[src] != src:
            errs.append("pred[src] != src")
        if np.any((pred == -1) != ~reached):
            errs.append("pred == -1 disagrees with dist == inf")
        vs = np.flatnonzero(need)
        p = pred[vs]
        if np.any((p < 0) | (p >= n)):
            errs.append("pred out of range")
        elif vs.size:
            # (p, v) must be an edge whose weight makes it tight
            key_all = s * n + C
            order = np.argsort(key_all, kind="stable")
            ks = key_all[order]
            key = p * n + vs
            lo = np.searchsorted(ks, key, side="left")
            hi = np.searchsorted(ks, key, side="right")
            if np.any(lo == hi):
                errs.append("(pred[v], v) is not an edge")
            else:
                # some parallel copy of (p, v) must be tight
                ok = np.zeros(vs.size, bool)
                for k in range(int((hi - lo).max())):
                    idx = np.minimum(lo + k, hi - 1)
                    ok |= (dist[p] + W[order][idx] == dist[vs]) & (lo + k < hi)
                if not ok.all():
                    errs.append("pred edge is not tight")
    return errs


def reached_edges(R, depth_or_dist, unreached) -> int:
    """m_reached: directed edges whose source is reached (TEPS numerator, A-14)."""
    R = _as(R, np.int64)
    x = np.asarray(depth_or_dist)
    deg = np.diff(R)
    return int(deg[x != unreached].sum())
