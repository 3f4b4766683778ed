"""Seeded synthetic graph inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no BFS, no shortest paths, no
frontier logic). It only draws graphs, weights and sources, the way the
paper's experiments prepared theirs:

* "we converted all datasets to undirected graphs" (PAPER.md P:1093-1094,
  §6) -> every generator symmetrises, drops self-loops and collapses
  duplicate edges (reading A-13);
* "edge weight values ... random values between 1 and 64"
  -> integer weights uniform on [1, 64], symmetric w(u,v) = w(v,u) (A-12);
* Table 1 fixes the SHAPES the synthetic stand-ins imitate
  (kron_g500-logn21, soc-orkut, a road network); the recipe is in DESIGN.md
  "Input recipe".

Determinism across devices: every random draw is a counter-based 32-bit hash
evaluated with int64 torch ops whose intermediate products stay below 2**63,
and every sort/unique is on distinct integer keys, so the same call gives the
bit-identical CSR on CPU and on CUDA (tests/test_graphgen.py checks this on
CPU against numpy re-evaluation). Graphs are returned as torch tensors on the
requested device; callers move them where they need them.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import torch

M32 = (1 << 32) - 1
_MUL = 0x45D9F3B  # < 2**31, so (x < 2**32) * _MUL < 2**63: no int64 overflow


def _mix32(x: torch.Tensor) -> torch.Tensor:
    """Bijective 32-bit integer hash on int64 tensors holding values < 2**32."""
    x = x ^ (x >> 16)
    x = (x * _MUL) & M32
    x = x ^ (x >> 16)
    x = (x * _MUL) & M32
    x = x ^ (x >> 16)
    return x


def _mix32_int(x: int) -> int:
    x &= M32
    x ^= x >> 16
    x = (x * _MUL) & M32
    x ^= x >> 16
    x = (x * _MUL) & M32
    x ^= x >> 16
    return x


def rand32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Counter-based uniform 32-bit draws: one value per (seed, stream, idx).

    idx: int64 tensor of non-negative counters (< 2**63). Returns int64 in
    [0, 2**32).
    """
    s1 = _mix32_int(seed * 0x9E3779B1 + stream * 0x85EBCA77 + 0x165667B1)
    s2 = _mix32_int(s1 ^ 0xC2B2AE3D ^ (stream << 7))
    lo = idx & M32
    hi = idx >> 32
    h = _mix32(lo ^ s1)
    h = _mix32(h ^ ((hi + s2) & M32))
    return h


@dataclasses.dataclass
class Graph:
    """A CSR graph. R: int64[n+1], C: int32[m], W: int32[m] (1..64) or None."""
    n: int
    R: torch.Tensor
    C: torch.Tensor
    W: Optional[torch.Tensor] = None
    symmetric: bool = True
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.C.numel())

    def to(self, device) -> "Graph":
        return Graph(self.n, self.R.to(device), self.C.to(device),
                     None if self.W is None else self.W.to(device),
                     self.symmetric, dict(self.meta))

    def numpy(self):
        """(R int64, C int32, W uint32 or None) as contiguous numpy arrays."""
        R = self.R.cpu().numpy().astype(np.int64, copy=False)
        C = self.C.cpu().numpy().astype(np.int32, copy=False)
        W = None if self.W is None else self.W.cpu().numpy().astype(np.uint32)
        return np.ascontiguousarray(R), np.ascontiguousarray(C), W

    def degrees(self) -> torch.Tensor:
        return self.R[1:] - self.R[:-1]


# --------------------------------------------------------------------------
# CSR assembly (symmetrise, drop self-loops, dedupe) -- input preparation only
# --------------------------------------------------------------------------

def csr_from_edges(n: int, src: torch.Tensor, dst: torch.Tensor, *,
                   symmetrize: bool = True, dedupe: bool = True,
                   drop_self_loops: bool = True) -> Graph:
    """Build a CSR with neighbour lists sorted ascending."""
    src = src.to(torch.int64)
    dst = dst.to(torch.int64)
    if symmetrize:
        src, dst = torch.cat([src, dst]), torch.cat([dst, src])
    if drop_self_loops:
        keep = src != dst
        src, dst = src[keep], dst[keep]
    key = src * n + dst
    if dedupe:
        key = torch.unique(key, sorted=True)
    else:
        key, _ = torch.sort(key)
    s = key // n
    d = key - s * n
    del key
    counts = torch.bincount(s, minlength=n)
    R = torch.zeros(n + 1, dtype=torch.int64, device=s.device)
    R[1:] = torch.cumsum(counts, 0)
    return Graph(n, R, d.to(torch.int32), None, symmetrize)


def assign_weights(g: Graph, seed: int = 2, lo: int = 1, hi: int = 64) -> Graph:
    """Symmetric integer weights uniform on [lo, hi] (A-12).

    w(u,v) is a hash of (min(u,v), max(u,v), seed), so w(u,v) = w(v,u).
    """
    n = g.n
    s = torch.repeat_interleave(torch.arange(n, device=g.R.device), g.degrees())
    d = g.C.to(torch.int64)
    a = torch.minimum(s, d)
    b = torch.maximum(s, d)
    key = a * n + b
    span = hi - lo + 1
    h = rand32(seed, 77, key)
    if span & (span - 1) == 0:
        w = lo + (h & (span - 1))
    else:
        w = lo + (h % span)
    return Graph(g.n, g.R, g.C, w.to(torch.int32), g.symmetric, dict(g.meta))


# --------------------------------------------------------------------------
# Large synthetic families (the five BASELINE.json configs)
# --------------------------------------------------------------------------

def _perm_pow2(x: torch.Tensor, scale: int, seed: int) -> torch.Tensor:
    """A seeded bijection of [0, 2**scale) (Graph500-style label permutation)."""
    mask = (1 << scale) - 1
    half = max(1, (scale + 1) // 2)
    for r in range(4):
        odd = (_mix32_int(seed * 31 + r) | 1) & 0x7FFFFFFF
        add = _mix32_int(seed * 131 + r + 17) & mask
        x = (x * odd) & mask
        x = x ^ (x >> half)
        x = (x + add) & mask
    return x


def kronecker(scale: int, edge_factor: int, *, seed: int = 1, permute: bool = True,
              abc=(0.57, 0.19, 0.19), device="cpu", chunk: int = 1 << 26) -> Graph:
    """Graph500 Kronecker / R-MAT tuples (A,B,C,D = .57,.19,.19,.05).

    Each of n*edge_factor tuples draws one quadrant per bit level with a
    counter-based hash; labels optionally permuted by a seeded bijection;
    then symmetrised / self-loops dropped / deduplicated (A-13).
    """
    n = 1 << scale
    ntup = n * edge_factor
    a, b, c = abc
    ta = int(a * (1 << 32))
    tab = int((a + b) * (1 << 32))
    tabc = int((a + b + c) * (1 << 32))
    srcs, dsts = [], []
    for start in range(0, ntup, chunk):
        idx = torch.arange(start, min(ntup, start + chunk), device=device, dtype=torch.int64)
        u = torch.zeros_like(idx)
        v = torch.zeros_like(idx)
        for bit in range(scale):
            r = rand32(seed, bit, idx)
            ub = (r >= tab).to(torch.int64)           # quadrants C, D -> row bit 1
            vb = ((r >= ta) & (r < tab)) | (r >= tabc)  # quadrants B, D -> col bit 1
            u |= ub << bit
            v |= vb.to(torch.int64) << bit
        if permute:
            u = _perm_pow2(u, scale, seed)
            v = _perm_pow2(v, scale, seed)
        srcs.append(u)
        dsts.append(v)
        del idx
    src = torch.cat(srcs)
    dst = torch.cat(dsts)
    del srcs, dsts
    g = csr_from_edges(n, src, dst)
    g.meta = dict(generator="kronecker", scale=scale, edge_factor=edge_factor,
                  seed=seed, permute=permute, abc=list(abc), tuples=ntup)
    return g


def rmat(scale: int, edge_factor: int, *, seed: int = 1, device="cpu") -> Graph:
    """Unpermuted R-MAT (config 1: vertex 0 is the hub; A-15)."""
    g = kronecker(scale, edge_factor, seed=seed, permute=False, device=device)
    g.meta["generator"] = "rmat"
    return g


def chung_lu(n: int = 3_072_441, pairs: int = 117_200_000, *, alpha: float = 0.6,
             i0: float = 32.2, seed: int = 1, device="cpu", chunk: int = 1 << 26) -> Graph:
    """Chung-Lu power-law graph shaped like soc-orkut (Table 1).

    Expected degree of vertex i proportional to (i + i0)^-alpha; both pair
    endpoints drawn proportional to that weight by inverse-CDF over a 32-bit
    integer table (computed once on the host in float64, then used as exact
    integers on either device); labels randomly permuted.
    """
    w = (np.arange(n, dtype=np.float64) + i0) ** (-alpha)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    table = np.minimum(np.round(cdf * float(1 << 32)).astype(np.int64), 1 << 32)
    table[-1] = 1 << 32
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n).astype(np.int64)
    table_t = torch.from_numpy(table).to(device)
    perm_t = torch.from_numpy(perm).to(device)
    srcs, dsts = [], []
    for start in range(0, pairs, chunk):
        idx = torch.arange(start, min(pairs, start + chunk), device=device, dtype=torch.int64)
        ru = rand32(seed, 1001, idx)
        rv = rand32(seed, 1002, idx)
        u = torch.searchsorted(table_t, ru, right=True)
        v = torch.searchsorted(table_t, rv, right=True)
        srcs.append(perm_t[u])
        dsts.append(perm_t[v])
    g = csr_from_edges(n, torch.cat(srcs), torch.cat(dsts))
    g.meta = dict(generator="chung_lu", n=n, pairs=pairs, alpha=alpha, i0=i0, seed=seed)
    return g


def mesh(L: int = 4899, *, p_vertical: float = 0.2, seed: int = 1, device="cpu") -> Graph:
    """Row-connected mesh shaped like road_usa (high diameter, max degree 4).

    Vertex (r, c) has id r*L + c. Every horizontal lattice edge is present;
    each vertical lattice edge is present with probability p_vertical. Every
    row is a path and row 0..L-1 are joined by the vertical edges, so the
    graph is connected with overwhelming probability (checked in tests).
    """
    n = L * L
    r = torch.arange(L, device=device, dtype=torch.int64)
    c = torch.arange(L - 1, device=device, dtype=torch.int64)
    hs = (r[:, None] * L + c[None, :]).reshape(-1)
    hd = hs + 1
    vs = torch.arange(n - L, device=device, dtype=torch.int64)
    thr = int(p_vertical * (1 << 32))
    keep = rand32(seed, 2001, vs) < thr
    vs = vs[keep]
    vd = vs + L
    g = csr_from_edges(n, torch.cat([hs, vs]), torch.cat([hd, vd]))
    g.meta = dict(generator="mesh", L=L, p_vertical=p_vertical, seed=seed)
    return g


# --------------------------------------------------------------------------
# Small families for tests (closed forms live in tests/, not here)
# --------------------------------------------------------------------------

def from_edges(n: int, edges, weights=None, *, symmetrize=True, dedupe=True,
               drop_self_loops=True) -> Graph:
    """Graph from a python edge list [(u, v), ...] with optional weights.

    With weights and dedupe, a duplicated (u,v) keeps the minimum weight (the
    SSSP answer is unchanged by that choice; the kept weight must be defined).
    """
    e = torch.tensor(list(edges), dtype=torch.int64).reshape(-1, 2)
    if weights is None:
        g = csr_from_edges(n, e[:, 0], e[:, 1], symmetrize=symmetrize, dedupe=dedupe,
                           drop_self_loops=drop_self_loops)
        return g
    w = torch.tensor(list(weights), dtype=torch.int64)
    src, dst = e[:, 0], e[:, 1]
    if symmetrize:
        src, dst, w = torch.cat([src, dst]), torch.cat([dst, src]), torch.cat([w, w])
    if drop_self_loops:
        keep = src != dst
        src, dst, w = src[keep], dst[keep], w[keep]
    key = (src * n + dst) * (1 << 20) + w  # sort by edge, then weight (w < 2**20)
    key, _ = torch.sort(key)
    ek = key >> 20
    wk = key & ((1 << 20) - 1)
    if dedupe and ek.numel():
        first = torch.ones_like(ek, dtype=torch.bool)
        first[1:] = ek[1:] != ek[:-1]
        ek, wk = ek[first], wk[first]
    s = ek // n
    d = ek - s * n
    R = torch.zeros(n + 1, dtype=torch.int64)
    R[1:] = torch.cumsum(torch.bincount(s, minlength=n), 0)
    return Graph(n, R, d.to(torch.int32), wk.to(torch.int32), symmetrize)


def path(n: int) -> Graph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)]) if n > 1 else empty(n)


def cycle(n: int) -> Graph:
    return from_edges(n, [(i, (i + 1) % n) for i in range(n)])


def grid(rows: int, cols: int) -> Graph:
    e = []
    for i in range(rows):
        for j in range(cols):
            v = i * cols + j
            if j + 1 < cols:
                e.append((v, v + 1))
            if i + 1 < rows:
                e.append((v, v + cols))
    return from_edges(rows * cols, e)


def complete(n: int) -> Graph:
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def star(leaves: int) -> Graph:
    return from_edges(leaves + 1, [(0, i) for i in range(1, leaves + 1)])


def binary_tree(n: int) -> Graph:
    """Heap-numbered complete binary tree: parent(i) = (i-1)//2."""
    return from_edges(n, [((i - 1) // 2, i) for i in range(1, n)]) if n > 1 else empty(n)


def hypercube(d: int) -> Graph:
    n = 1 << d
    return from_edges(n, [(v, v ^ (1 << b)) for v in range(n) for b in range(d) if v < v ^ (1 << b)])


def empty(n: int) -> Graph:
    return Graph(n, torch.zeros(n + 1, dtype=torch.int64), torch.zeros(0, dtype=torch.int32),
                 None, True)


def erdos_renyi(n: int, m_pairs: int, *, seed: int = 1, device="cpu") -> Graph:
    idx = torch.arange(m_pairs, device=device, dtype=torch.int64)
    u = rand32(seed, 3001, idx) % n
    v = rand32(seed, 3002, idx) % n
    g = csr_from_edges(n, u, v)
    g.meta = dict(generator="erdos_renyi", n=n, pairs=m_pairs, seed=seed)
    return g


def directed_random(n: int, m_pairs: int, *, seed: int = 1, device="cpu") -> Graph:
    """A NON-symmetric graph (exercises the CSC / in-edge pull path, A-18)."""
    idx = torch.arange(m_pairs, device=device, dtype=torch.int64)
    u = rand32(seed, 4001, idx) % n
    v = rand32(seed, 4002, idx) % n
    g = csr_from_edges(n, u, v, symmetrize=False)
    g.symmetric = False
    g.meta = dict(generator="directed_random", n=n, pairs=m_pairs, seed=seed)
    return g


def sources(g: Graph, k: int, *, seed: int = 3) -> list:
    """k distinct seeded sources with out-degree >= 1 (A-15)."""
    deg = g.degrees().cpu()
    out, seen = [], set()
    j = 0
    while len(out) < k and j < 64 * k + 4 * g.n:
        cand = rand32(seed, 5001, torch.arange(j, j + 256, dtype=torch.int64)) % g.n
        for v in cand.tolist():
            if deg[v] > 0 and v not in seen:
                seen.add(v)
                out.append(int(v))
                if len(out) == k:
                    break
        j += 256
    return out


# --------------------------------------------------------------------------
# The five BASELINE.json configs (recipe: DESIGN.md "Input recipe")
# --------------------------------------------------------------------------

CONFIGS = {
    "c1_rmat16": "BFS from vertex 0 on synthetic R-MAT scale 16, edge factor 16, undirected",
    "c2_kron21": "BFS push-pull on kron_g500-logn21-shaped Kronecker s21 ef48",
    "c3_orkut": "BFS + SSSP (weights 1..64) on soc-orkut-shaped Chung-Lu",
    "c4_road": "BFS + delta-stepping SSSP on road_usa-shaped mesh 4899^2",
    "c5_kron25": "BFS on Graph500 Kronecker scale 25, edge factor 16",
}


def make_config(name: str, device="cpu", *, weights: Optional[bool] = None, shrink: int = 0) -> Graph:
    """Generate one of the five configs. `shrink` > 0 scales it down for tests
    (Kronecker scale - shrink; Chung-Lu n / 4**shrink; mesh L / 2**shrink)."""
    if name == "c1_rmat16":
        g = rmat(16 - shrink, 16, seed=1, device=device)
    elif name == "c2_kron21":
        g = kronecker(21 - shrink, 48, seed=1, device=device)
    elif name == "c3_orkut":
        f = 4 ** shrink
        g = chung_lu(max(1000, 3_072_441 // f), max(1000, 117_200_000 // f), seed=1, device=device)
    elif name == "c4_road":
        g = mesh(max(8, 4899 >> shrink), seed=1, device=device)
    elif name == "c5_kron25":
        g = kronecker(25 - shrink, 16, seed=1, device=device)
    else:
        raise KeyError(name)
    want_w = weights if weights is not None else name in ("c3_orkut", "c4_road")
    if want_w:
        g = assign_weights(g, seed=2)
    g.meta["config"] = name
    g.meta["shrink"] = shrink
    return g
