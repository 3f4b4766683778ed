// frontier.cuh -- the advance/filter machinery shared by BFS and SSSP.
//
// Advance = "generates a new frontier from the current frontier by visiting
// the neighbors of the current frontier" (§4.1); filter = "choosing
// a subset of the current frontier" to compact duplicates or to split it
// (P:357-364). Both run FUSED in one kernel pass ("kernel fusion";
// no per-edge intermediate array is materialised).
//
// B200 design:
//  * The frontier is a queue of vertex ids PLUS the exclusive prefix of their
//    out-degrees (the "scanned edge offset queue" of P:753-754). The filter
//    that produces the next frontier writes that prefix itself: one 64-bit
//    atomicAdd per 32 appended vertices reserves both the queue slots and the
//    edge range, so the load-balanced advance never runs a separate scan.
//  * Load-balanced partitioning (Davidson): the frontier's edges
//    are split into equal contiguous ranges, one per warp of the persistent
//    grid; a warp finds its first vertex with a 32-ary cooperative search of
//    the prefix ("sorted search"), then walks 32-entry windows and maps each
//    edge to its owner with a 5-step shuffle binary search ("binary search to
//    find the node ID").
//  * Node-granular thread/warp/CTA expansion (Merrill TWC) is the
//    other strategy (expand_twc below); the selection rule is P:760-775.
#pragma once

#include "gr_internal.cuh"

namespace gr {

// ---------------------------------------------------------------------------
// Warp-staged append into a frontier queue (filter output).
// All 32 lanes must call push()/finish() together (warp-converged).
// With offsets: entries carry the exclusive prefix of their degree.
// ---------------------------------------------------------------------------
struct Appender {
    int32_t *sv;                    // smem staging [kStageCap]
    int64_t *sd;                    // smem staging degrees [kStageCap] (offsets mode)
    int cnt;                        // warp-uniform
    int32_t *qv;                    // destination queue
    int64_t *qo;                    // destination prefix (null: count-only queue)
    unsigned long long *counter;    // packed (edges << S) | count, or plain count
    int S;                          // count-field bits (offsets mode)
    int64_t cap;                    // queue capacity
    unsigned long long *overflow;

    __device__ __forceinline__ void flush(int k) {
        unsigned l = lane_id();
        int32_t v = 0;
        int64_t d = 0;
        if ((int)l < k) { v = sv[l]; if (qo) d = sd[l]; }
        unsigned long long base = 0;
        int64_t incl = 0, total = 0;
        if (qo) {
            incl = warp_incl_scan<int64_t>(d);
            total = __shfl_sync(0xffffffffu, incl, 31);
        }
        if (l == 0) {
            unsigned long long add = qo ? (((unsigned long long)total << S) | (unsigned long long)k)
                                        : (unsigned long long)k;
            base = atomicAdd(counter, add);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        unsigned long long cbase = qo ? (base & ((1ull << S) - 1)) : base;
        if ((int64_t)(cbase + k) > cap) {
            if (l == 0) atomicExch(overflow, 1ull);
        } else if ((int)l < k) {
            qv[cbase + l] = v;
            if (qo) qo[cbase + l] = (int64_t)(base >> S) + (incl - d);
        }
    }

    __device__ __forceinline__ void push(bool has, int32_t v, int64_t d) {
        unsigned mask = __ballot_sync(0xffffffffu, has);
        if (mask == 0) return;
        int pos = cnt + __popc(mask & lanemask_lt());
        if (has) { sv[pos] = v; if (qo) sd[pos] = d; }
        cnt += __popc(mask);
        __syncwarp();
        if (cnt >= 32) {
            flush(32);
            __syncwarp();
            unsigned l = lane_id();
            int rest = cnt - 32;
            int32_t tv = 0; int64_t td = 0;
            if ((int)l < rest) { tv = sv[32 + l]; if (qo) td = sd[32 + l]; }
            __syncwarp();
            if ((int)l < rest) { sv[l] = tv; if (qo) sd[l] = td; }
            __syncwarp();
            cnt = rest;
        }
    }

    __device__ __forceinline__ void finish() {
        if (cnt > 0) flush(cnt);
        __syncwarp();
        cnt = 0;
    }
};

// Largest i in [0, F) with qo[i] <= e (qo ascending, qo[0] = 0 <= e).
// 32-ary cooperative search: each round narrows the range 32x.
__device__ __forceinline__ int64_t warp_search(const int64_t *qo, int64_t F, int64_t e) {
    int64_t lo = 0, hi = F;  // answer in [lo, hi)
    unsigned l = lane_id();
    while (hi - lo > 32) {
        int64_t span = hi - lo;
        int64_t p = lo + (span * (int64_t)l) / 32;
        int64_t val = __ldcg(qo + p);
        unsigned b = __ballot_sync(0xffffffffu, val <= e);
        int k = 31 - __clz(b);                      // lane 0 always qualifies
        int64_t nlo = lo + (span * (int64_t)k) / 32;
        int64_t nhi = (k == 31) ? hi : lo + (span * (int64_t)(k + 1)) / 32;
        lo = nlo; hi = nhi;
    }
    int64_t p = lo + l;
    bool ok = p < hi && __ldcg(qo + p) <= e;
    unsigned b = __ballot_sync(0xffffffffu, ok);
    return lo + (31 - __clz(b));
}

// ---------------------------------------------------------------------------
// Load-balanced advance over the frontier queue (merge-path).
// Op must provide:
//   uint64_t entry(int32_t v)            per-source payload (e.g. dist[v])
//   void edges<U>(ok[], src[], pay[], dst[], eidx[])  process U edges per lane
// Each warp of the grid processes the contiguous edge range
//   [E*gw/nw, E*(gw+1)/nw).
// ---------------------------------------------------------------------------
constexpr int kUnroll = 4;

template <class Op>
__device__ __forceinline__ void expand_lb(const int32_t *__restrict__ qv, const int64_t *__restrict__ qo,
                                          int64_t F, int64_t E, const int64_t *__restrict__ R,
                                          const int32_t *__restrict__ C, int64_t gw, int64_t nw, Op &op) {
    if (E <= 0 || F <= 0) return;
    int64_t e0 = (E * gw) / nw;  // E < 2^40, nw < 2^20: no overflow
    int64_t e1 = (E * (gw + 1)) / nw;
    if (e0 >= e1) return;
    unsigned l = lane_id();
    int64_t i = warp_search(qo, F, e0);
    int64_t e = e0;
    while (e < e1) {
        int64_t j = i + l;
        bool valid = j < F;
        int32_t v = valid ? __ldcg(qv + j) : 0;
        int64_t o = valid ? __ldcg(qo + j) : E;
        int64_t rs = 0, re = 0;
        if (valid) { rs = R[v]; re = R[v + 1]; }
        unsigned long long pay = valid ? op.entry(v) : 0ull;
        int64_t end = valid ? o + (re - rs) : E;
        int64_t wend = __shfl_sync(0xffffffffu, end, 31);
        if (wend > e1) wend = e1;
        for (int64_t b = e; b < wend; b += 32 * kUnroll) {
            bool ok[kUnroll];
            int32_t src[kUnroll];
            unsigned long long sp[kUnroll];
            int64_t eidx[kUnroll];
            int32_t dst[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                int64_t my = b + u * 32 + l;
                int k = 0;
#pragma unroll
                for (int s = 16; s >= 1; s >>= 1) {
                    int64_t oc = __shfl_sync(0xffffffffu, o, k + s);
                    if (oc <= my) k += s;
                }
                ok[u] = my < wend;
                src[u] = __shfl_sync(0xffffffffu, v, k);
                sp[u] = __shfl_sync(0xffffffffu, pay, k);
                int64_t ok_o = __shfl_sync(0xffffffffu, o, k);
                int64_t ok_rs = __shfl_sync(0xffffffffu, rs, k);
                eidx[u] = ok_rs + (my - ok_o);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) dst[u] = ok[u] ? __ldg(C + eidx[u]) : 0;
            op.template edges<kUnroll>(ok, src, sp, dst, eidx);
        }
        e = wend;
        i += 32;
    }
}

}  // namespace gr
