// pull.cuh -- the pull (bottom-up) step and the frontier bitmap -> queue
// conversion shared by the single-GPU BFS kernel (bfs.cu) and the partitioned
// one (pbfs.cu). P:804-834 (push vs pull), P:821-825 (bitmap frontier).
#pragma once

#include "frontier.cuh"

namespace gr {

#ifndef GR_PULL_Q
#define GR_PULL_Q 2
#endif
constexpr int kPullQ = GR_PULL_Q;            // pull: candidates per lane per batch
constexpr int kPullBatch = 32 * kPullQ;      // pull: candidates per batch
constexpr int kPullList = kPullBatch + 32;   // pull: per-warp candidate list (< batch + 32 before a batch)
#ifndef GR_PULL_GRAB
#define GR_PULL_GRAB 4
#endif
constexpr int kPullGrab = GR_PULL_GRAB;  // pull: bitmap words per grab
#ifndef GR_PULL_LONG
#define GR_PULL_LONG 4
#endif
constexpr int64_t kPullLong = GR_PULL_LONG;  // pull: longer unresolved in-lists are scanned by the warp
#ifndef GR_PULL_AGG
#define GR_PULL_AGG 0  // warp-aggregated REDs: C2 -0.7%, C3 -0.3%, C5 +1.3% (noise): off
#endif
#ifndef GR_PULL_SCAN_U
#define GR_PULL_SCAN_U 1  // 4 and 8 measured slower (C2 0.130 -> 0.134 / 0.149 ms)
#endif
constexpr int kPullScanU = GR_PULL_SCAN_U;   // pull: 32-edge groups per warp-scan step

// ---------------------------------------------------------------------------
// Pull (bottom-up) step over in-edges: "pull starts with a
// frontier of unvisited vertices, generating the new frontier by filtering
// the unvisited frontier for vertices that have neighbors in the current
// frontier"; the current frontier is held as a bitmap.
// B200 design: each CTA owns a contiguous range of visited-bitmap words; its
// warps take 16 words at a time and COMPACT the unvisited vertices of those
// words into a per-warp shared-memory list (filter of the unvisited set, one
// ballot per round), so every lane of a batch works on a real candidate (a
// late pull step has ~1 candidate per 10 vertices: a lane-per-vertex sweep
// would leave 90% of the lanes idle through the whole dependent chain
// R' -> C' -> frontier bit). A batch is 64 candidates, two per lane, with
// the loads of both issued back to back. Each candidate stops at its first
// in-neighbour in the frontier (early exit; in-lists are ordered by neighbour
// degree, so hubs come first). Found vertices set their bits in the next
// frontier and visited bitmaps with fire-and-forget RED.OR.
// The next frontier is kept as a bitmap only ("lazy queue"): the step counts
// its size and edges (for the direction rule) and a following push step
// builds the queue from the bitmap (bitmap_to_queue), so pull -> pull
// sequences never write a queue.
// ---------------------------------------------------------------------------

struct PullCounts {
    unsigned long long ndisc = 0, insp = 0, qcnt = 0, qedges = 0;
    unsigned dmax = 0;
};

// A: any view with n, R, Rt, Ct, ph, visited, depth, pred (BfsArgs; the
// partitioned kernel's PullView, whose in-lists hold GLOBAL ids probed in the
// all-gathered frontier `fcur` while x, visited, depth, pred and fnext are
// local). [wb0, wb1): this CTA's range of visited-bitmap words.
template <class A>
__device__ __forceinline__ void pull_level(const A &a, const uint32_t *__restrict__ fcur,
                                           uint32_t *__restrict__ fnext, int32_t next_depth, int *swork,
                                           int32_t *wl, PullCounts &pc, uint32_t sbm, int64_t sbits,
                                           int64_t wb0, int64_t wb1, int grab = kPullGrab) {
    const int64_t nwords = (a.n + 31) / 32;
    const unsigned l = lane_id();
    const unsigned long long pol = policy_evict_first();
    const bool sym = a.Rt == a.R;
    const uint32_t tail = (a.n & 31) ? ((1u << (a.n & 31)) - 1u) : 0xffffffffu;
    // frontier word of u (u >= 0): loaded unconditionally by the callers and
    // tested afterwards, so the probes of a lane are in flight together (a
    // probe consumed inside a short-circuit branch costs a round trip each)
    auto fword = [&](int32_t u) -> uint32_t {
        return u < sbits ? lds_u32(sbm + 4u * (uint32_t)(u >> 5)) : __ldg(fcur + (u >> 5));
    };
    auto fbit = [&](int32_t u) -> bool { return (fword(u) >> (u & 31)) & 1u; };
    int cnt = 0;  // warp-uniform
    auto process = [&](int k) {  // candidates wl[0, k), k <= kPullBatch
        int32_t v[kPullQ], par[kPullQ], u0[kPullQ];
        int64_t beg[kPullQ], end[kPullQ];
        bool fnd[kPullQ];
#pragma unroll
        for (int q = 0; q < kPullQ; ++q) v[q] = ((int)l + 32 * q < k) ? wl[l + 32 * q] : -1;
        if (a.ph) {
            // pull head {first in-neighbour, in-degree}: one 8-byte load per
            // candidate (consecutive candidates -> coalesced) answers most of
            // them (in-lists are ordered by neighbour degree, hubs first);
            // only unresolved lists read their row offset
            int2 h[kPullQ];
            int64_t rt[kPullQ];
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) h[q] = v[q] >= 0 ? __ldg(a.ph + v[q]) : make_int2(-1, 0);
            // row offsets loaded speculatively with the heads (candidates are
            // sorted: coalesced), so an unresolved list starts its scan one
            // dependent round trip earlier
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) rt[q] = v[q] >= 0 ? __ldg(a.Rt + v[q]) : 0;
            uint32_t fw[kPullQ];
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) {
                u0[q] = h[q].x;
                fw[q] = u0[q] >= 0 ? fword(u0[q]) : 0u;
            }
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) {
                fnd[q] = u0[q] >= 0 && ((fw[q] >> (u0[q] & 31)) & 1u);
                par[q] = u0[q];
                pc.insp += (u0[q] >= 0);
            }
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) {
                beg[q] = (!fnd[q] && h[q].y > 1) ? rt[q] : 0;
                end[q] = beg[q] + h[q].y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) {
                beg[q] = v[q] >= 0 ? a.Rt[v[q]] : 0;
                end[q] = v[q] >= 0 ? a.Rt[v[q] + 1] : 0;
            }
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) u0[q] = beg[q] < end[q] ? ld_stream(a.Ct + beg[q], pol) : -1;
            uint32_t fw[kPullQ];
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) fw[q] = u0[q] >= 0 ? fword(u0[q]) : 0u;
#pragma unroll
            for (int q = 0; q < kPullQ; ++q) {
                fnd[q] = u0[q] >= 0 && ((fw[q] >> (u0[q] & 31)) & 1u);
                par[q] = u0[q];
                pc.insp += (u0[q] >= 0);
            }
        }
        // the rest of each unresolved list: first by its lane (4 edges a step,
        // at most kPullLong edges), then what is left of the long ones by the
        // whole warp, 32 edges a step with a ballot early exit (one lane
        // scanning a long list alone held its warp for 100+ us on C3)
        int64_t nxt[kPullQ];
#pragma unroll
        for (int q = 0; q < kPullQ; ++q) {
            nxt[q] = beg[q] + 1;
            if (fnd[q]) continue;
            const int64_t lim = (end[q] - nxt[q] > kPullLong) ? nxt[q] + kPullLong : end[q];
            for (int64_t e = nxt[q]; e < lim && !fnd[q]; e += 4) {
                int32_t u[4];
                uint32_t uw[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) u[j] = (e + j < lim) ? ld_stream(a.Ct + e + j, pol) : -1;
#pragma unroll
                for (int j = 0; j < 4; ++j) uw[j] = u[j] >= 0 ? fword(u[j]) : 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (!fnd[q] && u[j] >= 0) {
                        ++pc.insp;
                        if ((uw[j] >> (u[j] & 31)) & 1u) { fnd[q] = true; par[q] = u[j]; }
                    }
                }
            }
            nxt[q] = lim;
        }
        bool lng[kPullQ];
#pragma unroll
        for (int q = 0; q < kPullQ; ++q) lng[q] = !fnd[q] && nxt[q] < end[q];
#pragma unroll
        for (int q = 0; q < kPullQ; ++q) {
            unsigned lm = __ballot_sync(0xffffffffu, lng[q]);
            while (lm) {
                const int ld = __ffs(lm) - 1;
                lm &= lm - 1;
                const int64_t b = __shfl_sync(0xffffffffu, nxt[q], ld);
                const int64_t e = __shfl_sync(0xffffffffu, end[q], ld);
                int32_t hitu = -1;
                // kPullScanU x 32 edges per step, all loads of a step in flight
                // (one lane's unresolved long list was a chain of 2 dependent
                // round trips per 32 edges: the pull level's tail warp)
                for (int64_t x = b; x < e; x += 32 * kPullScanU) {
                    int32_t u[kPullScanU];
                    uint32_t uw[kPullScanU];
#pragma unroll
                    for (int k = 0; k < kPullScanU; ++k) {
                        const int64_t y = x + 32 * k + l;
                        u[k] = y < e ? ld_stream(a.Ct + y, pol) : -1;
                    }
#pragma unroll
                    for (int k = 0; k < kPullScanU; ++k) uw[k] = u[k] >= 0 ? fword(u[k]) : 0u;
                    bool done = false;
#pragma unroll
                    for (int k = 0; k < kPullScanU; ++k) {
                        if (done) break;
                        const bool hit = u[k] >= 0 && ((uw[k] >> (u[k] & 31)) & 1u);
                        const unsigned bm = __ballot_sync(0xffffffffu, hit);
                        const int first = bm ? __ffs(bm) - 1 : 32;
                        pc.insp += (u[k] >= 0 && (int)l <= first);
                        if (bm) {
                            hitu = __shfl_sync(0xffffffffu, u[k], first);
                            done = true;
                        }
                    }
                    if (done) break;
                }
                if ((int)l == ld && hitu >= 0) { fnd[q] = true; par[q] = hitu; }
            }
        }
#pragma unroll
        for (int q = 0; q < kPullQ; ++q) {
#if GR_PULL_AGG
            // the batch's candidates are sorted: its found vertices share a few
            // bitmap words; one RED per word and bitmap (warp OR-reduction)
            {
                const int32_t xw = v[q] >= 0 ? (v[q] >> 5) : -1;
                unsigned rem = __ballot_sync(0xffffffffu, fnd[q]);
                while (rem) {
                    const int w0 = __shfl_sync(0xffffffffu, xw, __ffs(rem) - 1);
                    const bool in = fnd[q] && xw == w0;
                    const unsigned bits = __reduce_or_sync(0xffffffffu, in ? 1u << (v[q] & 31) : 0u);
                    if ((int)l == __ffs(rem) - 1) {
                        atomicOr(fnext + w0, bits);      // RED.OR
                        atomicOr(a.visited + w0, bits);  // RED.OR
                    }
                    rem &= ~__ballot_sync(0xffffffffu, in);
                }
            }
#endif
            if (!fnd[q]) continue;
            const int32_t x = v[q];
            a.depth[x] = next_depth;
            if (a.pred) a.pred[x] = par[q];
#if !GR_PULL_AGG
            const uint32_t bit = 1u << (x & 31);
            atomicOr(fnext + (x >> 5), bit);      // RED.OR
            atomicOr(a.visited + (x >> 5), bit);  // RED.OR
#endif
            const int64_t deg = sym ? end[q] - beg[q] : a.R[x + 1] - a.R[x];
            ++pc.ndisc;
            if (deg > 0) {
                ++pc.qcnt;
                pc.qedges += (unsigned long long)deg;
                pc.dmax = max(pc.dmax, (unsigned)deg);
            }
        }
        // keep the unprocessed tail (cnt - k < 32 entries) at the front
        __syncwarp();
        const int rem = cnt - k;
        const int32_t t = ((int)l < rem) ? wl[k + l] : 0;
        __syncwarp();
        if ((int)l < rem) wl[l] = t;
        __syncwarp();
        cnt = rem;
    };
    for (;;) {
        int c = 0;
        if (l == 0) c = atomicAdd(swork, grab);
        c = __shfl_sync(0xffffffffu, c, 0);
        const int64_t w0 = wb0 + c;
        if (w0 >= wb1) break;
        const int64_t wi = w0 + l;
        uint32_t cm = ((int)l < grab && wi < wb1) ? ~a.visited[wi] : 0u;
        if (wi == nwords - 1) cm &= tail;
        // word by word, lane b takes bit b: the list stays sorted by vertex id,
        // so a batch's depth/pred stores and bitmap REDs touch few lines
        unsigned nz = __ballot_sync(0xffffffffu, cm != 0);
        while (nz) {
            const int j = __ffs(nz) - 1;
            nz &= nz - 1;
            const uint32_t w = __shfl_sync(0xffffffffu, cm, j);
            if ((w >> l) & 1u) wl[cnt + __popc(w & lanemask_lt())] = (int32_t)((w0 + j) * 32 + l);
            cnt += __popc(w);
            __syncwarp();
            if (cnt >= kPullBatch) process(kPullBatch);
        }
    }
    while (cnt > 0) process(cnt < kPullBatch ? cnt : kPullBatch);
}

// Frontier bitmap -> queue (the other direction of the
// conversion): the frontier of a pull step, needed as a queue when the next
// step pushes. Warp-strided over 32-word chunks; appends (v, degree prefix,
// R[v]) for every set bit with out-degree > 0.
template <class A, class App>
__device__ __forceinline__ void bitmap_to_queue(const A &a, const uint32_t *__restrict__ fb,
                                                int64_t gw, int64_t nw, App &app) {
    const int64_t nwords = (a.n + 31) / 32;
    const unsigned l = lane_id();
    for (int64_t w0 = gw * 32; w0 < nwords; w0 += nw * 32) {
        const int64_t wi = w0 + l;
        uint32_t bits = wi < nwords ? __ldcg(fb + wi) : 0u;
        while (__any_sync(0xffffffffu, bits != 0)) {
            const bool has = bits != 0;
            int32_t v = 0;
            int64_t rs = 0, deg = 0;
            if (has) {
                v = (int32_t)(wi * 32 + (__ffs(bits) - 1));
                bits &= bits - 1;
                rs = a.R[v];
                deg = a.R[v + 1] - rs;
            }
            app.push(has && deg > 0, v, deg, rs);
        }
    }
    app.finish();
}

// Direction rule (reading A-3). Pure function of global counters:
//   forced       0 auto, 1 push, 2 pull (gr_bfs_opts.direction)
//   switch_rule  1: paper-literal "unvisited < frontier"
//                0: Beamer -- push->pull when m_f > m_u / alpha (and m_f >=
//                   n/32: a pull step sweeps every bitmap word), pull->push when
//                   f < nonisolated / beta and the frontier shrinks
//   dir          direction of the previous step (1 push, 2 pull)
__device__ __forceinline__ int direction_rule(int forced, int switch_rule, double alpha, double beta,
                                              int64_t nonisolated, int dir, int64_t f, int64_t mf,
                                              int64_t u_cnt, int64_t m_u, int64_t prev_f, int64_t nwords,
                                              int64_t stay_f = 0) {
    if (forced != 0) return forced;
    if (switch_rule == 1) return (u_cnt < f) ? 2 : 1;
    if (dir == 1) {
        if ((double)mf > (double)m_u / alpha && mf >= nwords) return 2;
        return 1;
    }
    // ... unless fewer vertices are left unvisited than the frontier holds
    // (the literal rule's pull condition) and the frontier is at most stay_f:
    // one more pull step then touches fewer vertices than the push step and
    // saves the bitmap -> queue conversion (measured: stay_f
    // unlimited in bfs.cu, 0 -- plain Beamer -- in the partitioned kernel)
    if ((double)f < (double)nonisolated / beta && f < prev_f && !(f <= stay_f && u_cnt < f)) return 1;
    return 2;
}

}  // namespace gr
