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

// Debug trace (GR_TRACE builds only): thread 0 stamps %globaltimer at fixed
// points of the first levels; read back with gr_debug_trace().
#ifdef GR_TRACE
static __device__ long long *g_trace;
static __device__ int g_trace_L;
static __device__ long long *g_bal;   // [64 levels][grid][2]: first / last warp done (per CTA)
#define GR_TSTAMP(k)                                                                         \
    do {                                                                                    \
        if (g_trace && blockIdx.x == 0 && threadIdx.x == 0 && g_trace_L < 256) {            \
            long long t_;                                                                   \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
            g_trace[g_trace_L * 16 + (k)] = t_;                                             \
        }                                                                                   \
    } while (0)
// stamp k once the value x has ARRIVED (a load's result, not its issue):
// the volatile local store waits for x, the memory-clobbering timer read
// stays behind it
#define GR_TDEP(k, val)                                                                      \
    do {                                                                                    \
        if (g_trace && blockIdx.x == 0 && threadIdx.x == 0 && g_trace_L < 256) {            \
            volatile int d_ = (int)(val);                                                   \
            (void)d_;                                                                       \
            long long t_;                                                                   \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory");                \
            g_trace[g_trace_L * 16 + (k)] = t_;                                             \
        }                                                                                   \
    } while (0)
#else
#define GR_TSTAMP(k) do {} while (0)
#define GR_TDEP(k, val) do {} while (0)
#endif

// ---------------------------------------------------------------------------
// Warp-staged append into a frontier queue (filter output).
// All 32 lanes must call push()/finish() together (warp-converged).
// With offsets: entries carry the exclusive prefix of their degree.
// Entries are staged in shared memory and written kStageCap at a time, so one
// global atomicAdd reserves up to kStageCap queue slots (the counter is a
// single L2 address shared by the whole grid: fewer atomics, less contention).
// ---------------------------------------------------------------------------
template <int kCap>
struct AppenderT {
    int32_t *sv;                    // smem staging [kCap]
    int32_t *sd;                    // smem staging degrees [kCap] (offsets mode)
    int64_t *sr;                    // smem staging row starts [kCap] (offsets mode)
    int cnt;                        // warp-uniform
    int32_t *qv;                    // destination queue
    int64_t *qo;                    // destination prefix (null: count-only queue)
    int64_t *qr;                    // destination row starts R[v] (offsets mode): the
                                    // next level reads its lists without touching R
    unsigned long long *counter;    // packed (edges << S) | count, or plain count
    int S;                          // count-field bits (offsets mode)
    int64_t cap;                    // queue capacity
    unsigned long long *overflow;
    unsigned long long *dmax = nullptr;  // max appended degree (offsets mode; null: not tracked)
    bool stream = false;            // streaming (evict-first) queue stores: keep L2 for per-vertex state
    unsigned tag = 1;               // overflow code: which queue (diagnostics; any non-zero = overflow)
    const int64_t *Rl = nullptr;    // lazy row offsets (offsets mode): push() stages the vertex only and
                                    // the flush loads R[v], R[v+1] of all staged entries at once, so a
                                    // discovery costs no dependent load inside the edge loop

    // Lazy mode: row start and degree of every staged entry, loaded together
    // (one round trip per flush instead of one per discovering edge group);
    // entries of out-degree 0 are dropped (a frontier holds vertices with
    // edges to expand). Returns the new count.
    __device__ __forceinline__ int fill_from_R(int k) {
        const unsigned l = lane_id();
        constexpr int kR = kCap / 32;
        int32_t v[kR];
        int64_t r0[kR], r1[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            const int j = r * 32 + (int)l;
            v[r] = (j < k) ? sv[j] : -1;
            r0[r] = (v[r] >= 0) ? Rl[v[r]] : 0;
            r1[r] = (v[r] >= 0) ? Rl[v[r] + 1] : 0;
        }
        __syncwarp();
        int out = 0;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            const bool keep = r1[r] > r0[r];
            const unsigned bm = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int pos = out + __popc(bm & lanemask_lt());
                sv[pos] = v[r];
                sd[pos] = (int32_t)(r1[r] - r0[r]);
                sr[pos] = r0[r];
            }
            out += __popc(bm);
        }
        __syncwarp();
        return out;
    }

    __device__ __forceinline__ void flush() {
        const unsigned l = lane_id();
        if (Rl) cnt = fill_from_R(cnt);
        const int k = cnt;
        constexpr int kR = kCap / 32;
        // pass 1: total degree (and max) of the staged entries
        int64_t tot = 0;
        unsigned mx = 0;
        if (qo) {
#pragma unroll 4
            for (int r = 0; r < kR; ++r) {
                const int j = r * 32 + (int)l;
                const int64_t d = (j < k) ? (int64_t)sd[j] : 0;
                tot += d;
                mx = max(mx, (unsigned)d);
            }
            tot = warp_sum<int64_t>(tot);
            if (dmax) mx = __reduce_max_sync(0xffffffffu, mx);
        }
        unsigned long long base = 0;
        if (l == 0) {
            if (dmax && mx) atomicMax(dmax, (unsigned long long)mx);
            const unsigned long long add = qo ? (((unsigned long long)tot << S) | (unsigned long long)k)
                                              : (unsigned long long)k;
            base = atomicAdd(counter, add);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned long long cbase = qo ? (base & ((1ull << S) - 1)) : base;
        if ((int64_t)(cbase + k) > cap) {
            if (l == 0) atomicExch(overflow, (unsigned long long)tag | ((cbase + k) << 8));
        } else {
            // pass 2: exclusive degree prefix of each entry, then the writes
            int64_t run = qo ? (int64_t)(base >> S) : 0;
#pragma unroll 4
            for (int r = 0; r < kR; ++r) {
                if (r * 32 >= k) break;
                const int j = r * 32 + (int)l;
                if (qo) {
                    const int64_t d = (j < k) ? (int64_t)sd[j] : 0;
                    const int64_t x = warp_incl_scan<int64_t>(d);
                    if (j < k) {
                        if (stream) {
                            __stcs(qo + cbase + j, run + x - d);
                            __stcs(qr + cbase + j, sr[j]);
                        } else {
                            qo[cbase + j] = run + x - d;
                            qr[cbase + j] = sr[j];
                        }
                    }
                    run += __shfl_sync(0xffffffffu, x, 31);
                }
                if (j < k) {
                    if (stream) __stcs(qv + cbase + j, sv[j]);
                    else qv[cbase + j] = sv[j];
                }
            }
        }
        __syncwarp();
        cnt = 0;
    }

    // v: vertex, d: its out-degree, rs: R[v] (offsets mode; ignored in lazy mode)
    __device__ __forceinline__ void push(bool has, int32_t v, int64_t d, int64_t rs = 0) {
        const unsigned mask = __ballot_sync(0xffffffffu, has);
        if (mask == 0) return;
        const int pos = cnt + __popc(mask & lanemask_lt());
        if (has) { sv[pos] = v; if (qo && !Rl) { sd[pos] = (int32_t)d; sr[pos] = rs; } }
        cnt += __popc(mask);
        __syncwarp();
        if (cnt > kCap - 32) flush();
    }

    __device__ __forceinline__ void finish() {
        if (cnt > 0) flush();
        __syncwarp();
    }

    // End-of-step flush of ALL warps of the CTA with ONE global atomic: the
    // warps' packed (edges << S | count) totals are scanned in shared memory
    // and thread 0 reserves the CTA's range (and records the CTA's largest
    // degree). A grid step with few discoveries per warp otherwise ends with
    // one same-address atomicAdd (+ atomicMax) per warp of the grid on the
    // queue counter -- 4736 serialised L2 atomics per level (measured: the
    // 38K-edge second level of C2 took 27.6 us). Every thread of the CTA
    // must call it; sw: shared unsigned long long[2 * warps + 2].
    __device__ __forceinline__ void finish_cta(unsigned long long *sw) {
        const unsigned l = lane_id();
        const int wi = threadIdx.x >> 5, nwb = blockDim.x >> 5;
        if (Rl && cnt > 0) cnt = fill_from_R(cnt);
        const int k = cnt;
        constexpr int kR = kCap / 32;
        int64_t tot = 0;
        unsigned mx = 0;
        if (qo && k > 0) {
#pragma unroll 4
            for (int r = 0; r < kR; ++r) {
                const int j = r * 32 + (int)l;
                const int64_t d = (j < k) ? (int64_t)sd[j] : 0;
                tot += d;
                mx = max(mx, (unsigned)d);
            }
            tot = warp_sum<int64_t>(tot);
            mx = __reduce_max_sync(0xffffffffu, mx);
        }
        if (l == 0) {
            sw[wi] = qo ? (((unsigned long long)tot << S) | (unsigned long long)k) : (unsigned long long)k;
            sw[nwb + wi] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long run = 0, m = 0;
            for (int w = 0; w < nwb; ++w) {
                const unsigned long long x = sw[w];
                sw[w] = run;
                run += x;
                m = max(m, sw[nwb + w]);
            }
            sw[2 * nwb] = run ? atomicAdd(counter, run) : 0ull;
            if (dmax && m) atomicMax(dmax, m);
        }
        __syncthreads();
        if (k > 0) {
            const unsigned long long base = sw[2 * nwb] + sw[wi];
            const unsigned long long cbase = qo ? (base & ((1ull << S) - 1)) : base;
            if ((int64_t)(cbase + k) > cap) {
                if (l == 0) atomicExch(overflow, (unsigned long long)tag | ((cbase + k) << 8));
            } else {
                int64_t run = qo ? (int64_t)(base >> S) : 0;
#pragma unroll 4
                for (int r = 0; r < kR; ++r) {
                    if (r * 32 >= k) break;
                    const int j = r * 32 + (int)l;
                    if (qo) {
                        const int64_t d = (j < k) ? (int64_t)sd[j] : 0;
                        const int64_t x = warp_incl_scan<int64_t>(d);
                        if (j < k) {
                            qo[cbase + j] = run + x - d;
                            qr[cbase + j] = sr[j];
                        }
                        run += __shfl_sync(0xffffffffu, x, 31);
                    }
                    if (j < k) qv[cbase + j] = sv[j];
                }
            }
        }
        __syncwarp();
        cnt = 0;
        __syncthreads();  // sw may be reused
    }
};
using Appender = AppenderT<kStageCap>;

// Cache-policy loads (PTX createpolicy): the C / W streams are read once per
// traversal and must not evict the L2-resident per-vertex state (visited
// bitmap, depth, dist); that state is loaded with evict_last.
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *p, unsigned long long pol) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p, unsigned long long pol) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
// L1-allocating probe: may return a stale (older) word; used only as a filter
// where the bits it can miss are re-checked by an atomic.
__device__ __forceinline__ uint32_t ld_l1(const uint32_t *p) {
    uint32_t r;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
// L2-coherent probe of state updated by other SMs during the step.
__device__ __forceinline__ uint32_t ld_probe(const uint32_t *p, unsigned long long pol) {
    uint32_t r;
    asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ unsigned long long ld_probe(const unsigned long long *p, unsigned long long pol) {
    unsigned long long r;
    asm volatile("ld.global.cg.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
    return r;
}

// Shared-memory bitmap snapshot: a prefix of a
// global bitmap copied into shared memory at the start of a step, so the
// per-edge random probes of the step are shared-memory loads (bank conflicts
// only) instead of one 128-B L1TEX wavefront per distinct line.
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(saddr));
    return r;
}
__device__ __forceinline__ uint32_t atom_or_shared(uint32_t saddr, uint32_t v) {
    uint32_t r;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(r) : "r"(saddr), "r"(v) : "memory");
    return r;
}
// CTA-wide copy of words [0, words) of src into sbm (words % 4 == 0).
// The caller puts a __syncthreads() after it.
__device__ __forceinline__ void snapshot_bits(uint32_t *sbm, const uint32_t *src, int64_t words) {
    const int64_t n4 = words >> 2;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(sbm);
    constexpr int U = 4;
    for (int64_t i = threadIdx.x; i < n4; i += (int64_t)blockDim.x * U) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int64_t j = i + (int64_t)k * blockDim.x;
            if (j < n4) v[k] = __ldcg(s4 + j);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int64_t j = i + (int64_t)k * blockDim.x;
            if (j < n4) d4[j] = v[k];
        }
    }
}

// Smallest i in [0, F] with key(i) >= t, key non-decreasing, key(F) = +inf.
// 32-ary cooperative search: each round narrows the range 32x.
template <class Key>
__device__ __forceinline__ int64_t warp_lower_bound(int64_t F, int64_t t, Key key) {
    int64_t lo = 0, hi = F;  // answer in [lo, hi]
    const unsigned l = lane_id();
    while (hi - lo > 32) {
        // probes p_l = lo + (l+1)*step - 1, step = floor(span/32) >= 1: shifts only
        const int64_t step = (hi - lo) >> 5;
        const int64_t p = lo + (int64_t)(l + 1) * step - 1;
        const unsigned b = __ballot_sync(0xffffffffu, key(p) < t);
        const int k = __popc(b);  // probes [0,k) are < t
        const int64_t nlo = (k == 0) ? lo : lo + (int64_t)k * step;        // p_{k-1} + 1
        const int64_t nhi = (k == 32) ? hi : lo + (int64_t)(k + 1) * step - 1;  // p_k
        lo = nlo; hi = nhi;
    }
    const int64_t p = lo + l;
    const bool less = p < hi && key(p) < t;
    return lo + __popc(__ballot_sync(0xffffffffu, less));
}

// Both ends of a merge-path piece at once: the two half-warps run 16-ary
// searches side by side (one memory round trip per round for both), so a
// piece costs ceil(log16 F) dependent rounds instead of 2 ceil(log32 F) --
// e.g. 1 instead of 2 for a frontier of <= 16 hubs.
template <class Key>
__device__ __forceinline__ void warp_lower_bound2(int64_t F, int64_t t0, int64_t t1, Key key, int64_t &r0,
                                                  int64_t &r1) {
    const unsigned l = lane_id(), hl = l & 15;
    const unsigned hmask = (l >> 4) ? 0xffff0000u : 0x0000ffffu;
    const int64_t t = (l >> 4) ? t1 : t0;
    int64_t lo = 0, hi = F;  // answer in [lo, hi]
    for (;;) {
        const bool big = hi - lo > 16;
        if (!__any_sync(0xffffffffu, big)) break;
        const int64_t step = (hi - lo) >> 4;
        const int64_t p = lo + (int64_t)(hl + 1) * step - 1;
        const bool less = big && key(p) < t;
        const unsigned b = __ballot_sync(0xffffffffu, less) & hmask;
        if (big) {
            const int k = __popc(b);
            const int64_t nlo = (k == 0) ? lo : lo + (int64_t)k * step;
            const int64_t nhi = (k == 16) ? hi : lo + (int64_t)(k + 1) * step - 1;
            lo = nlo; hi = nhi;
        }
    }
    const int64_t p = lo + hl;
    const bool less = p < hi && key(p) < t;
    const int64_t res = lo + __popc(__ballot_sync(0xffffffffu, less) & hmask);
    r0 = __shfl_sync(0xffffffffu, res, 0);
    r1 = __shfl_sync(0xffffffffu, res, 16);
}

// ---------------------------------------------------------------------------
// Frontier views: where the queue of the current level lives.
//   GlobalFrontier: vertex ids, exclusive degree prefix and row starts R[v]
//                   in global memory (grid-wide levels). The filter wrote all
//                   three when it appended the vertex, so loading an entry is
//                   three independent coalesced loads (no dependent R[v]
//                   lookup: one memory round trip less per level). Entries are
//                   contiguous in edge space, so deg(j) = qo[j+1] - qo[j].
//   SmemFrontier:   the same three arrays in shared memory (single-CTA levels).
// ---------------------------------------------------------------------------
// The queue of a level was written by the previous level (before a grid
// barrier, whose fence makes it visible): plain loads, cached in L1, so the
// warps of an SM share one L2 request per line -- with a small frontier every
// warp of the grid searches and loads the SAME few lines (an L2 hot spot
// with L2-only loads).
struct GlobalFrontier {
    const int32_t *qv;
    const int64_t *qo;
    const int64_t *qr;
    int64_t F, E;
    __device__ __forceinline__ int64_t off(int64_t i) const { return qo[i]; }
    __device__ __forceinline__ void load(int64_t j, int32_t &v, int64_t &o, int64_t &rs, int64_t &end) const {
        v = qv[j];
        o = qo[j];
        rs = qr[j];
        end = (j + 1 < F) ? qo[j + 1] : E;
    }
};

struct SmemFrontier {
    const int32_t *qv;
    const int64_t *qo;
    const int64_t *rs;
    int64_t F, E;
    __device__ __forceinline__ int64_t off(int64_t i) const { return qo[i]; }
    __device__ __forceinline__ void load(int64_t j, int32_t &v, int64_t &o, int64_t &r, int64_t &end) const {
        v = qv[j];
        o = qo[j];
        r = rs[j];
        end = (j + 1 < F) ? qo[j + 1] : E;
    }
};

// ---------------------------------------------------------------------------
// Load-balanced advance over the frontier queue (merge-path).
// The merged sequence of frontier vertices and their edges (F + E items) is
// cut into equal pieces, one per warp (of the grid, or of one CTA), so every
// warp gets the same number of (vertex window loads + edge visits).
// Op must provide:
//   uint64_t entry(int32_t v)            per-source payload (e.g. dist[v])
//   void edges<U>(ok[], src[], pay[], dst[], eidx[])  process U edges per lane
// ---------------------------------------------------------------------------
constexpr int kUnroll = 4;
#ifndef GR_PF_AHEAD
#define GR_PF_AHEAD 2
#endif
constexpr int kPfAhead = GR_PF_AHEAD;
#ifndef GR_PIPE2
#define GR_PIPE2 0
#endif         // uniform groups: L2 prefetch of the C lines this many groups ahead
constexpr int64_t kMinChunk = 4096;           // dynamic merge-path: min items per piece
constexpr int64_t kTwcMaxDeg = 4096;          // auto strategy: TWC only without longer lists
constexpr int kGroup = 32 * kUnroll;          // edges per warp group

// Processes the merged items [d0, d1) (d0 < d1).
template <class Front, class Op>
__device__ __forceinline__ void expand_lb_range(const Front &fr, const int32_t *__restrict__ C, int64_t d0,
                                                int64_t d1, Op &op) {
    const int64_t F = fr.F, E = fr.E;
    auto mkey = [&](int64_t i) { return fr.off(i) + i; };  // merged position of vertex i
#ifndef GR_LB2
#define GR_LB2 1
#endif
#if GR_LB2
    int64_t i0, i1;
    warp_lower_bound2(F, d0, d1, mkey, i0, i1);
#else
    const int64_t i0 = warp_lower_bound(F, d0, mkey);
    const int64_t i1 = warp_lower_bound(F, d1, mkey);
#endif
    GR_TSTAMP(1);
    const int64_t e0 = d0 - i0, e1 = d1 - i1;
    if (e0 >= e1) return;
    const unsigned l = lane_id();
    const unsigned long long pol = policy_evict_first();
    // owner of edge e0: largest i with qo[i] <= e0 (i0 - 1, or i0 if its list starts at e0)
    int64_t i = (i0 < F && fr.off(i0) == e0) ? i0 : i0 - 1;
    int64_t e = e0;
    while (e < e1) {
        const int64_t j = i + l;
        const bool valid = j < F;
        int32_t v = 0;
        int64_t o = E, rs = 0, end = E;
        if (valid) fr.load(j, v, o, rs, end);
        const unsigned long long pay = valid ? op.entry(v) : 0ull;
        const int64_t shift = rs - o;               // C index of edge x of entry j = x + shift
        if (valid && end > o) {                     // first lines of every list of the window
            asm volatile("prefetch.global.L2 [%0];" ::"l"(C + rs));
            if (end - o > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + rs + 32));
        }
        int64_t wend = __shfl_sync(0xffffffffu, end, 31);
        GR_TSTAMP(2);
        if (wend > e1) wend = e1;
        // one group = 32 x kUnroll consecutive edges of the window: owner
        // search (uniform fast path or 5-step shuffle search) + C loads
        auto group = [&](int64_t b, bool *ok, int32_t *src, unsigned long long *sp, int64_t *eidx,
                         int32_t *dst) {
            // offsets relative to the batch start fit in 32 bits (clamped)
            const int64_t rel64 = o - b;
            const int32_t rel = rel64 < -0x7fffffffLL ? -0x7fffffff : (rel64 > 0x7fffffffLL ? 0x7fffffff : (int32_t)rel64);
            // uniform fast path: the whole group belongs to one entry
            const unsigned first = __ballot_sync(0xffffffffu, rel <= 0);
            const unsigned last = __ballot_sync(0xffffffffu, rel <= 32 * kUnroll - 1);
            const int kf = 31 - __clz(first), kl = 31 - __clz(last);
            if (kf == kl) {
                const int32_t sv = __shfl_sync(0xffffffffu, v, kf);
                const unsigned long long spv = __shfl_sync(0xffffffffu, pay, kf);
                const int64_t sh = __shfl_sync(0xffffffffu, shift, kf);
                // stream ahead: a later group (4 lines) into L2
                const int64_t pf = b + kPfAhead * 32 * kUnroll + (int64_t)l * 32;
                if (l < kUnroll && pf < wend) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + pf + sh));
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t my = b + u * 32 + l;
                    ok[u] = my < wend;
                    src[u] = sv;
                    sp[u] = spv;
                    eidx[u] = my + sh;
                }
            } else {
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int32_t myr = u * 32 + (int32_t)l;
                    int k = 0;
#pragma unroll
                    for (int s = 16; s >= 1; s >>= 1) {
                        const int32_t oc = __shfl_sync(0xffffffffu, rel, k + s);
                        if (oc <= myr) k += s;
                    }
                    const int64_t my = b + myr;
                    ok[u] = my < wend;
                    src[u] = __shfl_sync(0xffffffffu, v, k);
                    sp[u] = __shfl_sync(0xffffffffu, pay, k);
                    eidx[u] = my + __shfl_sync(0xffffffffu, shift, k);
                }
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) dst[u] = ok[u] ? ld_stream(C + eidx[u], pol) : 0;
        };
#if GR_PIPE2
        // two groups in flight: the C loads of group g+1 are issued before
        // group g's per-edge work (probes, claims, appends) starts
        bool ok[kUnroll];
        int32_t src[kUnroll];
        unsigned long long sp[kUnroll];
        int64_t eidx[kUnroll];
        int32_t dst[kUnroll];
        if (e < wend) group(e, ok, src, sp, eidx, dst);
        for (int64_t b = e; b < wend; b += 32 * kUnroll) {
            bool ok1[kUnroll];
            int32_t src1[kUnroll];
            unsigned long long sp1[kUnroll];
            int64_t eidx1[kUnroll];
            int32_t dst1[kUnroll];
            const bool more = b + 32 * kUnroll < wend;
            if (more) group(b + 32 * kUnroll, ok1, src1, sp1, eidx1, dst1);
            GR_TSTAMP(3);
            op.template edges<kUnroll>(ok, src, sp, dst, eidx);
            GR_TSTAMP(4);
            if (more) {
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    ok[u] = ok1[u]; src[u] = src1[u]; sp[u] = sp1[u]; eidx[u] = eidx1[u]; dst[u] = dst1[u];
                }
            }
        }
#else
        for (int64_t b = e; b < wend; b += 32 * kUnroll) {
            bool ok[kUnroll];
            int32_t src[kUnroll];
            unsigned long long sp[kUnroll];
            int64_t eidx[kUnroll];
            int32_t dst[kUnroll];
            group(b, ok, src, sp, eidx, dst);
            GR_TSTAMP(3);
            op.template edges<kUnroll>(ok, src, sp, dst, eidx);
            GR_TSTAMP(4);
        }
#endif
        e = wend;
        i += 32;
    }
}

// Static partition: warp gw of nw takes the gw-th equal piece of the merged
// sequence. With `work` (a zeroed grid-wide counter): dynamic partition, the
// merged sequence is cut into kChunks pieces per warp; warp gw starts with
// piece gw and then takes the next unclaimed piece (one atomic per piece), so
// a slow piece (measured: a few CTAs of a static partition finish 2-5x after
// the median on C2 push levels) no longer holds the whole grid at the barrier.
template <class Front, class Op>
__device__ __forceinline__ void expand_lb(const Front &fr, const int32_t *__restrict__ C, int64_t gw,
                                          int64_t nw, Op &op, unsigned long long *work = nullptr,
                                          int kChunks = 4) {
    const int64_t F = fr.F, E = fr.E;
    if (E <= 0 || F <= 0) return;
    const int64_t D = F + E;
    if (work == nullptr || D < nw * 256) {
        const int64_t d0 = (D * gw) / nw;  // D < 2^40, nw < 2^20: no overflow
        const int64_t d1 = (D * (gw + 1)) / nw;
        if (d0 < d1) expand_lb_range(fr, C, d0, d1, op);
        return;
    }
    const int64_t P0 = nw * kChunks;
    int64_t K = (D + P0 - 1) / P0;
    if (K < kMinChunk) {                   // two searches per piece: keep pieces long,
        const int64_t Kw = (D + nw - 1) / nw;  // but never fewer pieces than warps
        K = Kw < kMinChunk ? Kw : kMinChunk;
    }
    const int64_t P = (D + K - 1) / K;
    int64_t c = gw;
    while (c < P) {
        const int64_t d0 = c * K;
        const int64_t d1 = (d0 + K < D) ? d0 + K : D;
        if (d0 < d1) expand_lb_range(fr, C, d0, d1, op);
        unsigned long long t = 0;
        if (lane_id() == 0) t = atomicAdd(work, 1ull);
        c = nw + (int64_t)__shfl_sync(0xffffffffu, t, 0);
    }
}

// ---------------------------------------------------------------------------
// Node-granular thread/warp/CTA advance ("per-warp and per-CTA coarse-grained"
// mapping of Merrill et al., with the fine-grained per-thread class
// of P:693-706). Each CTA takes a contiguous slice of the frontier, one vertex
// per thread per round; lists are classified by size:
//   large  (> blockDim edges): threads arbitrate for the whole CTA, which
//          sweeps the winner's list (coalesced);
//   medium (> 32 edges):       lanes arbitrate for their warp;
//   small  (<= 32 edges):      the warp concatenates its small lists (warp
//          scan of degrees) and maps each edge to its owner with the 5-step
//          shuffle search, i.e. per-thread work balanced inside the warp.
// No frontier-wide prefix or search is needed (node-granular balancing; the
// paper selects it for frontiers below the 4096 threshold).
// All threads of the CTA must call it (CTA barriers inside).
// ---------------------------------------------------------------------------
template <class Front, class Op>
__device__ __forceinline__ void expand_twc(const Front &fr, const int32_t *__restrict__ C, Op &op,
                                           int *s_win) {
    const int64_t F = fr.F;
    const int64_t j0 = F * blockIdx.x / gridDim.x, j1 = F * (blockIdx.x + 1) / gridDim.x;
    const unsigned l = lane_id();
    const int wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const unsigned long long pol = policy_evict_first();
    for (int64_t base = j0; base < j1; base += blockDim.x) {  // uniform trip count in the CTA
        const int64_t j = base + threadIdx.x;
        int32_t v = 0;
        int64_t o = 0, rs = 0, end = 0;
        if (j < j1) fr.load(j, v, o, rs, end);
        int64_t deg = end - o;
        const unsigned long long pay = (j < j1) ? op.entry(v) : 0ull;
        // ---- large lists: the whole CTA ---------------------------------------
        for (;;) {
            if (threadIdx.x == 0) *s_win = -1;
            __syncthreads();
            if (deg > (int64_t)blockDim.x) atomicMax(s_win, (int)threadIdx.x);
            __syncthreads();
            const int win = *s_win;
            __syncthreads();
            if (win < 0) break;
            // broadcast the winner's list through shared memory
            __shared__ long long s_list[3];
            if ((int)threadIdx.x == win) { s_list[0] = rs; s_list[1] = deg; s_list[2] = ((long long)v << 32) | (unsigned)pay; deg = 0; }
            __syncthreads();
            const int64_t lrs = s_list[0], ldeg = s_list[1];
            const int32_t lv = (int32_t)(s_list[2] >> 32);
            const unsigned long long lpay = (unsigned)(s_list[2] & 0xffffffffu);
            __syncthreads();
            for (int64_t x = (int64_t)wib * kGroup; x < ldeg; x += (int64_t)nwb * kGroup) {
                bool ok[kUnroll];
                int32_t src[kUnroll], dst[kUnroll];
                unsigned long long sp[kUnroll];
                int64_t eidx[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t k = x + u * 32 + l;
                    ok[u] = k < ldeg;
                    src[u] = lv;
                    sp[u] = lpay;
                    eidx[u] = lrs + k;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) dst[u] = ok[u] ? ld_stream(C + eidx[u], pol) : 0;
                op.template edges<kUnroll>(ok, src, sp, dst, eidx);
            }
        }
        // ---- medium lists: the warp ----------------------------------------------
        for (;;) {
            const unsigned med = __ballot_sync(0xffffffffu, deg > 32);
            if (!med) break;
            const int ldr = __ffs(med) - 1;
            const int64_t lrs = __shfl_sync(0xffffffffu, rs, ldr);
            const int64_t ldeg = __shfl_sync(0xffffffffu, deg, ldr);
            const int32_t lv = __shfl_sync(0xffffffffu, v, ldr);
            const unsigned long long lpay = __shfl_sync(0xffffffffu, pay, ldr);
            if ((int)l == ldr) deg = 0;
            for (int64_t x = 0; x < ldeg; x += kGroup) {
                bool ok[kUnroll];
                int32_t src[kUnroll], dst[kUnroll];
                unsigned long long sp[kUnroll];
                int64_t eidx[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t k = x + u * 32 + l;
                    ok[u] = k < ldeg;
                    src[u] = lv;
                    sp[u] = lpay;
                    eidx[u] = lrs + k;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) dst[u] = ok[u] ? ld_stream(C + eidx[u], pol) : 0;
                op.template edges<kUnroll>(ok, src, sp, dst, eidx);
            }
        }
        // ---- small lists: warp-level concatenation ---------------------------
        const int32_t d32 = (int32_t)deg;  // <= 32
        const int32_t incl = warp_incl_scan<int32_t>(d32);
        const int32_t excl = incl - d32;
        const int32_t T = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t shift = rs - excl;
        for (int32_t x = 0; x < T; x += kGroup) {
            bool ok[kUnroll];
            int32_t src[kUnroll], dst[kUnroll];
            unsigned long long sp[kUnroll];
            int64_t eidx[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int32_t my = x + u * 32 + (int32_t)l;
                int k = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const int32_t oc = __shfl_sync(0xffffffffu, excl, k + st);
                    if (oc <= my) k += st;
                }
                ok[u] = my < T;
                src[u] = __shfl_sync(0xffffffffu, v, k);
                sp[u] = __shfl_sync(0xffffffffu, pay, k);
                eidx[u] = my + __shfl_sync(0xffffffffu, shift, k);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) dst[u] = ok[u] ? ld_stream(C + eidx[u], pol) : 0;
            op.template edges<kUnroll>(ok, src, sp, dst, eidx);
        }
    }
}

// ---------------------------------------------------------------------------
// Thread-block cluster helpers of the narrow-level kernels (bfs.cu / sssp.cu
// *_ell_cluster_kernel): one cluster of up to 16 CTAs x 1024 threads, the
// frontier queues in distributed shared memory.
// ---------------------------------------------------------------------------
constexpr int kClBlock = 1024;
constexpr int kClQ = 4 * kClBlock;   // per-CTA queue: <= 4 appends per thread per level
constexpr int kClMax = 16;
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long ld_dsmem_u64(const unsigned long long *p, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    unsigned long long v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(r) : "memory");
    return v;
}
__device__ __forceinline__ int32_t ld_dsmem_s32(const int32_t *p, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    int32_t v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(r) : "memory");
    return v;
}


// ---------------------------------------------------------------------------
// RemoveRedundant stamp of SSSP ("a bitmap flag array associated
// with the frontier", reading A-7): the key of iteration `base` = 2*it and
// slice is base + 1 for the near queue, base for the far pile, claimed with
// atomicMax. A far improvement that lands after a near one can then never
// re-open the near slot, so a vertex enters the near queue at most once per
// iteration (with atomicExch of alternating keys, the sequence near, far,
// near admitted it twice -- measured: near queue > n on a dense graph).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t stamp_key(int32_t base, bool far) { return base + (far ? 0 : 1); }

// ---------------------------------------------------------------------------
// Bounded-degree advance (Graph::ell, every out-degree <= 4): one frontier
// vertex per lane, its whole neighbour list in one aligned 16-byte load --
// the thread-granular class of P:693-706 with no prefix, search or row-offset
// lookup. Frontier entry j goes to lane j%32 of warp (j/32) of the grid,
// warps interleaved over the CTAs so a narrow frontier spreads over all SMs.
// Op must provide slots(valid, v, int4 s) (warp-converged).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int4 ld_ell(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <class Op>
__device__ __forceinline__ void expand_ell(const int32_t *qv, int64_t f, const int4 *__restrict__ ell, int64_t gw,
                                           int64_t nw, Op &op) {
    const unsigned l = lane_id();
    for (int64_t j0 = gw * 32; j0 < f; j0 += nw * 32) {
        const int64_t j = j0 + l;
        const bool valid = j < f;
        const int32_t v = valid ? qv[j] : 0;
        GR_TDEP(1, v);
        const int4 s = valid ? ld_ell(ell + v) : make_int4(-1, -1, -1, -1);
        GR_TDEP(2, s.x);
        op.slots(valid, v, s);
        GR_TSTAMP(4);
    }
}

// Weighted variant (SSSP, Graph::ellw): the frontier vertex's payload
// (op.entry, e.g. its distance) and its 32-byte record (ids, then
// (weight << 3) | degree per slot) are loaded in parallel.
// Op must provide entry(v) and slots(valid, v, pay, int4 ids, int4 wts).
template <class Op>
__device__ __forceinline__ void expand_ellw(const int32_t *qv, int64_t f, const int4 *__restrict__ ellw, int64_t gw,
                                            int64_t nw, Op &op) {
    const unsigned l = lane_id();
    for (int64_t j0 = gw * 32; j0 < f; j0 += nw * 32) {
        const int64_t j = j0 + l;
        const bool valid = j < f;
        const int32_t v = valid ? qv[j] : 0;
        const unsigned long long pay = valid ? op.entry(v) : 0ull;
        const int4 id = valid ? ld_ell(ellw + 2 * (int64_t)v) : make_int4(-1, -1, -1, -1);
        const int4 wt = valid ? ld_ell(ellw + 2 * (int64_t)v + 1) : make_int4(0, 0, 0, 0);
        op.slots(valid, v, pay, id, wt);
    }
}

// ---------------------------------------------------------------------------
// Pipelined load-balanced advance (grid levels). Same merge-path partition
// and owner mapping as expand_lb, but the neighbour ids (and weights) of the
// next kStages groups of 128 edges are copied global -> shared memory with
// cp.async (LDGSTS) while the current group is processed: the per-SM bytes in
// flight no longer depend on registers (64 per thread at 32 warps/SM), which
// made the C stream latency-bound. A group owned by one list (hub vertices:
// most edges of a power-law graph) is copied as 16-byte chunks of the aligned
// superset of its range; a mixed group element by element.
// ---------------------------------------------------------------------------
constexpr int kGroupBuf = kGroup + 8;         // aligned superset (16-byte chunks)

struct PipeStageMeta {
    long long b;       // first edge (frontier-edge index) of the group
    long long lim;     // end of the valid range of the group
    int mode;          // >= 0: single owner, element k at buf[mode + k]; -1: mixed
    int src;           // single owner vertex
    unsigned pay;      // single owner payload
    int pad;
};

template <int kStages, bool kW>   // kW: weights + per-source payload (SSSP)
struct PipeWarpSmem {
    int32_t dst[kStages][kGroupBuf];
    int32_t wt[kW ? kStages : 1][kW ? kGroupBuf : 4];
    int32_t src[kStages][kGroup];
    uint32_t pay[kW ? kStages : 1][kW ? kGroup : 4];
    PipeStageMeta meta[kStages];
};

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;
        default: cp_async_wait<7>(); break;
    }
}

// Op must provide entry(v) (payload, low 32 bits used) and
//   edges<U>(ok[], src[], pay[], dst[], wt[])
template <int kStages, bool kW, class Front, class Op>
__device__ __forceinline__ void expand_pipe(const Front &fr, const int32_t *__restrict__ C,
                                            const uint32_t *__restrict__ W, int64_t gw, int64_t nw,
                                            Op &op, PipeWarpSmem<kStages, kW> *ps) {
    const int64_t F = fr.F, E = fr.E;
    if (E <= 0 || F <= 0) return;
    const int64_t D = F + E;
    const int64_t d0 = (D * gw) / nw;
    const int64_t d1 = (D * (gw + 1)) / nw;
    if (d0 >= d1) return;
    auto mkey = [&](int64_t i) { return fr.off(i) + i; };
    const int64_t i0 = warp_lower_bound(F, d0, mkey);
    const int64_t i1 = warp_lower_bound(F, d1, mkey);
    const int64_t e0 = d0 - i0, e1 = d1 - i1;
    if (e0 >= e1) return;
    const unsigned l = lane_id();

    // ---- generator state: current window of 32 frontier entries -------------
    int64_t gi = (i0 < F && fr.off(i0) == e0) ? i0 : i0 - 1;
    int32_t v = 0;
    int64_t o = E, shift = 0, wend = E;
    uint32_t pay = 0;
    auto load_window = [&]() {
        const int64_t j = gi + l;
        const bool valid = j < F;
        int64_t rs = 0, end = E;
        v = 0;
        o = E;
        if (valid) fr.load(j, v, o, rs, end);
        pay = valid ? (uint32_t)op.entry(v) : 0u;
        shift = rs - o;
        wend = __shfl_sync(0xffffffffu, end, 31);
        if (wend > e1) wend = e1;
    };
    load_window();
    int64_t b = e0;  // next edge to issue

    auto issue = [&](int s) -> bool {
        while (b >= wend) {
            if (b >= e1) return false;
            gi += 32;
            load_window();
        }
        const int64_t lim = (wend < b + kGroup) ? wend : b + kGroup;
        const int64_t rel64 = o - b;
        const int32_t rel = rel64 < -0x7fffffffLL ? -0x7fffffff
                          : (rel64 > 0x7fffffffLL ? 0x7fffffff : (int32_t)rel64);
        const unsigned first = __ballot_sync(0xffffffffu, rel <= 0);
        const unsigned last = __ballot_sync(0xffffffffu, rel <= (int32_t)(lim - b) - 1);
        const int kf = 31 - __clz(first), kl = 31 - __clz(last);
        PipeStageMeta m;
        m.b = b;
        m.lim = lim;
        if (kf == kl) {
            const int64_t sh = __shfl_sync(0xffffffffu, shift, kf);
            m.src = __shfl_sync(0xffffffffu, v, kf);
            m.pay = __shfl_sync(0xffffffffu, pay, kf);
            const int64_t g0 = b + sh;           // C index of the first edge
            const int64_t A = g0 & ~3ll;         // 16-byte aligned start
            m.mode = (int)(g0 - A);
            const int n16 = (int)((m.mode + (lim - b) + 3) >> 2);  // <= 33 chunks
            for (int c = (int)l; c < n16; c += 32) {
                cp_async16(&ps->dst[s][4 * c], C + A + 4 * c);
                if (kW) cp_async16(&ps->wt[kW ? s : 0][4 * c], W + A + 4 * c);
            }
        } else {
            m.mode = -1;
            m.src = 0;
            m.pay = 0;
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int32_t myr = u * 32 + (int32_t)l;
                int k = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const int32_t oc = __shfl_sync(0xffffffffu, rel, k + st);
                    if (oc <= myr) k += st;
                }
                const int64_t my = b + myr;
                const int32_t sv = __shfl_sync(0xffffffffu, v, k);
                const uint32_t spv = __shfl_sync(0xffffffffu, pay, k);
                const int64_t ci = my + __shfl_sync(0xffffffffu, shift, k);
                if (my < lim) {
                    cp_async4(&ps->dst[s][myr], C + ci);
                    if (kW) cp_async4(&ps->wt[kW ? s : 0][myr], W + ci);
                    ps->src[s][myr] = sv;
                    if (kW) ps->pay[kW ? s : 0][myr] = spv;
                }
            }
        }
        cp_async_commit();
        if (l == 0) ps->meta[s] = m;
        b = lim;
        return true;
    };

    int issued = 0, consumed = 0;
    for (int s = 0; s < kStages; ++s) {
        if (!issue(s)) break;
        ++issued;
    }
    while (consumed < issued) {
        const int s = consumed % kStages;
        cp_async_wait_dyn(issued - consumed - 1);
        __syncwarp();
        const PipeStageMeta m = ps->meta[s];
        bool ok[kUnroll];
        int32_t src[kUnroll], dst[kUnroll];
        unsigned long long pp[kUnroll];
        uint32_t wt[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int k = u * 32 + (int)l;
            ok[u] = m.b + k < m.lim;
            const int idx = m.mode >= 0 ? m.mode + k : k;
            dst[u] = ok[u] ? ps->dst[s][idx] : 0;
            wt[u] = (kW && ok[u]) ? (uint32_t)ps->wt[kW ? s : 0][idx] : 0u;
            src[u] = m.mode >= 0 ? m.src : (ok[u] ? ps->src[s][k] : 0);
            pp[u] = !kW ? 0ull : (m.mode >= 0 ? m.pay : (ok[u] ? ps->pay[kW ? s : 0][k] : 0u));
        }
        __syncwarp();  // stage s may be refilled below
        ++consumed;
        if (issue(issued % kStages)) ++issued;
        op.template edges<kUnroll>(ok, src, pp, dst, wt);
    }
}

}  // namespace gr
