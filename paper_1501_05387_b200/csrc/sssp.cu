// sssp.cu -- single-source shortest paths, delta-stepping with Gunrock's
// two-level near/far priority queue, as ONE persistent cooperative kernel.
//
// Paper: Alg. 1: UpdateLabel = "new_label < atomicMin(labels[d],
// new_label)", SetPred, RemoveRedundant via an
// output-queue stamp ("a bitmap flag array associated with the
// frontier to remove redundant vertices" P:950-951); priority queue (P:838-857,
// "an additional filter pass between two iterations" P:941-942).
// Readings: A-7 (stamp keyed by iteration AND slice), A-8 (one fused relax
// kernel step per iteration + far re-split pass), A-9 (64-bit packed
// atomicMin keeps pred consistent with dist), A-10 (delta), A-11 (far pile:
// drop stale, jump threshold to the band of the minimum far distance).
#include "frontier.cuh"

namespace gr {

struct SsspArgs {
    int64_t n, m;
    const int64_t *R;
    const int32_t *C;
    const uint32_t *W;
    const uint32_t *CW;       // packed (C << 7) | W, or null
    const int64_t *Rt;        // in-list offsets (== R when symmetric)
    const uint32_t *CWt;      // packed weighted in-lists (u << 7) | w(u,v), or null: no pull steps
    const int4 *ellw;         // bounded-degree weighted adjacency (null: none; Graph::ellw)
    int32_t lazy_r;           // near queue: row offsets loaded at the appender's flush
    int32_t bar_ns;           // GridBar backoff cap (ns)
    int32_t resume;           // bounded-degree graphs: sssp_ell_cluster_kernel ran the first steps
    int32_t cl_stamp;         // cluster near iterations dedupe appends by stamp (1) or not (0)
    int32_t cl_farres;        // cluster near iterations reserve far slots before the atomicMin (1)
    uint32_t *fb;             // pull steps: bitmap of the near frontier [ceil(n/32)]
    int32_t direction;        // 0 auto, 1 push, 2 pull (near iterations; reading A-24)
    double alpha;             // auto: pull when m_f * alpha > m
    unsigned long long *dp;   // (dist << 32) | pred
    int32_t *stamp;
    int32_t *qv[2];
    int64_t *qo[2];
    int64_t *qr[2];
    int32_t *far[2];
    int64_t far_cap;
    Ctl *ctl;
    gr_level_stats *stats;
    int32_t src;
    uint64_t delta;
    int64_t lb_threshold;     // auto strategy: thread/warp/CTA only below this frontier size (A-4)
    int stream_queues;        // near/far queue stores with the streaming cache hint
    int S;
};

#ifndef GR_SSSP_PIPE
#define GR_SSSP_PIPE 0  // cp.async pipeline off: its shared memory displaces L1 (measured slower)
#endif
#if GR_SSSP_PIPE
constexpr int kSsspStages = 2;     // cp.async pipeline depth (C + W + payload per stage)
#endif
#ifndef GR_SSSP_STAGE
#define GR_SSSP_STAGE 64
#endif
constexpr int kSsspStage = GR_SSSP_STAGE;  // append staging per warp (near and far)
using SsspAppender = AppenderT<kSsspStage>;

struct SsspSmem {
#if GR_SSSP_PIPE
    PipeWarpSmem<kSsspStages, true> pipe[kWarpsPerBlock];
#endif
    int32_t sv[kWarpsPerBlock][kSsspStage];   // near staging
    int32_t sd[kWarpsPerBlock][kSsspStage];
    int64_t sr[kWarpsPerBlock][kSsspStage];
    int32_t fv[kWarpsPerBlock][kSsspStage];   // far staging
    unsigned long long ctl[8];
    unsigned long long bsum[4];
    unsigned long long wsum[2 * kWarpsPerBlock + 2];  // Appender::finish_cta
    int win;  // expand_twc: CTA arbitration
};

// Fused advance + compute + filter of one near iteration (a10).
// kPacked: the advance streams the packed edge array CW[e] = (C[e] << 7) | W[e]
// (graph.cu; n < 2^25, weights <= 127 -- the paper's are 1..64)
// instead of C and W: 4 bytes per relaxed edge instead of 8.
template <bool kPacked>
struct RelaxOpT {
    unsigned long long *dp;
    int32_t *stamp;
    const uint32_t *W;
    const int64_t *R;
    uint64_t thr;
    int32_t key_near;   // 2*it: stamp keys of this iteration (stamp_key, A-7)
    SsspAppender *nearq;
    SsspAppender *farq;
    unsigned long long nimp;
    unsigned long long pol_keep;  // evict_last for dist
    unsigned long long pol_stream;  // evict_first for the W stream (read once, like C)

    __device__ __forceinline__ unsigned long long entry(int32_t v) {
        return ld_probe(dp + v, pol_keep) >> 32;  // dist[u] read when the window is loaded
    }

    // x[]: the edge weights staged in shared memory by the pipelined advance
    // (uint32), or the edge indices (int64) from expand_lb / expand_twc
    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *du,
                                          const int32_t *dst, const T5 *x) {
        unsigned long long cur[U];
        uint32_t w[U];
        int32_t vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (kPacked) {
                vv[u] = (int32_t)((uint32_t)dst[u] >> 7);
                w[u] = (uint32_t)dst[u] & 127u;
            } else {
                vv[u] = dst[u];
                if constexpr (sizeof(T5) == 8) w[u] = ok[u] ? ld_stream(W + x[u], pol_stream) : 0u;
                else w[u] = (uint32_t)x[u];
            }
            cur[u] = ok[u] ? ld_probe(dp + vv[u], pol_keep) : 0ull;
        }
        // UpdateLabel for every edge of the lane in flight at once, then the
        // RemoveRedundant stamps of the improved ones at once (each atomic
        // consumed inside its own branch made them one dependent round trip
        // apiece), then the filter
        unsigned long long old[U];
        bool tr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long nd = du[u] + w[u];
            tr[u] = ok[u] && nd < (cur[u] >> 32);
            old[u] = tr[u] ? atomicMin(dp + vv[u], (nd << 32) | (unsigned int)src[u]) : 0ull;
        }
        bool imp[U];
        int32_t ex[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long nd = du[u] + w[u];
            imp[u] = tr[u] && nd < (old[u] >> 32);
            const int32_t key = stamp_key(key_near, nd >= thr);
            ex[u] = imp[u] ? atomicMax(stamp + vv[u], key) : key;
            if (imp[u]) ++nimp;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned long long nd = du[u] + w[u];
            const bool far = nd >= thr;
            const bool first = imp[u] && ex[u] < stamp_key(key_near, far);
            const bool to_near = first && !far;
            int64_t deg = 0, rs = 0;
            if (to_near && !nearq->Rl) { rs = R[vv[u]]; deg = R[vv[u] + 1] - rs; }
            nearq->push(to_near && (nearq->Rl || deg > 0), vv[u], deg, rs);
            farq->push(first && far, vv[u], 0);
        }
    }

    // Bounded-degree adjacency (expand_ellw, Graph::ellw): the four (v, w)
    // slots of frontier vertex u arrive in one 32-byte record whose weight
    // words also carry deg(v). No culling probe: on these graphs a relax step
    // is latency-bound, so the packed atomicMin is issued directly, with the
    // pred field all ones: it lowers dp[v] only for a STRICTLY smaller
    // distance (a tie leaves the current parent, as the probe-guarded push
    // relax does; with zero weights a tie-won parent could close a pred
    // cycle), and the winner then lowers the pred field to u with a
    // fire-and-forget RED.MIN (same distance, any later smaller distance
    // already beats both).
    const int4 *ellw = nullptr;
    __device__ __forceinline__ void slots(bool, int32_t u, unsigned long long du, int4 id4, int4 wt4) {
        const int32_t id[4] = {id4.x, id4.y, id4.z, id4.w};
        const int32_t wt[4] = {wt4.x, wt4.y, wt4.z, wt4.w};
        unsigned long long nd[4], old[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            nd[k] = du + (unsigned long long)((uint32_t)wt[k] >> 3);
            old[k] = id[k] >= 0 ? atomicMin(dp + id[k], (nd[k] << 32) | 0xffffffffull) : 0ull;
        }
        bool imp[4], far[4], first[4];
        int32_t ex[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            imp[k] = id[k] >= 0 && nd[k] < (old[k] >> 32);
            if (imp[k]) atomicMin(dp + id[k], (nd[k] << 32) | (unsigned int)u);  // result unused: RED.MIN
            far[k] = nd[k] >= thr;
            const int32_t key = stamp_key(key_near, far[k]);
            ex[k] = imp[k] ? atomicMax(stamp + id[k], key) : key;  // all in flight, read below
            if (imp[k]) ++nimp;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) first[k] = imp[k] && ex[k] < stamp_key(key_near, far[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t deg = wt[k] & 7;
            const bool to_near = first[k] && !far[k];
            if (to_near && deg) asm volatile("prefetch.global.L2 [%0];" ::"l"(ellw + 2 * (int64_t)id[k]));
            nearq->push(to_near && deg > 0, id[k], deg, 0);
            farq->push(first[k] && far[k], id[k], 0);
        }
    }
};

// Pull (bottom-up) near iteration (the paper names SSSP as a next
// user of pull; reading A-24): the near frontier as a bitmap, and
// every vertex v takes min over its in-edges (u, v) with u in the frontier of
// dist[u] + w(u, v) -- the same relaxations as the push step, computed at
// the receiver, so dp[v] needs no atomic (v is owned by one lane, or by one
// warp for lists longer than kSsspPullLane). An improved v joins the near
// queue (nd < thr) or the far pile, once (no stamp race: one owner).
constexpr int64_t kSsspPullLane = 8;

template <class App>
__device__ __forceinline__ unsigned long long sssp_pull_step(const SsspArgs &a, uint64_t thr, int32_t key_near,
                                                             int64_t gw, int64_t nw, App &nearq, App &farq,
                                                             unsigned long long pol) {
    const unsigned l = lane_id();
    unsigned long long nimp = 0;
    const unsigned long long pol_s = policy_evict_first();
    auto relax_in = [&](uint32_t x, unsigned long long &best) {  // one in-edge, packed (u << 7) | w
        const int32_t u = (int32_t)(x >> 7);
        if ((a.fb[u >> 5] >> (u & 31)) & 1u) {
            const unsigned long long du = ld_probe(a.dp + u, pol) >> 32;
            const unsigned long long cand = ((du + (x & 127u)) << 32) | (unsigned)u;
            best = cand < best ? cand : best;
        }
    };
    for (int64_t base = gw * 32; base < a.n; base += nw * 32) {
        const int64_t v = base + l;
        int64_t b = 0, e = 0;
        if (v < a.n) { b = a.Rt[v]; e = a.Rt[v + 1]; }
        unsigned long long best = ~0ull;  // (nd << 32) | parent: smallest nd, then smallest parent (A-9)
        const bool lane_list = e > b && e - b <= kSsspPullLane;
        if (lane_list) {
            for (int64_t x0 = b; x0 < e; x0 += 4) {
                uint32_t xx[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) xx[j] = x0 + j < e ? ld_stream(a.CWt + x0 + j, pol_s) : 0xffffffffu;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (x0 + j < e) relax_in(xx[j], best);
            }
        }
        unsigned lm = __ballot_sync(0xffffffffu, e - b > kSsspPullLane);
        while (lm) {
            const int ld = __ffs(lm) - 1;
            lm &= lm - 1;
            const int64_t lb = __shfl_sync(0xffffffffu, b, ld), le = __shfl_sync(0xffffffffu, e, ld);
            unsigned long long part = ~0ull;
            for (int64_t x = lb + l; x < le; x += 32) relax_in(ld_stream(a.CWt + x, pol_s), part);
#pragma unroll
            for (int sh = 16; sh > 0; sh >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, part, sh);
                part = o < part ? o : part;
            }
            if ((int)l == ld) best = part;
        }
        bool to_near = false, to_far = false;
        int64_t deg = 0, rs = 0;
        if (best != ~0ull) {
            const unsigned long long cur = ld_probe(a.dp + v, pol);
            if ((best >> 32) < (cur >> 32)) {
                a.dp[v] = best;  // v's owner: a plain 64-bit store
                const bool far = (best >> 32) >= thr;
                a.stamp[v] = stamp_key(key_near, far);
                if (far) to_far = true;
                else { to_near = true; if (!nearq.Rl) { rs = a.R[v]; deg = a.R[v + 1] - rs; } }
                ++nimp;
            }
        }
        nearq.push(to_near && (nearq.Rl || deg > 0), (int32_t)v, deg, rs);
        farq.push(to_far, (int32_t)v, 0);
    }
    return nimp;
}

__device__ __forceinline__ long long sssp_gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool kPacked>
__global__ void __launch_bounds__(kBlock, kMinBlocks) sssp_kernel(SsspArgs a) {
    using RelaxOp = RelaxOpT<kPacked>;
    const int32_t *Cs = kPacked ? reinterpret_cast<const int32_t *>(a.CW) : a.C;  // the advance's edge stream
    const bool env_stream = a.stream_queues;
    const GridBar grid{&a.ctl->gbar, a.bar_ns};
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SsspSmem *s = reinterpret_cast<SsspSmem *>(smem_raw);

    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gw = tid >> 5;
    const int64_t nw = nthreads >> 5;
    const int wib = threadIdx.x >> 5;
    const unsigned long long cmask = (1ull << a.S) - 1;

    uint64_t thr = a.delta;          // near band is [.., thr)
    int32_t it = 0;                  // stamp iteration (keys 2*it, 2*it+1)
    int fp = 0;                      // current far buffer
    int k = 0;                       // step index (slots, queue ping-pong)
    long long t_prev = 0;
    if (a.resume) {
        // the narrow first steps ran in sssp_ell_cluster_kernel: finished, or
        // the state of step bstate[0] handed over (queue, far piles, slots)
        if (threadIdx.x == 0) {
            long long x[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) x[q] = __ldcg(a.ctl->bstate + q);
#pragma unroll
            for (int q = 0; q < 5; ++q) s->ctl[q] = (unsigned long long)x[q];
            s->ctl[5] = __ldcg(&a.ctl->handoff);
        }
        __syncthreads();
        if (s->ctl[5] != 1ull) return;
        k = (int)(long long)s->ctl[0];
        it = (int32_t)(long long)s->ctl[1];
        thr = (uint64_t)s->ctl[2];
        fp = (int)(long long)s->ctl[3];
        if (tid == 0) t_prev = (long long)s->ctl[4];
        __syncthreads();
    } else {
    // ---- Set_Problem_Data, the source's entries written by their
    // owner thread in the same pass: one grid barrier ----------------------
    const int64_t d_src = a.R[a.src + 1] - a.R[a.src];
    for (int64_t v = tid; v < a.n; v += nthreads) {
        // dist = UINT32_MAX (inf), pred = -1; the source: dist 0, pred = src (A-1)
        a.dp[v] = (v == a.src) ? (unsigned long long)(unsigned int)a.src : ~0ull;
        a.stamp[v] = -1;
    }
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) {
        const int64_t word = tid % (int64_t)(sizeof(Slot) / 8);
        unsigned long long x = word == (int64_t)(offsetof(Slot, minfar) / 8) ? ~0ull : 0ull;
        if (tid == 0 && d_src > 0) x = ((unsigned long long)d_src << a.S) | 1ull;          // slot 0 qpack
        if (tid == (int64_t)(offsetof(Slot, dmax) / 8) && d_src > 0) x = (unsigned long long)d_src;
        ((unsigned long long *)a.ctl->slot)[tid] = x;
    }
    if (tid == 0) {
        a.ctl->overflow = 0ull;
        a.ctl->far_count[0] = 0ull;
        a.ctl->far_count[1] = 0ull;
        if (d_src > 0) {
            a.qv[0][0] = a.src;
            a.qo[0][0] = 0;
            a.qr[0][0] = a.R[a.src];
        }
    }
    grid.sync();
    if (tid == 0) t_prev = sssp_gtimer();
    }
    const int k0 = k;                // records below k0 were closed by the cluster kernel

    SsspAppender nearq, farq;
    nearq.sv = s->sv[wib]; nearq.sd = s->sd[wib]; nearq.sr = s->sr[wib]; nearq.cnt = 0; nearq.S = a.S;
    nearq.cap = a.n;
    nearq.overflow = &a.ctl->overflow;
    farq.sv = s->fv[wib]; farq.sd = nullptr; farq.cnt = 0; farq.qo = nullptr; farq.S = 0;
    nearq.stream = farq.stream = env_stream;
    nearq.Rl = (a.lazy_r && !a.ellw) ? a.R : nullptr;
    farq.cap = a.far_cap; farq.overflow = &a.ctl->overflow;
    farq.tag = 2;
    const unsigned long long pol_keep = policy_evict_last();

    for (;; ++k) {
        Slot &cur = a.ctl->slot[k & 3];
        Slot &nxt = a.ctl->slot[(k + 1) & 3];
        // ---- control words: one thread reads, the CTA shares ----------------
        if (threadIdx.x == 0) {
            s->ctl[0] = ld_relaxed(&cur.qpack);
            s->ctl[1] = ld_relaxed(&a.ctl->far_count[fp]);
            s->ctl[2] = ld_relaxed(&cur.ndisc);
            s->ctl[3] = ld_relaxed(&a.ctl->overflow);
            s->ctl[5] = ld_relaxed(&cur.dmax);
            s->bsum[0] = 0;
        }
        __syncthreads();
        const unsigned long long qp = s->ctl[0];
        const int64_t f = (int64_t)(qp & cmask);
        const int64_t mf = (int64_t)(qp >> a.S);
        const int64_t fc = (int64_t)s->ctl[1];
        if (k > k0 && tid == 0 && k - 1 < kMaxStatRecords) {
            a.stats[k - 1].discovered = (int64_t)s->ctl[2];
            const long long t = sssp_gtimer();
            a.stats[k - 1].ns = t - t_prev;
            t_prev = t;
        }
        if (s->ctl[3]) break;
        if (f == 0 && fc == 0) break;
        if (tid == 0) {
            Slot &rst = a.ctl->slot[(k + 2) & 3];
            rst.qpack = 0; rst.ndisc = 0; rst.fpack = 0; rst.work = 0; rst.minfar = ~0ull;
            rst.insp = 0; rst.dmax = 0;
            if (k < kMaxStatRecords) {
                gr_level_stats &st = a.stats[k];
                st.level = k; st.direction = f > 0 ? 3 : 4; st.frontier = f > 0 ? f : fc;
                st.frontier_edges = mf; st.discovered = 0; st.inspected_edges = mf; st.aux = fc;
                st.ns = 0;
            }
        }
        nearq.qv = a.qv[(k + 1) & 1];
        nearq.qo = a.qo[(k + 1) & 1];
        nearq.qr = a.qr[(k + 1) & 1];
        nearq.counter = &nxt.qpack;
        nearq.dmax = &nxt.dmax;

        if (f > 0) {
            // ---- near iteration: Advance(UpdateLabel, SetPred) + Filter ----
            ++it;
            farq.qv = a.far[fp];
            farq.counter = &a.ctl->far_count[fp];
            RelaxOp op{a.dp, a.stamp, a.W, a.R, thr, 2 * it, &nearq, &farq, 0ull, pol_keep, policy_evict_first(),
                       a.ellw};
            GlobalFrontier fr{a.qv[k & 1], a.qo[k & 1], a.qr[k & 1], f, mf};
            const bool pull = a.CWt && (a.direction == 2 || (a.direction == 0 && (double)mf * a.alpha > (double)a.m));
            if (pull && tid == 0 && k < kMaxStatRecords) a.stats[k].direction = 5;  // pull relax
            if (pull) {
                // frontier queue -> bitmap, then every vertex pulls over its in-edges
                const int64_t nwords = (a.n + 31) / 32;
                for (int64_t w = tid; w < nwords; w += nthreads) a.fb[w] = 0u;
                grid.sync();
                const int32_t *qc = a.qv[k & 1];
                for (int64_t j = tid; j < f; j += nthreads) {
                    const int32_t v = qc[j];
                    atomicOr(a.fb + (v >> 5), 1u << (v & 31));
                }
                grid.sync();
                op.nimp = sssp_pull_step(a, thr, 2 * it, gw, nw, nearq, farq, pol_keep);
            } else if (a.ellw) {
                // bounded-degree graphs: one vertex per lane, warps spread over the SMs
                expand_ellw(a.qv[k & 1], f, a.ellw, (int64_t)wib * gridDim.x + blockIdx.x, nw, op);
            } else
            // same auto rule as BFS (reading A-4): short lists -> thread/warp/CTA
            if (f < a.lb_threshold && mf <= 16 * f && (int64_t)s->ctl[5] <= kTwcMaxDeg)  // no long list (see bfs.cu)
                expand_twc(fr, Cs, op, &s->win);
            else
#if GR_SSSP_PIPE
                expand_pipe<kSsspStages, true>(fr, a.C, a.W, gw, nw, op, &s->pipe[wib]);
#else
                expand_lb(fr, Cs, gw, nw, op, &a.ctl->slot[k & 3].work, 4);
#endif
            if (mf >= 16384) {  // wide step: one queue atomic per CTA (see bfs.cu kCtaFlushEdges)
                nearq.finish_cta(s->wsum);
                farq.finish_cta(s->wsum);
            } else {
                nearq.finish();
                farq.finish();
            }
            const unsigned long long ni = warp_sum<unsigned long long>(op.nimp);
            if (lane_id() == 0 && ni) atomicAdd(&s->bsum[0], ni);
            __syncthreads();
            if (threadIdx.x == 0 && s->bsum[0]) atomicAdd(&nxt.ndisc, s->bsum[0]);
            grid.sync();
        } else {
            // ---- near slice exhausted: "update the priority function and
            // operate on the far slice". Re-split (A-11). --------
            const int32_t *far_c = a.far[fp];
            if (threadIdx.x == 0) s->bsum[1] = ~0ull;
            __syncthreads();
            unsigned long long mymin = ~0ull;
            for (int64_t j = tid; j < fc; j += nthreads) {
                const int32_t v = far_c[j];
                if (v < 0) continue;  // sentinel of the cluster kernel's reserved far slots
                const unsigned long long d = ld_probe(a.dp + v, pol_keep) >> 32;
                if (d >= thr && d < mymin) mymin = d;
            }
            for (int sh = 16; sh > 0; sh >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, mymin, sh);
                mymin = o < mymin ? o : mymin;
            }
            if (lane_id() == 0 && mymin != ~0ull) atomicMin(&s->bsum[1], mymin);
            __syncthreads();
            if (threadIdx.x == 0 && s->bsum[1] != ~0ull) atomicMin(&cur.minfar, s->bsum[1]);
            grid.sync();
            if (threadIdx.x == 0) s->ctl[4] = ld_relaxed(&cur.minfar);
            if (tid == 0) a.ctl->far_count[fp] = 0ull;
            __syncthreads();
            const unsigned long long mn = s->ctl[4];
            if (mn == ~0ull) {  // every far entry was stale: the next step
                grid.sync();        // sees f == 0 and an empty far pile and stops
                fp ^= 1;
                continue;
            }
            const uint64_t thr_old = thr;
            const uint64_t band = (mn / a.delta + 1);
            thr = (band > (0xFFFFFFFFFFFFFFFFull / a.delta)) ? 0xFFFFFFFFFFFFFFFFull : band * a.delta;
            ++it;
            farq.qv = a.far[fp ^ 1];
            farq.counter = &a.ctl->far_count[fp ^ 1];
            for (int64_t base = gw * 32; base < fc; base += nw * 32) {
                const int64_t j = base + lane_id();
                bool to_near = false, to_far = false;
                int32_t v = 0;
                int64_t deg = 0, rs = 0;
                if (j < fc && far_c[j] >= 0) {
                    v = far_c[j];
                    const unsigned long long d = ld_probe(a.dp + v, pol_keep) >> 32;
                    const int64_t r0 = nearq.Rl ? 0 : a.R[v], r1 = nearq.Rl ? 0 : a.R[v + 1];  // with d
                    if (d >= thr_old) {  // else stale: already expanded below thr_old
                        const bool nearb = d < thr;
                        const int32_t key = stamp_key(2 * it, !nearb);
                        if (atomicMax(a.stamp + v, key) < key) {
                            if (nearb) { to_near = true; rs = r0; deg = r1 - r0; }
                            else to_far = true;
                        }
                    }
                }
                nearq.push(to_near && (nearq.Rl || deg > 0), v, deg, rs);
                farq.push(to_far, v, 0);
            }
            if (fc >= 16384) {
                nearq.finish_cta(s->wsum);
                farq.finish_cta(s->wsum);
            } else {
                nearq.finish();
                farq.finish();
            }
            grid.sync();
            fp ^= 1;
        }
    }
    if (tid == 0) {
        a.ctl->levels = (unsigned long long)k;
        if (a.ctl->overflow) a.ctl->sticky = 1ull;
    }
}

__global__ void unpack_kernel(const unsigned long long *dp, int64_t n, uint32_t *dist, int32_t *pred) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) {
        unsigned long long x = dp[v];
        if (dist) dist[v] = (uint32_t)(x >> 32);
        if (pred) pred[v] = (int32_t)(uint32_t)(x & 0xffffffffu);
    }
}


// ---------------------------------------------------------------------------
// Narrow steps of bounded-degree SSSP in ONE thread-block cluster (the SSSP
// counterpart of bfs_ell_cluster_kernel, bfs.cu): the near queue lives in the
// cluster's distributed shared memory, the far piles stay in global memory;
// a near iteration relaxes one frontier vertex per thread (entries
// interleaved over the CTAs), a far re-split (A-11) reduces the minimum live
// far distance over the cluster and splits the pile. The traversal is handed
// to the grid kernel (sssp_kernel, resume) when a near frontier exceeds one
// entry per thread, a far pile could overflow a CTA's queue, or the direction
// rule (A-24) asks for a pull step. Semantics of the grid path: packed
// (dist << 32 | pred) atomicMin (A-9) with strict improvement (RelaxOpT::
// slots), monotone stamp keys (A-7), drop of stale far entries (A-11).
// ---------------------------------------------------------------------------
struct SClSmem {
    int32_t q[2][kClQ];              // near queue appended by this CTA, by step parity
    unsigned long long cnt[3];       // (edges << 32) | count near appends, by step mod 3
    unsigned long long imp[3];       // improvements (stats), by step mod 3
    unsigned long long mn;           // re-split: this CTA's minimum live far distance
    int pfx[kClMax + 1];
    long long tot[4];                // F, MF, improvements of the previous step, far count
};

__global__ void sssp_init_kernel(SsspArgs a) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < a.n; v += nthreads) {
        a.dp[v] = ~0ull;   // dist = UINT32_MAX (inf), pred = -1
        a.stamp[v] = -1;
    }
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (tid == 0) {
        a.ctl->overflow = 0ull;
        a.ctl->far_count[0] = 0ull;
        a.ctl->far_count[1] = 0ull;
        a.ctl->handoff = 0ull;
    }
}

// warp-aggregated append of v into the global far pile fq (count *fc)
__device__ __forceinline__ void cl_far_push(bool has, int32_t v, int32_t *fq, unsigned long long *fc, int64_t cap,
                                            unsigned long long *overflow) {
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (!m) return;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(fc, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (has) {
        const unsigned long long pos = base + __popc(m & lanemask_lt());
        if ((int64_t)pos < cap) fq[pos] = v;
        else atomicExch(overflow, 2ull);
    }
}

__global__ void __launch_bounds__(kClBlock, 1) sssp_ell_cluster_kernel(SsspArgs a) {
    __shared__ SClSmem s;
    const unsigned K = cluster_nctarank();
    const unsigned rank = cluster_ctarank();
    const int t = threadIdx.x;
    const unsigned l = lane_id();
    if (t < 3) { s.cnt[t] = 0ull; s.imp[t] = 0ull; }
    const int64_t deg_src = a.R[a.src + 1] - a.R[a.src];
    __syncthreads();
    if (rank == 0 && t == 0) {
        a.dp[a.src] = (unsigned long long)(unsigned int)a.src;  // dist 0, pred = src (A-1)
        if (deg_src > 0) { s.q[0][0] = a.src; s.cnt[0] = ((unsigned long long)deg_src << 32) | 1ull; }
    }
    cluster_barrier();
    uint64_t thr = a.delta;
    int32_t it = 0;
    int fp = 0;
    long long tp = 0;
    if (rank == 0 && t == 0) tp = sssp_gtimer();
    const unsigned long long pol = policy_evict_last();
    int k = 0;
    for (;; ++k) {
        const int c0 = k % 3, c1 = (k + 1) % 3, c2 = (k + 2) % 3, p = k & 1;
        if (t < 32) {
            unsigned long long x = 0, y = 0;
            // the far count's global load issued first, in flight with the DSMEM loads
            const unsigned long long fcv = (l == 0) ? __ldcg(&a.ctl->far_count[fp]) : 0ull;
            if (l < K) { x = ld_dsmem_u64(&s.cnt[c0], l); y = ld_dsmem_u64(&s.imp[c0], l); }
            const int cn = (int)(x & 0xffffffffu);
            const int incl = warp_incl_scan<int>(cn);
            const long long e = warp_sum<long long>((long long)(x >> 32));
            const long long d = warp_sum<long long>((long long)y);
            if (l < K) s.pfx[l + 1] = incl;
            if (l == 0) { s.pfx[0] = 0; s.tot[1] = e; s.tot[2] = d; s.tot[3] = (long long)fcv; }
            if (l == 31) s.tot[0] = incl;
        }
        __syncthreads();
        const int64_t F = s.tot[0], MF = s.tot[1], NI = s.tot[2], fc = s.tot[3];
        if (rank == 0 && t == 0 && k > 0 && k - 1 < kMaxStatRecords) {
            const long long tn = sssp_gtimer();
            a.stats[k - 1].discovered = NI;
            a.stats[k - 1].ns = tn - tp;
            tp = tn;
        }
        if (F == 0 && fc == 0) {
            if (rank == 0 && t == 0) { a.ctl->levels = (unsigned long long)k; a.ctl->handoff = 2ull; }
            break;
        }
        const bool pull = F > 0 && a.CWt && (a.direction == 2 || (a.direction == 0 && (double)MF * a.alpha > (double)a.m));
        if ((F > 0 && (F > (int64_t)K * kClBlock || pull)) || (F == 0 && fc > (int64_t)K * kClQ)) {
            // ---- hand the step to the grid kernel -------------------------
            for (int64_t j = (int64_t)t * K + rank; j < F; j += (int64_t)K * kClBlock) {
                int o = 0;
                while (o + 1 < (int)K && s.pfx[o + 1] <= j) ++o;
                a.qv[k & 1][j] = ld_dsmem_s32(&s.q[p][j - s.pfx[o]], o);
            }
            if (rank == 0 && t == 0) {
                for (int q = 0; q < kSlots; ++q) {
                    Slot &r = a.ctl->slot[q];
                    r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull; r.dmax = 0;
                }
                a.ctl->slot[k & 3].qpack = ((unsigned long long)MF << a.S) | (unsigned long long)F;
                a.ctl->slot[k & 3].dmax = 4ull;
                long long *bs = a.ctl->bstate;
                bs[0] = k; bs[1] = it; bs[2] = (long long)thr; bs[3] = fp; bs[4] = tp;
                a.ctl->handoff = 1ull;
            }
            break;
        }
        if (rank == 0 && t == 0 && k < kMaxStatRecords) {
            gr_level_stats &st = a.stats[k];
            st.level = k; st.direction = F > 0 ? 3 : 4; st.frontier = F > 0 ? F : fc;
            st.frontier_edges = MF; st.discovered = 0; st.inspected_edges = MF; st.aux = fc; st.ns = 0;
        }
        if (t == 0) { s.cnt[c2] = 0ull; s.imp[c2] = 0ull; }
        int na = 0;
        long long ea = 0;
        int32_t nv[4];
        unsigned long long nimp = 0;
        if (F > 0) {
            // ---- near iteration: UpdateLabel + SetPred + RemoveRedundant ----
            ++it;
            const int64_t j = (int64_t)t * K + rank;
            int32_t u = 0;
            unsigned long long du = 0;
            int4 id4 = make_int4(-1, -1, -1, -1), wt4 = make_int4(0, 0, 0, 0);
            if (j < F) {
                int o = 0;
#pragma unroll 1
                while (o + 1 < (int)K && s.pfx[o + 1] <= j) ++o;
                u = ld_dsmem_s32(&s.q[p][j - s.pfx[o]], o);
                du = ld_probe(a.dp + u, pol) >> 32;
                id4 = ld_ell(a.ellw + 2 * (int64_t)u);
                wt4 = ld_ell(a.ellw + 2 * (int64_t)u + 1);
            }
            const int32_t id[4] = {id4.x, id4.y, id4.z, id4.w};
            const int32_t wt[4] = {wt4.x, wt4.y, wt4.z, wt4.w};
            unsigned long long nd[4], old[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) nd[q] = du + (unsigned long long)((uint32_t)wt[q] >> 3);
            // far-pile slots for every relaxation that WOULD go far, reserved now
            // (one atomic per warp, in flight with the atomicMins below); slots of
            // relaxations that do not improve get the sentinel -1, which the
            // re-splits skip -- the far append costs no round trip of its own
            int npf = 0;
            if (a.cl_farres) {
#pragma unroll
                for (int q = 0; q < 4; ++q) npf += (id[q] >= 0 && nd[q] >= thr);
            }
            const int pfi = warp_incl_scan<int>(npf);
            unsigned long long fbase = 0;
            if (l == 31 && pfi > 0) fbase = atomicAdd(&a.ctl->far_count[fp], (unsigned long long)pfi);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                old[q] = id[q] >= 0 ? atomicMin(a.dp + id[q], (nd[q] << 32) | 0xffffffffull) : 0ull;
            bool imp[4], far[4];
            int32_t ex[4];
            const int32_t key_base = 2 * it;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                imp[q] = id[q] >= 0 && nd[q] < (old[q] >> 32);
                if (imp[q]) atomicMin(a.dp + id[q], (nd[q] << 32) | (unsigned int)u);  // RED.MIN: the pred
                far[q] = nd[q] >= thr;
                const int32_t key = stamp_key(key_base, far[q]);
                // RemoveRedundant by stamp (A-7), or (cl_stamp = 0) every strict
                // improvement appends: a duplicate re-relaxes with the same
                // distance and appends nothing, one dependent atomic less
                ex[q] = (imp[q] && a.cl_stamp) ? atomicMax(a.stamp + id[q], key) : (imp[q] ? key - 1 : key);
                nimp += imp[q];
            }
            bool tofar[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool first = imp[q] && ex[q] < stamp_key(key_base, far[q]);
                const int32_t deg = wt[q] & 7;
                const bool tonear = first && !far[q] && deg > 0;
                tofar[q] = first && far[q];
                nv[q] = tonear ? id[q] : -1;
                na += tonear;
                ea += tonear ? deg : 0;
                if (tonear) {  // the next iteration reads its record and its distance
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.ellw + 2 * (int64_t)id[q]));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.dp + id[q]));
                }
            }
            if (a.cl_farres) {
                fbase = __shfl_sync(0xffffffffu, fbase, 31);
                int64_t pos = (int64_t)fbase + pfi - npf;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (id[q] >= 0 && nd[q] >= thr) {
                        if (pos < a.far_cap) a.far[fp][pos] = tofar[q] ? id[q] : -1;
                        else atomicExch(&a.ctl->overflow, 2ull);
                        ++pos;
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    cl_far_push(tofar[q], id[q], a.far[fp], &a.ctl->far_count[fp], a.far_cap, &a.ctl->overflow);
            }
        } else {
            // ---- far re-split (A-11): minimum live far distance, then split --
            const int32_t *far_c = a.far[fp];
            unsigned long long mymin = ~0ull;
            for (int64_t j = (int64_t)t * K + rank; j < fc; j += (int64_t)K * kClBlock) {
                const int32_t v = far_c[j];
                if (v < 0) continue;  // reserved slot of a relaxation that did not improve
                const unsigned long long d = ld_probe(a.dp + v, pol) >> 32;
                if (d >= thr && d < mymin) mymin = d;
            }
#pragma unroll
            for (int sh = 16; sh > 0; sh >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, mymin, sh);
                mymin = o < mymin ? o : mymin;
            }
            if (t == 0) s.mn = ~0ull;
            __syncthreads();
            if (l == 0 && mymin != ~0ull) atomicMin(&s.mn, mymin);
            cluster_barrier();
            if (t < 32) {
                unsigned long long x = (l < K) ? ld_dsmem_u64(&s.mn, l) : ~0ull;
#pragma unroll
                for (int sh = 16; sh > 0; sh >>= 1) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, x, sh);
                    x = o < x ? o : x;
                }
                if (l == 0) s.tot[0] = (long long)x;
            }
            __syncthreads();
            const unsigned long long mn = (unsigned long long)s.tot[0];
            cluster_barrier();  // every CTA read every s.mn before it is reused
            if (rank == 0 && t == 0) a.ctl->far_count[fp] = 0ull;  // consumed below (all read fc)
            if (mn != ~0ull) {
                const uint64_t thr_old = thr;
                const uint64_t band = mn / a.delta + 1;
                thr = (band > (0xFFFFFFFFFFFFFFFFull / a.delta)) ? 0xFFFFFFFFFFFFFFFFull : band * a.delta;
                ++it;
                const int32_t key_base = 2 * it;
                for (int64_t j0 = 0; j0 < fc; j0 += (int64_t)K * kClBlock) {  // warp-uniform trip count
                    const int64_t j = j0 + (int64_t)t * K + rank;
                    bool tonear = false, tofar = false;
                    int32_t v = 0;
                    int64_t deg = 0;
                    if (j < fc && far_c[j] >= 0) {
                        v = far_c[j];
                        const unsigned long long d = ld_probe(a.dp + v, pol) >> 32;
                        const int64_t r0 = a.R[v], r1 = a.R[v + 1];
                        if (d >= thr_old) {  // else stale: already expanded below thr_old
                            const bool nearb = d < thr;
                            const int32_t key = stamp_key(key_base, !nearb);
                            if (atomicMax(a.stamp + v, key) < key) {
                                deg = r1 - r0;
                                tonear = nearb && deg > 0;
                                tofar = !nearb;
                            }
                        }
                    }
                    // near entries of a re-split: appended right here (<= 4 per thread: fc <= 4 x threads)
                    const int incl = warp_incl_scan<int>(tonear ? 1 : 0);
                    const long long et = warp_sum<long long>(tonear ? deg : 0);
                    unsigned long long base = 0;
                    if (l == 31 && incl > 0) base = atomicAdd(&s.cnt[c1], ((unsigned long long)et << 32) | (unsigned)incl);
                    base = __shfl_sync(0xffffffffu, base, 31);
                    if (tonear) s.q[p ^ 1][(int)(base & 0xffffffffu) + incl - 1] = v;
                    cl_far_push(tofar, v, a.far[fp ^ 1], &a.ctl->far_count[fp ^ 1], a.far_cap, &a.ctl->overflow);
                }
            }
            fp ^= 1;
        }
        // near appends of the iteration: one packed shared-memory atomic per warp
        if (F > 0) {
            const int incl = warp_incl_scan<int>(na);
            const long long etot = warp_sum<long long>(ea);
            unsigned long long base = 0;
            if (l == 31 && incl > 0) base = atomicAdd(&s.cnt[c1], ((unsigned long long)etot << 32) | (unsigned)incl);
            base = __shfl_sync(0xffffffffu, base, 31);
            int pos = (int)(base & 0xffffffffu) + incl - na;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (nv[q] >= 0) s.q[p ^ 1][pos++] = nv[q];
        }
        const unsigned long long nw = warp_sum<unsigned long long>(nimp);
        if (l == 0 && nw) atomicAdd(&s.imp[c1], nw);
        cluster_barrier();
    }
    cluster_barrier();  // no CTA exits while another reads its shared memory
}

// Largest cluster (16, else 8) of sssp_ell_cluster_kernel CTAs the device
// can run (0: none; GR_ELL_CLUSTER_SIZE forces one).
static int sssp_cluster_size() {
    static int k = -1;
    if (k >= 0) return k;
    k = 0;
    const int want = (int)env_int("GR_ELL_CLUSTER_SIZE", 0);
    cudaFuncSetAttribute(sssp_ell_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8}) {
        if (want > 0 && c != want) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)c);
        cfg.blockDim = dim3(kClBlock);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, sssp_ell_cluster_kernel, &cfg) == cudaSuccess && ncl >= 1) {
            k = c;
            break;
        }
    }
    cudaGetLastError();
    return k;
}

gr_status run_sssp(Graph *g, int32_t src, uint32_t *dist, int32_t *pred, uint64_t delta, int32_t direction,
                   double alpha, int *launches) {
    if (direction != 1 && !g->CWt) {  // weighted in-lists for pull steps, built on first use
        gr_status st = build_pull_weights(g);
        if (st != GR_OK) return st;
    }
    SsspArgs a;
    a.n = g->n; a.m = g->m;
    a.R = g->R; a.C = g->C; a.W = g->W; a.CW = g->CW;
    a.Rt = g->Rt; a.CWt = g->CWt; a.fb = g->fbuf[0];
    a.ellw = g->ellw;
    a.lazy_r = (int32_t)env_int("GR_LAZY_R", 1);
    a.bar_ns = (int32_t)env_int("GR_BAR_NS", 128);
    a.cl_stamp = (int32_t)env_int("GR_CL_STAMP", 0);  // measured: C4 SSSP 104 -> 94 ms without
    a.cl_farres = (int32_t)env_int("GR_CL_FARRES", 1);
    a.direction = direction;
    a.alpha = alpha > 0 ? alpha : 2.0;  // measured on C3: pull pays only when m_f > m / 2
    a.dp = g->dp; a.stamp = g->stamp;
    for (int i = 0; i < 2; ++i) {
        a.qv[i] = g->qv[i]; a.qo[i] = g->qo[i]; a.qr[i] = g->qr[i]; a.far[i] = g->farq[i];
    }
    a.far_cap = g->far_cap;
    a.ctl = g->ctl; a.stats = g->stats_dev;
    a.src = src;
    a.delta = delta;
    a.lb_threshold = env_int("GR_SSSP_LB_THRESHOLD", 65536);
    a.stream_queues = (int)env_int("GR_SSSP_STREAMQ", 0);
    a.S = g->pack_shift;
    const bool packed = g->CW != nullptr;
    const void *fn = packed ? (const void *)sssp_kernel<true> : (const void *)sssp_kernel<false>;
    static int per_sm_v[2] = {0, 0};
    int &per_sm = per_sm_v[packed ? 1 : 0];
    const size_t smem = sizeof(SsspSmem);
    if (per_sm == 0) {
        GR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, smem));
    }
    if (per_sm < 1) { set_error("sssp_kernel cannot be resident"); return GR_ERR_CUDA; }
    int64_t ctas = (int64_t)g->num_sms * per_sm;
    const int64_t cap_ctas = env_int("GR_SSSP_CTAS", 0);  // experiment: fewer persistent CTAs
    if (cap_ctas > 0 && cap_ctas < ctas) ctas = cap_ctas;
    // bounded-degree graphs: the narrow steps run in one thread-block cluster
    // (sssp_ell_cluster_kernel); the grid kernel resumes only if they outgrow it
    int nl = 0;
    a.resume = 0;
    const int kcl = (g->ellw && direction != 2 && env_int("GR_ELL_CLUSTER", 1)) ? sssp_cluster_size() : 0;
    if (kcl > 0) {
        sssp_init_kernel<<<g->num_sms * 4, 512, 0, g->stream>>>(a);
        GR_CUDA(cudaGetLastError());
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)kcl);
        cfg.blockDim = dim3(kClBlock);
        cfg.stream = g->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)kcl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        GR_CUDA(cudaLaunchKernelEx(&cfg, sssp_ell_cluster_kernel, a));
        count_launch(2);
        nl += 2;
        a.resume = 1;
    }
    dim3 grid((unsigned)ctas), block(kBlock);
    void *args[] = {&a};
    GR_CUDA(cudaLaunchCooperativeKernel(fn, grid, block, args, smem, g->stream));
    unpack_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(g->dp, g->n, dist, pred);
    GR_CUDA(cudaGetLastError());
    count_launch(2);
    *launches = nl + 2;
    return GR_OK;
}

}  // namespace gr
