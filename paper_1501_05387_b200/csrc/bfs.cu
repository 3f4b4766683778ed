// bfs.cu -- breadth-first search, push and direction-optimizing push-pull,
// as ONE persistent cooperative kernel per traversal (device-side iteration
// control: no host round trip per level).
//
// Paper: BFS §5.1; advance/filter; fusion;
// load balancing; idempotent vs atomic discovery (P:793-802,
// P:916-921); push vs pull. Readings A-1..A-6 in DESIGN.md.
//
// Level modes:
//  * grid push  -- merge-path advance over the global queue, every warp of the
//                  grid (expand_lb + BfsPushOp); also sets the next frontier's
//                  bits in a rotating frontier bitmap so a following pull
//                  level needs no conversion;
//  * grid pull  -- bottom-up sweep over the frontier bitmap (pull_level);
//  * small push -- frontier <= kSmallF vertices and <= kSmallE edges: CTA 0
//                  alone runs consecutive levels with the frontier queue in
//                  SHARED memory and CTA barriers (tiny levels are pure
//                  latency: a grid barrier and L2 round trips per control
//                  word would dominate).
// Control words every block needs (frontier size, counters) are read by one
// thread per CTA and broadcast through shared memory: thousands of warps
// reading one L2 address serialise on its slice.
#include "frontier.cuh"

namespace gr {

#ifndef GR_SMALL_CAP
#define GR_SMALL_CAP 512  // measured: smaller shared memory leaves more L1 for probes/spills
#endif
constexpr int64_t kSmallF = GR_SMALL_CAP;  // small mode: queue capacity (shared memory)
constexpr int64_t kSmallFDefault = 512;   // small mode: default max frontier (swept on C4)
constexpr int64_t kSmallE = 16384;  // small mode: max frontier edges
#ifndef GR_BFS_STAGES
#define GR_BFS_STAGES 0  // measured on C2 push: 2 and 4 stages are slower (smem displaces L1)
#endif
constexpr int kBfsStages = GR_BFS_STAGES;  // cp.async pipeline depth of the grid push advance (0: off)
constexpr int kSmallCntBits = 24;   // count field of the small-mode packed counter
constexpr unsigned long long kSmallCntMask = (1ull << kSmallCntBits) - 1;

struct BfsArgs {
    int64_t n, m;
    const int64_t *R;
    const int32_t *C;
    const int64_t *Rt;   // in-edges for pull (== R when symmetric)
    const int32_t *Ct;
    uint32_t *visited;
    const uint32_t *noin;  // vertices with in-degree 0
    uint32_t *fbuf[3];     // rotating frontier bitmaps
    int32_t *qv[2];
    int64_t *qo[2];
    int64_t *qr[2];
    int32_t *depth;
    int32_t *pred;       // may be null
    Ctl *ctl;
    gr_level_stats *stats;
    int32_t src;
    int32_t direction;   // 0 auto, 1 push, 2 pull
    int32_t switch_rule; // 0 Beamer, 1 paper-literal
    int32_t idempotent;
    double alpha, beta;
    int64_t nonisolated;
    int S;
    int64_t small_f, small_e;  // small-mode thresholds (<= kSmallF, tuning knobs)
    int32_t strategy;          // 0 auto, 1 thread/warp/CTA, 2 merge-path (gr_bfs_opts)
    int64_t lb_threshold;      // auto: frontiers below it use thread/warp/CTA
};

struct BfsSmem {
    union {
        struct {  // grid levels: per-warp append staging + cp.async pipeline
            PipeWarpSmem<(kBfsStages > 0 ? kBfsStages : 1), false> pipe[kBfsStages > 0 ? kWarpsPerBlock : 1];
            int32_t sv[kWarpsPerBlock][kStageCap];
            int32_t sd[kWarpsPerBlock][kStageCap];
            int64_t sr[kWarpsPerBlock][kStageCap];
        } stage;
        struct {  // small mode: the frontier lives here (double-buffered)
            int64_t rs[2][kSmallF];   // row start of each entry
            int64_t off[2][kSmallF];  // exclusive degree prefix (reserved at append time)
            int32_t q[2][kSmallF];    // vertex ids
        } small;
    } u;
    unsigned long long ctl[8];
    long long scan[kWarpsPerBlock];
    unsigned long long bsum[4];
    unsigned long long pk[3];   // small mode: packed (edges << kSmallCntBits) | count, per level mod 3
    unsigned long long nd[3];   // small mode: discovered per level mod 3
    int work;
    int win;     // expand_twc: CTA arbitration
};

// ---------------------------------------------------------------------------
// Per-edge op of the grid push advance: the fused cond/apply + filter of BFS.
// cond: "is d unvisited" (bitmap probe, culling heuristic P:797-799);
// claim: atomicOr on the visited word returns the old bit, so each vertex is
// discovered exactly once ("non-idempotent advance ... uses atomic
// operations to guarantee each element appears only once"); apply: depth and
// pred; filter: warp-staged append into the next queue.
// With idempotent=1 the claim is atomic-free: depth[] (not the bitmap) is the
// authoritative visited test, plain stores write it, the bitmap is updated
// with a fire-and-forget red.or and only filters (reading A-6); duplicates may
// enter the queue and are harmless (same depth).
// ---------------------------------------------------------------------------
struct BfsPushOp {
    uint32_t *visited;
    uint32_t *fbn;       // next frontier bitmap (null: not maintained this level)
    int32_t *depth;
    int32_t *pred;
    const int64_t *R;
    int32_t next_depth;
    int32_t idempotent;
    Appender *app;
    unsigned long long ndisc;
    unsigned long long pol_keep;   // evict_last policy for the visited bitmap
    int probe;           // culling probe before the claim: 0 none (small levels claim
                         // directly: one L2 round trip less on the critical path),
                         // 1 L2-coherent, 2 through L1 (most targets already visited
                         // before the level: L1 hits, stale words only cost an atomic)

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const T5 *) {
        uint32_t word[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            word[u] = !ok[u] ? 0xffffffffu
                    : probe == 1 ? ld_probe(visited + (dst[u] >> 5), pol_keep)
                    : probe == 2 ? ld_l1(visited + (dst[u] >> 5)) : 0u;
        bool disc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t w = dst[u];
            const uint32_t bit = 1u << (w & 31);
            disc[u] = false;
            bool cand = ok[u] && !(word[u] & bit);
            if (idempotent) {
                // warp-level culling heuristic (A-5 i): lanes of one warp that
                // target the same vertex keep only the lowest lane
                const unsigned peers = __match_any_sync(0xffffffffu, cand ? w : -1 - (int)lane_id());
                cand = cand && (__ffs(peers) - 1 == (int)lane_id());
            }
            if (cand) {
                if (idempotent) {
                    if (*(volatile int32_t *)(depth + w) < 0) {
                        disc[u] = true;
                        atomicOr(visited + (w >> 5), bit);  // result unused -> RED.OR
                    }
                } else {
                    const uint32_t old = atomicOr(visited + (w >> 5), bit);
                    disc[u] = !(old & bit);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!__any_sync(0xffffffffu, disc[u])) continue;
            const int32_t w = dst[u];
            int64_t deg = 0, rs = 0;
            if (disc[u]) {
                depth[w] = next_depth;
                if (pred) pred[w] = src[u];
                if (fbn) atomicOr(fbn + (w >> 5), 1u << (w & 31));  // RED.OR
                rs = R[w];
                deg = R[w + 1] - rs;
                ++ndisc;
            }
            app->push(disc[u] && deg > 0, w, deg, rs);
        }
    }
};

// Small-mode op: claim directly with atomicOr (one L2 round trip instead of
// probe + claim) while the target's row offsets are loaded speculatively in
// parallel, then append (vertex, row start, degree) into the shared-memory
// queue of the next level and prefetch the head of its neighbour list into L2
// (the next level reads it a few microseconds later). Entries beyond kSmallF
// spill to the global queue, which then ends small mode.
struct SmallPushOp {
    uint32_t *visited;
    int32_t *depth;
    int32_t *pred;
    const int64_t *R;
    const int32_t *C;
    int32_t next_depth;
    int32_t *sq_next;            // smem vertex ids
    int64_t *srs_next;           // smem row starts
    int64_t *soff_next;          // smem degree prefix
    unsigned long long *spk;     // smem packed counter (edges << kSmallCntBits) | count
    int32_t *gq_next;            // global spill queue (entries >= kSmallF)
    int64_t *go_next;
    int64_t *gr_next;
    unsigned long long ndisc;

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const int64_t *) {
        uint32_t old[U];
        int64_t rs[U], re[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            old[u] = ok[u] ? atomicOr(visited + (dst[u] >> 5), 1u << (dst[u] & 31)) : 0xffffffffu;
            rs[u] = ok[u] ? R[dst[u]] : 0;
            re[u] = ok[u] ? R[dst[u] + 1] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t w = dst[u];
            const bool disc = !((old[u] >> (w & 31)) & 1u);
            const unsigned mask = __ballot_sync(0xffffffffu, disc);
            if (!mask) continue;
            // one packed shared-memory atomic reserves the queue slots AND the
            // edge range: the next level's degree prefix comes out of the append
            const int64_t deg = disc ? re[u] - rs[u] : 0;
            const int64_t incl = warp_incl_scan<int64_t>(deg);
            const int64_t tot = __shfl_sync(0xffffffffu, incl, 31);
            unsigned long long base = 0;
            if (lane_id() == 0)
                base = atomicAdd(spk, ((unsigned long long)tot << kSmallCntBits) | (unsigned long long)__popc(mask));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (disc) {
                depth[w] = next_depth;
                if (pred) pred[w] = src[u];
                const int64_t pos = (int64_t)(base & kSmallCntMask) + __popc(mask & lanemask_lt());
                const int64_t off = (int64_t)(base >> kSmallCntBits) + incl - deg;
                if (pos < kSmallF) {
                    sq_next[pos] = w;
                    srs_next[pos] = rs[u];
                    soff_next[pos] = off;
                } else {
                    gq_next[pos] = w;
                    go_next[pos] = off;
                    gr_next[pos] = rs[u];
                }
                if (deg > 0) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(C + rs[u]));
                    if (deg > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + rs[u] + 32));
                }
                ++ndisc;
            }
        }
    }
};

// ---------------------------------------------------------------------------
// Pull (bottom-up) step over in-edges: "pull starts with a
// frontier of unvisited vertices, generating the new frontier by filtering
// the unvisited frontier for vertices that have neighbors in the current
// frontier"; the current frontier is held as a bitmap. A warp
// owns 32 consecutive vertices = one bitmap word, so the next-frontier word
// and the visited word are written with one plain store from a ballot: no
// atomics. Each lane stops at its first in-neighbour in the frontier (early
// exit). Each CTA owns a contiguous range of words; its warps take words from
// a shared-memory counter (per-vertex scan lengths vary widely).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pull_level(const BfsArgs &a, const uint32_t *__restrict__ fcur,
                                           uint32_t *__restrict__ fnext, int32_t next_depth,
                                           int *swork, Appender &app, unsigned long long &ndisc,
                                           unsigned long long &insp) {
    const int64_t nwords = (a.n + 31) / 32;
    const int64_t wb0 = nwords * blockIdx.x / gridDim.x;
    const int64_t wb1 = nwords * (blockIdx.x + 1) / gridDim.x;
    const unsigned l = lane_id();
    const unsigned long long pol = policy_evict_first();
    const bool sym = a.Rt == a.R;
    // kPW words per grab, processed in phases so their loads overlap: row
    // offsets of all kPW vertices, then their FIRST in-neighbour and its
    // frontier bit (most candidates resolve there: C2 averages 1.8 inspected
    // edges per candidate), then the remaining lists of the unresolved ones.
#ifndef GR_PULL_WORDS
#define GR_PULL_WORDS 2
#endif
    constexpr int kPW = GR_PULL_WORDS;
    for (;;) {
        int c = 0;
        if (l == 0) c = atomicAdd(swork, kPW);
        c = __shfl_sync(0xffffffffu, c, 0);
        const int64_t w0 = wb0 + c;
        if (w0 >= wb1) break;
        uint32_t visw[kPW];
        int64_t beg[kPW], end[kPW];
        int32_t parent[kPW];
        bool found[kPW];
#pragma unroll
        for (int k = 0; k < kPW; ++k) visw[k] = (w0 + k < wb1) ? a.visited[w0 + k] : 0xffffffffu;
#pragma unroll
        for (int k = 0; k < kPW; ++k) {
            const int64_t v = (w0 + k) * 32 + l;
            const bool cand = v < a.n && !((visw[k] >> l) & 1u);
            beg[k] = cand ? a.Rt[v] : 0;
            end[k] = cand ? a.Rt[v + 1] : 0;
        }
        int32_t u0[kPW];
#pragma unroll
        for (int k = 0; k < kPW; ++k) u0[k] = beg[k] < end[k] ? ld_stream(a.Ct + beg[k], pol) : -1;
#pragma unroll
        for (int k = 0; k < kPW; ++k) {
            const uint32_t fw = u0[k] >= 0 ? __ldg(fcur + (u0[k] >> 5)) : 0u;
            found[k] = u0[k] >= 0 && ((fw >> (u0[k] & 31)) & 1u);
            parent[k] = u0[k];
            insp += (u0[k] >= 0);
        }
#pragma unroll
        for (int k = 0; k < kPW; ++k) {
            if (found[k]) continue;
            for (int64_t e = beg[k] + 1; e < end[k] && !found[k]; e += 4) {
                int32_t u[4];
                uint32_t fw[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) u[q] = (e + q < end[k]) ? ld_stream(a.Ct + e + q, pol) : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q) fw[q] = (u[q] >= 0) ? __ldg(fcur + (u[q] >> 5)) : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!found[k] && u[q] >= 0) {
                        ++insp;
                        if ((fw[q] >> (u[q] & 31)) & 1u) {
                            found[k] = true;
                            parent[k] = u[q];
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kPW; ++k) {
            const int64_t wi = w0 + k;
            if (wi >= wb1) break;
            const int64_t v = wi * 32 + l;
            const unsigned nb = __ballot_sync(0xffffffffu, found[k]);
            if (l == 0) {
                fnext[wi] = nb;
                if (nb) a.visited[wi] = visw[k] | nb;
            }
            if (nb == 0) continue;
            int64_t deg = 0, rs = 0;
            if (found[k]) {
                a.depth[v] = next_depth;
                if (a.pred) a.pred[v] = parent[k];
                rs = sym ? beg[k] : a.R[v];
                deg = sym ? end[k] - beg[k] : a.R[v + 1] - rs;
            }
            ndisc += found[k];
            app.push(found[k] && deg > 0, (int32_t)v, deg, rs);
        }
    }
}

// Direction decision (reading A-3). Pure function of counters
// every block reads after the same barrier, so all blocks agree.
__device__ __forceinline__ int decide_direction(const BfsArgs &a, int dir, int64_t f, int64_t mf,
                                                int64_t u_cnt, int64_t m_u, int64_t prev_f,
                                                int64_t nwords) {
    if (a.direction != 0) return a.direction;
    if (a.switch_rule == 1) return (u_cnt < f) ? 2 : 1;  // paper-literal: unvisited < frontier
    if (dir == 1) {
        // Beamer: pull when the frontier's edges exceed the unvisited edges / alpha;
        // plus: a pull step sweeps every bitmap word, so require m_f >= n/32.
        if ((double)mf > (double)m_u / a.alpha && mf >= nwords) return 2;
        return 1;
    }
    if ((double)f < (double)a.nonisolated / a.beta && f < prev_f) return 1;
    return 2;
}

struct BfsState {  // per-traversal heuristic state, identical in every CTA
    int L;
    int dir, prev_dir;
    int64_t u_cnt, m_u, prev_f;
    int fb_valid;       // fbuf[L%3] holds the frontier of level L
    int fbn_clean;      // fbuf[(L+1)%3] is all zero
    int closed;         // stats records below this level are closed
};

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Block-wide exclusive scan of one int64 per thread; returns the exclusive
// prefix, total in *total. Uses s->scan; contains two __syncthreads.
__device__ __forceinline__ int64_t block_excl_scan(int64_t x, int64_t *total, BfsSmem *s) {
    const int wib = threadIdx.x >> 5;
    const int64_t incl = warp_incl_scan<int64_t>(x);
    __syncthreads();  // s->scan / s->bsum[3] may still be read by a previous scan
    if (lane_id() == 31) s->scan[wib] = incl;
    __syncthreads();
    if (wib == 0) {
        const int64_t y = (lane_id() < kWarpsPerBlock) ? s->scan[lane_id()] : 0;
        const int64_t yi = warp_incl_scan<int64_t>(y);
        if (lane_id() < kWarpsPerBlock) s->scan[lane_id()] = yi - y;
        if (lane_id() == 31) s->bsum[3] = (unsigned long long)yi;
    }
    __syncthreads();
    *total = (int64_t)s->bsum[3];
    return s->scan[wib] + incl - x;
}

__global__ void __launch_bounds__(kBlock, kMinBlocks) bfs_kernel(BfsArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BfsSmem *s = reinterpret_cast<BfsSmem *>(smem_raw);

    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gw = tid >> 5;
    const int64_t nw = nthreads >> 5;
    const int wib = threadIdx.x >> 5;
    const int64_t nwords = (a.n + 31) / 32;
    const unsigned long long cmask = (1ull << a.S) - 1;

    // ---- Set_Problem_Data: depth = -1 (A-2), pred = -1, src -----
    for (int64_t v = tid; v < a.n; v += nthreads) {
        a.depth[v] = -1;
        if (a.pred) a.pred[v] = -1;
    }
    // vertices with no in-edge can never be discovered: pre-mark them visited
    // so pull skips them (they keep depth -1; the bitmap is internal)
    for (int64_t w = tid; w < nwords; w += nthreads) a.visited[w] = a.noin[w];
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (tid == 0) a.ctl->overflow = 0ull;
    grid.sync();
    const int64_t deg_src = a.R[a.src + 1] - a.R[a.src];
    if (tid == 0) {
        a.depth[a.src] = 0;
        if (a.pred) a.pred[a.src] = a.src;  // A-1
        a.visited[a.src >> 5] |= 1u << (a.src & 31);
        a.qv[0][0] = a.src;
        a.qo[0][0] = 0;
        a.qr[0][0] = a.R[a.src];
        a.ctl->slot[0].qpack = (deg_src > 0) ? (((unsigned long long)deg_src << a.S) | 1ull) : 0ull;
    }
    grid.sync();

    // Heuristic state. u = unvisited vertices that have an in-edge, m_u =
    // edges incident to them (reading A-3).
    const bool src_has_in = !((a.noin[a.src >> 5] >> (a.src & 31)) & 1u);
    BfsState st;
    st.L = 0;
    st.dir = (a.direction == 2) ? 2 : 1;
    st.prev_dir = 1;
    st.u_cnt = a.nonisolated - (src_has_in ? 1 : 0);
    st.m_u = a.m - deg_src;
    st.prev_f = 0;
    st.fb_valid = 0;
    st.fbn_clean = 0;
    st.closed = 0;
    const unsigned long long pol_keep = policy_evict_last();
    long long t_prev = 0;
    if (tid == 0) t_prev = gtimer();
    bool pending = false;  // counters of the last grid level not yet applied to u, m_u

    Appender app;
    app.sv = s->u.stage.sv[wib];
    app.sd = s->u.stage.sd[wib];
    app.sr = s->u.stage.sr[wib];
    app.cnt = 0;
    app.S = a.S;
    app.cap = 2 * a.n;  // queues hold 2n entries (idempotent duplicates)
    app.overflow = &a.ctl->overflow;

    for (;;) {
        // ---- control words of level L: one thread reads, the CTA shares ----
        const int L = st.L;
        if (threadIdx.x == 0) {
            const Slot &cur = a.ctl->slot[L & 3];
            // independent relaxed loads: issued back to back, one round trip
            const unsigned long long q0 = ld_relaxed(&cur.qpack), q1 = ld_relaxed(&cur.ndisc),
                                     q2 = ld_relaxed(&cur.insp), q3 = ld_relaxed(&a.ctl->overflow);
            s->ctl[0] = q0; s->ctl[1] = q1; s->ctl[2] = q2; s->ctl[3] = q3;
            // per-level CTA counters, reset before the barrier below (racecheck)
            s->work = 0; s->bsum[0] = 0; s->bsum[1] = 0;
        }
        __syncthreads();
        const unsigned long long qp = s->ctl[0];
        const int64_t f = (int64_t)(qp & cmask);
        const int64_t mf = (int64_t)(qp >> a.S);
        if (pending) {
            st.u_cnt -= (int64_t)s->ctl[1];
            st.m_u -= mf;
            pending = false;
        }
        if (tid == 0 && L > st.closed && L - 1 < kMaxStatRecords) {
            gr_level_stats &sr = a.stats[L - 1];
            sr.discovered = (int64_t)s->ctl[1];
            if (sr.direction == 2) sr.inspected_edges = (int64_t)s->ctl[2];
            const long long t = gtimer();
            sr.ns = t - t_prev;
            t_prev = t;
        }
        const bool stop = (f == 0 || s->ctl[3]);
        __syncthreads();  // s->ctl is rewritten below
        if (stop) break;
        const int dir = decide_direction(a, st.dir, f, mf, st.u_cnt, st.m_u, st.prev_f, nwords);

        if (dir == 1 && f <= a.small_f && mf <= a.small_e) {
            // ================= small mode: CTA 0 alone ===========================
            if (blockIdx.x == 0) {
                int c = 0, r = 0;
                for (int64_t j = threadIdx.x; j < f; j += kBlock) {
                    const int32_t v = a.qv[L & 1][j];
                    s->u.small.q[0][j] = v;
                    s->u.small.off[0][j] = a.qo[L & 1][j];
                    s->u.small.rs[0][j] = a.qr[L & 1][j];
                }
                if (threadIdx.x < 3) { s->pk[threadIdx.x] = 0; s->nd[threadIdx.x] = 0; }
                __syncthreads();
                int64_t cf = f, E = mf;
                bool mu_pending = false;
                bool done = false;
                long long tp = t_prev;
                for (;;) {
                    if (cf > a.small_f) break;  // too large (or spilled to the global queue)
#ifdef GR_TRACE
                    if (threadIdx.x == 0) g_trace_L = st.L;
#endif
                    GR_TSTAMP(0);
                    if (mu_pending) { st.m_u -= E; mu_pending = false; }
                    if (cf == 0) { done = true; break; }
                    const int d = decide_direction(a, st.dir, cf, E, st.u_cnt, st.m_u, st.prev_f, nwords);
                    if (!(d == 1 && E <= a.small_e)) break;
                    st.dir = d;
                    const int Lc = st.L;
                    const int r1 = (r + 1) % 3, r2 = (r + 2) % 3;
                    if (threadIdx.x == 0) {
                        s->pk[r2] = 0;  // counter of level Lc + 2 (last read at level Lc - 1)
                        s->nd[r2] = 0;
                        if (Lc < kMaxStatRecords) {
                            gr_level_stats &sr = a.stats[Lc];
                            sr.level = Lc; sr.direction = 1; sr.frontier = cf; sr.frontier_edges = E;
                            sr.discovered = 0; sr.inspected_edges = E; sr.aux = st.u_cnt; sr.ns = 0;
                        }
                    }
                    SmallPushOp op{a.visited, a.depth, a.pred, a.R, a.C, Lc + 1, s->u.small.q[c ^ 1],
                                   s->u.small.rs[c ^ 1], s->u.small.off[c ^ 1], &s->pk[r1],
                                   a.qv[(Lc + 1) & 1], a.qo[(Lc + 1) & 1], a.qr[(Lc + 1) & 1], 0ull};
                    SmemFrontier fr{s->u.small.q[c], s->u.small.off[c], s->u.small.rs[c], cf, E};
                    GR_TSTAMP(9);
                    expand_lb(fr, a.C, (int64_t)wib, (int64_t)kWarpsPerBlock, op);
                    GR_TSTAMP(5);
                    const unsigned long long ndw = warp_sum<unsigned long long>(op.ndisc);
                    if (lane_id() == 0 && ndw) atomicAdd(&s->nd[r1], ndw);
                    __syncthreads();
                    const unsigned long long pk = s->pk[r1];
                    const unsigned long long ndl = s->nd[r1];
                    GR_TSTAMP(6);
                    if (threadIdx.x == 0 && Lc < kMaxStatRecords) {
                        const long long t = gtimer();
                        a.stats[Lc].discovered = (int64_t)ndl;
                        a.stats[Lc].ns = t - tp;
                        tp = t;
                    }
                    st.u_cnt -= (int64_t)ndl;
                    st.prev_f = cf;
                    st.prev_dir = 1;
                    st.L = Lc + 1;
                    c ^= 1;
                    r = r1;
                    cf = (int64_t)(pk & kSmallCntMask);
                    E = (int64_t)(pk >> kSmallCntBits);
                    mu_pending = true;
                }
                // hand the frontier of level st.L back to the grid
                if (!done) {
                    // the frontier of level st.L: entries below kSmallF are in shared
                    // memory, the rest were spilled (with their offsets) to the global queue
                    for (int64_t j = threadIdx.x; j < cf && j < kSmallF; j += kBlock) {
                        a.qv[st.L & 1][j] = s->u.small.q[c][j];
                        a.qo[st.L & 1][j] = s->u.small.off[c][j];
                        a.qr[st.L & 1][j] = s->u.small.rs[c][j];
                    }
                    if (mu_pending) st.m_u -= E;
                    if (threadIdx.x == 0) {
                        a.ctl->slot[st.L & 3].qpack = ((unsigned long long)E << a.S) | (unsigned long long)cf;
                        a.ctl->slot[st.L & 3].ndisc = 0;
                        a.ctl->slot[st.L & 3].insp = 0;
                    }
                } else if (threadIdx.x == 0) {
                    a.ctl->slot[st.L & 3].qpack = 0;
                }
                if (threadIdx.x == 0) {
                    for (int k = 1; k <= 2; ++k) {
                        Slot &r = a.ctl->slot[(st.L + k) & 3];
                        r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull;
                    }
                    long long *bs = a.ctl->bstate;
                    bs[0] = st.L; bs[1] = st.dir; bs[2] = st.prev_dir; bs[3] = st.u_cnt;
                    bs[4] = st.m_u; bs[5] = st.prev_f; bs[6] = tp;
                }
            }
            grid.sync();
            if (threadIdx.x == 0) {
                const volatile long long *bs = a.ctl->bstate;
                for (int k = 0; k < 7; ++k) s->ctl[k] = (unsigned long long)bs[k];
            }
            __syncthreads();
            st.L = (int)(long long)s->ctl[0];
            st.dir = (int)(long long)s->ctl[1];
            st.prev_dir = (int)(long long)s->ctl[2];
            st.u_cnt = (long long)s->ctl[3];
            st.m_u = (long long)s->ctl[4];
            st.prev_f = (long long)s->ctl[5];
            if (tid == 0) t_prev = (long long)s->ctl[6];
            st.closed = st.L;      // records below st.L are closed
            st.fb_valid = 0;       // small mode keeps no frontier bitmap
            st.fbn_clean = 0;
            pending = false;
            __syncthreads();
            continue;
        }

        // ===================== grid level ======================================
#ifdef GR_TRACE
        if (tid == 0) g_trace_L = L;
#endif
        GR_TSTAMP(0);
        st.dir = dir;
        if (tid == 0) {
            Slot &rst = a.ctl->slot[(L + 2) & 3];
            rst.qpack = 0; rst.ndisc = 0; rst.fpack = 0; rst.work = 0; rst.minfar = ~0ull; rst.insp = 0;
            if (L < kMaxStatRecords) {
                gr_level_stats &sr = a.stats[L];
                sr.level = L; sr.direction = dir; sr.frontier = f; sr.frontier_edges = mf;
                sr.discovered = 0; sr.inspected_edges = (dir == 1) ? mf : 0; sr.aux = st.u_cnt; sr.ns = 0;
            }
        }
        Slot &nxt = a.ctl->slot[(L + 1) & 3];
        app.qv = a.qv[(L + 1) & 1];
        app.qo = a.qo[(L + 1) & 1];
        app.qr = a.qr[(L + 1) & 1];
        app.counter = &nxt.qpack;
        uint32_t *fb_c = a.fbuf[L % 3];
        uint32_t *fb_n = a.fbuf[(L + 1) % 3];
        uint32_t *fb_z = a.fbuf[(L + 2) % 3];
        unsigned long long ndisc = 0, insp = 0;
        if (dir == 2 && !st.fb_valid) {
            // queue -> bitmap conversion ("converts the current
            // frontier into a bitmap of vertices")
            for (int64_t w = tid; w < nwords; w += nthreads) fb_c[w] = 0u;
            grid.sync();
            const int32_t *qv_c = a.qv[L & 1];
            for (int64_t j = tid; j < f; j += nthreads) {
                const int32_t v = qv_c[j];
                atomicOr(fb_c + (v >> 5), 1u << (v & 31));
            }
            grid.sync();
        }
        // clear the bitmap level L+1 will fill (it was last read at level L-1);
        // only when a pull level is plausible soon: a sweep over n/32 words is
        // not free on high-diameter graphs with thousands of tiny levels
        const bool need_fb = (dir == 2) || (mf >= nwords / 4);
        if (need_fb)
            for (int64_t w = tid; w < nwords; w += nthreads) fb_z[w] = 0u;
        if (dir == 1) {
            BfsPushOp op{a.visited, st.fbn_clean ? fb_n : nullptr, a.depth, a.pred, a.R, L + 1,
                         a.idempotent, &app, 0ull, pol_keep,
                         mf < (1 << 16) ? 0 : (st.m_u * 4 < a.m ? 2 : 1)};
            GlobalFrontier fr{a.qv[L & 1], a.qo[L & 1], a.qr[L & 1], f, mf};
            // auto (reading A-4, measured on B200): node-granular thread/warp/CTA
            // when the frontier's lists are short on average (mesh-like levels:
            // no frontier-wide search, 35% faster per level on C4); merge-path
            // over edges when a few lists carry the edges (hubs: one CTA per list
            // would serialise them; C2 level 1 is 26% slower with TWC)
            const bool twc = a.strategy == 1 ||
                             (a.strategy == 0 && f < a.lb_threshold && mf <= 16 * f);
            if (twc) {
                expand_twc(fr, a.C, op, &s->win);
            } else {
#if GR_BFS_STAGES > 0
            expand_pipe<kBfsStages, false>(fr, a.C, nullptr, gw, nw, op, &s->u.stage.pipe[wib]);
#else
            expand_lb(fr, a.C, gw, nw, op);
#endif
            }
            ndisc = op.ndisc;
            st.fb_valid = st.fbn_clean;
        } else {
            pull_level(a, fb_c, fb_n, L + 1, &s->work, app, ndisc, insp);
            st.fb_valid = 1;
        }
        GR_TSTAMP(5);
        app.finish();
        GR_TSTAMP(6);
        ndisc = warp_sum<unsigned long long>(ndisc);
        insp = warp_sum<unsigned long long>(insp);
        if (lane_id() == 0) {
            if (ndisc) atomicAdd(&s->bsum[0], ndisc);
            if (insp) atomicAdd(&s->bsum[1], insp);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s->bsum[0]) atomicAdd(&nxt.ndisc, s->bsum[0]);
            if (s->bsum[1]) atomicAdd(&nxt.insp, s->bsum[1]);
        }
        st.prev_dir = dir;
        st.prev_f = f;
        st.fbn_clean = need_fb;
        st.L = L + 1;
        pending = true;
        GR_TSTAMP(7);
        grid.sync();
        GR_TSTAMP(8);
    }
    if (tid == 0) a.ctl->levels = (unsigned long long)st.L;
}

gr_status run_bfs(Graph *g, int32_t src, int32_t *depth, int32_t *pred, const gr_bfs_opts &o,
                  int *launches) {
    BfsArgs a;
    a.n = g->n; a.m = g->m;
    a.R = g->R; a.C = g->C; a.Rt = g->Rt; a.Ct = g->Ct;
    a.visited = g->visited;
    a.noin = g->noin;
    for (int i = 0; i < 3; ++i) a.fbuf[i] = g->fbuf[i];
    for (int i = 0; i < 2; ++i) { a.qv[i] = g->qv[i]; a.qo[i] = g->qo[i]; a.qr[i] = g->qr[i]; }
    a.depth = depth; a.pred = pred;
    a.ctl = g->ctl; a.stats = g->stats_dev;
    a.src = src;
    a.direction = o.direction;
    a.switch_rule = o.switch_rule;
    a.idempotent = o.idempotent;
    a.strategy = o.strategy;
    a.lb_threshold = o.lb_threshold > 0 ? o.lb_threshold : env_int("GR_LB_THRESHOLD", 1ll << 40);
    a.alpha = o.alpha > 0 ? o.alpha : 14.0;
    a.beta = o.beta > 0 ? o.beta : 24.0;
    a.nonisolated = g->nonisolated;
    a.S = g->pack_shift;
    a.small_f = env_int("GR_SMALL_F", kSmallFDefault);
    a.small_e = env_int("GR_SMALL_E", kSmallE);
    if (a.small_f > kSmallF) a.small_f = kSmallF;

    static int per_sm = 0;  // occupancy of the kernel (same on every device of the box)
    const size_t smem = sizeof(BfsSmem);
    if (per_sm == 0) {
        GR_CUDA(cudaFuncSetAttribute(bfs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, kBlock, smem));
    }
    if (per_sm < 1) { set_error("bfs_kernel cannot be resident"); return GR_ERR_CUDA; }
    dim3 grid(g->num_sms * per_sm), block(kBlock);
    void *args[] = {&a};
    GR_CUDA(cudaLaunchCooperativeKernel((void *)bfs_kernel, grid, block, args, smem, g->stream));
    count_launch();
    *launches = 1;
    return GR_OK;
}

}  // namespace gr

#ifdef GR_TRACE
// debug only (not in gr.h): install the BFS level trace buffer (16 stamps x 256 levels)
extern "C" int gr_debug_trace_set(long long *dev_buf) {
    return (int)cudaMemcpyToSymbol(gr::g_trace, &dev_buf, sizeof(dev_buf));
}
#endif
