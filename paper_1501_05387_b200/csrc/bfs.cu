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
#include "pull.cuh"

namespace gr {

#ifndef GR_SMALL_CAP
#define GR_SMALL_CAP 512  // measured: smaller shared memory leaves more L1 for probes/spills
#endif
constexpr int64_t kSmallF = GR_SMALL_CAP;  // small mode: queue capacity (shared memory)
constexpr int64_t kSmallFDefault = 512;   // small mode: default max frontier (swept on C4)
constexpr int64_t kSmallE = 4096;   // small mode: max frontier edges (swept round 2: 4096 / 16384 / 65536: C1 0.079 / 0.086 / 0.086 ms, C2-C5 equal or better at 4096)
#ifndef GR_BFS_STAGES
#define GR_BFS_STAGES 0  // measured on C2 push: 2 and 4 stages are slower (smem displaces L1)
#endif
constexpr int kBfsStages = GR_BFS_STAGES;  // cp.async pipeline depth of the grid push advance (0: off)
#ifndef GR_SPEC_R
#define GR_SPEC_R 0  // 1: small push steps load the targets' row offsets in parallel with the claims
                     // (measured slower everywhere: C4 BFS 98.5 -> 106 ms, C2 0.144 -> 0.153 ms; spills)
#endif
constexpr int kSmallCntBits = 24;
constexpr int64_t kCtaFlushEdges = 16384;  // steps with at least this many frontier edges flush per CTA   // count field of the small-mode packed counter
constexpr unsigned long long kSmallCntMask = (1ull << kSmallCntBits) - 1;

struct BfsArgs {
    int64_t n, m;
    const int64_t *R;
    const int32_t *C;
    const int64_t *Rt;   // in-edges for pull (== R when symmetric)
    const int32_t *Ct;
    const int2 *ph;      // pull head {first in-neighbour, in-degree} per vertex (null: none)
    const int4 *ell;     // bounded-degree adjacency (null: none; Graph::ell)
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
    int64_t sbm_words;         // words of the shared-memory bitmap snapshot (0: off)
    int64_t snap_min_edges;    // push steps with at least this many frontier edges use it
    int32_t lb_chunks;         // dynamic merge-path pieces per warp (0: static partition)
    int32_t claim_cas;         // push claim: CAS on depth[] (1) or atomicOr on the bitmap (0)
    int64_t probe_skip_pct;    // push steps skip the culling probe while m_u >= this % of m
    int32_t lazy_r;            // grid push: row offsets of discovered vertices loaded at the flush
    int32_t bar_ns;            // GridBar backoff cap (ns)
    int32_t pull_stay;         // direction rule: stay in pull for tiny frontiers with fewer unvisited (A-3)
    int64_t sparse_grab;       // pull sweeps grab 32 words when u_cnt * sparse_grab < n (0: never)
    int64_t sparse_grab_maxw;  // ... and the bitmap has at most this many words (measured: C5's 2^20 prefer 4)
    int32_t resume;            // bounded-degree graphs: the cluster kernel ran the first levels
                               // (bfs_ell_cluster_kernel); continue from ctl->bstate, no init
};

template <int kNW>
struct BfsSmemT {
    union {
        struct {  // grid levels: per-warp append staging + cp.async pipeline
            PipeWarpSmem<(kBfsStages > 0 ? kBfsStages : 1), false> pipe[kBfsStages > 0 ? kNW : 1];
            int32_t sv[kNW][kStageCap];
            int32_t sd[kNW][kStageCap];
            int64_t sr[kNW][kStageCap];
        } stage;
        int32_t plist[kNW][kPullList];  // pull steps: per-warp candidate lists
        struct {  // small mode: the frontier lives here (double-buffered)
            int64_t rs[2][kSmallF];   // row start of each entry
            int64_t off[2][kSmallF];  // exclusive degree prefix (reserved at append time)
            int32_t q[2][kSmallF];    // vertex ids
        } small;
    } u;
    unsigned long long ctl[8];
    unsigned long long wsum[2 * kNW + 2];  // Appender::finish_cta
    long long scan[kNW];
    unsigned long long bsum[6];
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
    int claim_cas;       // non-idempotent claim by CAS on depth (1) or atomicOr on the bitmap (0)
    uint32_t sbm;        // shared address of the visited snapshot (targets < sbits)
    int64_t sbits;       // 0: no snapshot this step

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const T5 *) {
        uint32_t word[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            word[u] = !ok[u] ? 0xffffffffu
                    : dst[u] < sbits ? lds_u32(sbm + 4u * (uint32_t)(dst[u] >> 5))
                    : probe == 1 ? ld_probe(visited + (dst[u] >> 5), pol_keep)
                    : probe == 2 ? ld_l1(visited + (dst[u] >> 5)) : 0u;
        bool disc[U];
        // small steps (no probe): the row offsets of every target are loaded
        // speculatively, in parallel with the claims -- one dependent round trip
        // less per level (high-diameter graphs run thousands of such levels)
        int64_t spec[U];
        const bool specr = GR_SPEC_R && probe == 0 && !idempotent && !claim_cas;
        if (specr) {
#pragma unroll
            for (int u = 0; u < U; ++u) spec[u] = ok[u] ? __ldg(R + dst[u]) : 0;
        }
        // candidates first, then every claim of the lane in flight before any
        // result is read (a claim consumed inside its own branch made the U
        // atomics of a lane one dependent round trip each: measured ~0.45 us
        // apiece on B200, the largest term of a narrow level)
        bool cand[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t w = dst[u];
            const uint32_t bit = 1u << (w & 31);
            cand[u] = ok[u] && !(word[u] & bit);
            // snapshot: the first warp of this CTA to reach w sets its bit in
            // shared memory; the CTA's later visitors of w stop here (culling
            // inside the CTA is exact; the global claim below stays the truth)
            if (cand[u] && w < sbits) cand[u] = !(atom_or_shared(sbm + 4u * (uint32_t)(w >> 5), bit) & bit);
            if (idempotent) {
                // warp-level culling heuristic (A-5 i): lanes of one warp that
                // target the same vertex keep only the lowest lane
                const unsigned peers = __match_any_sync(0xffffffffu, cand[u] ? w : -1 - (int)lane_id());
                cand[u] = cand[u] && (__ffs(peers) - 1 == (int)lane_id());
            }
        }
        if (idempotent) {
            int32_t dv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) dv[u] = cand[u] ? *(volatile int32_t *)(depth + dst[u]) : 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                disc[u] = cand[u] && dv[u] < 0;
                if (disc[u]) atomicOr(visited + (dst[u] >> 5), 1u << (dst[u] & 31));  // result unused -> RED.OR
            }
        } else if (claim_cas) {
            // exactly-once per VERTEX: contention only between claims of
            // the same vertex, not of the 32 vertices sharing a bitmap word
            int32_t r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = cand[u] ? atomicCAS(depth + dst[u], -1, next_depth) : 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                disc[u] = cand[u] && r[u] == -1;
                if (disc[u]) atomicOr(visited + (dst[u] >> 5), 1u << (dst[u] & 31));  // RED.OR
            }
        } else {
            uint32_t old[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                old[u] = cand[u] ? atomicOr(visited + (dst[u] >> 5), 1u << (dst[u] & 31)) : 0xffffffffu;
#pragma unroll
            for (int u = 0; u < U; ++u) disc[u] = !((old[u] >> (dst[u] & 31)) & 1u);
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
                if (!app->Rl) {
                    rs = specr ? spec[u] : R[w];
                    deg = __ldg(R + w + 1) - rs;
                }
                ++ndisc;
            }
            // lazy appender: the row offsets of the staged vertices are loaded
            // at the flush, all at once (no dependent load per group here)
            app->push(disc[u] && (app->Rl || deg > 0), w, deg, rs);
        }
    }
};

// Grid push step over the bounded-degree adjacency (expand_ell): the same
// cond/claim/apply/filter as BfsPushOp, but each slot
// carries the neighbour's out-degree, so a discovered vertex is appended
// without loading R; its own ELL record is prefetched into L2 for the next
// level (high-diameter graphs: one dependent DRAM round trip less per level).
struct BfsEllOp {
    uint32_t *visited;
    uint32_t *fbn;       // next frontier bitmap (null: not maintained this level)
    int32_t *depth;
    int32_t *pred;
    const int4 *ell;
    int32_t next_depth;
    int32_t idempotent;
    Appender *app;
    unsigned long long ndisc;
    unsigned long long pol_keep;
    int probe;           // as BfsPushOp::probe

    __device__ __forceinline__ void slots(bool, int32_t v, int4 s4) {
        const int32_t sl[4] = {s4.x, s4.y, s4.z, s4.w};
        uint32_t word[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t w = sl[k] >> 3;
            word[k] = sl[k] < 0 ? 0xffffffffu
                    : probe == 1 ? ld_probe(visited + (w >> 5), pol_keep)
                    : probe == 2 ? ld_l1(visited + (w >> 5)) : 0u;
        }
        bool disc[4], cand[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t w = sl[k] >> 3;
            cand[k] = sl[k] >= 0 && !(word[k] & (1u << (w & 31)));
        }
        if (idempotent) {
            int32_t dv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t w = sl[k] >> 3;
                const unsigned peers = __match_any_sync(0xffffffffu, cand[k] ? w : -1 - (int)lane_id());
                cand[k] = cand[k] && (__ffs(peers) - 1 == (int)lane_id());
                dv[k] = cand[k] ? *(volatile int32_t *)(depth + w) : 0;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t w = sl[k] >> 3;
                disc[k] = cand[k] && dv[k] < 0;
                if (disc[k]) atomicOr(visited + (w >> 5), 1u << (w & 31));  // RED.OR
            }
        } else {
            // all claims of the lane in flight before any result is read
            uint32_t old[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t w = sl[k] >> 3;
                old[k] = cand[k] ? atomicOr(visited + (w >> 5), 1u << (w & 31)) : 0xffffffffu;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) disc[k] = !((old[k] >> ((sl[k] >> 3) & 31)) & 1u);
        }
        GR_TDEP(3, disc[0] + 2 * disc[1] + 4 * disc[2] + 8 * disc[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!__any_sync(0xffffffffu, disc[k])) continue;
            const int32_t w = sl[k] >> 3;
            const int32_t deg = sl[k] & 7;
            if (disc[k]) {
                depth[w] = next_depth;
                if (pred) pred[w] = v;
                if (fbn) atomicOr(fbn + (w >> 5), 1u << (w & 31));  // RED.OR
                if (deg) asm volatile("prefetch.global.L2 [%0];" ::"l"(ell + w));
                ++ndisc;
            }
            app->push(disc[k] && deg > 0, w, deg, 0);
        }
    }
};

// Small-mode op: claim directly with atomicOr (one L2 round trip instead of
// probe + claim) while the target's row offsets are loaded speculatively in
// parallel, then append (vertex, row start, degree) into the shared-memory
// queue of the next level and prefetch the head of its neighbour list into L2
// (the next level reads it a few microseconds later). Entries beyond kSmallF
// spill to the global queue, which then ends small mode.
template <bool kEll>
struct SmallPushOpT {
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
    const int4 *ell;             // bounded-degree adjacency (slots(); null: edges())

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
        append<U>(old, rs, re, dst, src);
    }

    // bounded-degree adjacency (expand_ell): the degree rides in the slot, the
    // discovered vertex's ELL record is what the next level loads
    __device__ __forceinline__ void slots(bool, int32_t v, int4 s4) {
        const int32_t sl[4] = {s4.x, s4.y, s4.z, s4.w};
        uint32_t old[4];
        int64_t rs[4], re[4];
        int32_t dst[4], src[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            dst[k] = sl[k] >> 3;
            src[k] = v;
            rs[k] = 0;
            re[k] = sl[k] & 7;
            old[k] = sl[k] >= 0 ? atomicOr(visited + (dst[k] >> 5), 1u << (dst[k] & 31)) : 0xffffffffu;
        }
        append<4>(old, rs, re, dst, src);
    }

    template <int U>
    __device__ __forceinline__ void append(const uint32_t *old, const int64_t *rs, const int64_t *re,
                                           const int32_t *dst, const int32_t *src) {
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
                    if constexpr (kEll) {
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(ell + w));
                    } else {
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(C + rs[u]));
                        if (deg > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + rs[u] + 32));
                    }
                }
                ++ndisc;
            }
        }
    }
};

// Direction decision (reading A-3): direction_rule (pull.cuh) on
// counters every block reads after the same barrier, so all blocks agree.
__device__ __forceinline__ int decide_direction(const BfsArgs &a, int dir, int64_t f, int64_t mf,
                                                int64_t u_cnt, int64_t m_u, int64_t prev_f,
                                                int64_t nwords) {
    return direction_rule(a.direction, a.switch_rule, a.alpha, a.beta, a.nonisolated, dir, f, mf, u_cnt, m_u,
                          prev_f, nwords, a.pull_stay == 2 ? INT64_MAX : a.pull_stay ? a.small_f : 0);
}

struct BfsState {  // per-traversal heuristic state, identical in every CTA
    int L;
    int dir, prev_dir;
    int64_t u_cnt, m_u, prev_f;
    int fb_valid;       // fbuf[L%3] holds the frontier of level L
    int fbn_clean;      // fbuf[(L+1)%3] is all zero
    int closed;         // stats records below this level are closed
    int q_valid;        // the queue of level L is materialised (a pull step keeps a bitmap only)
};

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int kBlk>
__host__ __device__ constexpr size_t bfs_sbm_offset() { return (sizeof(BfsSmemT<kBlk / kWarp>) + 127) & ~(size_t)127; }

// kPush: direction forced to push (gr_bfs_opts.direction = 1): the pull and
// bitmap-conversion paths are compiled out, which frees registers for the
// push advance (fewer spills at the 64-register cap).
// kEll: the graph has the bounded-degree adjacency (Graph::ell); its push
// steps use expand_ell (a separate instantiation: the general kernel keeps
// its register allocation)
template <int kBlk, int kMinB, bool kPush = false, bool kEll = false>
__global__ void __launch_bounds__(kBlk, kMinB) bfs_kernel(BfsArgs a) {
    constexpr int kNW = kBlk / kWarp;
    using BfsSmem = BfsSmemT<kNW>;
    const GridBar grid{&a.ctl->gbar, a.bar_ns};
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BfsSmem *s = reinterpret_cast<BfsSmem *>(smem_raw);
    uint32_t *sbm_p = reinterpret_cast<uint32_t *>(smem_raw + bfs_sbm_offset<kBlk>());
    const uint32_t sbm = (uint32_t)__cvta_generic_to_shared(sbm_p);
    const int64_t sbits = a.sbm_words * 32;

    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gw = tid >> 5;
    const int64_t nw = nthreads >> 5;
    const int wib = threadIdx.x >> 5;
    const int64_t nwords = (a.n + 31) / 32;
    const unsigned long long cmask = (1ull << a.S) - 1;

    BfsState st;
    long long t_prev = 0;
    if (kEll && a.resume) {
        // the narrow first levels ran in bfs_ell_cluster_kernel: it either
        // finished the traversal or left the frontier of level bstate[0] in
        // the queue with its descriptor in the level's slot
        if (threadIdx.x == 0) {
            long long x[7];
#pragma unroll
            for (int k = 0; k < 7; ++k) x[k] = __ldcg(a.ctl->bstate + k);
#pragma unroll
            for (int k = 0; k < 7; ++k) s->ctl[k] = (unsigned long long)x[k];
            s->ctl[7] = __ldcg(&a.ctl->handoff);
        }
        __syncthreads();
        if (s->ctl[7] != 1ull) return;  // finished in cluster mode
        st.L = (int)(long long)s->ctl[0];
        st.dir = (int)(long long)s->ctl[1];
        st.prev_dir = (int)(long long)s->ctl[2];
        st.u_cnt = (long long)s->ctl[3];
        st.m_u = (long long)s->ctl[4];
        st.prev_f = (long long)s->ctl[5];
        if (tid == 0) t_prev = (long long)s->ctl[6];
        st.closed = st.L;
        st.fb_valid = 0;
        st.fbn_clean = 0;
        st.q_valid = 1;
        __syncthreads();
    } else {
    // ---- Set_Problem_Data: depth = -1 (A-2), pred = -1, and the
    // source's entries written by the thread that owns them in the same pass
    // (one grid barrier instead of init-barrier-source-barrier) -------------
    const int64_t deg_src = a.R[a.src + 1] - a.R[a.src];
    for (int64_t v = tid; v < a.n; v += nthreads) {
        a.depth[v] = (v == a.src) ? 0 : -1;
        if (a.pred) a.pred[v] = (v == a.src) ? a.src : -1;  // A-1
    }
    // vertices with no in-edge can never be discovered: pre-mark them visited
    // so pull skips them (they keep depth -1; the bitmap is internal)
    for (int64_t w = tid; w < nwords; w += nthreads)
        a.visited[w] = a.noin[w] | ((w == (a.src >> 5)) ? 1u << (a.src & 31) : 0u);
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) {
        unsigned long long x = 0ull;  // slot 0 (words 0 and 6): the source's frontier descriptor
        if (tid == 0 && deg_src > 0) x = ((unsigned long long)deg_src << a.S) | 1ull;
        if (tid == (int64_t)(offsetof(Slot, dmax) / 8)) x = (unsigned long long)deg_src;
        ((unsigned long long *)a.ctl->slot)[tid] = x;
    }
    if (tid == 0) {
        a.ctl->overflow = 0ull;
        a.qv[0][0] = a.src;
        a.qo[0][0] = 0;
        a.qr[0][0] = a.R[a.src];
    }
    grid.sync();

    // Heuristic state. u = unvisited vertices that have an in-edge, m_u =
    // edges incident to them (reading A-3).
    const bool src_has_in = !((a.noin[a.src >> 5] >> (a.src & 31)) & 1u);
    st.L = 0;
    st.dir = (a.direction == 2) ? 2 : 1;
    st.prev_dir = 1;
    st.u_cnt = a.nonisolated - (src_has_in ? 1 : 0);
    st.m_u = a.m - deg_src;
    st.prev_f = 0;
    st.fb_valid = 0;
    st.fbn_clean = 0;
    st.closed = 0;
    st.q_valid = 1;
    if (tid == 0) t_prev = gtimer();
    }
    const unsigned long long pol_keep = policy_evict_last();
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
                                     q2 = ld_relaxed(&cur.insp), q3 = ld_relaxed(&a.ctl->overflow),
                                     q4 = ld_relaxed(&cur.dmax);
            s->ctl[0] = q0; s->ctl[1] = q1; s->ctl[2] = q2; s->ctl[3] = q3; s->ctl[4] = q4;
            // per-level CTA counters, reset before the barrier below (racecheck)
            s->work = 0; s->bsum[0] = 0; s->bsum[1] = 0; s->bsum[4] = 0; s->bsum[5] = 0;
#ifdef GR_TRACE
            s->bsum[2] = ~0ull; s->bsum[3] = 0;
#endif
        }
        __syncthreads();
        const unsigned long long qp = s->ctl[0];
        const int64_t f = (int64_t)(qp & cmask);
        const int64_t mf = (int64_t)(qp >> a.S);
        const int64_t dmax = (int64_t)s->ctl[4];
        if (pending) {
            st.u_cnt -= (int64_t)s->ctl[1];
            st.m_u -= mf;
            pending = false;
        }
        if (tid == 0 && L > st.closed && L - 1 < kMaxStatRecords) {
            gr_level_stats &sr = a.stats[L - 1];
            sr.discovered = (int64_t)s->ctl[1];
            // the level's direction is in a register: reading sr.direction back
            // was a dependent global load on CTA 0's critical path every level
            if (st.prev_dir == 2) sr.inspected_edges = (int64_t)s->ctl[2];
            const long long t = gtimer();
            sr.ns = t - t_prev;
            t_prev = t;
        }
        const bool stop = (f == 0 || s->ctl[3]);
        __syncthreads();  // s->ctl is rewritten below
        if (stop) break;
        const int dir = kPush ? 1 : decide_direction(a, st.dir, f, mf, st.u_cnt, st.m_u, st.prev_f, nwords);
        if (dir == 1 && !st.q_valid) {
            // the frontier of the last pull step exists as a bitmap only
            Appender conv = app;
            Slot &cs = a.ctl->slot[L & 3];
            conv.qv = a.qv[L & 1]; conv.qo = a.qo[L & 1]; conv.qr = a.qr[L & 1];
            conv.counter = &cs.fpack;
            conv.dmax = nullptr;
            conv.cnt = 0;
            conv.Rl = nullptr;
            bitmap_to_queue(a, a.fbuf[L % 3], gw, nw, conv);
            grid.sync();
            st.q_valid = 1;
        }

        if (dir == 1 && f <= a.small_f && mf <= a.small_e) {
            // ================= small mode: CTA 0 alone ===========================
            if (blockIdx.x == 0) {
                int c = 0, r = 0;
                for (int64_t j = threadIdx.x; j < f; j += kBlk) {
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
                    const int d = kPush ? 1 : decide_direction(a, st.dir, cf, E, st.u_cnt, st.m_u, st.prev_f, nwords);
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
                    SmallPushOpT<kEll> op{a.visited, a.depth, a.pred, a.R, a.C, Lc + 1, s->u.small.q[c ^ 1],
                                   s->u.small.rs[c ^ 1], s->u.small.off[c ^ 1], &s->pk[r1],
                                   a.qv[(Lc + 1) & 1], a.qo[(Lc + 1) & 1], a.qr[(Lc + 1) & 1], 0ull, a.ell};
                    SmemFrontier fr{s->u.small.q[c], s->u.small.off[c], s->u.small.rs[c], cf, E};
                    GR_TSTAMP(9);
                    if constexpr (kEll) expand_ell(s->u.small.q[c], cf, a.ell, (int64_t)wib, (int64_t)kNW, op);
                    else expand_lb(fr, a.C, (int64_t)wib, (int64_t)kNW, op);
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
                    for (int64_t j = threadIdx.x; j < cf && j < kSmallF; j += kBlk) {
                        a.qv[st.L & 1][j] = s->u.small.q[c][j];
                        a.qo[st.L & 1][j] = s->u.small.off[c][j];
                        a.qr[st.L & 1][j] = s->u.small.rs[c][j];
                    }
                    if (mu_pending) st.m_u -= E;
                    if (threadIdx.x == 0) {
                        a.ctl->slot[st.L & 3].qpack = ((unsigned long long)E << a.S) | (unsigned long long)cf;
                        a.ctl->slot[st.L & 3].ndisc = 0;
                        a.ctl->slot[st.L & 3].insp = 0;
                        a.ctl->slot[st.L & 3].work = 0;
                        a.ctl->slot[st.L & 3].dmax = (unsigned long long)E;  // bound: max deg <= E
                    }
                } else if (threadIdx.x == 0) {
                    a.ctl->slot[st.L & 3].qpack = 0;
                }
                if (threadIdx.x == 0) {
                    for (int k = 1; k <= 2; ++k) {
                        Slot &r = a.ctl->slot[(st.L + k) & 3];
                        r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull; r.dmax = 0;
                    }
                    long long *bs = a.ctl->bstate;
                    bs[0] = st.L; bs[1] = st.dir; bs[2] = st.prev_dir; bs[3] = st.u_cnt;
                    bs[4] = st.m_u; bs[5] = st.prev_f; bs[6] = tp;
                }
            } else if (gridDim.x > 1) {
                // the idle CTAs zero the three frontier bitmaps meanwhile, so
                // the grid level that follows records its next frontier in a
                // clean bitmap (a push -> pull switch then needs no
                // queue -> bitmap conversion pass and its two grid barriers)
                const int64_t nb = (int64_t)(gridDim.x - 1) * blockDim.x;
                for (int64_t w = (int64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x; w < nwords; w += nb) {
                    a.fbuf[0][w] = 0u; a.fbuf[1][w] = 0u; a.fbuf[2][w] = 0u;
                }
            }
            grid.sync();
            if (threadIdx.x == 0) {
                // independent L2 loads issued back to back (volatile loads were
                // serialised: 7 round trips while the CTA waits at the barrier)
                long long x[7];
#pragma unroll
                for (int k = 0; k < 7; ++k) x[k] = __ldcg(a.ctl->bstate + k);
#pragma unroll
                for (int k = 0; k < 7; ++k) s->ctl[k] = (unsigned long long)x[k];
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
            st.fbn_clean = gridDim.x > 1 ? 1 : 0;  // zeroed by the idle CTAs above
            st.q_valid = 1;
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
            rst.dmax = 0;
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
        app.dmax = &nxt.dmax;
        app.Rl = (!kEll && a.lazy_r) ? a.R : nullptr;
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
        const bool snap = a.sbm_words > 0 && (dir == 2 || mf >= a.snap_min_edges);
        if (snap) {
            // bitmap snapshot for this step: visited (push culling) or the
            // current frontier (pull probes); read-only global state now
            snapshot_bits(sbm_p, dir == 1 ? a.visited : fb_c, a.sbm_words);
            __syncthreads();
        }
        if (kEll && dir == 1) {
            BfsEllOp op{a.visited, st.fbn_clean ? fb_n : nullptr, a.depth, a.pred, a.ell, L + 1, a.idempotent,
                        &app, 0ull, pol_keep,
                        (mf < (1 << 16) || st.m_u * 100 >= a.m * a.probe_skip_pct) ? 0 : (st.m_u * 4 >= a.m ? 1 : 2)};
            // warps interleaved over the CTAs: a narrow frontier uses every SM
            expand_ell(a.qv[L & 1], f, a.ell, (int64_t)wib * gridDim.x + blockIdx.x, nw, op);
            ndisc = op.ndisc;
            st.fb_valid = st.fbn_clean;
        } else if (dir == 1) {
            BfsPushOp op{a.visited, st.fbn_clean ? fb_n : nullptr, a.depth, a.pred, a.R, L + 1,
                         a.idempotent, &app, 0ull, pol_keep,
                         // probe: none for small steps and when most edges still lead to
                         // unvisited vertices (the claim's old bit answers anyway: one random
                         // line per edge less); L2 while many do; L1 late (mostly visited)
                         (mf < (1 << 16) || st.m_u * 100 >= a.m * a.probe_skip_pct) ? 0
                             : (snap || st.m_u * 4 >= a.m ? 1 : 2), a.claim_cas, sbm,
                         snap ? sbits : 0};
            GlobalFrontier fr{a.qv[L & 1], a.qo[L & 1], a.qr[L & 1], f, mf};
            // auto (reading A-4, measured on B200): node-granular thread/warp/CTA
            // when the frontier's lists are short on average (mesh-like levels:
            // no frontier-wide search, 35% faster per level on C4); merge-path
            // over edges when a few lists carry the edges (hubs: one CTA per list
            // would serialise them; C2 level 1 is 26% slower with TWC)
            // ... but never with a long list in the frontier: thread/warp/CTA
            // gives a whole list to one CTA (measured on C2: one hub in a
            // frontier of 1.07M short lists held the level at 576 us vs 89 us median)
            const bool twc = a.strategy == 1 ||
                             (a.strategy == 0 && f < a.lb_threshold && mf <= 16 * f && dmax <= kTwcMaxDeg);
            if (twc) {
                expand_twc(fr, a.C, op, &s->win);
            } else {
#if GR_BFS_STAGES > 0
            expand_pipe<kBfsStages, false>(fr, a.C, nullptr, gw, nw, op, &s->u.stage.pipe[wib]);
#else
            expand_lb(fr, a.C, gw, nw, op, a.lb_chunks > 0 ? &a.ctl->slot[L & 3].work : nullptr,
                      a.lb_chunks);
#endif
            }
            ndisc = op.ndisc;
            st.fb_valid = st.fbn_clean;
        } else {
            if (!st.fbn_clean) {  // RED.OR targets must start at zero
                for (int64_t w = tid; w < nwords; w += nthreads) fb_n[w] = 0u;
                grid.sync();
            }
            PullCounts pc;
            // few unvisited vertices left (late levels): a warp grabs 32 bitmap
            // words at a time, so the sweep is not a chain of 4-word grabs
            pull_level(a, fb_c, fb_n, L + 1, &s->work, s->u.plist[wib], pc, sbm, snap ? sbits : 0,
                       nwords * blockIdx.x / gridDim.x, nwords * (blockIdx.x + 1) / gridDim.x,
                       (st.u_cnt * a.sparse_grab < a.n && nwords <= a.sparse_grab_maxw) ? 32 : kPullGrab);
            ndisc = pc.ndisc;
            insp = pc.insp;
            // lazy queue: only the size, edges and max degree of the next frontier
            const unsigned long long qc = warp_sum<unsigned long long>(pc.qcnt);
            const unsigned long long qe = warp_sum<unsigned long long>(pc.qedges);
            const unsigned dm = __reduce_max_sync(0xffffffffu, pc.dmax);
            if (lane_id() == 0) {
                if (qc) atomicAdd(&s->bsum[4], (qe << a.S) | qc);
                if (dm) atomicMax(&s->bsum[5], (unsigned long long)dm);
            }
            st.fb_valid = 1;
            st.q_valid = 0;
        }
        GR_TSTAMP(5);
        ndisc = warp_sum<unsigned long long>(ndisc);
        insp = warp_sum<unsigned long long>(insp);
        if (lane_id() == 0) {
            if (ndisc) atomicAdd(&s->bsum[0], ndisc);
            if (insp) atomicAdd(&s->bsum[1], insp);
#ifdef GR_TRACE
            const unsigned long long tw = (unsigned long long)gtimer();
            atomicMin(&s->bsum[2], tw);
            atomicMax(&s->bsum[3], tw);
#endif
        }
        // wide steps: one queue atomic per CTA (finish_cta); narrow steps (a few
        // warps hold entries): per-warp flushes, no extra CTA barriers (measured
        // on C4: +1.1 us per level with finish_cta on its 512-4K-vertex levels)
        if (mf >= kCtaFlushEdges) app.finish_cta(s->wsum);  // its CTA barriers also complete the counters
        else { app.finish(); __syncthreads(); }
        GR_TSTAMP(6);
#ifdef GR_TRACE
        if (g_bal && threadIdx.x == 0 && L < 64) {
            g_bal[((int64_t)L * gridDim.x + blockIdx.x) * 2] = (long long)s->bsum[2];
            g_bal[((int64_t)L * gridDim.x + blockIdx.x) * 2 + 1] = (long long)s->bsum[3];
        }
#endif
        if (threadIdx.x == 0) {
            if (s->bsum[0]) atomicAdd(&nxt.ndisc, s->bsum[0]);
            if (s->bsum[4]) atomicAdd(&nxt.qpack, s->bsum[4]);
            if (s->bsum[5]) atomicMax(&nxt.dmax, s->bsum[5]);
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
    if (tid == 0) {
        a.ctl->levels = (unsigned long long)st.L;
        if (a.ctl->overflow) a.ctl->sticky = 1ull;
    }
}


// ---------------------------------------------------------------------------
// Narrow levels of bounded-degree graphs in ONE thread-block cluster
// (high-diameter graphs, C4: ~10.6K levels of a few hundred to ~8K
// vertices). A level of the grid kernel is a chain of L2 round trips plus a
// 296-CTA barrier (~8 us); here the frontier lives in the cluster's
// distributed shared memory and a level costs one DSMEM read of the CTAs'
// counters, the entry (DSMEM) and its ELL record, one batch of claims, a
// shared-memory append and a hardware cluster barrier.
//  * every CTA appends the vertices its threads discover to its own
//    shared-memory queue (one packed (edges << 32) | count atomic per warp);
//  * the next level's entry j is owned by the CTA whose count prefix covers
//    j: each thread takes global index j = rank * 1024 + tid, so the work of
//    a level is spread evenly over the cluster whatever CTA discovered it;
//  * a level runs here only if its frontier fits one entry per thread
//    (then no CTA can append more than 4 x 1024 entries) and the direction
//    rule (A-3) says push; otherwise the frontier is written to the global
//    queue and the grid kernel resumes at that level (Ctl::handoff, bstate).
// Same semantics as the grid push step: atomicOr claim (exactly once),
// depth = L + 1, pred = the frontier vertex.
// ---------------------------------------------------------------------------

struct ClSmem {
    int32_t q[2][kClQ];               // appended vertices, by level parity
    unsigned long long cnt[3];        // (edges << 32) | count appended, by level mod 3
    unsigned long long nd[3];         // vertices discovered (degree 0 too), by level mod 3
    int pfx[kClMax + 1];              // exclusive prefix of the CTAs' counts (current level)
    long long tot[3];                 // F, MF, discovered by the previous level
};

// Set_Problem_Data for the cluster path: the whole GPU writes the
// O(n) arrays; the cluster kernel then places the source.
__global__ void bfs_init_kernel(BfsArgs a) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t nwords = (a.n + 31) / 32;
    for (int64_t v = tid; v < a.n; v += nthreads) {
        a.depth[v] = -1;
        if (a.pred) a.pred[v] = -1;
    }
    for (int64_t w = tid; w < nwords; w += nthreads) a.visited[w] = a.noin[w];
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (tid == 0) { a.ctl->overflow = 0ull; a.ctl->handoff = 0ull; }
}

__global__ void __launch_bounds__(kClBlock, 1) bfs_ell_cluster_kernel(BfsArgs a) {
    __shared__ ClSmem s;
    const unsigned K = cluster_nctarank();
    const unsigned rank = cluster_ctarank();
    const int t = threadIdx.x;
    const unsigned l = lane_id();
    const int64_t nwords = (a.n + 31) / 32;
    if (t < 3) { s.cnt[t] = 0ull; s.nd[t] = 0ull; }
    const int64_t deg_src = a.R[a.src + 1] - a.R[a.src];
    __syncthreads();
    if (rank == 0 && t == 0) {
        a.depth[a.src] = 0;
        if (a.pred) a.pred[a.src] = a.src;  // A-1
        atomicOr(a.visited + (a.src >> 5), 1u << (a.src & 31));
        if (deg_src > 0) { s.q[0][0] = a.src; s.cnt[0] = ((unsigned long long)deg_src << 32) | 1ull; }
    }
    cluster_barrier();
    const bool src_has_in = !((a.noin[a.src >> 5] >> (a.src & 31)) & 1u);
    int64_t u_cnt = a.nonisolated - (src_has_in ? 1 : 0);
    int64_t m_u = a.m - deg_src;
    int64_t prev_f = 0;
    long long tp = 0;
    if (rank == 0 && t == 0) tp = gtimer();
    int L = 0;
    for (;;) {
        const int c0 = L % 3, c1 = (L + 1) % 3, c2 = (L + 2) % 3, p = L & 1;
        // ---- the level's counters from every CTA of the cluster (DSMEM) ----
        if (t < 32) {
            unsigned long long x = 0, y = 0;
            if (l < K) { x = ld_dsmem_u64(&s.cnt[c0], l); y = ld_dsmem_u64(&s.nd[c0], l); }
            const int cn = (int)(x & 0xffffffffu);
            const int incl = warp_incl_scan<int>(cn);
            const long long e = warp_sum<long long>((long long)(x >> 32));
            const long long d = warp_sum<long long>((long long)y);
            if (l < K) s.pfx[l + 1] = incl;
            if (l == 0) { s.pfx[0] = 0; s.tot[1] = e; s.tot[2] = d; }
            if (l == 31) s.tot[0] = incl;
        }
        __syncthreads();
        const int64_t F = s.tot[0], MF = s.tot[1], ND = s.tot[2];
        if (L > 0) { u_cnt -= ND; m_u -= MF; }
        if (rank == 0 && t == 0 && L > 0 && L - 1 < kMaxStatRecords) {
            const long long tn = gtimer();
            a.stats[L - 1].discovered = ND;
            a.stats[L - 1].ns = tn - tp;
            tp = tn;
        }
        if (F == 0) {
            if (rank == 0 && t == 0) { a.ctl->levels = (unsigned long long)L; a.ctl->handoff = 2ull; }
            break;
        }
        const int dir = decide_direction(a, 1, F, MF, u_cnt, m_u, prev_f, nwords);
        if (dir != 1 || F > (int64_t)K * kClBlock) {
            // ---- hand the frontier of level L to the grid kernel ----------
            for (int64_t j = (int64_t)t * K + rank; j < F; j += (int64_t)K * kClBlock) {
                int o = 0;
                while (o + 1 < (int)K && s.pfx[o + 1] <= j) ++o;
                a.qv[L & 1][j] = ld_dsmem_s32(&s.q[p][j - s.pfx[o]], o);
            }
            if (rank == 0 && t == 0) {
                a.ctl->slot[L & 3].qpack = ((unsigned long long)MF << a.S) | (unsigned long long)F;
                a.ctl->slot[L & 3].dmax = 4ull;
                a.ctl->slot[L & 3].ndisc = 0; a.ctl->slot[L & 3].insp = 0; a.ctl->slot[L & 3].work = 0;
                for (int k = 1; k <= 2; ++k) {
                    Slot &r = a.ctl->slot[(L + k) & 3];
                    r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull; r.dmax = 0;
                }
                long long *bs = a.ctl->bstate;
                bs[0] = L; bs[1] = 1; bs[2] = 1; bs[3] = u_cnt; bs[4] = m_u; bs[5] = prev_f; bs[6] = tp;
                a.ctl->handoff = 1ull;
            }
            break;
        }
        if (rank == 0 && t == 0 && L < kMaxStatRecords) {
            gr_level_stats &sr = a.stats[L];
            sr.level = L; sr.direction = 1; sr.frontier = F; sr.frontier_edges = MF;
            sr.discovered = 0; sr.inspected_edges = MF; sr.aux = u_cnt; sr.ns = 0;
        }
        // counters of level L+2 were last read at level L-1 (before its barrier)
        if (t == 0) { s.cnt[c2] = 0ull; s.nd[c2] = 0ull; }
        // ---- expand: global entry j of the level, one per thread -----------
        // entries interleaved over the CTAs (j = t * K + rank): a narrow level
        // spreads over every SM of the cluster (its scattered record loads,
        // claims and stores are issue-limited per SM: with j = rank * 1024 + t
        // a 2K-vertex level ran on two SMs, 6.2 us per level on C4)
        const int64_t j = (int64_t)t * K + rank;
        int32_t v = 0;
        int4 rec = make_int4(-1, -1, -1, -1);
        if (j < F) {
            int o = 0;
#pragma unroll 1
            while (o + 1 < (int)K && s.pfx[o + 1] <= j) ++o;
            v = ld_dsmem_s32(&s.q[p][j - s.pfx[o]], o);
            rec = ld_ell(a.ell + v);
        }
        const int32_t sl[4] = {rec.x, rec.y, rec.z, rec.w};
        uint32_t old[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t w = sl[k] >> 3;
            old[k] = sl[k] >= 0 ? atomicOr(a.visited + (w >> 5), 1u << (w & 31)) : 0xffffffffu;
        }
        int na = 0, nd = 0;
        long long ea = 0;
        bool ap[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t w = sl[k] >> 3;
            const bool disc = !((old[k] >> (w & 31)) & 1u);
            ap[k] = disc && (sl[k] & 7) != 0;
            if (disc) {
                a.depth[w] = L + 1;
                if (a.pred) a.pred[w] = v;
                ++nd;
                if (ap[k]) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.ell + w));
            }
            na += ap[k];
            ea += ap[k] ? (sl[k] & 7) : 0;
        }
        // one packed shared-memory atomic per warp reserves the slots and the edges
        const int incl = warp_incl_scan<int>(na);
        const long long etot = warp_sum<long long>(ea);
        const int ndw = warp_sum<int>(nd);
        unsigned long long base = 0;
        if (l == 31 && incl > 0) base = atomicAdd(&s.cnt[c1], ((unsigned long long)etot << 32) | (unsigned)incl);
        if (l == 0 && ndw > 0) atomicAdd(&s.nd[c1], (unsigned long long)ndw);
        base = __shfl_sync(0xffffffffu, base, 31);
        int pos = (int)(base & 0xffffffffu) + incl - na;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (ap[k]) s.q[p ^ 1][pos++] = sl[k] >> 3;
        prev_f = F;
        ++L;
        cluster_barrier();
    }
    // no CTA may exit while another still reads its shared memory (the last
    // level's counters, the handed-off queue): every CTA leaves the loop at
    // the same level (identical decisions), then waits for the others here
    cluster_barrier();
}

// Largest cluster (16, else 8) of bfs_ell_cluster_kernel CTAs the device can
// run (0: none; GR_ELL_CLUSTER_SIZE forces one).
static int ell_cluster_size() {
    static int k = -1;
    if (k >= 0) return k;
    k = 0;
    const int want = (int)env_int("GR_ELL_CLUSTER_SIZE", 0);
    cudaFuncSetAttribute(bfs_ell_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
        if (cudaOccupancyMaxActiveClusters(&ncl, bfs_ell_cluster_kernel, &cfg) == cudaSuccess && ncl >= 1) {
            k = c;
            break;
        }
    }
    cudaGetLastError();  // an unsupported size leaves an error behind
    return k;
}

gr_status run_bfs(Graph *g, int32_t src, int32_t *depth, int32_t *pred, const gr_bfs_opts &o,
                  int *launches) {
    BfsArgs a;
    a.n = g->n; a.m = g->m;
    a.R = g->R; a.C = g->C; a.Rt = g->Rt; a.Ct = g->Ct; a.ph = g->ph;
    a.ell = g->ell;
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
    a.lb_threshold = o.lb_threshold > 0 ? o.lb_threshold : env_int("GR_LB_THRESHOLD", 65536);
    // alpha 20 (Beamer's CPU value is 14): swept on B200 over {6..30}, C2 -3%,
    // C3 -1%, C5 within noise for 17..24 (A-3)
    a.alpha = o.alpha > 0 ? o.alpha : (double)env_int("GR_ALPHA", 20);
    a.beta = o.beta > 0 ? o.beta : (double)env_int("GR_BETA", 24);
    a.nonisolated = g->nonisolated;
    a.S = g->pack_shift;
    a.small_f = env_int("GR_SMALL_F", kSmallFDefault);
    a.small_e = env_int("GR_SMALL_E", kSmallE);
    a.lb_chunks = (int32_t)env_int("GR_LB_CHUNKS", 4);
    a.claim_cas = (int32_t)env_int("GR_CLAIM_CAS", 0);
    a.probe_skip_pct = env_int("GR_PROBE_SKIP_PCT", 75);
    a.lazy_r = (int32_t)env_int("GR_LAZY_R", 1);
    a.bar_ns = (int32_t)env_int("GR_BAR_NS", 128);
    a.pull_stay = (int32_t)env_int("GR_PULL_STAY", 2);
    a.sparse_grab = env_int("GR_SPARSE_GRAB", 16);
    a.sparse_grab_maxw = env_int("GR_SPARSE_GRAB_MAXW", 1 << 18);
    if (a.small_f > kSmallF) a.small_f = kSmallF;

    // Kernel variant: graphs whose bitmap no
    // longer fits in L1 run 1024-thread CTAs (1 per SM) with most of the
    // shared memory holding a bitmap snapshot; small graphs keep 512 x 2 CTAs.
    const int64_t nwords = (g->n + 31) / 32;
    const bool use_snap = env_int("GR_SNAPSHOT", 0) != 0 && nwords * 4 > env_int("GR_SNAP_MIN_BYTES", 64 << 10);
    static int optin = 0;
    if (optin == 0) GR_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
    const bool push_only = a.direction == 1 && !use_snap && env_int("GR_PUSH_KERNEL", 0) != 0;  // measured 3% slower: off
    const void *fn = use_snap ? (const void *)bfs_kernel<1024, 1>
                   : g->ell ? (const void *)bfs_kernel<kBlock, kMinBlocks, false, true>
                   : push_only ? (const void *)bfs_kernel<kBlock, kMinBlocks, true>
                               : (const void *)bfs_kernel<kBlock, kMinBlocks>;
    const int block = use_snap ? 1024 : kBlock;
    size_t smem;
    a.sbm_words = 0;
    a.snap_min_edges = env_int("GR_SNAP_MIN_EDGES", 1 << 20);
    if (use_snap) {
        const size_t off = bfs_sbm_offset<1024>();
        int64_t w = ((int64_t)optin - (int64_t)off - 1024) / 4;  // 1 KB reserve
        if (w > nwords) w = nwords;
        a.sbm_words = w & ~3ll;
        smem = off + (size_t)a.sbm_words * 4;
    } else {
        smem = sizeof(BfsSmemT<kBlock / kWarp>);
    }
    static bool attr_set[4] = {false, false, false, false};
    const int variant = use_snap ? 1 : g->ell ? 3 : push_only ? 2 : 0;
    if (!attr_set[variant]) {
        GR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        attr_set[variant] = true;
    }
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
    if (per_sm < 1) { set_error("bfs_kernel cannot be resident"); return GR_ERR_CUDA; }
    if (per_sm > (use_snap ? 1 : kMinBlocks)) per_sm = use_snap ? 1 : kMinBlocks;
    int64_t ctas = (int64_t)g->num_sms * per_sm;
    const int64_t cap_ctas = env_int("GR_BFS_CTAS", 0);  // experiment: fewer persistent CTAs
    if (cap_ctas > 0 && cap_ctas < ctas) ctas = cap_ctas;
    // bounded-degree graphs: the narrow levels run in one thread-block cluster
    // (bfs_ell_cluster_kernel), the grid kernel resumes only if a frontier
    // outgrows it or the direction rule turns to pull
    int nl = 0;
    a.resume = 0;
    const int kcl = (g->ell && !use_snap && a.direction != 2 && env_int("GR_ELL_CLUSTER", 1)) ? ell_cluster_size() : 0;
    if (kcl > 0) {
        bfs_init_kernel<<<g->num_sms * 4, 512, 0, g->stream>>>(a);
        GR_CUDA(cudaGetLastError());
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)kcl);
        cfg.blockDim = dim3(kClBlock);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = g->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)kcl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        GR_CUDA(cudaLaunchKernelEx(&cfg, bfs_ell_cluster_kernel, a));
        count_launch(2);
        nl += 2;
        a.resume = 1;
    }
    dim3 grid((unsigned)ctas), blk(block);
    void *args[] = {&a};
    GR_CUDA(cudaLaunchCooperativeKernel(fn, grid, blk, args, smem, g->stream));
    count_launch();
    *launches = nl + 1;
    return GR_OK;
}

}  // namespace gr

#ifdef GR_TRACE
// debug only (not in gr.h): install the BFS level trace buffer (16 stamps x 256 levels)
extern "C" int gr_debug_trace_set(long long *dev_buf) {
    return (int)cudaMemcpyToSymbol(gr::g_trace, &dev_buf, sizeof(dev_buf));
}
// debug only: per-level per-CTA [first, last] warp completion times (64 levels x grid x 2)
extern "C" int gr_debug_balance_set(long long *dev_buf) {
    return (int)cudaMemcpyToSymbol(gr::g_bal, &dev_buf, sizeof(dev_buf));
}
#endif
