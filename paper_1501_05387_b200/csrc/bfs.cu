// bfs.cu -- breadth-first search, push and direction-optimizing push-pull,
// as ONE persistent cooperative kernel per traversal (device-side iteration
// control: no host round trip per level).
//
// Paper: BFS §5.1; advance/filter; fusion;
// load balancing; idempotent vs atomic discovery (P:793-802,
// P:916-921); push vs pull. Readings A-1..A-6 in DESIGN.md.
#include "frontier.cuh"

namespace gr {

struct BfsArgs {
    int64_t n, m;
    const int64_t *R;
    const int32_t *C;
    const int64_t *Rt;   // in-edges for pull (== R when symmetric)
    const int32_t *Ct;
    uint32_t *visited;
    uint32_t *fbuf0, *fbuf1;
    int32_t *qv0, *qv1;
    int64_t *qo0, *qo1;
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
};

// Per-edge op of the push advance: the fused cond/apply + filter of BFS.
// cond: "is d unvisited" (bitmap probe, culling heuristic P:797-799);
// claim: atomicOr on the visited word returns the old bit, so each vertex is
// discovered exactly once ("non-idempotent advance ... uses atomic
// operations to guarantee each element appears only once"); apply: depth and
// pred; filter: warp-staged append into the next queue.
// With idempotent=1 the claim is atomic-free: depth[] (not the bitmap) is the
// authoritative visited test, plain stores write it, the bitmap is updated
// with a fire-and-forget red.or and only filters (reading A-6); duplicates may
// enter the queue and are harmless (same depth).
struct BfsPushOp {
    uint32_t *visited;
    int32_t *depth;
    int32_t *pred;
    const int64_t *R;
    int32_t next_depth;
    int32_t idempotent;
    Appender *app;
    unsigned long long ndisc;

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const int64_t *) {
        uint32_t word[U];
#pragma unroll
        for (int u = 0; u < U; ++u) word[u] = ok[u] ? ld_cg(visited + (dst[u] >> 5)) : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int32_t w = dst[u];
            uint32_t bit = 1u << (w & 31);
            bool disc = false;
            int64_t deg = 0;
            if (ok[u] && !(word[u] & bit)) {
                if (idempotent) {
                    if (*(volatile int32_t *)(depth + w) < 0) {
                        disc = true;
                        depth[w] = next_depth;
                        atomicOr(visited + (w >> 5), bit);  // result unused -> RED.OR
                    }
                } else {
                    uint32_t old = atomicOr(visited + (w >> 5), bit);
                    if (!(old & bit)) {
                        disc = true;
                        depth[w] = next_depth;
                    }
                }
                if (disc) {
                    if (pred) pred[w] = src[u];
                    deg = R[w + 1] - R[w];
                }
            }
            ndisc += disc;
            app->push(disc && deg > 0, w, deg);
        }
    }
};

// Pull (bottom-up) step over in-edges: "pull starts with a
// frontier of unvisited vertices, generating the new frontier by filtering
// the unvisited frontier for vertices that have neighbors in the current
// frontier"; the current frontier is held as a bitmap. A warp
// owns 32 consecutive vertices = one bitmap word, so the next-frontier word
// and the visited word are written with one plain store from a ballot: no
// atomics. Each lane stops at its first in-neighbour in the frontier (early
// exit).
__device__ __forceinline__ void pull_level(const BfsArgs &a, const uint32_t *__restrict__ fcur,
                                           uint32_t *__restrict__ fnext, int32_t next_depth,
                                           int64_t gw, int64_t nw, Appender &app,
                                           unsigned long long &ndisc, unsigned long long &insp) {
    const int64_t nwords = (a.n + 31) / 32;
    const unsigned l = lane_id();
    for (int64_t wi = gw; wi < nwords; wi += nw) {
        int64_t v = wi * 32 + l;
        uint32_t visw = a.visited[wi];
        bool cand = v < a.n && !((visw >> l) & 1u);
        bool found = false;
        int32_t parent = -1;
        if (cand) {
            int64_t beg = a.Rt[v], end = a.Rt[v + 1];
            for (int64_t e = beg; e < end && !found; e += 4) {
                int32_t u[4];
                uint32_t fw[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) u[k] = (e + k < end) ? __ldg(a.Ct + e + k) : -1;
#pragma unroll
                for (int k = 0; k < 4; ++k) fw[k] = (u[k] >= 0) ? __ldg(fcur + (u[k] >> 5)) : 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!found && u[k] >= 0) {
                        ++insp;
                        if ((fw[k] >> (u[k] & 31)) & 1u) {
                            found = true;
                            parent = u[k];
                        }
                    }
                }
            }
        }
        unsigned nb = __ballot_sync(0xffffffffu, found);
        if (l == 0) {
            fnext[wi] = nb;
            if (nb) a.visited[wi] = visw | nb;
        }
        int64_t deg = 0;
        if (found) {
            a.depth[v] = next_depth;
            if (a.pred) a.pred[v] = parent;
            deg = a.R[v + 1] - a.R[v];
        }
        ndisc += found;
        app.push(found && deg > 0, (int32_t)v, deg);
    }
}

__global__ void __launch_bounds__(kBlock) bfs_kernel(BfsArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t s_v[kWarpsPerBlock][kStageCap];
    __shared__ int64_t s_d[kWarpsPerBlock][kStageCap];

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
    for (int64_t w = tid; w < nwords; w += nthreads) a.visited[w] = 0u;
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (tid == 0) a.ctl->overflow = 0ull;
    grid.sync();
    const int64_t deg_src = a.R[a.src + 1] - a.R[a.src];
    if (tid == 0) {
        a.depth[a.src] = 0;
        if (a.pred) a.pred[a.src] = a.src;  // A-1
        a.visited[a.src >> 5] = 1u << (a.src & 31);
        if (deg_src > 0) {
            a.qv0[0] = a.src;
            a.qo0[0] = 0;
            a.ctl->slot[0].qpack = ((unsigned long long)deg_src << a.S) | 1ull;
        }
    }
    grid.sync();

    // Heuristic state (identical in every block: computed from the same
    // counters after each grid barrier). u = unvisited non-isolated vertices,
    // m_u = edges incident to them (reading A-3).
    int64_t u_cnt = a.nonisolated - 1;
    int64_t m_u = a.m - deg_src;
    int dir = (a.direction == 2) ? 2 : 1;
    int prev_dir = 1;  // the initial frontier is a queue
    int64_t prev_f = 0;

    Appender app;
    app.sv = s_v[wib];
    app.sd = s_d[wib];
    app.cnt = 0;
    app.S = a.S;
    app.cap = a.n;
    app.overflow = &a.ctl->overflow;

    int L = 0;
    for (;; ++L) {
        Slot &cur = a.ctl->slot[L & 3];
        Slot &nxt = a.ctl->slot[(L + 1) & 3];
        const unsigned long long qp = ld_volatile(&cur.qpack);
        const int64_t f = (int64_t)(qp & cmask);
        const int64_t mf = (int64_t)(qp >> a.S);
        if (L > 0 && tid == 0 && L - 1 < kMaxStatRecords) {
            gr_level_stats &st = a.stats[L - 1];
            st.discovered = (int64_t)ld_volatile(&cur.ndisc);
            if (st.direction == 2) st.inspected_edges = (int64_t)ld_volatile(&cur.insp);
        }
        if (f == 0 || ld_volatile(&a.ctl->overflow)) break;

        // ---- direction decision (reading A-3) -------------------
        if (a.direction == 0) {
            if (a.switch_rule == 1) {
                dir = (u_cnt < f) ? 2 : 1;  // paper-literal: unvisited < frontier
            } else if (dir == 1) {
                if ((double)mf > (double)m_u / a.alpha) dir = 2;
            } else {
                if ((double)f < (double)a.nonisolated / a.beta && f < prev_f) dir = 1;
            }
        }
        if (tid == 0) {
            Slot &rst = a.ctl->slot[(L + 2) & 3];
            rst.qpack = 0; rst.ndisc = 0; rst.fpack = 0; rst.work = 0; rst.minfar = ~0ull;
            rst.insp = 0;
            if (L < kMaxStatRecords) {
                gr_level_stats &st = a.stats[L];
                st.level = L; st.direction = dir; st.frontier = f; st.frontier_edges = mf;
                st.discovered = 0; st.inspected_edges = (dir == 1) ? mf : 0; st.aux = u_cnt;
            }
        }

        int32_t *qv_c = (L & 1) ? a.qv1 : a.qv0;
        int64_t *qo_c = (L & 1) ? a.qo1 : a.qo0;
        int32_t *qv_n = (L & 1) ? a.qv0 : a.qv1;
        int64_t *qo_n = (L & 1) ? a.qo0 : a.qo1;
        uint32_t *fb_c = (L & 1) ? a.fbuf1 : a.fbuf0;
        uint32_t *fb_n = (L & 1) ? a.fbuf0 : a.fbuf1;

        app.qv = qv_n;
        app.qo = qo_n;
        app.counter = &nxt.qpack;
        unsigned long long ndisc = 0;

        if (dir == 1) {
            BfsPushOp op{a.visited, a.depth, a.pred, a.R, L + 1, a.idempotent, &app, 0ull};
            expand_lb(qv_c, qo_c, f, mf, a.R, a.C, gw, nw, op);
            ndisc = op.ndisc;
        } else {
            if (prev_dir == 1) {
                // queue -> bitmap conversion ("converts the current
                // frontier into a bitmap of vertices")
                for (int64_t w = tid; w < nwords; w += nthreads) fb_c[w] = 0u;
                grid.sync();
                for (int64_t j = tid; j < f; j += nthreads) {
                    int32_t v = qv_c[j];
                    atomicOr(fb_c + (v >> 5), 1u << (v & 31));
                }
                grid.sync();
            }
            unsigned long long insp = 0;
            pull_level(a, fb_c, fb_n, L + 1, gw, nw, app, ndisc, insp);
            insp = warp_sum<unsigned long long>(insp);
            if (lane_id() == 0 && insp) atomicAdd(&nxt.insp, insp);
        }
        app.finish();
        ndisc = warp_sum<unsigned long long>(ndisc);
        if (lane_id() == 0 && ndisc) atomicAdd(&nxt.ndisc, ndisc);
        prev_dir = dir;
        prev_f = f;
        grid.sync();
        const unsigned long long nq = ld_volatile(&nxt.qpack);
        const unsigned long long nd = ld_volatile(&nxt.ndisc);
        u_cnt -= (int64_t)nd;
        m_u -= (int64_t)(nq >> a.S);
    }
    if (tid == 0) a.ctl->levels = (unsigned long long)L;
}

gr_status run_bfs(Graph *g, int32_t src, int32_t *depth, int32_t *pred, const gr_bfs_opts &o,
                  int *launches) {
    BfsArgs a;
    a.n = g->n; a.m = g->m;
    a.R = g->R; a.C = g->C; a.Rt = g->Rt; a.Ct = g->Ct;
    a.visited = g->visited;
    a.fbuf0 = g->fbuf[0]; a.fbuf1 = g->fbuf[1];
    a.qv0 = g->qv[0]; a.qv1 = g->qv[1];
    a.qo0 = g->qo[0]; a.qo1 = g->qo[1];
    a.depth = depth; a.pred = pred;
    a.ctl = g->ctl; a.stats = g->stats_dev;
    a.src = src;
    a.direction = o.direction;
    a.switch_rule = o.switch_rule;
    a.idempotent = o.idempotent;
    a.alpha = o.alpha > 0 ? o.alpha : 14.0;
    a.beta = o.beta > 0 ? o.beta : 24.0;
    a.nonisolated = g->nonisolated;
    a.S = g->pack_shift;

    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, kBlock, 0));
    if (per_sm < 1) { set_error("bfs_kernel cannot be resident"); return GR_ERR_CUDA; }
    dim3 grid(g->num_sms * per_sm), block(kBlock);
    void *args[] = {&a};
    GR_CUDA(cudaLaunchCooperativeKernel((void *)bfs_kernel, grid, block, args, 0, g->stream));
    count_launch();
    *launches = 1;
    return GR_OK;
}

}  // namespace gr
