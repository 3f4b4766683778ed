// pbfs.cu -- BFS over a 1D vertex partition as ONE persistent kernel per rank
// (SURVEY §8(b) gr_bfs on a partitioned graph, §8(e); SURVEY §5 Tier 2 "fused
// compute + exchange"). The paper is single-GPU (multi-GPU is its future
// work); every step of a level is the single-GPU hot path of
// bfs.cu (advance + filter P:326-364; merge-path balancing
// P:748-758; pull P:804-834; direction rule A-3), extended with an exchange
// that happens INSIDE the kernel over peer memory (NVLink on an NVSwitch box):
//
//  push level  local merge-path advance; an owned target is claimed here; a
//              remote target is culled by this rank's "already sent" bitmap and
//              its (vertex, parent) pair is stored straight into the OWNER's
//              inbox (slots reserved with a system-scope atomicAdd on the
//              owner's inbox counter, warp-aggregated per owner) -> barrier ->
//              the owner claims its inbox entries;
//  pull level  each rank stores its frontier-bitmap shard into every rank's
//              global frontier bitmap (an all-gather done with peer stores)
//              -> barrier -> bottom-up step over the owned unvisited vertices;
//  every level each rank publishes (f, m_f, discovered, ...) of its next local
//              frontier into every rank's counter table -> barrier -> every
//              rank sums the same table, takes the same direction decision
//              and stops at the same level.
// No host round trip and no NCCL call per level. Barriers: a cooperative grid
// barrier inside a process; across processes, epoch flags in the peers'
// symmetric regions (release / acquire at system scope). A loopback group (all
// ranks in one process on one GPU) runs every rank in ONE cooperative launch,
// CTA block [r*ctas, (r+1)*ctas) acting as rank r: the multi-rank logic is the
// same code, tested on one GPU.
#include "part.cuh"
#include "pull.cuh"

namespace gr {

gr_status graph_create(int64_t n, int64_t m, const int64_t *R, const int32_t *C, const uint32_t *W,
                       uint32_t flags, int device, void *stream, Graph **out, int64_t ncols);
bool ptr_on_device(const void *p);
gr_status sort_lists_by_degree(Graph *g, cudaStream_t s, int blocks, const int32_t *deg);
gr_status build_pull_head(Graph *g);

// ---------------------------------------------------------------- kernel arguments
struct PRank {                 // everything the CTAs of one rank need
    int32_t rank, S;
    int64_t n_local, v_begin, m_local, nonisolated;
    const int64_t *R;
    const int32_t *C;          // push lists (global ids)
    const int32_t *Cp;         // pull lists (global ids, ordered by global neighbour degree)
    const int2 *ph;            // pull head {first pull-list entry, degree} per owned vertex
    uint32_t *visited;         // local bitmap (authoritative claims of owned vertices)
    const uint32_t *noin;      // local: vertices without in-edges (pre-visited)
    uint32_t *sent;            // global bitmap: remote vertices this rank already shipped
    uint32_t *fb[3];           // local frontier bitmaps (rotating, as in bfs.cu)
    int32_t *qv[2];            // local frontier queues (LOCAL ids)
    int64_t *qo[2];
    int64_t *qr[2];
    int32_t *depth, *pred;     // outputs of the owned block (pred: GLOBAL ids)
    Ctl *ctl;
    gr_level_stats *stats;
    char *sym[kMaxRanks];      // every rank's symmetric region, as mapped by this rank
};

struct PBfsArgs {
    PRank ranks[kMaxRanks];    // the ranks this launch hosts (1, or all of a loopback group)
    int32_t vranks, nranks, multiproc, ctas;
    int64_t n_global, block, src;
    size_t off_gfront[2], off_inbox;
    int64_t inbox_cap;
    int32_t direction, switch_rule, lb_chunks;
    double alpha, beta;
};

struct PullView {              // pull_level / bitmap_to_queue view of a partition
    int64_t n;
    const int64_t *R, *Rt;
    const int32_t *Ct;
    const int2 *ph;
    uint32_t *visited;
    int32_t *depth, *pred;
};

// ---------------------------------------------------------------------------
// Fused cond/apply + filter + exchange of a push level (per edge (s, w)):
// owned w: culling probe, atomicOr claim on the local visited word, depth /
// pred / next-frontier bit, warp-staged append (as BfsPushOp); remote w:
// test-and-set in the "already sent" bitmap, then (w, parent) goes into the
// owner's inbox -- lanes with the same owner share one system-scope atomicAdd
// on the owner's counter and store their pairs contiguously.
// ---------------------------------------------------------------------------
struct PPushOp {
    const PRank *a;
    uint32_t *fbn;          // next local frontier bitmap (null: not maintained)
    int32_t next_depth;
    Appender *app;
    int64_t block, inbox_cap;
    size_t off_inbox;
    int probe;              // probe the claim word first (most targets already visited)
    unsigned long long pol_keep;
    unsigned long long ndisc, shipped;

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const T5 *) {
        // probes of all U edges, then all claims in flight, then the results
        // (an atomic consumed inside its own branch costs a round trip apiece)
        bool disc[U], ship[U], own[U];
        uint32_t word[U], *cw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t w = dst[u];
            const int64_t lw = (int64_t)w - a->v_begin;
            own[u] = lw >= 0 && lw < a->n_local;
            cw[u] = own[u] ? a->visited + (lw >> 5) : a->sent + (w >> 5);  // claim word
            word[u] = !ok[u] ? 0xffffffffu : (own[u] && !probe) ? 0u : ld_probe(cw[u], pol_keep);
        }
        uint32_t old[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t bit = 1u << ((own[u] ? (int32_t)((int64_t)dst[u] - a->v_begin) : dst[u]) & 31);
            old[u] = !(word[u] & bit) ? atomicOr(cw[u], bit) : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t bit = 1u << ((own[u] ? (int32_t)((int64_t)dst[u] - a->v_begin) : dst[u]) & 31);
            const bool got = !(old[u] & bit);
            disc[u] = got && own[u];
            ship[u] = got && !own[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t w = dst[u];
            const int32_t parent = (int32_t)(a->v_begin + src[u]);
            if (__any_sync(0xffffffffu, disc[u])) {
                const int64_t lw = (int64_t)w - a->v_begin;
                if (disc[u]) {
                    a->depth[lw] = next_depth;
                    if (a->pred) a->pred[lw] = parent;
                    if (fbn) atomicOr(fbn + (lw >> 5), 1u << (lw & 31));  // RED.OR
                    ++ndisc;
                }
                app->push(disc[u], (int32_t)lw, 0, 0);  // lazy appender: R loaded at the flush
            }
            const unsigned shm = __ballot_sync(0xffffffffu, ship[u]);
            if (shm) {
                const int q = ship[u] ? (int)((int64_t)w / block) : -1;
                const unsigned peers = __match_any_sync(0xffffffffu, q);
                if (ship[u]) {
                    const int leader = __ffs(peers) - 1;
                    SymHdr *h = reinterpret_cast<SymHdr *>(a->sym[q]);
                    unsigned long long base = 0;
                    if ((int)lane_id() == leader) base = atomicAdd_system(&h->inbox_count, (unsigned long long)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    const unsigned long long pos = base + __popc(peers & lanemask_lt());
                    if ((int64_t)pos < inbox_cap) {
                        int2 *ib = reinterpret_cast<int2 *>(a->sym[q] + off_inbox);
                        ib[pos] = make_int2(w, parent);
                    } else {
                        atomicExch(&a->ctl->overflow, 1ull);
                    }
                    ++shipped;
                }
            }
        }
    }
};

template <int kNW>
struct PSmem {
    union {
        struct {
            int32_t sv[kNW][kStageCap];
            int32_t sd[kNW][kStageCap];
            int64_t sr[kNW][kStageCap];
        } stage;
        int32_t plist[kNW][kPullList];
    } u;
    PRank r;
    unsigned long long wsum[2 * kNW + 2];  // Appender::finish_cta
    unsigned long long ctl[16];
    unsigned long long bsum[8];
    int work;
};

constexpr int kPBlock = 512;
constexpr int kPMinB = 2;

template <int kBlk, int kMinB>
__global__ void __launch_bounds__(kBlk, kMinB) pbfs_kernel(const __grid_constant__ PBfsArgs A) {
    constexpr int kNW = kBlk / kWarp;
    __shared__ PSmem<kNW> sm;
    cg::grid_group grid = cg::this_grid();
    const int vr = blockIdx.x / A.ctas;
    const int bid = blockIdx.x - vr * A.ctas;
    if (threadIdx.x == 0) sm.r = A.ranks[vr];
    __syncthreads();
    const PRank &a = sm.r;
    const int64_t tid = (int64_t)bid * kBlk + threadIdx.x;      // rank-local thread id
    const int64_t nthreads = (int64_t)A.ctas * kBlk;
    const int64_t gw = tid >> 5, nw = nthreads >> 5;
    const int wib = threadIdx.x >> 5;
    const int64_t nwl = (a.n_local + 31) / 32;                  // local bitmap words
    const int64_t gwords = (A.n_global + 31) / 32;              // global bitmap words
    const unsigned long long cmask = (1ull << a.S) - 1;
    const bool lead = bid == 0 && threadIdx.x == 0;             // one thread per rank
    RankSync rs{&grid, a.sym, a.rank, A.nranks, A.multiproc, bid, a.ctl, a.ctl->epoch};
    auto hdr = [&](int q) { return rs.hdr(q); };
    auto gbar = [&]() { rs.bar(); };
    auto publish = [&](int par, const unsigned long long *vals) { rs.publish(par, vals); };

    // ---- Set_Problem_Data on the owned block ------------------
    for (int64_t v = tid; v < a.n_local; v += nthreads) {
        a.depth[v] = -1;
        if (a.pred) a.pred[v] = -1;
    }
    for (int64_t w = tid; w < nwl; w += nthreads) a.visited[w] = a.noin[w];
    for (int64_t w = tid; w < gwords; w += nthreads) a.sent[w] = 0u;
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (lead) {
        a.ctl->overflow = 0ull;
        hdr(a.rank)->inbox_count = 0ull;
    }
    gbar();  // every rank is in this run (its previous run's tables are no longer read)
    {
        unsigned long long vals[8] = {0, 0, 0, 0, (unsigned long long)a.m_local, 0, 0,
                                      (unsigned long long)a.nonisolated};
        if (lead) {
            a.sent[A.src >> 5] |= 1u << (A.src & 31);  // nobody ships the source
            const int64_t ls = A.src - a.v_begin;
            if (ls >= 0 && ls < a.n_local) {
                const int64_t d = a.R[ls + 1] - a.R[ls];
                a.depth[ls] = 0;
                if (a.pred) a.pred[ls] = (int32_t)A.src;  // A-1, global id
                a.visited[ls >> 5] |= 1u << (ls & 31);
                a.qv[0][0] = (int32_t)ls;
                a.qo[0][0] = 0;
                a.qr[0][0] = a.R[ls];
                if (d > 0) {
                    a.ctl->slot[0].qpack = ((unsigned long long)d << a.S) | 1ull;
                    vals[kStF] = 1;
                    vals[kStMf] = (unsigned long long)d;
                    vals[kStDmax] = (unsigned long long)d;
                }
            }
        }
        __syncthreads();
        publish(0, vals);
    }

    Appender app;
    app.sv = sm.u.stage.sv[wib];
    app.sd = sm.u.stage.sd[wib];
    app.sr = sm.u.stage.sr[wib];
    app.cnt = 0;
    app.S = a.S;
    app.cap = 2 * a.n_local;
    app.overflow = &a.ctl->overflow;
    app.Rl = a.R;  // lazy: every pushed id is local; its row offsets are loaded at the flush
    const unsigned long long pol_keep = policy_evict_last();
    const PullView view{a.n_local, a.R, a.R, a.Cp, a.ph, a.visited, a.depth, a.pred};
    const uint32_t *gfront_own[2] = {reinterpret_cast<const uint32_t *>(a.sym[a.rank] + A.off_gfront[0]),
                                     reinterpret_cast<const uint32_t *>(a.sym[a.rank] + A.off_gfront[1])};
    const int2 *inbox = reinterpret_cast<const int2 *>(a.sym[a.rank] + A.off_inbox);

    int L = 0, dir = (A.direction == 2) ? 2 : 1;
    int64_t u_cnt = 0, m_u = 0, prev_f = 0, M = 0, NONISO = 0;
    bool fb_valid = false, fbn_clean = false, q_valid = true;
    unsigned long long istart = 0;
    long long t_prev = lead ? pgtimer() : 0;

    for (;;) {
        const int par = L & 1;
        if (threadIdx.x == 0) {
            unsigned long long t[8];
            rs.read(par, t, kStDmax, kStOvf);
            for (int k = 0; k < 8; ++k) sm.ctl[k] = t[k];
            sm.ctl[8] = ld_relaxed(&a.ctl->slot[L & 3].qpack);
            sm.work = 0;
            for (int k = 0; k < 8; ++k) sm.bsum[k] = 0;
        }
        __syncthreads();
        const int64_t F = (int64_t)sm.ctl[kStF], MF = (int64_t)sm.ctl[kStMf];
        const int64_t f_loc = (int64_t)(sm.ctl[8] & cmask), mf_loc = (int64_t)(sm.ctl[8] >> a.S);
        if (L == 0) {
            M = (int64_t)sm.ctl[kStInsp];
            NONISO = (int64_t)sm.ctl[kStAux];
            u_cnt = NONISO - (MF > 0 ? 1 : 0);
            m_u = M - MF;
        } else {
            u_cnt -= (int64_t)sm.ctl[kStDisc];
            m_u -= MF;
            if (lead && L - 1 < kMaxStatRecords) {
                gr_level_stats &sr = a.stats[L - 1];
                sr.discovered = (int64_t)sm.ctl[kStDisc];
                if (sr.direction == 2) sr.inspected_edges = (int64_t)sm.ctl[kStInsp];
                else sr.aux = 8 * (int64_t)sm.ctl[kStShip];
                const long long tn = pgtimer();
                sr.ns = tn - t_prev;
                t_prev = tn;
            }
        }
        const bool stop = F == 0 || sm.ctl[kStOvf] != 0;
        __syncthreads();  // sm.ctl is rewritten below
        if (stop) break;
        const int d = direction_rule(A.direction, A.switch_rule, A.alpha, A.beta, NONISO, dir, F, MF, u_cnt, m_u,
                                     prev_f, gwords);
        if (lead && L < kMaxStatRecords) {
            gr_level_stats &sr = a.stats[L];
            sr.level = L; sr.direction = d; sr.frontier = F; sr.frontier_edges = MF;
            sr.discovered = 0; sr.inspected_edges = d == 1 ? MF : 0;
            // bytes over the interconnect: push = 8 B per shipped pair (filled
            // at the next level); pull = every rank's shard to every other rank
            sr.aux = d == 2 ? (int64_t)(A.nranks - 1) * A.nranks * (A.block / 8) : 0;
            sr.ns = 0;
        }
        if (tid == 0) {
            Slot &rst = a.ctl->slot[(L + 2) & 3];
            rst.qpack = 0; rst.ndisc = 0; rst.fpack = 0; rst.work = 0; rst.insp = 0; rst.dmax = 0; rst.pad[0] = 0;
        }
        Slot &nxt = a.ctl->slot[(L + 1) & 3];
        app.qv = a.qv[(L + 1) & 1];
        app.qo = a.qo[(L + 1) & 1];
        app.qr = a.qr[(L + 1) & 1];
        app.counter = &nxt.qpack;
        app.dmax = &nxt.dmax;
        uint32_t *fb_c = a.fb[L % 3];
        uint32_t *fb_n = a.fb[(L + 1) % 3];
        uint32_t *fb_z = a.fb[(L + 2) % 3];
        // keep the frontier bitmap of level L+1 only when a pull step is plausible soon
        const bool need_fb = d == 2 || MF >= gwords / 4;
        if (need_fb)
            for (int64_t w = tid; w < nwl; w += nthreads) fb_z[w] = 0u;
        unsigned long long ndisc = 0, insp = 0, shipped = 0;
        if (d == 1) {
            if (!q_valid) {  // the last pull step left its frontier as a bitmap only
                Appender conv = app;
                conv.qv = a.qv[L & 1]; conv.qo = a.qo[L & 1]; conv.qr = a.qr[L & 1];
                conv.counter = &a.ctl->slot[L & 3].fpack;
                conv.dmax = nullptr;
                conv.cnt = 0;
                conv.Rl = nullptr;
                bitmap_to_queue(view, fb_c, gw, nw, conv);
                grid.sync();
                q_valid = true;
            }
            PPushOp op{&a, fbn_clean ? fb_n : nullptr, L + 1, &app, A.block, A.inbox_cap, A.off_inbox,
                       (m_u * 4 < M * 3) ? 1 : 0, pol_keep, 0ull, 0ull};
            GlobalFrontier fr{a.qv[L & 1], a.qo[L & 1], a.qr[L & 1], f_loc, mf_loc};
            expand_lb(fr, a.C, gw, nw, op, A.lb_chunks > 0 ? &a.ctl->slot[L & 3].work : nullptr, A.lb_chunks);
            app.finish_cta(sm.wsum);
            ndisc = op.ndisc;
            shipped = op.shipped;
            if (A.nranks > 1) {
                gbar();  // every pair of this level is in its owner's inbox
                if (threadIdx.x == 0) sm.ctl[9] = __ldcg(&hdr(a.rank)->inbox_count);
                __syncthreads();
                unsigned long long iend = sm.ctl[9];
                if ((int64_t)iend > A.inbox_cap) iend = (unsigned long long)A.inbox_cap;
                // absorb: the owner claims what the other ranks discovered
                for (int64_t base = (int64_t)istart + gw * 32; base < (int64_t)iend; base += nw * 32) {
                    const int64_t j = base + lane_id();
                    bool disc = false;
                    int64_t lw = 0, deg = 0, rs = 0;
                    if (j < (int64_t)iend) {
                        const int2 pr = __ldcg(inbox + j);
                        lw = (int64_t)pr.x - a.v_begin;
                        if (lw < 0 || lw >= a.n_local) {
                            atomicExch(&a.ctl->overflow, 2ull);  // misrouted pair
                        } else {
                            const uint32_t bit = 1u << (lw & 31);
                            disc = !(atomicOr(a.visited + (lw >> 5), bit) & bit);
                            if (disc) {
                                a.depth[lw] = L + 1;
                                if (a.pred) a.pred[lw] = pr.y;
                                if (fbn_clean) atomicOr(fb_n + (lw >> 5), bit);  // RED.OR
                                ++ndisc;
                            }
                        }
                    }
                    app.push(disc, (int32_t)lw, deg, rs);  // lazy appender: R at the flush
                }
                app.finish_cta(sm.wsum);
                istart = iend;
            }
            fb_valid = fbn_clean;
        } else {
            if (!fb_valid) {  // queue -> bitmap
                for (int64_t w = tid; w < nwl; w += nthreads) fb_c[w] = 0u;
                grid.sync();
                const int32_t *qc = a.qv[L & 1];
                for (int64_t j = tid; j < f_loc; j += nthreads) {
                    const int32_t v = qc[j];
                    atomicOr(fb_c + (v >> 5), 1u << (v & 31));
                }
                grid.sync();
            }
            if (!fbn_clean)  // RED.OR targets must start at zero (ordered by the barrier below)
                for (int64_t w = tid; w < nwl; w += nthreads) fb_n[w] = 0u;
            // all-gather of the frontier shards with peer stores: my words go to
            // word rank*block/32 of every rank's global bitmap of this parity
            const int64_t w0 = (int64_t)a.rank * (A.block / 32);
            for (int q = 0; q < A.nranks; ++q) {
                uint32_t *dst = reinterpret_cast<uint32_t *>(a.sym[q] + A.off_gfront[par]) + w0;
                for (int64_t w = tid; w < nwl; w += nthreads) dst[w] = __ldcg(fb_c + w);
            }
            gbar();
            PullCounts pc;
            pull_level(view, gfront_own[par], fb_n, L + 1, &sm.work, sm.u.plist[wib], pc, 0u, 0,
                       nwl * bid / A.ctas, nwl * (bid + 1) / A.ctas);
            ndisc = pc.ndisc;
            insp = pc.insp;
            const unsigned long long qc = warp_sum<unsigned long long>(pc.qcnt);
            const unsigned long long qe = warp_sum<unsigned long long>(pc.qedges);
            const unsigned dm = __reduce_max_sync(0xffffffffu, pc.dmax);
            if (lane_id() == 0) {
                if (qc) atomicAdd(&sm.bsum[4], (qe << a.S) | qc);
                if (dm) atomicMax(&sm.bsum[5], (unsigned long long)dm);
            }
            fb_valid = true;
            q_valid = false;
        }
        ndisc = warp_sum<unsigned long long>(ndisc);
        insp = warp_sum<unsigned long long>(insp);
        shipped = warp_sum<unsigned long long>(shipped);
        if (lane_id() == 0) {
            if (ndisc) atomicAdd(&sm.bsum[0], ndisc);
            if (insp) atomicAdd(&sm.bsum[1], insp);
            if (shipped) atomicAdd(&sm.bsum[2], shipped);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (sm.bsum[0]) atomicAdd(&nxt.ndisc, sm.bsum[0]);
            if (sm.bsum[1]) atomicAdd(&nxt.insp, sm.bsum[1]);
            if (sm.bsum[2]) atomicAdd(&nxt.pad[0], sm.bsum[2]);
            if (sm.bsum[4]) atomicAdd(&nxt.qpack, sm.bsum[4]);
            if (sm.bsum[5]) atomicMax(&nxt.dmax, sm.bsum[5]);
        }
        grid.sync();  // this rank's counters of level L+1 are final
        unsigned long long vals[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (lead) {
            const unsigned long long qp = ld_relaxed(&nxt.qpack);
            vals[kStF] = qp & cmask;
            vals[kStMf] = qp >> a.S;
            vals[kStDisc] = ld_relaxed(&nxt.ndisc);
            vals[kStOvf] = ld_relaxed(&a.ctl->overflow);
            vals[kStInsp] = ld_relaxed(&nxt.insp);
            vals[kStShip] = ld_relaxed(&nxt.pad[0]);
            vals[kStDmax] = ld_relaxed(&nxt.dmax);
        }
        publish((L + 1) & 1, vals);
        prev_f = F;
        dir = d;
        fbn_clean = need_fb;
        ++L;
    }
    if (lead) {
        a.ctl->levels = (unsigned long long)L;
        a.ctl->epoch = rs.ep;
        if (a.ctl->overflow) a.ctl->sticky = 1ull;
    }
}

// ---------------------------------------------------------------- host side

static void fill_rank(Graph *g, PRank &r, int32_t *depth, int32_t *pred) {
    r.rank = g->comm->rank;
    r.S = g->pack_shift;
    r.n_local = g->n; r.v_begin = g->v_begin; r.m_local = g->m; r.nonisolated = g->nonisolated;
    r.R = g->R; r.C = g->C; r.Cp = g->Ct; r.ph = g->ph;
    r.visited = g->visited; r.noin = g->noin; r.sent = g->sent;
    for (int i = 0; i < 3; ++i) r.fb[i] = g->fbuf[i];
    for (int i = 0; i < 2; ++i) { r.qv[i] = g->qv[i]; r.qo[i] = g->qo[i]; r.qr[i] = g->qr[i]; }
    r.depth = depth; r.pred = pred;
    r.ctl = g->ctl; r.stats = g->stats_dev;
    for (int q = 0; q < kMaxRanks; ++q) r.sym[q] = g->sym_peer[q];
}

__global__ void pdeg_kernel(const int64_t *R, int64_t n, int64_t block, int32_t *deg) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < block; v += nt) {
        const int64_t d = v < n ? R[v + 1] - R[v] : 0;
        deg[v] = (int32_t)(d > 0x7fffffffll ? 0x7fffffffll : d);
    }
}

// Pull lists ordered by the GLOBAL degree of the neighbour (descending), so
// bottom-up scans exit early as on one GPU (a7); needs every rank's degrees:
// an NCCL all-gather for real ranks, device copies inside a loopback group.
static gr_status order_pull_lists(Graph **gs, int k, const int32_t *deg_global) {
    for (int i = 0; i < k; ++i) {
        Graph *g = gs[i];
        if (g->m == 0 || g->m >= (1ll << 31)) continue;  // segmented sort limit: keep the caller's order
        if (g->Ct == g->C) {
            gr_status st = dev_alloc(g, (void **)&g->Ct, g->m * sizeof(int32_t));
            if (st != GR_OK) { g->Ct = g->C; return st; }
            GR_CUDA(cudaMemcpyAsync(g->Ct, g->C, g->m * sizeof(int32_t), cudaMemcpyDeviceToDevice, g->stream));
        }
        gr_status st = sort_lists_by_degree(g, g->stream, g->num_sms * 4, deg_global);
        if (st != GR_OK) return st;
    }
    return GR_OK;
}

gr_status prepare_real(Graph *g) {
    Comm *c = g->comm;
    int32_t *deg = nullptr;
    const size_t per = (size_t)g->block * sizeof(int32_t);
    GR_CUDA(cudaMalloc((void **)&deg, per * (c->nranks + 1)));
    pdeg_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(g->R, g->n, g->block, deg);
    count_launch();
    gr_status st = comm_allgather_bytes(c, deg, deg + g->block, per, g->stream);
    if (st == GR_OK) {  // global totals: m, max weight, non-isolated vertices
        long long mine[3] = {(long long)g->m, (long long)g->max_w, (long long)g->nonisolated};
        long long *d3 = nullptr;
        GR_CUDA(cudaMalloc((void **)&d3, sizeof(mine) * (c->nranks + 1)));
        GR_CUDA(cudaMemcpy(d3, mine, sizeof(mine), cudaMemcpyHostToDevice));
        st = comm_allgather_bytes(c, d3, d3 + 3, sizeof(mine), g->stream);
        long long all[3 * kMaxRanks];
        if (st == GR_OK) GR_CUDA(cudaMemcpy(all, d3 + 3, sizeof(mine) * c->nranks, cudaMemcpyDeviceToHost));
        cudaFree(d3);
        g->m_global = 0; g->maxw_global = 0; g->nonisolated_global = 0;
        for (int q = 0; q < c->nranks && st == GR_OK; ++q) {
            g->m_global += all[3 * q];
            g->maxw_global = all[3 * q + 1] > (long long)g->maxw_global ? (uint32_t)all[3 * q + 1] : g->maxw_global;
            g->nonisolated_global += all[3 * q + 2];
        }
    }
    if (st == GR_OK && !(g->flags_keep_order)) st = order_pull_lists(&g, 1, deg + g->block);
    if (st == GR_OK) st = build_pull_head(g);
    cudaStreamSynchronize(g->stream);
    cudaFree(deg);
    if (st == GR_OK) g->prepared = true;
    return st;
}

gr_status prepare_loopback(LoopGroup *grp) {
    Graph *g0 = grp->graphs[0];
    const int P = grp->P;
    int64_t mg = 0, nig = 0;
    uint32_t mw = 0;
    for (int q = 0; q < P; ++q) {
        mg += grp->graphs[q]->m;
        nig += grp->graphs[q]->nonisolated;
        mw = grp->graphs[q]->max_w > mw ? grp->graphs[q]->max_w : mw;
    }
    for (int r = 0; r < P; ++r) {
        for (int q = 0; q < P; ++q) grp->graphs[r]->sym_peer[q] = grp->graphs[q]->sym;
        grp->graphs[r]->m_global = mg;
        grp->graphs[r]->nonisolated_global = nig;
        grp->graphs[r]->maxw_global = mw;
    }
    int32_t *deg = nullptr;
    GR_CUDA(cudaMalloc((void **)&deg, (size_t)g0->block * P * sizeof(int32_t)));
    for (int q = 0; q < P; ++q) {
        Graph *g = grp->graphs[q];
        pdeg_kernel<<<g->num_sms * 4, 256, 0, g0->stream>>>(g->R, g->n, g->block, deg + (size_t)q * g->block);
        count_launch();
    }
    GR_CUDA(cudaStreamSynchronize(g0->stream));
    gr_status st = GR_OK;
    if (!g0->flags_keep_order) st = order_pull_lists(grp->graphs, P, deg);
    for (int r = 0; r < P && st == GR_OK; ++r) st = build_pull_head(grp->graphs[r]);
    cudaDeviceSynchronize();
    cudaFree(deg);
    if (st == GR_OK)
        for (int r = 0; r < P; ++r) grp->graphs[r]->prepared = true;
    return st;
}

// One collective BFS: the `k` ranks of gs (one real rank, or a whole loopback
// group) in one cooperative launch on gs[0]'s stream.
static gr_status launch_pbfs(Graph **gs, int k, int64_t src, int32_t **depth, int32_t **pred, const gr_bfs_opts &o) {
    Graph *g0 = gs[0];
    Comm *c = g0->comm;
    const SymLayout Ly = sym_layout(c->nranks, g0->block, g0->has_w && g0->W);
    PBfsArgs A;
    memset(&A, 0, sizeof(A));
    for (int i = 0; i < k; ++i) fill_rank(gs[i], A.ranks[i], depth[i], pred[i]);
    A.vranks = k;
    A.nranks = c->nranks;
    A.multiproc = (c->group == nullptr && c->nranks > 1) ? 1 : 0;
    A.n_global = g0->n_global;
    A.block = g0->block;
    A.src = src;
    A.off_gfront[0] = Ly.gfront[0];
    A.off_gfront[1] = Ly.gfront[1];
    A.off_inbox = Ly.inbox;
    A.inbox_cap = Ly.inbox_cap;
    A.direction = o.direction;
    A.switch_rule = o.switch_rule;
    A.alpha = o.alpha > 0 ? o.alpha : (double)env_int("GR_PALPHA", 14);
    A.beta = o.beta > 0 ? o.beta : 24.0;
    A.lb_chunks = (int32_t)env_int("GR_LB_CHUNKS", 4);
    const void *fn = (const void *)pbfs_kernel<kPBlock, kPMinB>;
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPBlock, 0));
    if (per_sm < 1) { set_error("pbfs_kernel cannot be resident"); return GR_ERR_CUDA; }
    if (per_sm > kPMinB) per_sm = kPMinB;
    const int64_t total = (int64_t)g0->num_sms * per_sm;
    A.ctas = (int32_t)(total / k);
    if (A.ctas < 1) { set_error("too many ranks for one GPU"); return GR_ERR_INVALID_ARGUMENT; }
    dim3 grid((unsigned)(A.ctas * k)), blk(kPBlock);
    void *args[] = {(void *)&A};
    GR_CUDA(cudaLaunchCooperativeKernel(fn, grid, blk, args, 0, g0->stream));
    count_launch();
    return GR_OK;
}

static gr_status finish_pbfs(Graph *g) {
    unsigned long long levels = 0, overflow = 0;
    GR_CUDA(cudaMemcpyAsync(&levels, &g->ctl->levels, sizeof(levels), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemcpyAsync(&overflow, &g->ctl->overflow, sizeof(overflow), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemsetAsync(&g->ctl->sticky, 0, sizeof(unsigned long long), g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    g->stats_levels = (int)levels;
    g->stats_records = (int)(levels < (unsigned long long)kMaxStatRecords ? levels : kMaxStatRecords);
    g->stats_records = -1 - g->stats_records;
    g->last_launches = 1;
    g->last_delta = 0;
    g->last_kind = 1;
    g->reached = -2;
    if (overflow == 3) { set_error("partitioned BFS: a peer rank did not reach a barrier within 20 s"); return GR_ERR_NCCL; }
    if (overflow == 2) { set_error("partitioned BFS: received a vertex this rank does not own"); return GR_ERR_OVERFLOW; }
    if (overflow) { set_error("partitioned BFS: a queue exceeded its capacity"); return GR_ERR_OVERFLOW; }
    return GR_OK;
}

// gr_bfs on a partitioned graph: collective over the comm's ranks.
gr_status pbfs_collective(Graph *g, int64_t src, int32_t *depth_out, int32_t *pred_out, const gr_bfs_opts &o) {
    Comm *c = g->comm;
    GR_CUDA(cudaSetDevice(g->device));
    const bool dev_d = ptr_on_device(depth_out);
    const bool dev_p = pred_out && ptr_on_device(pred_out);
    auto stage = [&](Graph *x, int32_t *dout, int32_t *pout, bool dd, bool dp, int32_t **d, int32_t **p) -> gr_status {
        *d = dout;
        *p = pout;
        if (!dd) {
            if (!x->depth_buf) { gr_status st = dev_alloc(x, (void **)&x->depth_buf, x->n * 4); if (st != GR_OK) return st; }
            *d = x->depth_buf;
        }
        if (pout && !dp) {
            if (!x->pred_buf) { gr_status st = dev_alloc(x, (void **)&x->pred_buf, x->n * 4); if (st != GR_OK) return st; }
            *p = x->pred_buf;
        }
        return GR_OK;
    };
    auto copy_back = [&](Graph *x, int32_t *dout, int32_t *pout, int32_t *d, int32_t *p) -> gr_status {
        if (d != dout) GR_CUDA(cudaMemcpyAsync(dout, d, x->n * 4, cudaMemcpyDeviceToHost, x->stream));
        if (pout && p != pout) GR_CUDA(cudaMemcpyAsync(pout, p, x->n * 4, cudaMemcpyDeviceToHost, x->stream));
        GR_CUDA(cudaStreamSynchronize(x->stream));
        return GR_OK;
    };
    gr_status st;
    if (!c->group) {  // a real rank: every rank of the comm makes this call
        if (!g->prepared && (st = prepare_real(g)) != GR_OK) return st;
        int32_t *d, *p;
        if ((st = stage(g, depth_out, pred_out, dev_d, dev_p, &d, &p)) != GR_OK) return st;
        Graph *gs[1] = {g};
        if ((st = launch_pbfs(gs, 1, src, &d, &p, o)) != GR_OK) return st;
        g->last_src = (int32_t)(src - g->v_begin);
        if ((st = finish_pbfs(g)) != GR_OK) return st;
        return copy_back(g, depth_out, pred_out, d, p);
    }
    // loopback: the call of the group's last rank launches every rank
    LoopGroup *grp = c->group;
    if (grp->joined == 0) { grp->kind = 1; grp->src = src; grp->bopts = o; }
    else if (grp->kind != 1 || grp->src != src) {
        grp->joined = 0;
        set_error("loopback collective mismatch: every rank must call gr_bfs with the same source");
        return GR_ERR_INVALID_ARGUMENT;
    }
    grp->out0[c->rank] = depth_out;
    grp->out1[c->rank] = pred_out;
    grp->joined |= 1 << c->rank;
    if (grp->joined != (1 << grp->P) - 1) return GR_OK;
    grp->joined = 0;
    for (int r = 0; r < grp->P; ++r)
        if (!grp->graphs[r]) { set_error("loopback rank %d has no partitioned graph", r); return GR_ERR_INVALID_ARGUMENT; }
    if (!g->prepared && (st = prepare_loopback(grp)) != GR_OK) return st;
    int32_t *d[kMaxRanks], *p[kMaxRanks];
    for (int r = 0; r < grp->P; ++r) {
        int32_t *dout = (int32_t *)grp->out0[r], *pout = (int32_t *)grp->out1[r];
        if ((st = stage(grp->graphs[r], dout, pout, ptr_on_device(dout), pout && ptr_on_device(pout), &d[r], &p[r])) != GR_OK)
            return st;
    }
    Graph *g0 = grp->graphs[0];
    GR_CUDA(cudaStreamSynchronize(g->stream));  // the caller's work on its stream precedes the launch
    if ((st = launch_pbfs(grp->graphs, grp->P, src, d, p, grp->bopts)) != GR_OK) return st;
    GR_CUDA(cudaStreamSynchronize(g0->stream));
    gr_status first = GR_OK;
    for (int r = 0; r < grp->P; ++r) {
        Graph *x = grp->graphs[r];
        x->last_src = (int32_t)(src - x->v_begin);
        st = finish_pbfs(x);
        if (st != GR_OK && first == GR_OK) first = st;
        st = copy_back(x, (int32_t *)grp->out0[r], (int32_t *)grp->out1[r], d[r], p[r]);
        if (st != GR_OK && first == GR_OK) first = st;
    }
    return first;
}

}  // namespace gr

using namespace gr;

extern "C" {

gr_status gr_graph_create_partitioned(gr_comm *ch, int64_t n_global, int64_t v_begin, int64_t v_end, int64_t m_local,
                                      const int64_t *row_offsets, const int32_t *col_indices,
                                      const uint32_t *weights, uint32_t flags, void *cuda_stream, gr_graph **out) {
    Comm *c = (Comm *)ch;
    if (!c || !out || n_global < 1 || n_global > 0x7fffffffll) {
        set_error("invalid gr_graph_create_partitioned arguments");
        return GR_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    const int P = c->nranks;
    const int64_t block = 32 * ((n_global + 32 * (int64_t)P - 1) / (32 * (int64_t)P));
    const int64_t vb = (int64_t)c->rank * block, ve = vb + block < n_global ? vb + block : n_global;
    if (v_begin != vb || v_end != ve || ve <= vb) {
        set_error("rank %d of %d must own [%lld, %lld), got [%lld, %lld)", c->rank, P, (long long)vb, (long long)ve,
                  (long long)v_begin, (long long)v_end);
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (!(flags & GR_SYMMETRIC)) {
        set_error("a partitioned graph must be symmetric (GR_SYMMETRIC): its out-lists are the pull steps' in-lists");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (c->group && c->group->graphs[c->rank]) {
        set_error("loopback rank %d already has a partitioned graph", c->rank);
        return GR_ERR_INVALID_ARGUMENT;
    }
    Graph *g = nullptr;
    gr_status st = graph_create(v_end - v_begin, m_local, row_offsets, col_indices, weights,
                                flags | GR_KEEP_ORDER, c->device, cuda_stream, &g, n_global);
    if (st != GR_OK) return st;
    g->comm = c;
    g->part = true;
    g->n_global = n_global; g->v_begin = v_begin; g->v_end = v_end; g->block = block;
    g->nparts = P; g->rank = c->rank;
    g->has_w = weights != nullptr || m_local == 0;
    g->flags_keep_order = (flags & GR_KEEP_ORDER) != 0;
    const SymLayout Ly = sym_layout(P, block, weights != nullptr && m_local > 0);
    if ((st = dev_alloc(g, (void **)&g->sent, ((n_global + 31) / 32) * sizeof(uint32_t))) != GR_OK ||
        (st = comm_sym_alloc(c, g, Ly.bytes)) != GR_OK) {
        comm_sym_free(g);
        dev_free_all(g);
        delete g;
        return st;
    }
    if (c->group) c->group->graphs[c->rank] = g;
    *out = (gr_graph *)g;
    return GR_OK;
}

}  // extern "C"
