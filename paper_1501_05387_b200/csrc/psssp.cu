// psssp.cu -- delta-stepping SSSP over a 1D vertex partition as ONE
// persistent kernel per rank (SURVEY §8(b) gr_sssp on a partitioned graph,
// §8(e), §8(f) f2). The paper's SSSP is single-GPU (Alg. 1; the
// near/far priority queue P:838-857 implemented "as an additional filter pass
// between two iterations" P:941-942; multi-GPU is future work P:1383-1396).
// Per partition the step structure and readings are the single-GPU ones
// (sssp.cu: A-7 slice-keyed stamp, A-9 packed dist|pred atomicMin, A-11 far
// pile maintenance); reading A-21 adds one exchange per near iteration, done
// inside the kernel over peer memory:
//
//  near step   relax the owned near queue; an owned target is relaxed here;
//              a remote target lowers this rank's "best shipped" value of the
//              vertex (packed atomicMin) and a strict improvement puts the
//              vertex once per step on this rank's ship list -> (grid
//              barrier: every improvement of the step is in `best`) -> each
//              shipped vertex's FINAL best value goes into its owner's inbox
//              of this step parity as a (vertex, dist, parent) record (slots
//              reserved by a system-scope atomicAdd on the owner's counter,
//              warp-aggregated per owner) -> group barrier -> the owner relaxes
//              its inbox records (same stamp / near-far filter);
//  re-split    (the near queue is empty on every rank) each rank's minimum far
//              distance >= threshold is published -> barrier -> every rank
//              takes the global minimum, jumps the threshold to its band and
//              splits its far pile (stale entries dropped);
//  every step  (near count, its edges, far count, overflow, improvements) of
//              every rank are published into every rank's table -> barrier ->
//              every rank takes the same decision (relax / re-split / stop).
// Culling by "best shipped" is exact: the owner's dist never exceeds a value
// shipped to it, so a candidate that does not beat this rank's best cannot
// improve the owner's label.
#include "part.cuh"
#include "frontier.cuh"

namespace gr {

bool ptr_on_device(const void *p);
gr_status prepare_real(Graph *g);
gr_status prepare_loopback(LoopGroup *grp);

constexpr int kPsCap = 64;   // near / far staging per warp
using PsApp = AppenderT<kPsCap>;

struct SRank {
    int32_t rank, S;
    int64_t n_local, v_begin;
    const int64_t *R;
    const int32_t *C;            // GLOBAL ids
    const uint32_t *W;
    const uint32_t *CW;          // packed (C << 7) | W, or null
    unsigned long long *dp;      // [n_local] (dist << 32) | global pred (A-9)
    int32_t *stamp;              // [n_local] RemoveRedundant stamp (A-7)
    unsigned long long *best;    // [n_global] best value shipped to the owner (A-21)
    int32_t *sstamp;             // [n_global] step of the last shipment
    int32_t *ship;               // [n_global] vertices shipped in the current step
    int32_t *qv[2];              // near queues (LOCAL ids)
    int64_t *qo[2];
    int64_t *qr[2];
    int32_t *far[2];             // far piles (LOCAL ids)
    int64_t far_cap;
    uint32_t *dist;              // outputs of the owned block
    int32_t *pred;
    Ctl *ctl;
    gr_level_stats *stats;
    char *sym[kMaxRanks];
};

struct PSsspArgs {
    SRank ranks[kMaxRanks];
    int32_t vranks, nranks, multiproc, ctas;
    int64_t n_global, block, src;
    uint64_t delta;
    size_t off_sinbox[2];
    int64_t inbox_cap;
};

// published counters of a step (RankSync table)
enum { kSsF = 0, kSsMf = 1, kSsFar = 2, kSsOvf = 3, kSsImp = 4, kSsShip = 5, kSsMin = 6, kSsPad = 7 };

// Owner-side relaxation of local vertex lv with candidate (nd, parent):
// UpdateLabel + SetPred (packed atomicMin, A-9), RemoveRedundant (A-7) and
// the near/far split. 1 near, 2 far, 0 nothing to append.
__device__ __forceinline__ int sp_relax(const SRank &a, int64_t lv, unsigned long long nd, uint32_t parent,
                                        uint64_t thr, int32_t key_near, unsigned long long cur) {
    if (nd >= (cur >> 32)) return 0;
    const unsigned long long old = atomicMin(a.dp + lv, (nd << 32) | parent);
    if (nd >= (old >> 32)) return 0;
    const bool far = nd >= thr;
    const int32_t key = stamp_key(key_near, far);
    if (atomicMax(a.stamp + lv, key) >= key) return 0;
    return far ? 2 : 1;
}

template <bool kPacked>  // kPacked: the edge stream is (C << 7) | W (graph.cu), 4 B per edge
struct PSRelaxOp {
    const SRank *a;
    uint64_t thr;
    int32_t key_near;   // 2 * it
    int32_t step;
    PsApp *nearq, *farq;
    unsigned long long *ship_count;
    unsigned long long pol, pol_stream;
    unsigned long long nimp;

    __device__ __forceinline__ unsigned long long entry(int32_t v) { return ld_probe(a->dp + v, pol) >> 32; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *du,
                                          const int32_t *dst, const T5 *x) {
        uint32_t w[U];
        int32_t vv[U];
        unsigned long long cur[U];
        // weight loads and pre-check probes of all U edges before any atomic
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (kPacked) {
                vv[u] = (int32_t)((uint32_t)dst[u] >> 7);
                w[u] = (uint32_t)dst[u] & 127u;
            } else {
                vv[u] = dst[u];
                w[u] = ok[u] ? ld_stream(a->W + x[u], pol_stream) : 0u;
            }
            const int64_t lv = (int64_t)vv[u] - a->v_begin;
            const bool owned = lv >= 0 && lv < a->n_local;
            cur[u] = ok[u] ? ld_probe(owned ? a->dp + lv : a->best + vv[u], pol) : 0ull;
        }
        // UpdateLabel (owned: dp, remote: best) of all U edges in flight, then
        // the stamps of the improved ones in flight, then the filter -- each
        // atomic consumed inside its own branch was a round trip apiece
        unsigned long long old[U];
        bool tr[U], own[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t lv = (int64_t)vv[u] - a->v_begin;
            own[u] = lv >= 0 && lv < a->n_local;
            const unsigned long long nd = du[u] + w[u];
            const uint32_t parent = (uint32_t)(a->v_begin + src[u]);
            tr[u] = ok[u] && nd < (cur[u] >> 32);
            old[u] = tr[u] ? atomicMin(own[u] ? a->dp + lv : a->best + vv[u], (nd << 32) | parent) : 0ull;
        }
        int32_t ex[U], key[U];
        bool imp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t lv = (int64_t)vv[u] - a->v_begin;
            const unsigned long long nd = du[u] + w[u];
            imp[u] = tr[u] && nd < (old[u] >> 32);
            key[u] = own[u] ? stamp_key(key_near, nd >= thr) : step;
            // owned: near/far stamp (atomicMax, stamp_key); remote: one shipment per step
            ex[u] = !imp[u] ? key[u] : own[u] ? atomicMax(a->stamp + lv, key[u]) : atomicExch(a->sstamp + vv[u], key[u]);
            if (imp[u] && own[u]) ++nimp;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t v = vv[u];
            const int64_t lv = (int64_t)v - a->v_begin;
            const bool first = imp[u] && (own[u] ? ex[u] < key[u] : ex[u] != key[u]);
            const bool far = du[u] + w[u] >= thr;
            const int kind = (first && own[u]) ? (far ? 2 : 1) : 0;
            const bool ship = first && !own[u];
            nearq->push(kind == 1, (int32_t)lv, 0, 0);  // lazy appender: R at the flush
            farq->push(kind == 2, (int32_t)lv, 0);
            const unsigned sm = __ballot_sync(0xffffffffu, ship);
            if (sm) {  // this step's ship list (one atomic per warp)
                unsigned long long base = 0;
                if (lane_id() == 0) base = atomicAdd(ship_count, (unsigned long long)__popc(sm));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (ship) a->ship[base + __popc(sm & lanemask_lt())] = v;
            }
        }
    }
};

template <int kNW>
struct SSmem {
    int32_t sv[kNW][kPsCap];
    int32_t sd[kNW][kPsCap];
    int64_t sr[kNW][kPsCap];
    int32_t fv[kNW][kPsCap];
    SRank r;
    unsigned long long wsum[2 * kNW + 2];
    unsigned long long ctl[16];
    unsigned long long bsum[4];
};

constexpr int kSBlock = 512;
constexpr int kSMinB = 2;

template <int kBlk, int kMinB, bool kPacked>
__global__ void __launch_bounds__(kBlk, kMinB) psssp_kernel(const __grid_constant__ PSsspArgs A) {
    constexpr int kNW = kBlk / kWarp;
    __shared__ SSmem<kNW> sm;
    cg::grid_group grid = cg::this_grid();
    const int vr = blockIdx.x / A.ctas;
    const int bid = blockIdx.x - vr * A.ctas;
    if (threadIdx.x == 0) sm.r = A.ranks[vr];
    __syncthreads();
    const SRank &a = sm.r;
    const int64_t tid = (int64_t)bid * kBlk + threadIdx.x;
    const int64_t nthreads = (int64_t)A.ctas * kBlk;
    const int64_t gw = tid >> 5, nw = nthreads >> 5;
    const int wib = threadIdx.x >> 5;
    const unsigned long long cmask = (1ull << a.S) - 1;
    const bool lead = bid == 0 && threadIdx.x == 0;
    RankSync rs{&grid, a.sym, a.rank, A.nranks, A.multiproc, bid, a.ctl, a.ctl->epoch};

    // ---- Set_Problem_Data ------------------------------------
    for (int64_t v = tid; v < a.n_local; v += nthreads) {
        a.dp[v] = ~0ull;   // dist = UINT32_MAX, pred = -1 (A-2)
        a.stamp[v] = -1;
    }
    for (int64_t v = tid; v < A.n_global; v += nthreads) {
        a.best[v] = ~0ull;
        a.sstamp[v] = -1;
    }
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (lead) {
        a.ctl->overflow = 0ull;
        a.ctl->far_count[0] = 0ull;
        a.ctl->far_count[1] = 0ull;
        a.ctl->reached = 0ull;  // ship-list length of the current step
        rs.hdr(a.rank)->sin_count[0] = 0ull;
        rs.hdr(a.rank)->sin_count[1] = 0ull;
    }
    rs.bar();  // every rank is in this run
    {
        unsigned long long vals[8] = {0, 0, 0, 0, 0, 0, ~0ull, 0};
        if (tid < kSlots) a.ctl->slot[tid].minfar = ~0ull;
        if (lead) {
            const int64_t ls = A.src - a.v_begin;
            if (ls >= 0 && ls < a.n_local) {
                a.dp[ls] = (unsigned long long)(uint32_t)A.src;  // dist 0, pred = src (A-1, global id)
                const int64_t d = a.R[ls + 1] - a.R[ls];
                if (d > 0) {
                    a.qv[0][0] = (int32_t)ls;
                    a.qo[0][0] = 0;
                    a.qr[0][0] = a.R[ls];
                    a.ctl->slot[0].qpack = ((unsigned long long)d << a.S) | 1ull;
                    vals[kSsF] = 1;
                    vals[kSsMf] = (unsigned long long)d;
                }
            }
        }
        __syncthreads();
        rs.publish(0, vals);
    }

    PsApp nearq, farq;
    nearq.sv = sm.sv[wib]; nearq.sd = sm.sd[wib]; nearq.sr = sm.sr[wib]; nearq.cnt = 0; nearq.S = a.S;
    nearq.cap = 2 * a.n_local;
    nearq.Rl = a.R;  // lazy: every near id is local; row offsets loaded at the flush
    nearq.overflow = &a.ctl->overflow;
    farq.sv = sm.fv[wib]; farq.sd = nullptr; farq.sr = nullptr; farq.cnt = 0; farq.S = 0;
    farq.qo = nullptr; farq.qr = nullptr;
    farq.cap = a.far_cap;
    farq.overflow = &a.ctl->overflow;
    const unsigned long long pol = policy_evict_last(), pol_stream = policy_evict_first();

    uint64_t thr = A.delta;  // near band is [.., thr)
    int32_t it = 0;          // stamp iteration (keys 2*it, 2*it+1)
    int fp = 0;              // current far pile
    int par = 0;             // parity of the last published table
    long long t_prev = lead ? pgtimer() : 0;
    int k = 0;
    for (;; ++k) {
        Slot &cur = a.ctl->slot[k & 3];
        Slot &nxt = a.ctl->slot[(k + 1) & 3];
        if (threadIdx.x == 0) {
            unsigned long long t[8];
            rs.read(par, t, -1, kSsOvf, kSsMin);
            for (int i = 0; i < 8; ++i) sm.ctl[i] = t[i];
            sm.ctl[8] = ld_relaxed(&cur.qpack);
            sm.ctl[9] = ld_relaxed(&a.ctl->far_count[fp]);
            sm.bsum[0] = 0;
            sm.bsum[1] = ~0ull;
        }
        __syncthreads();
        const int64_t F = (int64_t)sm.ctl[kSsF], MF = (int64_t)sm.ctl[kSsMf], FAR = (int64_t)sm.ctl[kSsFar];
        const int64_t f_loc = (int64_t)(sm.ctl[8] & cmask), mf_loc = (int64_t)(sm.ctl[8] >> a.S);
        const int64_t fc_loc = (int64_t)sm.ctl[9];
        if (k > 0 && lead && k - 1 < kMaxStatRecords) {
            a.stats[k - 1].discovered = (int64_t)sm.ctl[kSsImp];
            a.stats[k - 1].aux = 16 * (int64_t)sm.ctl[kSsShip];  // bytes of (vertex, dist, parent) records sent
            const long long tn = pgtimer();
            a.stats[k - 1].ns = tn - t_prev;
            t_prev = tn;
        }
        const bool stop = sm.ctl[kSsOvf] != 0 || (F == 0 && FAR == 0);
        __syncthreads();
        if (stop) break;
        if (lead) {
            Slot &rst = a.ctl->slot[(k + 2) & 3];
            rst.qpack = 0; rst.ndisc = 0; rst.fpack = 0; rst.work = 0; rst.minfar = ~0ull; rst.insp = 0;
            rst.dmax = 0;
            if (k < kMaxStatRecords) {
                gr_level_stats &st = a.stats[k];
                st.level = k; st.direction = F > 0 ? 3 : 4; st.frontier = F > 0 ? F : FAR;
                st.frontier_edges = MF; st.discovered = 0; st.inspected_edges = MF; st.aux = 0; st.ns = 0;
            }
        }
        nearq.qv = a.qv[(k + 1) & 1];
        nearq.qo = a.qo[(k + 1) & 1];
        nearq.qr = a.qr[(k + 1) & 1];
        nearq.counter = &nxt.qpack;
        nearq.dmax = &nxt.dmax;
        unsigned long long nimp = 0;
        int64_t nship = 0;
        if (F > 0) {
            // ---- near iteration: Advance(UpdateLabel, SetPred) + Filter --------
            ++it;
            farq.qv = a.far[fp];
            farq.counter = &a.ctl->far_count[fp];
            PSRelaxOp<kPacked> op{&a, thr, 2 * it, k, &nearq, &farq, &a.ctl->reached, pol, pol_stream, 0ull};
            GlobalFrontier fr{a.qv[k & 1], a.qo[k & 1], a.qr[k & 1], f_loc, mf_loc};
            expand_lb(fr, kPacked ? reinterpret_cast<const int32_t *>(a.CW) : a.C, gw, nw, op, &cur.work, 4);
            nimp = op.nimp;
            nearq.finish_cta(sm.wsum);
            farq.finish_cta(sm.wsum);
            if (A.nranks > 1) {
                grid.sync();  // every improvement of the step is in `best`, the ship list is complete
                if (threadIdx.x == 0) sm.ctl[10] = ld_relaxed(&a.ctl->reached);
                __syncthreads();
                const int64_t ns = (int64_t)sm.ctl[10];
                nship = ns;
                // the FINAL best value of each shipped vertex into its owner's inbox
                for (int64_t base = gw * 32; base < ns; base += nw * 32) {
                    const int64_t j = base + lane_id();
                    const bool has = j < ns;
                    const int32_t v = has ? a.ship[j] : 0;
                    const int q = has ? (int)((int64_t)v / A.block) : -1;
                    const unsigned peers = __match_any_sync(0xffffffffu, q);
                    if (has) {
                        const int leader = __ffs(peers) - 1;
                        unsigned long long pos = 0;
                        if ((int)lane_id() == leader)
                            pos = atomicAdd_system(&rs.hdr(q)->sin_count[k & 1], (unsigned long long)__popc(peers));
                        pos = __shfl_sync(peers, pos, leader) + __popc(peers & lanemask_lt());
                        if ((int64_t)pos < A.inbox_cap) {
                            const unsigned long long b = __ldcg(a.best + v);
                            int4 *ib = reinterpret_cast<int4 *>(a.sym[q] + A.off_sinbox[k & 1]);
                            ib[pos] = make_int4(v, (int32_t)(uint32_t)(b >> 32), (int32_t)(uint32_t)b, 0);
                        } else {
                            atomicExch(&a.ctl->overflow, 1ull);
                        }
                    }
                }
                rs.bar();  // every record of this step is in its owner's inbox
                if (threadIdx.x == 0) sm.ctl[11] = __ldcg(&rs.hdr(a.rank)->sin_count[k & 1]);
                __syncthreads();
                int64_t nrecv = (int64_t)sm.ctl[11];
                if (nrecv > A.inbox_cap) nrecv = A.inbox_cap;
                const int4 *ib = reinterpret_cast<const int4 *>(a.sym[a.rank] + A.off_sinbox[k & 1]);
                for (int64_t base = gw * 32; base < nrecv; base += nw * 32) {
                    const int64_t j = base + lane_id();
                    int kind = 0;
                    int64_t lv = 0, deg = 0, rs0 = 0;
                    if (j < nrecv) {
                        const int4 t = __ldcg(ib + j);
                        lv = (int64_t)t.x - a.v_begin;
                        if (lv < 0 || lv >= a.n_local) {
                            atomicExch(&a.ctl->overflow, 2ull);  // misrouted record
                        } else {
                            kind = sp_relax(a, lv, (unsigned long long)(uint32_t)t.y, (uint32_t)t.z, thr, 2 * it,
                                            ld_probe(a.dp + lv, pol));
                            if (kind) ++nimp;

                        }
                    }
                    nearq.push(kind == 1, (int32_t)lv, deg, rs0);  // lazy: R at the flush
                    farq.push(kind == 2, (int32_t)lv, 0);
                }
                nearq.finish_cta(sm.wsum);
                farq.finish_cta(sm.wsum);
                if (lead) a.ctl->reached = 0ull;  // ship list of the next step
            }
        } else {
            // ---- near slice exhausted everywhere: "update the priority function
            // and operate on the far slice". Re-split (A-11). -----
            const int32_t *far_c = a.far[fp];
            unsigned long long mymin = ~0ull;
            for (int64_t j = tid; j < fc_loc; j += nthreads) {
                const unsigned long long d = ld_probe(a.dp + far_c[j], pol) >> 32;
                if (d >= thr && d < mymin) mymin = d;
            }
            for (int sh = 16; sh > 0; sh >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, mymin, sh);
                mymin = o < mymin ? o : mymin;
            }
            if (lane_id() == 0 && mymin != ~0ull) atomicMin(&sm.bsum[1], mymin);
            __syncthreads();
            if (threadIdx.x == 0 && sm.bsum[1] != ~0ull) atomicMin(&cur.minfar, sm.bsum[1]);
            grid.sync();
            unsigned long long vals[8] = {0, 0, 0, 0, 0, 0, ~0ull, 0};
            if (lead) vals[kSsMin] = ld_relaxed(&cur.minfar);
            par ^= 1;
            rs.publish(par, vals);
            if (threadIdx.x == 0) {
                unsigned long long t[8];
                rs.read(par, t, -1, kSsOvf, kSsMin);
                sm.ctl[12] = t[kSsMin];
            }
            if (lead) a.ctl->far_count[fp] = 0ull;
            __syncthreads();
            const unsigned long long mn = sm.ctl[12];
            if (mn == ~0ull) break;  // every far entry of every rank was stale: done
            const uint64_t thr_old = thr;
            const uint64_t band = mn / A.delta + 1;
            thr = (band > (0xFFFFFFFFFFFFFFFFull / A.delta)) ? 0xFFFFFFFFFFFFFFFFull : band * A.delta;
            ++it;
            farq.qv = a.far[fp ^ 1];
            farq.counter = &a.ctl->far_count[fp ^ 1];
            for (int64_t base = gw * 32; base < fc_loc; base += nw * 32) {
                const int64_t j = base + lane_id();
                bool to_near = false, to_far = false;
                int32_t v = 0;
                int64_t deg = 0, rs0 = 0;
                if (j < fc_loc) {
                    v = far_c[j];
                    const unsigned long long d = ld_probe(a.dp + v, pol) >> 32;
                    if (d >= thr_old) {  // else stale: already expanded below thr_old
                        const bool nearb = d < thr;
                        const int32_t key = stamp_key(2 * it, !nearb);
                        if (atomicMax(a.stamp + v, key) < key) {
                            if (nearb) to_near = true;
                            else to_far = true;
                        }
                    }
                }
                nearq.push(to_near, v, deg, rs0);  // lazy: R at the flush
                farq.push(to_far, v, 0);
            }
            nearq.finish_cta(sm.wsum);
            farq.finish_cta(sm.wsum);
            fp ^= 1;
        }
        nimp = warp_sum<unsigned long long>(nimp);
        if (lane_id() == 0 && nimp) atomicAdd(&sm.bsum[0], nimp);
        __syncthreads();
        if (threadIdx.x == 0 && sm.bsum[0]) atomicAdd(&nxt.ndisc, sm.bsum[0]);
        grid.sync();  // this rank's counters of step k+1 are final
        unsigned long long vals[8] = {0, 0, 0, 0, 0, 0, ~0ull, 0};
        if (lead) {
            const unsigned long long qp = ld_relaxed(&nxt.qpack);
            vals[kSsF] = qp & cmask;
            vals[kSsMf] = qp >> a.S;
            vals[kSsFar] = ld_relaxed(&a.ctl->far_count[fp]);
            vals[kSsOvf] = ld_relaxed(&a.ctl->overflow);
            vals[kSsImp] = ld_relaxed(&nxt.ndisc);
            vals[kSsShip] = (unsigned long long)nship;
            rs.hdr(a.rank)->sin_count[(k + 1) & 1] = 0ull;  // consumed at step k-1; refilled at step k+1
        }
        par ^= 1;
        rs.publish(par, vals);
    }
    // outputs of the owned block: dist (UINT32_MAX unreached) and pred (global ids)
    for (int64_t v = tid; v < a.n_local; v += nthreads) {
        const unsigned long long x = a.dp[v];
        a.dist[v] = (uint32_t)(x >> 32);
        if (a.pred) a.pred[v] = (int32_t)(uint32_t)(x & 0xffffffffu);
    }
    if (lead) {
        a.ctl->levels = (unsigned long long)k;
        a.ctl->epoch = rs.ep;
        if (a.ctl->overflow) a.ctl->sticky = 1ull;
    }
}

// ---------------------------------------------------------------- host side

static gr_status psssp_scratch(Graph *g) {
    if (g->dp) return GR_OK;
    gr_status st;
    g->far_cap = 2 * g->m + 2 * g->n + 1024;
    if ((st = dev_alloc(g, (void **)&g->dp, g->n * sizeof(unsigned long long))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->stamp, g->n * sizeof(int32_t))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->farq[0], g->far_cap * sizeof(int32_t))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->farq[1], g->far_cap * sizeof(int32_t))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->ps_best, g->n_global * sizeof(unsigned long long))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->ps_sstamp, g->n_global * sizeof(int32_t))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->ps_ship, g->n_global * sizeof(int32_t))) != GR_OK)
        return st;
    return GR_OK;
}

static void fill_srank(Graph *g, SRank &r, uint32_t *dist, int32_t *pred) {
    r.rank = g->comm->rank;
    r.S = g->pack_shift;
    r.n_local = g->n; r.v_begin = g->v_begin;
    r.R = g->R; r.C = g->C; r.W = g->W; r.CW = g->CW;
    r.dp = g->dp; r.stamp = g->stamp; r.best = g->ps_best; r.sstamp = g->ps_sstamp; r.ship = g->ps_ship;
    for (int i = 0; i < 2; ++i) {
        r.qv[i] = g->qv[i]; r.qo[i] = g->qo[i]; r.qr[i] = g->qr[i]; r.far[i] = g->farq[i];
    }
    r.far_cap = g->far_cap;
    r.dist = dist; r.pred = pred;
    r.ctl = g->ctl; r.stats = g->stats_dev;
    for (int q = 0; q < kMaxRanks; ++q) r.sym[q] = g->sym_peer[q];
}

// delta: reading A-10 (the single-GPU auto rule on the GLOBAL graph)
static uint64_t auto_delta(Graph *g, uint32_t delta) {
    if (delta) return delta;
    const double avg = (double)g->m_global / (double)g->n_global;
    const uint64_t mw = g->maxw_global ? g->maxw_global : 1;
    uint64_t d = avg >= 8.0 ? (mw + 10) / 21 : mw * 32;
    return d ? d : 1;
}

static gr_status launch_psssp(Graph **gs, int k, int64_t src, uint32_t **dist, int32_t **pred, uint64_t delta) {
    Graph *g0 = gs[0];
    Comm *c = g0->comm;
    const SymLayout Ly = sym_layout(c->nranks, g0->block, true);
    PSsspArgs A;
    memset(&A, 0, sizeof(A));
    for (int i = 0; i < k; ++i) fill_srank(gs[i], A.ranks[i], dist[i], pred[i]);
    A.vranks = k;
    A.nranks = c->nranks;
    A.multiproc = (c->group == nullptr && c->nranks > 1) ? 1 : 0;
    A.n_global = g0->n_global;
    A.block = g0->block;
    A.src = src;
    A.delta = delta;
    A.off_sinbox[0] = Ly.sinbox[0];
    A.off_sinbox[1] = Ly.sinbox[1];
    A.inbox_cap = Ly.inbox_cap;
    bool packed = true;
    for (int i = 0; i < k; ++i) packed = packed && gs[i]->CW != nullptr;
    const void *fn = packed ? (const void *)psssp_kernel<kSBlock, kSMinB, true>
                            : (const void *)psssp_kernel<kSBlock, kSMinB, false>;
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSBlock, 0));
    if (per_sm < 1) { set_error("psssp_kernel cannot be resident"); return GR_ERR_CUDA; }
    if (per_sm > kSMinB) per_sm = kSMinB;
    A.ctas = (int32_t)((int64_t)g0->num_sms * per_sm / k);
    if (A.ctas < 1) { set_error("too many ranks for one GPU"); return GR_ERR_INVALID_ARGUMENT; }
    dim3 grid((unsigned)(A.ctas * k)), blk(kSBlock);
    void *args[] = {(void *)&A};
    GR_CUDA(cudaLaunchCooperativeKernel(fn, grid, blk, args, 0, g0->stream));
    count_launch();
    return GR_OK;
}

static gr_status finish_psssp(Graph *g, uint64_t delta) {
    unsigned long long levels = 0, overflow = 0;
    GR_CUDA(cudaMemcpyAsync(&levels, &g->ctl->levels, sizeof(levels), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemcpyAsync(&overflow, &g->ctl->overflow, sizeof(overflow), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemsetAsync(&g->ctl->sticky, 0, sizeof(unsigned long long), g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    g->stats_levels = (int)levels;
    g->stats_records = (int)(levels < (unsigned long long)kMaxStatRecords ? levels : kMaxStatRecords);
    g->stats_records = -1 - g->stats_records;
    g->last_launches = 1;
    g->last_delta = (uint32_t)(delta > 0xFFFFFFFFull ? 0xFFFFFFFFull : delta);
    g->last_kind = 2;
    g->reached = -2;
    if (overflow == 3) { set_error("partitioned SSSP: a peer rank did not reach a barrier within 20 s"); return GR_ERR_NCCL; }
    if (overflow == 2) { set_error("partitioned SSSP: received a vertex this rank does not own"); return GR_ERR_OVERFLOW; }
    if (overflow) { set_error("partitioned SSSP: a queue exceeded its capacity"); return GR_ERR_OVERFLOW; }
    return GR_OK;
}

// gr_sssp on a partitioned graph: collective over the comm's ranks.
gr_status psssp_collective(Graph *g, int64_t src, uint32_t *dist_out, int32_t *pred_out, uint32_t delta_opt) {
    Comm *c = g->comm;
    GR_CUDA(cudaSetDevice(g->device));
    gr_status st;
    auto stage = [&](Graph *x, uint32_t *dout, int32_t *pout, uint32_t **d, int32_t **p) -> gr_status {
        *d = dout;
        *p = pout;
        if (!ptr_on_device(dout)) {
            if (!x->dist_buf) { gr_status s2 = dev_alloc(x, (void **)&x->dist_buf, x->n * 4); if (s2 != GR_OK) return s2; }
            *d = x->dist_buf;
        }
        if (pout && !ptr_on_device(pout)) {
            if (!x->pred_buf) { gr_status s2 = dev_alloc(x, (void **)&x->pred_buf, x->n * 4); if (s2 != GR_OK) return s2; }
            *p = x->pred_buf;
        }
        return GR_OK;
    };
    auto copy_back = [&](Graph *x, uint32_t *dout, int32_t *pout, uint32_t *d, int32_t *p) -> gr_status {
        if (d != dout) GR_CUDA(cudaMemcpyAsync(dout, d, x->n * 4, cudaMemcpyDeviceToHost, x->stream));
        if (pout && p != pout) GR_CUDA(cudaMemcpyAsync(pout, p, x->n * 4, cudaMemcpyDeviceToHost, x->stream));
        GR_CUDA(cudaStreamSynchronize(x->stream));
        return GR_OK;
    };
    auto checks = [&](Graph *x) -> gr_status {
        if (!x->has_w || (!x->W && x->m > 0)) { set_error("partitioned graph was created without weights"); return GR_ERR_NO_WEIGHTS; }
        if ((unsigned long long)x->maxw_global * (unsigned long long)(x->n_global - 1) >= 0xFFFFFFFFull) {
            set_error("max_w=%u * (n-1)=%lld may overflow uint32 distances", x->maxw_global, (long long)(x->n_global - 1));
            return GR_ERR_OVERFLOW;
        }
        return psssp_scratch(x);
    };
    if (!g->has_w || (!g->W && g->m > 0)) { set_error("partitioned graph was created without weights"); return GR_ERR_NO_WEIGHTS; }
    if (!c->group) {
        if (!g->prepared && (st = prepare_real(g)) != GR_OK) return st;
        if ((st = checks(g)) != GR_OK) return st;
        uint32_t *d;
        int32_t *p;
        if ((st = stage(g, dist_out, pred_out, &d, &p)) != GR_OK) return st;
        const uint64_t delta = auto_delta(g, delta_opt);
        Graph *gs[1] = {g};
        if ((st = launch_psssp(gs, 1, src, &d, &p, delta)) != GR_OK) return st;
        g->last_src = (int32_t)(src - g->v_begin);
        if ((st = finish_psssp(g, delta)) != GR_OK) return st;
        return copy_back(g, dist_out, pred_out, d, p);
    }
    LoopGroup *grp = c->group;
    if (grp->joined == 0) { grp->kind = 2; grp->src = src; grp->sopts.delta = delta_opt; }
    else if (grp->kind != 2 || grp->src != src || grp->sopts.delta != delta_opt) {
        grp->joined = 0;
        set_error("loopback collective mismatch: every rank must call gr_sssp with the same source and delta");
        return GR_ERR_INVALID_ARGUMENT;
    }
    grp->out0[c->rank] = dist_out;
    grp->out1[c->rank] = pred_out;
    grp->joined |= 1 << c->rank;
    if (grp->joined != (1 << grp->P) - 1) return GR_OK;
    grp->joined = 0;
    for (int r = 0; r < grp->P; ++r)
        if (!grp->graphs[r]) { set_error("loopback rank %d has no partitioned graph", r); return GR_ERR_INVALID_ARGUMENT; }
    if (!g->prepared && (st = prepare_loopback(grp)) != GR_OK) return st;
    uint32_t *d[kMaxRanks];
    int32_t *p[kMaxRanks];
    for (int r = 0; r < grp->P; ++r) {
        if ((st = checks(grp->graphs[r])) != GR_OK) return st;
        if ((st = stage(grp->graphs[r], (uint32_t *)grp->out0[r], (int32_t *)grp->out1[r], &d[r], &p[r])) != GR_OK)
            return st;
    }
    const uint64_t delta = auto_delta(g, delta_opt);
    Graph *g0 = grp->graphs[0];
    GR_CUDA(cudaStreamSynchronize(g->stream));
    if ((st = launch_psssp(grp->graphs, grp->P, src, d, p, delta)) != GR_OK) return st;
    GR_CUDA(cudaStreamSynchronize(g0->stream));
    gr_status first = GR_OK;
    for (int r = 0; r < grp->P; ++r) {
        Graph *x = grp->graphs[r];
        x->last_src = (int32_t)(src - x->v_begin);
        st = finish_psssp(x, delta);
        if (st != GR_OK && first == GR_OK) first = st;
        st = copy_back(x, (uint32_t *)grp->out0[r], (int32_t *)grp->out1[r], d[r], p[r]);
        if (st != GR_OK && first == GR_OK) first = st;
    }
    return first;
}

}  // namespace gr
