// partition_sssp.cu -- 1D-partitioned delta-stepping SSSP (multi-GPU,
// SURVEY §8(f) f2). The paper's SSSP is single-GPU (Alg. 1; near/far
// priority queue P:838-857; multi-GPU is future work P:1383-1396).
// This keeps its step structure per partition and adds one exchange:
//
//   relax (step k, near iteration it, far pile fp, threshold thr)
//       merge-path advance over the owned near queue; per edge
//       nd = dist[u] + w (UpdateLabel):
//         owned target  -> 64-bit packed atomicMin on (dist<<32 | pred) (A-9),
//                          stamp keyed by iteration AND slice (A-7), append to
//                          near (nd < thr) or far -- exactly as on one GPU;
//         remote target -> atomicMin into this rank's "best shipped" value of
//                          the vertex; a strict improvement claims the vertex
//                          for this step's bucket of its owner (one entry per
//                          vertex per step, so a bucket never exceeds `block`);
//       a pack pass then writes each bucket entry's FINAL best value as a
//       (vertex, dist, parent) triple;
//   (exchange)  the caller's all-to-all moves the triples to their owners;
//   absorb      the owner relaxes the received triples against its
//               authoritative dist, same stamp / near-far filter;
//   re-split    when the global near queue is empty: min over the far piles
//               (all-reduced by the caller), threshold jumps to its band, the
//               far pile splits into near / far, stale entries dropped (A-11).
//
// Culling by "best shipped" is exact: the owner's dist is never above a value
// this rank shipped before, so a candidate that does not beat it cannot
// improve the owner's label.
#include "frontier.cuh"

namespace gr {

bool ptr_on_device(const void *p);

constexpr int kPsBlock = 256;
constexpr int kPsWarps = kPsBlock / 32;
constexpr int kPsStage = 64;
using PsAppender = AppenderT<kPsStage>;

struct PsArgs {
    int64_t n_local, v_begin, block, n_global;
    int nparts;
    const int64_t *R;
    const int32_t *C;
    const uint32_t *W;
    unsigned long long *dp;     // [n_local] (dist << 32) | global pred
    int32_t *stamp;             // [n_local] RemoveRedundant stamp (A-7)
    unsigned long long *best;   // [n_global] best value shipped to the owner
    int32_t *sstamp;            // [n_global] step of the last shipment
    int32_t *send;              // [3 * nparts * block]
    long long *send_counts;     // [nparts]
    int32_t *qv[2];
    int64_t *qo[2];
    int64_t *qr[2];
    int32_t *far[2];
    int64_t far_cap;
    Ctl *ctl;
    int S;
};

struct PsSmem {
    int32_t sv[kPsWarps][kPsStage];
    int32_t sd[kPsWarps][kPsStage];
    int64_t sr[kPsWarps][kPsStage];
    int32_t fv[kPsWarps][kPsStage];
};

__device__ __forceinline__ void ps_queues(const PsArgs &a, PsSmem &s, int wib, int step, int fp,
                                          PsAppender &nearq, PsAppender &farq) {
    nearq.sv = s.sv[wib]; nearq.sd = s.sd[wib]; nearq.sr = s.sr[wib]; nearq.cnt = 0; nearq.S = a.S;
    nearq.cap = 2 * a.n_local;
    nearq.overflow = &a.ctl->overflow;
    nearq.qv = a.qv[(step + 1) & 1];
    nearq.qo = a.qo[(step + 1) & 1];
    nearq.qr = a.qr[(step + 1) & 1];
    nearq.counter = &a.ctl->slot[(step + 1) & 3].qpack;
    farq.sv = s.fv[wib]; farq.sd = nullptr; farq.sr = nullptr; farq.cnt = 0; farq.S = 0;
    farq.qo = nullptr; farq.qr = nullptr;
    farq.cap = a.far_cap;
    farq.overflow = &a.ctl->overflow;
    farq.qv = a.far[fp];
    farq.counter = &a.ctl->far_count[fp];
}

__device__ __forceinline__ void ps_reset_slot(const PsArgs &a, int step) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // slot of step+2 is idle now
        Slot &r = a.ctl->slot[(step + 2) & 3];
        r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull; r.dmax = 0;
    }
}

// Owner-side relaxation of local vertex lv with candidate (nd, parent):
// UpdateLabel + SetPred (packed atomicMin, A-9) + RemoveRedundant (A-7) +
// near/far split. Returns 1 near, 2 far, 0 nothing to append.
__device__ __forceinline__ int ps_relax_owned_cur(const PsArgs &a, int64_t lv, unsigned long long nd, uint32_t parent,
                                                  uint64_t thr, int32_t key_near, unsigned long long cur) {
    if (nd >= (cur >> 32)) return 0;  // plain pre-check against the value loaded by the caller
    const unsigned long long old = atomicMin(a.dp + lv, (nd << 32) | parent);
    if (nd >= (old >> 32)) return 0;
    const bool far = nd >= thr;
    const int32_t key = key_near + (far ? 1 : 0);
    if (atomicExch(a.stamp + lv, key) == key) return 0;
    return far ? 2 : 1;
}
__device__ __forceinline__ int ps_relax_owned(const PsArgs &a, int64_t lv, unsigned long long nd, uint32_t parent,
                                              uint64_t thr, int32_t key_near, unsigned long long pol) {
    return ps_relax_owned_cur(a, lv, nd, parent, thr, key_near, ld_probe(a.dp + lv, pol));
}

struct PsRelaxOp {
    const PsArgs *a;
    uint64_t thr;
    int32_t key_near;   // 2 * it
    int32_t step;
    PsAppender *nearq, *farq;
    unsigned long long pol;

    __device__ __forceinline__ unsigned long long entry(int32_t v) { return ld_probe(a->dp + v, pol) >> 32; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *du,
                                          const int32_t *dst, const T5 *x) {
        uint32_t w[U];
        unsigned long long cur[U];
        // all weight loads and all pre-check probes (dist of owned targets,
        // best-shipped of remote ones) issued before any dependent atomic, as
        // in the single-GPU RelaxOp
#pragma unroll
        for (int u = 0; u < U; ++u) {
            w[u] = ok[u] ? __ldg(a->W + x[u]) : 0u;
            const int64_t lv = (int64_t)dst[u] - a->v_begin;
            const bool owned = lv >= 0 && lv < a->n_local;
            cur[u] = ok[u] ? ld_probe(owned ? a->dp + lv : a->best + dst[u], pol) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t v = dst[u];
            const int64_t lv = (int64_t)v - a->v_begin;
            const bool owned = lv >= 0 && lv < a->n_local;
            const unsigned long long nd = du[u] + w[u];
            const uint32_t parent = (uint32_t)(a->v_begin + src[u]);
            int kind = 0;
            bool ship = false;
            int64_t deg = 0, rs = 0;
            if (ok[u] && owned) {
                kind = ps_relax_owned_cur(*a, lv, nd, parent, thr, key_near, cur[u]);
                if (kind == 1) { rs = a->R[lv]; deg = a->R[lv + 1] - rs; }
            } else if (ok[u] && nd < (cur[u] >> 32)) {
                const unsigned long long old = atomicMin(a->best + v, (nd << 32) | parent);
                if (nd < (old >> 32)) ship = atomicExch(a->sstamp + v, step) != step;
            }
            nearq->push(kind == 1 && deg > 0, (int32_t)lv, deg, rs);
            farq->push(kind == 2, (int32_t)lv, 0);
            const unsigned shipm = __ballot_sync(0xffffffffu, ship);
            if (shipm) {  // bucket v for its owner q: one atomic per owner per warp
                const int q = ship ? (int)(v / a->block) : -1;
                const unsigned peers = __match_any_sync(0xffffffffu, q);
                if (ship) {
                    const int leader = __ffs(peers) - 1;
                    long long base = 0;
                    if ((int)lane_id() == leader)
                        base = (long long)atomicAdd((unsigned long long *)(a->send_counts + q),
                                                    (unsigned long long)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    const long long pos = base + __popc(peers & lanemask_lt());
                    a->send[3 * ((int64_t)q * a->block + pos)] = v;  // value filled by the pack pass
                }
            }
        }
    }
};

__global__ void ps_init_kernel(PsArgs a) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < a.n_local; v += nt) {  // Set_Problem_Data
        a.dp[v] = ~0ull;   // dist = UINT32_MAX, pred = -1 (A-2)
        a.stamp[v] = -1;
    }
    for (int64_t v = tid; v < a.n_global; v += nt) {
        a.best[v] = ~0ull;
        a.sstamp[v] = -1;
    }
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (tid == 0) {
        a.ctl->overflow = 0ull;
        a.ctl->far_count[0] = 0ull;
        a.ctl->far_count[1] = 0ull;
    }
}

__global__ void ps_seed_kernel(PsArgs a, int64_t src) {
    for (int i = 0; i < kSlots; ++i) a.ctl->slot[i].minfar = ~0ull;
    const int64_t s = src - a.v_begin;
    if (s < 0 || s >= a.n_local) return;
    a.dp[s] = (unsigned long long)(uint32_t)src;  // dist 0, pred = src (A-1, global id)
    const int64_t d = a.R[s + 1] - a.R[s];
    if (d > 0) {
        a.qv[0][0] = (int32_t)s;
        a.qo[0][0] = 0;
        a.qr[0][0] = a.R[s];
        a.ctl->slot[0].qpack = ((unsigned long long)d << a.S) | 1ull;
    }
}

__global__ void __launch_bounds__(kPsBlock, 4) ps_relax_kernel(PsArgs a, int step, int it, int fp, uint64_t thr) {
    __shared__ PsSmem s;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned long long qp = ld_relaxed(&a.ctl->slot[step & 3].qpack);
    const int64_t f = (int64_t)(qp & ((1ull << a.S) - 1));
    const int64_t mf = (int64_t)(qp >> a.S);
    ps_reset_slot(a, step);
    PsAppender nearq, farq;
    ps_queues(a, s, wib, step, fp, nearq, farq);
    PsRelaxOp op{&a, thr, 2 * it, step, &nearq, &farq, policy_evict_last()};
    GlobalFrontier fr{a.qv[step & 1], a.qo[step & 1], a.qr[step & 1], f, mf};
    expand_lb(fr, a.C, gw, nw, op);
    nearq.finish();
    farq.finish();
}

// Fills the (dist, parent) words of every bucket entry from the final best
// value. Grid: x strides the entries of owner q = blockIdx.y.
__global__ void ps_pack_kernel(PsArgs a) {
    const int64_t q = blockIdx.y;
    const int64_t cnt = (int64_t)a.send_counts[q];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += (int64_t)gridDim.x * blockDim.x) {
        int32_t *t = a.send + 3 * (q * a.block + j);
        const unsigned long long b = a.best[t[0]];
        t[1] = (int32_t)(uint32_t)(b >> 32);
        t[2] = (int32_t)(uint32_t)(b & 0xffffffffu);
    }
}

__global__ void __launch_bounds__(kPsBlock) ps_absorb_kernel(PsArgs a, int step, int it, int fp, uint64_t thr,
                                                             const int32_t *trip, int64_t nrecv) {
    __shared__ PsSmem s;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    PsAppender nearq, farq;
    ps_queues(a, s, wib, step, fp, nearq, farq);
    const unsigned long long pol = policy_evict_last();
    for (int64_t base = gw * 32; base < nrecv; base += nw * 32) {
        const int64_t j = base + lane_id();
        int kind = 0;
        int64_t lv = 0, deg = 0, rs = 0;
        if (j < nrecv) {
            const int32_t v = trip[3 * j];
            const unsigned long long nd = (uint32_t)trip[3 * j + 1];
            const uint32_t parent = (uint32_t)trip[3 * j + 2];
            lv = (int64_t)v - a.v_begin;
            if (lv < 0 || lv >= a.n_local) {
                atomicExch((unsigned long long *)&a.ctl->overflow, 2ull);  // misrouted triple
            } else {
                kind = ps_relax_owned(a, lv, nd, parent, thr, 2 * it, pol);
                if (kind == 1) { rs = a.R[lv]; deg = a.R[lv + 1] - rs; }
            }
        }
        nearq.push(kind == 1 && deg > 0, (int32_t)lv, deg, rs);
        farq.push(kind == 2, (int32_t)lv, 0);
    }
    nearq.finish();
    farq.finish();
}

// min over the far pile of dist >= thr (entries below thr are stale, A-11)
__global__ void ps_far_min_kernel(PsArgs a, int step, int fp, uint64_t thr) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    const int64_t fc = (int64_t)ld_relaxed(&a.ctl->far_count[fp]);
    unsigned long long mymin = ~0ull;
    for (int64_t j = tid; j < fc; j += nt) {
        const unsigned long long d = a.dp[a.far[fp][j]] >> 32;
        if (d >= thr && d < mymin) mymin = d;
    }
    for (int sh = 16; sh > 0; sh >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, mymin, sh);
        mymin = o < mymin ? o : mymin;
    }
    if (lane_id() == 0 && mymin != ~0ull) atomicMin(&a.ctl->slot[step & 3].minfar, mymin);
}

// "update the priority function and operate on the far slice"
__global__ void __launch_bounds__(kPsBlock) ps_resplit_kernel(PsArgs a, int step, int it, int fp, uint64_t thr_old,
                                                              uint64_t thr) {
    __shared__ PsSmem s;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t fc = (int64_t)ld_relaxed(&a.ctl->far_count[fp]);
    ps_reset_slot(a, step);
    PsAppender nearq, farq;
    ps_queues(a, s, wib, step, fp ^ 1, nearq, farq);
    const int32_t *far_c = a.far[fp];
    for (int64_t base = gw * 32; base < fc; base += nw * 32) {
        const int64_t j = base + lane_id();
        bool to_near = false, to_far = false;
        int32_t v = 0;
        int64_t deg = 0, rs = 0;
        if (j < fc) {
            v = far_c[j];
            const unsigned long long d = a.dp[v] >> 32;
            if (d >= thr_old) {  // else stale: already expanded below thr_old
                const bool nearb = d < thr;
                const int32_t key = 2 * it + (nearb ? 0 : 1);
                if (atomicExch(a.stamp + v, key) != key) {
                    if (nearb) { to_near = true; rs = a.R[v]; deg = a.R[v + 1] - rs; }
                    else to_far = true;
                }
            }
        }
        nearq.push(to_near && deg > 0, v, deg, rs);
        farq.push(to_far, v, 0);
    }
    nearq.finish();
    farq.finish();
}

__global__ void ps_unpack_kernel(const unsigned long long *dp, int64_t n, uint32_t *dist, int32_t *pred) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) {
        const unsigned long long x = dp[v];
        dist[v] = (uint32_t)(x >> 32);
        if (pred) pred[v] = (int32_t)(uint32_t)(x & 0xffffffffu);
    }
}

static PsArgs ps_args(Graph *g) {
    PsArgs a;
    a.n_local = g->n; a.v_begin = g->v_begin; a.block = g->block; a.n_global = g->n_global;
    a.nparts = g->nparts;
    a.R = g->R; a.C = g->C; a.W = g->W;
    a.dp = g->dp; a.stamp = g->stamp; a.best = g->ps_best; a.sstamp = g->ps_sstamp;
    a.send = g->ps_send; a.send_counts = g->send_counts;
    for (int i = 0; i < 2; ++i) {
        a.qv[i] = g->qv[i]; a.qo[i] = g->qo[i]; a.qr[i] = g->qr[i]; a.far[i] = g->farq[i];
    }
    a.far_cap = g->far_cap;
    a.ctl = g->ctl;
    a.S = g->pack_shift;
    return a;
}

static gr_status ps_check(Graph *g, bool begun = true) {
    if (!g || !g->part) { set_error("not a partitioned graph"); return GR_ERR_INVALID_ARGUMENT; }
    if (!g->has_w || (!g->W && g->m > 0)) { set_error("partition was created without weights"); return GR_ERR_NO_WEIGHTS; }
    if (begun && !g->ps_dist) { set_error("gr_part_sssp_begin was not called"); return GR_ERR_INVALID_ARGUMENT; }
    return GR_OK;
}

}  // namespace gr

using namespace gr;

// Device-side counters (no host synchronisation): out = {near count of step,
// far count of pile fp, overflow code}; summed over ranks by the caller.
__global__ void ps_counts_kernel(const gr::Ctl *ctl, int step, int fp, int S, long long *out) {
    out[0] = (long long)(ctl->slot[step & 3].qpack & ((1ull << S) - 1));
    out[1] = (long long)ctl->far_count[fp];
    out[2] = (long long)ctl->overflow;
}

extern "C" {

gr_status gr_part_sssp_begin(gr_graph *h, int64_t src, uint32_t *dist_out, int32_t *pred_out) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g, false);
    if (st != GR_OK) return st;
    if (!dist_out) { set_error("dist_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    if (src < 0 || src >= g->n_global) {
        set_error("src=%lld not in [0, n=%lld)", (long long)src, (long long)g->n_global);
        return GR_ERR_OUT_OF_RANGE;
    }
    if ((unsigned long long)g->max_w * (unsigned long long)(g->n_global - 1) >= 0xFFFFFFFFull) {
        set_error("max_w=%u * (n-1)=%lld may overflow uint32 distances", g->max_w, (long long)(g->n_global - 1));
        return GR_ERR_OVERFLOW;
    }
    GR_CUDA(cudaSetDevice(g->device));
    if (!ptr_on_device(dist_out) || (pred_out && !ptr_on_device(pred_out))) {
        set_error("partitioned SSSP outputs must be device memory");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (!g->dp) {
        const int64_t P = g->nparts, B = g->block;
        g->far_cap = 2 * g->m + 2 * g->n + 1024;
        if ((st = dev_alloc(g, (void **)&g->dp, g->n * sizeof(unsigned long long))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->stamp, g->n * sizeof(int32_t))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->farq[0], g->far_cap * sizeof(int32_t))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->farq[1], g->far_cap * sizeof(int32_t))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->ps_best, g->n_global * sizeof(unsigned long long))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->ps_sstamp, g->n_global * sizeof(int32_t))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->ps_send, 3 * P * B * sizeof(int32_t))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->ps_recv, 3 * P * B * sizeof(int32_t))) != GR_OK)
            return st;
    }
    g->ps_dist = dist_out;
    g->ps_pred = pred_out;
    PsArgs a = ps_args(g);
    ps_init_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(a);
    ps_seed_kernel<<<1, 1, 0, g->stream>>>(a, src);
    count_launch(2);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_sssp_buffers(gr_graph *h, int32_t **send_triples, int64_t **send_counts, int32_t **recv_triples,
                               int64_t *block) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (send_triples) *send_triples = g->ps_send;
    if (send_counts) *send_counts = (int64_t *)g->send_counts;
    if (recv_triples) *recv_triples = g->ps_recv;
    if (block) *block = g->block;
    return GR_OK;
}

gr_status gr_part_sssp_relax(gr_graph *h, int32_t step, int32_t it, int32_t fp, uint64_t thr) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (step < 0 || it < 1 || (fp & ~1)) { set_error("invalid step/it/fp"); return GR_ERR_INVALID_ARGUMENT; }
    PsArgs a = ps_args(g);
    GR_CUDA(cudaMemsetAsync(g->send_counts, 0, g->nparts * sizeof(long long), g->stream));
    ps_relax_kernel<<<g->num_sms * 8, kPsBlock, 0, g->stream>>>(a, step, it, fp, thr);
    ps_pack_kernel<<<dim3(g->num_sms, g->nparts), 256, 0, g->stream>>>(a);
    count_launch(2);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_sssp_absorb(gr_graph *h, int32_t step, int32_t it, int32_t fp, uint64_t thr,
                              const int32_t *recv_triples, int64_t nrecv) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (step < 0 || it < 1 || (fp & ~1) || nrecv < 0 || (nrecv > 0 && !recv_triples)) {
        set_error("invalid argument");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (nrecv == 0) return GR_OK;
    PsArgs a = ps_args(g);
    const int64_t blocks = (nrecv + kPsBlock - 1) / kPsBlock;
    ps_absorb_kernel<<<(int)(blocks < g->num_sms * 8 ? blocks : g->num_sms * 8), kPsBlock, 0, g->stream>>>(
        a, step, it, fp, thr, recv_triples, nrecv);
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_sssp_counts(gr_graph *h, int32_t step, int32_t fp, int64_t *near_count, int64_t *far_count) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (step < 0 || (fp & ~1)) { set_error("invalid step/fp"); return GR_ERR_INVALID_ARGUMENT; }
    unsigned long long qp = 0, fc = 0, ov = 0;
    GR_CUDA(cudaMemcpyAsync(&qp, &g->ctl->slot[step & 3].qpack, sizeof(qp), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemcpyAsync(&fc, &g->ctl->far_count[fp], sizeof(fc), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemcpyAsync(&ov, &g->ctl->overflow, sizeof(ov), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    if (ov) {
        set_error(ov == 2 ? "received a vertex this rank does not own" : "a near/far queue exceeded its capacity");
        return GR_ERR_OVERFLOW;
    }
    if (near_count) *near_count = (int64_t)(qp & ((1ull << g->pack_shift) - 1));
    if (far_count) *far_count = (int64_t)fc;
    return GR_OK;
}

gr_status gr_part_sssp_far_min(gr_graph *h, int32_t step, int32_t fp, uint64_t thr, uint64_t *min_out) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (step < 0 || (fp & ~1) || !min_out) { set_error("invalid argument"); return GR_ERR_INVALID_ARGUMENT; }
    PsArgs a = ps_args(g);
    ps_far_min_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(a, step, fp, thr);
    count_launch();
    unsigned long long mn = ~0ull;
    GR_CUDA(cudaMemcpyAsync(&mn, &g->ctl->slot[step & 3].minfar, sizeof(mn), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    *min_out = mn;
    return GR_OK;
}

gr_status gr_part_sssp_resplit(gr_graph *h, int32_t step, int32_t it, int32_t fp, uint64_t thr_old, uint64_t thr) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (step < 0 || it < 1 || (fp & ~1) || thr <= thr_old) { set_error("invalid argument"); return GR_ERR_INVALID_ARGUMENT; }
    PsArgs a = ps_args(g);
    ps_resplit_kernel<<<g->num_sms * 8, kPsBlock, 0, g->stream>>>(a, step, it, fp, thr_old, thr);
    GR_CUDA(cudaMemsetAsync(&g->ctl->far_count[fp], 0, sizeof(unsigned long long), g->stream));
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_sssp_end(gr_graph *h) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    ps_unpack_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(g->dp, g->n, g->ps_dist, g->ps_pred);
    count_launch();
    GR_CUDA(cudaGetLastError());
    GR_CUDA(cudaStreamSynchronize(g->stream));
    return GR_OK;
}

gr_status gr_part_sssp_counts_async(gr_graph *h, int32_t step, int32_t fp, int64_t *out3) {
    Graph *g = (Graph *)h;
    gr_status st = ps_check(g);
    if (st != GR_OK) return st;
    if (step < 0 || (fp & ~1) || !out3 || !ptr_on_device(out3)) {
        set_error("invalid step/fp or out3 (device int64[3])");
        return GR_ERR_INVALID_ARGUMENT;
    }
    ps_counts_kernel<<<1, 1, 0, g->stream>>>(g->ctl, step, fp, g->pack_shift, (long long *)out3);
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

}  // extern "C"
