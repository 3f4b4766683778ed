// partition.cu -- 1D-partitioned BFS (multi-GPU). The paper is
// single-GPU (multi-GPU is future work); this extends its push
// advance + filter with an exchange step: remote
// discoveries are bucketed per owner in the same fused kernel and claimed by
// the owner after the caller's all-to-all.
//
// One level = gr_part_bfs_expand (this rank's frontier) -> caller exchange ->
// gr_part_bfs_absorb (received pairs). Both append into the local next
// frontier queue with the same packed (edges << S | count) counter, so the
// next level's merge-path prefix is produced by the filter, as on one GPU.
#include "frontier.cuh"

namespace gr {

gr_status graph_create(int64_t n, int64_t m, const int64_t *R, const int32_t *C, const uint32_t *W,
                       uint32_t flags, int device, void *stream, Graph **out, int64_t ncols);
bool ptr_on_device(const void *p);
gr_status sort_lists_by_degree(Graph *g, cudaStream_t s, int blocks, const int32_t *deg);

constexpr int kPartBlock = 256;
constexpr int kPartWarps = kPartBlock / 32;
constexpr int kPartStage = 128;
using PartAppender = AppenderT<kPartStage>;

struct PartArgs {
    int64_t n_local, v_begin, block;
    int nparts;
    const int64_t *R;
    const int32_t *C;
    const int32_t *Cp;   // pull lists: C, or its copy ordered by neighbour degree
    uint32_t *visited;   // local bitmap
    uint32_t *sent;      // global bitmap
    int32_t *send_pairs;
    long long *send_counts;
    int32_t *depth, *pred;
    int32_t *qv[2];
    int64_t *qo[2];
    int64_t *qr[2];
    Ctl *ctl;
    int S;
};

__global__ void part_init_kernel(PartArgs a, int64_t nwords_global) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < a.n_local; v += nt) {
        a.depth[v] = -1;
        if (a.pred) a.pred[v] = -1;
    }
    for (int64_t w = tid; w < (a.n_local + 31) / 32; w += nt) a.visited[w] = 0u;
    for (int64_t w = tid; w < nwords_global; w += nt) a.sent[w] = 0u;
    if (tid < kSlots * (int64_t)(sizeof(Slot) / 8)) ((unsigned long long *)a.ctl->slot)[tid] = 0ull;
    if (tid == 0) a.ctl->overflow = 0ull;
}

__global__ void part_seed_kernel(PartArgs a, int64_t src) {
    // every rank marks src as sent (no one ships it to its owner); the owner seeds it
    a.sent[src >> 5] |= 1u << (src & 31);
    const int64_t s = src - a.v_begin;
    if (s < 0 || s >= a.n_local) return;
    a.depth[s] = 0;
    if (a.pred) a.pred[s] = (int32_t)src;  // A-1, global id
    a.visited[s >> 5] |= 1u << (s & 31);
    const int64_t d = a.R[s + 1] - a.R[s];
    a.qv[0][0] = (int32_t)s;
    a.qo[0][0] = 0;
    a.qr[0][0] = a.R[s];
    a.ctl->slot[0].qpack = d > 0 ? (((unsigned long long)d << a.S) | 1ull) : 0ull;
}

// Fused cond/apply + filter of the partitioned push advance.
struct PartPushOp {
    PartArgs *a;
    int32_t next_depth;
    PartAppender *app;

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const T5 *) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t w = dst[u];
            const int64_t lw = (int64_t)w - a->v_begin;
            const bool owned = ok[u] && lw >= 0 && lw < a->n_local;
            bool disc = false, ship = false;
            if (owned) {
                const uint32_t bit = 1u << (lw & 31);
                if (!(__ldcg(a->visited + (lw >> 5)) & bit))
                    disc = !(atomicOr(a->visited + (lw >> 5), bit) & bit);
            } else if (ok[u]) {
                const uint32_t bit = 1u << (w & 31);
                if (!(__ldcg(a->sent + (w >> 5)) & bit))
                    ship = !(atomicOr(a->sent + (w >> 5), bit) & bit);
            }
            const int32_t parent = (int32_t)(a->v_begin + src[u]);
            int64_t deg = 0, rs = 0;
            if (disc) {
                a->depth[lw] = next_depth;
                if (a->pred) a->pred[lw] = parent;
                rs = a->R[lw];
                deg = a->R[lw + 1] - rs;
            }
            app->push(disc && deg > 0, (int32_t)lw, deg, rs);
            // remote: bucket (w, parent) for owner q, one atomic per owner per warp
            const unsigned shipm = __ballot_sync(0xffffffffu, ship);
            if (shipm) {
                const int q = ship ? (int)(w / a->block) : -1;
                const unsigned peers = __match_any_sync(0xffffffffu, q);
                if (ship) {
                    const int leader = __ffs(peers) - 1;
                    long long base = 0;
                    if ((int)lane_id() == leader)
                        base = (long long)atomicAdd((unsigned long long *)(a->send_counts + q),
                                                    (unsigned long long)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    const long long pos = base + __popc(peers & lanemask_lt());
                    int32_t *dstp = a->send_pairs + 2 * ((int64_t)q * a->block + pos);
                    dstp[0] = w;
                    dstp[1] = parent;
                }
            }
        }
    }
};

__global__ void __launch_bounds__(kPartBlock) part_expand_kernel(PartArgs a, int level) {
    __shared__ int32_t s_v[kPartWarps][kPartStage];
    __shared__ int32_t s_d[kPartWarps][kPartStage];
    __shared__ int64_t s_r[kPartWarps][kPartStage];
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned long long qp = ld_relaxed(&a.ctl->slot[level & 3].qpack);
    const int64_t f = (int64_t)(qp & ((1ull << a.S) - 1));
    const int64_t mf = (int64_t)(qp >> a.S);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // slot of level+2 is idle now
        Slot &r = a.ctl->slot[(level + 2) & 3];
        r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull;
    }
    PartAppender app;
    app.sv = s_v[wib]; app.sd = s_d[wib]; app.sr = s_r[wib]; app.cnt = 0; app.S = a.S;
    app.cap = 2 * a.n_local;
    app.overflow = &a.ctl->overflow;
    app.qv = a.qv[(level + 1) & 1];
    app.qo = a.qo[(level + 1) & 1];
    app.qr = a.qr[(level + 1) & 1];
    app.counter = &a.ctl->slot[(level + 1) & 3].qpack;
    PartPushOp op{&a, level + 1, &app};
    GlobalFrontier fr{a.qv[level & 1], a.qo[level & 1], a.qr[level & 1], f, mf};
    expand_lb(fr, a.C, gw, nw, op);
    app.finish();
}

__global__ void __launch_bounds__(kPartBlock) part_absorb_kernel(PartArgs a, int level, const int32_t *pairs,
                                                                 int64_t nrecv) {
    __shared__ int32_t s_v[kPartWarps][kPartStage];
    __shared__ int32_t s_d[kPartWarps][kPartStage];
    __shared__ int64_t s_r[kPartWarps][kPartStage];
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    PartAppender app;
    app.sv = s_v[wib]; app.sd = s_d[wib]; app.sr = s_r[wib]; app.cnt = 0; app.S = a.S;
    app.cap = 2 * a.n_local;
    app.overflow = &a.ctl->overflow;
    app.qv = a.qv[(level + 1) & 1];
    app.qo = a.qo[(level + 1) & 1];
    app.qr = a.qr[(level + 1) & 1];
    app.counter = &a.ctl->slot[(level + 1) & 3].qpack;
    for (int64_t base = gw * 32; base < nrecv; base += nw * 32) {
        const int64_t j = base + lane_id();
        bool disc = false;
        int64_t lw = 0, deg = 0, rs = 0;
        if (j < nrecv) {
            const int32_t w = pairs[2 * j], parent = pairs[2 * j + 1];
            lw = (int64_t)w - a.v_begin;
            if (lw < 0 || lw >= a.n_local) {
                atomicExch((unsigned long long *)&a.ctl->overflow, 2ull);  // misrouted pair
            } else {
                const uint32_t bit = 1u << (lw & 31);
                disc = !(atomicOr(a.visited + (lw >> 5), bit) & bit);
                if (disc) {
                    a.depth[lw] = level + 1;
                    if (a.pred) a.pred[lw] = parent;
                    rs = a.R[lw];
                    deg = a.R[lw + 1] - rs;
                }
            }
        }
        app.push(disc && deg > 0, (int32_t)lw, deg, rs);
    }
    app.finish();
}

// frontier bitmap shard of level `level` from the local queue
__global__ void part_shard_clear_kernel(uint32_t *shard, int64_t words) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w = tid; w < words; w += nt) shard[w] = 0u;
}
__global__ void part_shard_fill_kernel(PartArgs a, int level, uint32_t *shard) {
    const unsigned long long qp = ld_relaxed(&a.ctl->slot[level & 3].qpack);
    const int64_t f = (int64_t)(qp & ((1ull << a.S) - 1));
    const int32_t *q = a.qv[level & 1];
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = tid; j < f; j += nt) {
        const int32_t v = q[j];
        atomicOr(shard + (v >> 5), 1u << (v & 31));
    }
}

// Bottom-up step of a partition: owned unvisited vertices look for
// a parent in the GLOBAL frontier bitmap. As the single-GPU pull_level: each
// warp compacts the unvisited vertices of 32 words of the local visited bitmap
// into a shared-memory candidate list (ascending ids), then resolves 64
// candidates at a time (2 per lane, the row-offset and first-neighbour loads
// of both issued together); a lane scans up to kPartPullLong more edges of an
// unresolved list, and whatever is left of the long lists is scanned by the
// whole warp, 32 edges a step with a ballot early exit. Found vertices: depth /
// pred, RED.OR into the local visited bitmap and into `nshard` (the level+1
// frontier shard, cleared before the launch), and the local queue of level + 1
// (merge-path prefix via the packed counter).
constexpr int64_t kPartPullLong = 4;
constexpr int kPartPullBatch = 64;

__global__ void __launch_bounds__(kPartBlock) part_pull_kernel(PartArgs a, int level, const uint32_t *gfront,
                                                              uint32_t *nshard) {
    __shared__ int32_t s_v[kPartWarps][kPartStage];
    __shared__ int32_t s_d[kPartWarps][kPartStage];
    __shared__ int64_t s_r[kPartWarps][kPartStage];
    __shared__ int32_t s_wl[kPartWarps][kPartPullBatch + 32];
    const int wib = threadIdx.x >> 5;
    const unsigned l = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Slot &r = a.ctl->slot[(level + 2) & 3];
        r.qpack = 0; r.ndisc = 0; r.fpack = 0; r.work = 0; r.insp = 0; r.minfar = ~0ull;
    }
    PartAppender app;
    app.sv = s_v[wib]; app.sd = s_d[wib]; app.sr = s_r[wib]; app.cnt = 0; app.S = a.S;
    app.cap = 2 * a.n_local;
    app.overflow = &a.ctl->overflow;
    app.qv = a.qv[(level + 1) & 1];
    app.qo = a.qo[(level + 1) & 1];
    app.qr = a.qr[(level + 1) & 1];
    app.counter = &a.ctl->slot[(level + 1) & 3].qpack;
    int32_t *wl = s_wl[wib];
    const unsigned long long pol = policy_evict_first();
    const int64_t nwords = (a.n_local + 31) / 32;
    const uint32_t tail = (a.n_local & 31) ? ((1u << (a.n_local & 31)) - 1u) : 0xffffffffu;
    auto fbit = [&](int32_t u) -> bool { return (__ldg(gfront + (u >> 5)) >> (u & 31)) & 1u; };
    int cnt = 0;  // warp-uniform
    auto process = [&](int k) {  // candidates wl[0, k), k <= kPartPullBatch
        int32_t v[2], par[2], u0[2];
        int64_t beg[2], end[2], nxt[2];
        bool fnd[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) v[q] = ((int)l + 32 * q < k) ? wl[l + 32 * q] : -1;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            beg[q] = v[q] >= 0 ? a.R[v[q]] : 0;
            end[q] = v[q] >= 0 ? a.R[v[q] + 1] : 0;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) u0[q] = beg[q] < end[q] ? ld_stream(a.Cp + beg[q], pol) : -1;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            fnd[q] = u0[q] >= 0 && fbit(u0[q]);
            par[q] = u0[q];
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            nxt[q] = beg[q] + 1;
            if (fnd[q]) continue;
            const int64_t lim = (end[q] - nxt[q] > kPartPullLong) ? nxt[q] + kPartPullLong : end[q];
            for (int64_t e = nxt[q]; e < lim && !fnd[q]; e += 4) {
                int32_t u[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) u[j] = (e + j < lim) ? ld_stream(a.Cp + e + j, pol) : -1;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (!fnd[q] && u[j] >= 0 && fbit(u[j])) { fnd[q] = true; par[q] = u[j]; }
            }
            nxt[q] = lim;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            unsigned lm = __ballot_sync(0xffffffffu, !fnd[q] && nxt[q] < end[q]);
            while (lm) {
                const int ld = __ffs(lm) - 1;
                lm &= lm - 1;
                const int64_t b = __shfl_sync(0xffffffffu, nxt[q], ld);
                const int64_t e = __shfl_sync(0xffffffffu, end[q], ld);
                int32_t hitu = -1;
                for (int64_t x = b; x < e; x += 32) {
                    const int32_t u = (x + l < e) ? ld_stream(a.Cp + x + l, pol) : -1;
                    const unsigned bm = __ballot_sync(0xffffffffu, u >= 0 && fbit(u));
                    if (bm) {
                        hitu = __shfl_sync(0xffffffffu, u, __ffs(bm) - 1);
                        break;
                    }
                }
                if ((int)l == ld && hitu >= 0) { fnd[q] = true; par[q] = hitu; }
            }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (fnd[q]) {
                const int32_t x = v[q];
                a.depth[x] = level + 1;
                if (a.pred) a.pred[x] = par[q];
                const uint32_t bit = 1u << (x & 31);
                atomicOr(nshard + (x >> 5), bit);     // RED.OR
                atomicOr(a.visited + (x >> 5), bit);  // RED.OR
            }
            // found vertices have an in-edge, hence out-degree > 0 (symmetric)
            app.push(fnd[q], fnd[q] ? v[q] : 0, end[q] - beg[q], beg[q]);
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
    for (int64_t w0 = gw * 32; w0 < nwords; w0 += nw * 32) {
        const int64_t wi = w0 + l;
        uint32_t cm = wi < nwords ? ~a.visited[wi] : 0u;
        if (wi == nwords - 1) cm &= tail;
        unsigned nz = __ballot_sync(0xffffffffu, cm != 0);
        while (nz) {
            const int j = __ffs(nz) - 1;
            nz &= nz - 1;
            const uint32_t w = __shfl_sync(0xffffffffu, cm, j);
            if ((w >> l) & 1u) wl[cnt + __popc(w & lanemask_lt())] = (int32_t)((w0 + j) * 32 + l);
            cnt += __popc(w);
            __syncwarp();
            if (cnt >= kPartPullBatch) process(kPartPullBatch);
        }
    }
    while (cnt > 0) process(cnt < kPartPullBatch ? cnt : kPartPullBatch);
    app.finish();
}

static PartArgs part_args(Graph *g) {
    PartArgs a;
    a.n_local = g->n; a.v_begin = g->v_begin; a.block = g->block; a.nparts = g->nparts;
    a.R = g->R; a.C = g->C; a.Cp = g->Ct; a.visited = g->visited; a.sent = g->sent;
    a.send_pairs = g->send_pairs; a.send_counts = g->send_counts;
    a.depth = g->part_depth; a.pred = g->part_pred;
    for (int i = 0; i < 2; ++i) { a.qv[i] = g->qv[i]; a.qo[i] = g->qo[i]; a.qr[i] = g->qr[i]; }
    a.ctl = g->ctl;
    a.S = g->pack_shift;
    return a;
}

}  // namespace gr

using namespace gr;

// Device-side frontier readout (no host synchronisation): out[0] = f,
// out[1] = m_f of level `level`, out[2] = overflow code (0 none, 1 queue, 2
// misrouted pair). The caller sums out[] over ranks on the device and reads
// the totals once per level.
__global__ void part_frontier_kernel(const Ctl *ctl, int level, int S, long long *out) {
    const unsigned long long qp = ctl->slot[level & 3].qpack;
    out[0] = (long long)(qp & ((1ull << S) - 1));
    out[1] = (long long)(qp >> S);
    out[2] = (long long)ctl->overflow;
}

extern "C" {

static gr_status create_part(int64_t n_global, int32_t nparts, int32_t rank, int64_t v_begin, int64_t v_end,
                             int64_t m_local, const int64_t *row_offsets, const int32_t *col_indices,
                             const uint32_t *weights, uint32_t flags, int device, void *cuda_stream,
                             gr_graph **out) {
    if (!out || nparts < 1 || rank < 0 || rank >= nparts || n_global < 1) {
        set_error("invalid partition arguments (nparts=%d rank=%d n_global=%lld)", nparts, rank, (long long)n_global);
        return GR_ERR_INVALID_ARGUMENT;
    }
    const int64_t block = 32 * ((n_global + 32 * (int64_t)nparts - 1) / (32 * (int64_t)nparts));
    const int64_t vb = (int64_t)rank * block, ve = vb + block < n_global ? vb + block : n_global;
    if (v_begin != vb || v_end != ve || ve <= vb) {
        set_error("rank %d of %d must own [%lld, %lld), got [%lld, %lld)", rank, nparts, (long long)vb,
                  (long long)ve, (long long)v_begin, (long long)v_end);
        return GR_ERR_INVALID_ARGUMENT;
    }
    Graph *g = nullptr;
    gr_status st = graph_create(v_end - v_begin, m_local, row_offsets, col_indices, weights, flags, device,
                                cuda_stream, &g, n_global);
    if (st != GR_OK) return st;
    g->part = true;
    g->n_global = n_global; g->v_begin = v_begin; g->v_end = v_end; g->block = block;
    g->nparts = nparts; g->rank = rank;
    if ((st = dev_alloc(g, (void **)&g->sent, ((n_global + 31) / 32) * sizeof(uint32_t))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->send_pairs, 2 * (size_t)nparts * block * sizeof(int32_t))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->send_counts, nparts * sizeof(long long))) != GR_OK ||
        (st = dev_alloc(g, (void **)&g->recv_pairs, 2 * (size_t)n_global * sizeof(int32_t))) != GR_OK) {
        dev_free_all(g);
        delete g;
        return st;
    }
    *out = (gr_graph *)g;
    return GR_OK;
}

gr_status gr_graph_create_part(int64_t n_global, int32_t nparts, int32_t rank, int64_t v_begin, int64_t v_end,
                               int64_t m_local, const int64_t *row_offsets, const int32_t *col_indices,
                               uint32_t flags, int device, void *cuda_stream, gr_graph **out) {
    return create_part(n_global, nparts, rank, v_begin, v_end, m_local, row_offsets, col_indices, nullptr, flags,
                       device, cuda_stream, out);
}

gr_status gr_graph_create_part_w(int64_t n_global, int32_t nparts, int32_t rank, int64_t v_begin, int64_t v_end,
                                 int64_t m_local, const int64_t *row_offsets, const int32_t *col_indices,
                                 const uint32_t *weights, uint32_t flags, int device, void *cuda_stream,
                                 gr_graph **out) {
    if (!weights && m_local > 0) { set_error("weights is NULL"); return GR_ERR_NO_WEIGHTS; }
    gr_status st = create_part(n_global, nparts, rank, v_begin, v_end, m_local, row_offsets, col_indices, weights,
                               flags, device, cuda_stream, out);
    if (st == GR_OK) ((Graph *)*out)->has_w = true;  // m_local = 0: no weight is ever read
    return st;
}

gr_status gr_part_buffers(gr_graph *h, int32_t **send_pairs, int64_t **send_counts, int32_t **recv_pairs,
                          int64_t *block) {
    Graph *g = (Graph *)h;
    if (!g || !g->part) { set_error("not a partitioned graph"); return GR_ERR_INVALID_ARGUMENT; }
    if (send_pairs) *send_pairs = g->send_pairs;
    if (send_counts) *send_counts = (int64_t *)g->send_counts;
    if (recv_pairs) *recv_pairs = g->recv_pairs;
    if (block) *block = g->block;
    return GR_OK;
}

gr_status gr_part_bfs_begin(gr_graph *h, int64_t src, int32_t *depth_out, int32_t *pred_out) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || !depth_out) { set_error("not a partitioned graph / depth_out NULL"); return GR_ERR_INVALID_ARGUMENT; }
    if (src < 0 || src >= g->n_global) {
        set_error("src=%lld not in [0, n=%lld)", (long long)src, (long long)g->n_global);
        return GR_ERR_OUT_OF_RANGE;
    }
    GR_CUDA(cudaSetDevice(g->device));
    if (!ptr_on_device(depth_out) || (pred_out && !ptr_on_device(pred_out))) {
        set_error("partitioned BFS outputs must be device memory");
        return GR_ERR_INVALID_ARGUMENT;
    }
    g->part_depth = depth_out;
    g->part_pred = pred_out;
    g->pull_shard_level = -1;
    PartArgs a = part_args(g);
    part_init_kernel<<<g->num_sms * 4, 256, 0, g->stream>>>(a, (g->n_global + 31) / 32);
    part_seed_kernel<<<1, 1, 0, g->stream>>>(a, src);
    count_launch(2);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_bfs_expand(gr_graph *h, int32_t level) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || level < 0) { set_error("invalid argument"); return GR_ERR_INVALID_ARGUMENT; }
    if (g->pull_shard_level == level + 1) g->pull_shard_level = -1;  // level+1 is rebuilt by push
    PartArgs a = part_args(g);
    GR_CUDA(cudaMemsetAsync(g->send_counts, 0, g->nparts * sizeof(long long), g->stream));
    part_expand_kernel<<<g->num_sms * 8, kPartBlock, 0, g->stream>>>(a, level);
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_bfs_absorb(gr_graph *h, int32_t level, const int32_t *recv_pairs, int64_t nrecv) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || level < 0 || nrecv < 0 || (nrecv > 0 && !recv_pairs)) {
        set_error("invalid argument");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (nrecv == 0) return GR_OK;
    PartArgs a = part_args(g);
    const int64_t blocks = (nrecv + kPartBlock - 1) / kPartBlock;
    part_absorb_kernel<<<(int)(blocks < g->num_sms * 8 ? blocks : g->num_sms * 8), kPartBlock, 0, g->stream>>>(
        a, level, recv_pairs, nrecv);
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_bfs_shard(gr_graph *h, int32_t level, uint32_t *shard) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || level < 0 || !shard) { set_error("invalid argument"); return GR_ERR_INVALID_ARGUMENT; }
    if (g->pull_shard_level == level) {  // written by the pull step that built this frontier
        GR_CUDA(cudaMemcpyAsync(shard, g->pull_shard, (g->block / 32) * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                g->stream));
        return GR_OK;
    }
    PartArgs a = part_args(g);
    part_shard_clear_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(shard, g->block / 32);
    part_shard_fill_kernel<<<g->num_sms * 2, 256, 0, g->stream>>>(a, level, shard);
    count_launch(2);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_bfs_pull(gr_graph *h, int32_t level, const uint32_t *global_frontier) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || level < 0 || !global_frontier) { set_error("invalid argument"); return GR_ERR_INVALID_ARGUMENT; }
    if (!g->pull_shard) {
        gr_status st = dev_alloc(g, (void **)&g->pull_shard, (g->block / 32) * sizeof(uint32_t));
        if (st != GR_OK) return st;
        GR_CUDA(cudaMemsetAsync(g->pull_shard, 0, (g->block / 32) * sizeof(uint32_t), g->stream));
    }
    GR_CUDA(cudaMemsetAsync(g->pull_shard, 0, (g->block / 32) * sizeof(uint32_t), g->stream));
    PartArgs a = part_args(g);
    part_pull_kernel<<<g->num_sms * 8, kPartBlock, 0, g->stream>>>(a, level, global_frontier, g->pull_shard);
    count_launch();
    g->pull_shard_level = level + 1;
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_bfs_frontier(gr_graph *h, int32_t level, int64_t *f, int64_t *mf) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || level < 0) { set_error("invalid argument"); return GR_ERR_INVALID_ARGUMENT; }
    unsigned long long qp = 0, ov = 0;
    GR_CUDA(cudaMemcpyAsync(&qp, &g->ctl->slot[level & 3].qpack, sizeof(qp), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemcpyAsync(&ov, &g->ctl->overflow, sizeof(ov), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    if (ov) {
        set_error(ov == 2 ? "received a vertex this rank does not own" : "local frontier queue overflow");
        return GR_ERR_OVERFLOW;
    }
    if (f) *f = (int64_t)(qp & ((1ull << g->pack_shift) - 1));
    if (mf) *mf = (int64_t)(qp >> g->pack_shift);
    return GR_OK;
}

gr_status gr_part_bfs_frontier_async(gr_graph *h, int32_t level, int64_t *out3) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || level < 0 || !out3 || !ptr_on_device(out3)) {
        set_error("invalid argument (out3 must be device int64[3])");
        return GR_ERR_INVALID_ARGUMENT;
    }
    part_frontier_kernel<<<1, 1, 0, g->stream>>>(g->ctl, level, g->pack_shift, (long long *)out3);
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

gr_status gr_part_order_pull_lists(gr_graph *h, const int32_t *deg_global) {
    Graph *g = (Graph *)h;
    if (!g || !g->part || !deg_global || !ptr_on_device(deg_global)) {
        set_error("invalid argument (deg_global must be device int32[n_global])");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (g->Rt != g->R) {
        set_error("pull-list order needs a symmetric partition (out-lists double as in-lists)");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (g->m == 0) return GR_OK;
    if (g->m >= (1ll << 31)) {
        set_error("pull-list order: m_local >= 2^31 is not supported by the segmented sort");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (g->Ct == g->C) {
        gr_status st = dev_alloc(g, (void **)&g->Ct, g->m * sizeof(int32_t));
        if (st != GR_OK) { g->Ct = g->C; return st; }
        GR_CUDA(cudaMemcpyAsync(g->Ct, g->C, g->m * sizeof(int32_t), cudaMemcpyDeviceToDevice, g->stream));
    }
    return sort_lists_by_degree(g, g->stream, g->num_sms * 4, deg_global);
}

}  // extern "C"
