// bc.cu -- betweenness centrality, Brandes's two-pass formulation as the
// paper's second consumer of the advance operator.
//
// Paper §5.3: "The first phase has an advance step identical to
// the original BFS and a computation step that computes the number of
// shortest paths from source to each vertex. The second phase uses an
// advance step to iterate over the BFS frontier backwards with a computation
// step to compute the dependency scores." Brandes (cited P:962-963):
//   sigma[s] = 1, sigma[w] = sum over (v,w) in E with d[w] = d[v]+1 of sigma[v]
//   delta[v] = sum over (v,w) in E with d[w] = d[v]+1 of sigma[v]/sigma[w] (1 + delta[w])
//   bc[v]   += delta[v]  for v != s.
//
// B200 design:
//  * forward level L: merge-path advance (expand_lb) over the level-L queue;
//    per edge (v,w): claim w by CAS on depth (-1 -> L+1, the winner appends
//    w to the level-(L+1) queue with its degree prefix), and every edge whose
//    target sits at L+1 adds sigma[v] (carried as the window payload) with a
//    double atomicAdd ("atomicAdd" accumulation);
//  * the queues of all levels are kept back to back (each vertex is appended
//    exactly once, so n entries suffice) -- the "BFS frontier" the second
//    phase iterates backwards (SPEC S:445 reading: retained frontiers);
//  * backward level L (deepest first): the same advance over the level-L
//    queue, each edge (v,w) with d[w] = L+1 contributes sigma[v]/sigma[w]
//    (1 + delta[w]) to delta[v]; a warp whose 32 edges share v (long lists:
//    the common case on hubs) reduces in registers and issues one atomic.
// sigma / delta / bc are fp64 (the oracle's precision; path counts exceed
// fp32's 24-bit mantissa on the paper's graphs).
#include <vector>

#include "frontier.cuh"

namespace gr {

bool ptr_on_device(const void *p);

constexpr int kBcBlock = 256;
constexpr int kBcWarps = kBcBlock / 32;
constexpr int kBcStage = 64;
using BcAppender = AppenderT<kBcStage>;

// Per-vertex BC state in ONE 16-byte record, so the random per-edge accesses
// of both passes touch one 32-B sector: depth (probe + CAS claim) and sigma
// (atomicAdd) in the forward pass; depth and coef = (1 + delta) / sigma of
// the successor in the backward pass (val holds sigma until the vertex's
// level has been processed backwards, then coef).
struct __align__(16) BcVert {
    double val;
    int32_t depth;
    int32_t pad;
};

struct BcArgs {
    int64_t n;
    const int64_t *R;
    const int32_t *C;
    const int64_t *Rt;         // in-lists (the CSR itself when symmetric): pull levels
    const int32_t *Ct;
    BcVert *bv;
    double *delta;
    int32_t *qv;               // all levels back to back
    int64_t *qo;
    int64_t *qr;
    unsigned long long *cnt;   // per level: (edges << S) | count
    int S;
};

struct BcFwdOp {
    const BcArgs *a;
    int32_t next;              // L + 1
    BcAppender *app;

    __device__ __forceinline__ unsigned long long entry(int32_t v) {
        return (unsigned long long)__double_as_longlong(__ldcg(&a->bv[v].val));
    }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *, const unsigned long long *pay,
                                          const int32_t *dst, const T5 *) {
        int32_t d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) d[u] = ok[u] ? __ldcg(&a->bv[dst[u]].depth) : -2;
        // the claims of all U edges in flight, then the row offsets of the
        // discovered ones in flight (each consumed inside its own branch was
        // a dependent round trip apiece)
        int32_t c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = d[u] == -1 ? atomicCAS(&a->bv[dst[u]].depth, -1, next) : d[u];
        bool disc[U];
        int64_t r0[U], r1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            disc[u] = d[u] == -1 && c[u] == -1;
            const int32_t dw = disc[u] ? next : c[u];
            if (dw == next) atomicAdd(&a->bv[dst[u]].val, __longlong_as_double((long long)pay[u]));  // RED
            r0[u] = disc[u] ? a->R[dst[u]] : 0;
            r1[u] = disc[u] ? a->R[dst[u] + 1] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            // every discovered vertex joins its level's queue (degree 0 too:
            // the backward pass converts its sigma into coef)
            app->push(disc[u], dst[u], r1[u] - r0[u], r0[u]);
    }
};

struct BcBwdOp {
    const BcArgs *a;
    int32_t next;              // L + 1

    __device__ __forceinline__ unsigned long long entry(int32_t v) {
        return (unsigned long long)__double_as_longlong(__ldcg(&a->bv[v].val));  // sigma[v]
    }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *pay,
                                          const int32_t *dst, const T5 *) {
        double2 r[U];  // {val, (depth, pad)} of the successor candidate: one 16-B load
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = ok[u] ? __ldcg(reinterpret_cast<const double2 *>(a->bv + dst[u]))
                                                 : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double c = 0.0;
            const int32_t dw = ok[u] ? (int32_t)(__double_as_longlong(r[u].y) & 0xffffffffll) : -2;
            if (dw == next)  // w is a successor of v: sigma[v] * (1 + delta[w]) / sigma[w]
                c = __longlong_as_double((long long)pay[u]) * r[u].x;
            const int32_t s0 = __shfl_sync(0xffffffffu, src[u], 0);
            if (__all_sync(0xffffffffu, src[u] == s0)) {
                c = warp_sum<double>(c);
                if (lane_id() == 0 && c != 0.0) atomicAdd(a->delta + s0, c);
            } else if (c != 0.0) {
                atomicAdd(a->delta + src[u], c);
            }
        }
    }
};

__global__ void bc_init_kernel(BcArgs a, int32_t s) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < a.n; v += nt) {
        BcVert x;
        x.val = v == s ? 1.0 : 0.0;   // sigma
        x.depth = v == s ? 0 : -1;
        x.pad = 0;
        a.bv[v] = x;
        a.delta[v] = 0.0;
    }
    if (tid == 0) {
        const int64_t d = a.R[s + 1] - a.R[s];
        a.qv[0] = s;
        a.qo[0] = 0;
        a.qr[0] = a.R[s];
        a.cnt[0] = ((unsigned long long)d << a.S) | 1ull;
        a.cnt[1] = 0ull;
    }
}

// level L processed backwards: val = sigma -> coef = (1 + delta) / sigma
__global__ void bc_coef_kernel(BcArgs a, int64_t off, int64_t f) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = tid; j < f; j += nt) {
        const int32_t v = a.qv[off + j];
        a.bv[v].val = (1.0 + a.delta[v]) / a.bv[v].val;
    }
}

__global__ void bc_sigma_kernel(const BcVert *bv, int64_t n, double *sigma) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) sigma[v] = bv[v].depth >= 0 ? bv[v].val : 0.0;
}

__global__ void __launch_bounds__(kBcBlock) bc_fwd_kernel(BcArgs a, int L, int64_t off, int64_t f, int64_t mf) {
    __shared__ int32_t s_v[kBcWarps][kBcStage];
    __shared__ int32_t s_d[kBcWarps][kBcStage];
    __shared__ int64_t s_r[kBcWarps][kBcStage];
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.cnt[L + 2] = 0ull;  // read by level L+1
    BcAppender app;
    app.sv = s_v[wib]; app.sd = s_d[wib]; app.sr = s_r[wib]; app.cnt = 0; app.S = a.S;
    app.cap = a.n - (off + f);
    app.overflow = a.cnt + a.n + 2;  // never set: each vertex is appended once
    app.qv = a.qv + off + f;
    app.qo = a.qo + off + f;
    app.qr = a.qr + off + f;
    app.counter = a.cnt + L + 1;
    BcFwdOp op{&a, L + 1, &app};
    GlobalFrontier fr{a.qv + off, a.qo + off, a.qr + off, f, mf};
    expand_lb(fr, a.C, gw, nw, op);
    app.finish();
}

// Pull (bottom-up) forward level L -> L+1 (paper P:804-834, named for BC in
// "more sophisticated BC and SSSP implementations could benefit
// from it"): every unvisited vertex v with in-edges sums sigma over its
// in-neighbours at depth L -- sigma[v] = sum over (u,v) in E, d[u] = L of
// sigma[u], Brandes's forward recurrence read from the receiver's side. No
// early exit (every parent counts) but no atomics: v is owned by one lane
// (lists of <= kBcPullLane edges) or one warp (longer lists, 32 edges a step
// with a warp reduction). Found vertices join the level-(L+1) queue.
constexpr int64_t kBcPullLane = 8;

__global__ void __launch_bounds__(kBcBlock) bc_fwd_pull_kernel(BcArgs a, int L, int64_t off, int64_t f) {
    __shared__ int32_t s_v[kBcWarps][kBcStage];
    __shared__ int32_t s_d[kBcWarps][kBcStage];
    __shared__ int64_t s_r[kBcWarps][kBcStage];
    const int wib = threadIdx.x >> 5;
    const unsigned l = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.cnt[L + 2] = 0ull;  // read by level L+1
    BcAppender app;
    app.sv = s_v[wib]; app.sd = s_d[wib]; app.sr = s_r[wib]; app.cnt = 0; app.S = a.S;
    app.cap = a.n - (off + f);
    app.overflow = a.cnt + a.n + 2;
    app.qv = a.qv + off + f;
    app.qo = a.qo + off + f;
    app.qr = a.qr + off + f;
    app.counter = a.cnt + L + 1;
    const unsigned long long pol = policy_evict_first();
    for (int64_t base = gw * 32; base < a.n; base += nw * 32) {
        const int64_t v = base + l;
        int64_t b = 0, e = 0;
        bool cand = false;
        if (v < a.n && __ldcg(&a.bv[v].depth) == -1) {
            b = a.Rt[v];
            e = a.Rt[v + 1];
            cand = e > b;
        }
        double sum = 0.0;
        const bool lane_list = cand && e - b <= kBcPullLane;
        if (lane_list) {  // short list: this lane, 4 neighbour loads then 4 record loads in flight
            for (int64_t x = b; x < e; x += 4) {
                int32_t u[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) u[j] = x + j < e ? ld_stream(a.Ct + x + j, pol) : -1;
                double2 r[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    r[j] = u[j] >= 0 ? __ldcg(reinterpret_cast<const double2 *>(a.bv + u[j])) : make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (u[j] >= 0 && (int32_t)(__double_as_longlong(r[j].y) & 0xffffffffll) == L) sum += r[j].x;
            }
        }
        unsigned lm = __ballot_sync(0xffffffffu, cand && !lane_list);
        while (lm) {  // long lists: the whole warp, one list at a time
            const int ld = __ffs(lm) - 1;
            lm &= lm - 1;
            const int64_t lb = __shfl_sync(0xffffffffu, b, ld), le = __shfl_sync(0xffffffffu, e, ld);
            double part = 0.0;
            for (int64_t x = lb + l; x < le; x += 32) {
                const int32_t u = ld_stream(a.Ct + x, pol);
                const double2 r = __ldcg(reinterpret_cast<const double2 *>(a.bv + u));
                if ((int32_t)(__double_as_longlong(r.y) & 0xffffffffll) == L) part += r.x;
            }
            part = warp_sum<double>(part);
            if ((int)l == ld) sum = part;
        }
        const bool found = cand && sum > 0.0;
        int64_t deg = 0, rs = 0;
        if (found) {
            BcVert x;
            x.val = sum;
            x.depth = L + 1;
            x.pad = 0;
            a.bv[v] = x;
            rs = a.R[v];
            deg = a.R[v + 1] - rs;
        }
        app.push(found, (int32_t)v, deg, rs);
    }
    app.finish();
}

__global__ void __launch_bounds__(kBcBlock) bc_bwd_kernel(BcArgs a, int L, int64_t off, int64_t f, int64_t mf) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    BcBwdOp op{&a, L + 1};
    GlobalFrontier fr{a.qv + off, a.qo + off, a.qr + off, f, mf};
    expand_lb(fr, a.C, gw, nw, op);
}

__global__ void bc_accum_kernel(const double *delta, int64_t n, int32_t s, double *bc) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt)
        if (v != s) bc[v] += delta[v];
}

__global__ void bc_zero_kernel(double *x, int64_t n) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) x[v] = 0.0;
}

}  // namespace gr

using namespace gr;

extern "C" {

gr_status gr_bc_ex(gr_graph *h, const int32_t *sources, int64_t nsrc, double *bc_out, double *sigma_out,
                   const gr_bc_opts *opts) {
    Graph *g = (Graph *)h;
    gr_bc_opts o = opts ? *opts : gr_bc_opts{};
    if (o.direction < 0 || o.direction > 2 || o.alpha < 0) { set_error("invalid gr_bc_opts"); return GR_ERR_INVALID_ARGUMENT; }
    const double alpha = o.alpha > 0 ? o.alpha : 2.0;
    if (!g || !bc_out || nsrc < 0 || (nsrc > 0 && !sources)) {
        set_error("graph / bc_out / sources is NULL or nsrc < 0");
        return GR_ERR_INVALID_ARGUMENT;
    }
    if (g->part) { set_error("gr_bc needs a whole (unpartitioned) graph"); return GR_ERR_INVALID_ARGUMENT; }
    if (ptr_on_device(sources)) { set_error("sources must be host memory"); return GR_ERR_INVALID_ARGUMENT; }
    for (int64_t i = 0; i < nsrc; ++i)
        if (sources[i] < 0 || sources[i] >= g->n) {
            set_error("sources[%lld]=%d not in [0, n=%lld)", (long long)i, sources[i], (long long)g->n);
            return GR_ERR_OUT_OF_RANGE;
        }
    GR_CUDA(cudaSetDevice(g->device));
    if (g->pending && gr_graph_sync(h) != GR_OK) return GR_ERR_OVERFLOW;
    gr_status st;
    const int64_t n = g->n;
    if (!g->bc_vert) {
        if ((st = dev_alloc(g, &g->bc_vert, n * sizeof(BcVert))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->bc_delta, n * sizeof(double))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->bc_cnt, (n + 3) * sizeof(unsigned long long))) != GR_OK)
            return st;
    }
    const bool dev_bc = ptr_on_device(bc_out);
    double *bc = bc_out;
    if (!dev_bc) {
        if (!g->bc_buf && (st = dev_alloc(g, (void **)&g->bc_buf, n * sizeof(double))) != GR_OK) return st;
        bc = g->bc_buf;
    }
    BcArgs a;
    a.n = n; a.R = g->R; a.C = g->C; a.Rt = g->Rt; a.Ct = g->Ct;
    a.bv = (BcVert *)g->bc_vert; a.delta = g->bc_delta;
    double *sig = nullptr;  // sigma of the last source, saved before the backward pass overwrites it
    if (sigma_out && nsrc > 0) {
        if (ptr_on_device(sigma_out)) sig = sigma_out;
        else {
            if (!g->bc_sig && (st = dev_alloc(g, (void **)&g->bc_sig, n * sizeof(double))) != GR_OK) return st;
            sig = g->bc_sig;
        }
    }
    a.qv = g->qv[0]; a.qo = g->qo[0]; a.qr = g->qr[0];
    a.cnt = g->bc_cnt; a.S = g->pack_shift;
    const int grid = g->num_sms * 8;
    cudaStream_t s = g->stream;
    bc_zero_kernel<<<g->num_sms * 4, 256, 0, s>>>(bc, n);
    int launches = 1;
    std::vector<int64_t> off, fs, mfs;
    int levels_total = 0;
    for (int64_t i = 0; i < nsrc; ++i) {
        const int32_t src = sources[i];
        bc_init_kernel<<<g->num_sms * 4, 256, 0, s>>>(a, src);
        ++launches;
        off.assign(1, 0);
        fs.clear();
        mfs.clear();
        int64_t m_u = g->m;  // out-edges of vertices not yet discovered (their in-lists on symmetric graphs)
        for (int L = 0;; ++L) {  // forward phase: BFS + sigma (one host read per level)
            unsigned long long qp = 0;
            GR_CUDA(cudaMemcpyAsync(&qp, a.cnt + L, sizeof(qp), cudaMemcpyDeviceToHost, s));
            GR_CUDA(cudaStreamSynchronize(s));
            const int64_t f = (int64_t)(qp & ((1ull << a.S) - 1)), mf = (int64_t)(qp >> a.S);
            if (f == 0) break;
            fs.push_back(f);
            mfs.push_back(mf);
            m_u -= mf;
            // direction (A-24): pull when the frontier's edges exceed the
            // unvisited vertices' edges / alpha (no early exit in a BC pull:
            // it reads every unvisited list in full, hence a small alpha)
            const bool pull = o.direction == 2 || (o.direction == 0 && (double)mf > (double)m_u / alpha);
            if (pull) bc_fwd_pull_kernel<<<grid, kBcBlock, 0, s>>>(a, L, off[L], f);
            else bc_fwd_kernel<<<grid, kBcBlock, 0, s>>>(a, L, off[L], f, mf);
            if (i == nsrc - 1 && L < kMaxStatRecords) {  // per-level records of the last source
                gr_level_stats rec{};
                rec.level = L; rec.direction = pull ? 2 : 1; rec.frontier = f; rec.frontier_edges = mf;
                rec.aux = m_u;
                g->stats_host[L] = rec;
            }
            ++launches;
            off.push_back(off[L] + f);
        }
        levels_total += (int)fs.size();
        if (sig && i == nsrc - 1) {
            bc_sigma_kernel<<<g->num_sms * 4, 256, 0, s>>>(a.bv, n, sig);
            ++launches;
        }
        // backward phase: the stored frontiers, deepest first (the deepest
        // level has no successors: only its coef; level 0 = the source, whose
        // dependency is not accumulated)
        for (int L = (int)fs.size() - 1; L >= 1; --L) {
            if (L + 1 < (int)fs.size()) {
                bc_bwd_kernel<<<grid, kBcBlock, 0, s>>>(a, L, off[L], fs[L], mfs[L]);
                ++launches;
            }
            if (L > 1) {  // coef of level L is read by level L - 1 >= 1 only
                bc_coef_kernel<<<g->num_sms * 2, 256, 0, s>>>(a, off[L], fs[L]);
                ++launches;
            }
        }
        bc_accum_kernel<<<g->num_sms * 4, 256, 0, s>>>(a.delta, n, src, bc);
        ++launches;
    }
    GR_CUDA(cudaGetLastError());
    if (!dev_bc) GR_CUDA(cudaMemcpyAsync(bc_out, bc, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (sig && sig != sigma_out) GR_CUDA(cudaMemcpyAsync(sigma_out, sig, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    GR_CUDA(cudaStreamSynchronize(s));
    count_launch(launches);
    g->last_launches = launches;
    g->stats_levels = levels_total;
    g->stats_records = nsrc > 0 ? (int)(fs.size() < (size_t)kMaxStatRecords ? fs.size() : kMaxStatRecords) : 0;
    g->last_kind = 0;  // run totals are not counted for BC
    return GR_OK;
}

gr_status gr_bc(gr_graph *h, const int32_t *sources, int64_t nsrc, double *bc_out, double *sigma_out) {
    return gr_bc_ex(h, sources, nsrc, bc_out, sigma_out, nullptr);
}

}  // extern "C"
