// pagerank.cu -- PageRank with a converging-vertex frontier (
// paper §5.5).
//
// Paper: "we begin with a frontier that contains all vertices in the graph
// and end when all vertices have converged. Each iteration contains one
// advance operator to compute the PageRank value on the frontier of vertices,
// and one filter operator to remove the vertices whose PageRanks have already
// converged. We accumulate PageRank values with AtomicAdd operations."
//
// Reading A-23: PR(v) = (1-d)/n + d * sum over in-edges (u,v) of
// PR(u)/outdeg(u), d = damping (0.85 default), start PR = 1/n, no dangling
// redistribution (the paper is silent; on the symmetrised configs only
// isolated vertices dangle). A vertex leaves the frontier once its update
// |PR_new - PR_old| <= tol * PR_new; it keeps its value and other vertices keep
// reading it.
// B200 design: the advance runs over IN-lists (CSC; the CSR itself for
// symmetric graphs) of the frontier vertices with the merge-path balancer;
// per edge the contribution y[u] = PR(u) / outdeg(u) (kept per vertex by the
// filter, so one random 8-B load per edge) is summed into acc[v] -- a
// warp whose 32 edges share v reduces in registers and issues one fp64
// atomicAdd (the paper's AtomicAdd, aggregated). The filter kernel turns acc
// into the new rank (Jacobi within an iteration: all reads of a step happen
// before any rank of that step changes) and appends the still-moving vertices
// with their in-degree prefix for the next step's balancer.
#include "frontier.cuh"

namespace gr {

bool ptr_on_device(const void *p);

constexpr int kPrBlock = 256;
constexpr int kPrWarps = kPrBlock / 32;
constexpr int kPrStage = 64;
using PrAppender = AppenderT<kPrStage>;

struct PrAccOp {
    const double *y;      // y[u] = PR(u) / outdeg(u) (0 for dangling u), kept by the filter
    double *acc;

    __device__ __forceinline__ unsigned long long entry(int32_t) { return 0ull; }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *,
                                          const int32_t *dst, const T5 *) {
        double c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = ok[u] ? __ldg(y + dst[u]) : 0.0;  // one random sector per edge
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t s0 = __shfl_sync(0xffffffffu, src[u], 0);
            if (__all_sync(0xffffffffu, src[u] == s0)) {
                const double t = warp_sum<double>(c[u]);
                if (lane_id() == 0 && t != 0.0) atomicAdd(acc + s0, t);
            } else if (c[u] != 0.0) {
                atomicAdd(acc + src[u], c[u]);
            }
        }
    }
};

__global__ void pr_init_kernel(const int64_t *R, const int64_t *Rt, int64_t n, double *x, double *inv, double *y,
                               double *acc,
                               int32_t *qv, int64_t *qr, int64_t *qo, unsigned long long *cnt, int S) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) {
        const int64_t od = R[v + 1] - R[v];
        x[v] = 1.0 / (double)n;
        inv[v] = od > 0 ? 1.0 / (double)od : 0.0;
        y[v] = x[v] * inv[v];
        acc[v] = 0.0;
        qv[v] = (int32_t)v;        // frontier 0 = every vertex, in-list prefix = Rt
        qr[v] = Rt[v];
        qo[v] = Rt[v];
    }
    if (tid == 0) cnt[0] = ((unsigned long long)Rt[n] << S) | (unsigned long long)n;
}

__global__ void __launch_bounds__(kPrBlock) pr_advance_kernel(const int32_t *Ct, const int32_t *qv,
                                                              const int64_t *qo, const int64_t *qr, int64_t f,
                                                              int64_t mf, PrAccOp op) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    GlobalFrontier fr{qv, qo, qr, f, mf};
    expand_lb(fr, Ct, gw, nw, op);
}

// frontier = every vertex again (the convergence check sweep)
__global__ void pr_refill_kernel(const int64_t *Rt, int64_t n, int32_t *qv, int64_t *qr, int64_t *qo,
                                 unsigned long long *cnt, int S) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) {
        qv[v] = (int32_t)v;
        qr[v] = Rt[v];
        qo[v] = Rt[v];
    }
    if (tid == 0) *cnt = ((unsigned long long)Rt[n] << S) | (unsigned long long)n;
}

// filter: new rank, converged vertices leave the frontier
__global__ void __launch_bounds__(kPrBlock) pr_filter_kernel(const int64_t *Rt, const int32_t *qv, int64_t f,
                                                             double *x, const double *inv, double *y, double *acc,
                                                             double base, double d, double tol, PrAppender app) {
    __shared__ int32_t s_v[kPrWarps][kPrStage];
    __shared__ int32_t s_d[kPrWarps][kPrStage];
    __shared__ int64_t s_r[kPrWarps][kPrStage];
    const int wib = threadIdx.x >> 5;
    app.sv = s_v[wib]; app.sd = s_d[wib]; app.sr = s_r[wib]; app.cnt = 0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = tid - lane_id(); b < f; b += nt) {
        const int64_t j = b + lane_id();
        bool keep = false;
        int32_t v = 0;
        int64_t deg = 0, rs = 0;
        if (j < f) {
            v = qv[j];
            const double xn = base + d * acc[v];
            acc[v] = 0.0;
            keep = fabs(xn - x[v]) > tol * xn;
            x[v] = xn;
            y[v] = xn * inv[v];
            if (keep) { rs = Rt[v]; deg = Rt[v + 1] - rs; }
        }
        app.push(keep, v, deg, rs);
    }
    app.finish();
}

}  // namespace gr

using namespace gr;

extern "C" {

gr_status gr_pagerank(gr_graph *h, double damping, double tol, int32_t max_iter, double *rank_out,
                      int32_t *iterations) {
    Graph *g = (Graph *)h;
    if (!g || !rank_out) { set_error("graph or rank_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    if (g->part) { set_error("gr_pagerank needs a whole (unpartitioned) graph"); return GR_ERR_INVALID_ARGUMENT; }
    if (!(damping >= 0.0 && damping < 1.0) || !(tol >= 0.0) || max_iter < 1) {
        set_error("need 0 <= damping < 1, tol >= 0, max_iter >= 1");
        return GR_ERR_INVALID_ARGUMENT;
    }
    GR_CUDA(cudaSetDevice(g->device));
    if (g->pending && gr_graph_sync(h) != GR_OK) return GR_ERR_OVERFLOW;
    gr_status st;
    const int64_t n = g->n;
    if (!g->pr_inv) {
        if ((st = dev_alloc(g, (void **)&g->pr_inv, 2 * n * sizeof(double))) != GR_OK ||  // inv | y
            (st = dev_alloc(g, (void **)&g->pr_acc, n * sizeof(double))) != GR_OK ||
            (st = dev_alloc(g, (void **)&g->pr_cnt, 4 * sizeof(unsigned long long))) != GR_OK)
            return st;
    }
    const bool dev_out = ptr_on_device(rank_out);
    double *x = rank_out;
    if (!dev_out) {
        if (!g->bc_buf && (st = dev_alloc(g, (void **)&g->bc_buf, n * sizeof(double))) != GR_OK) return st;
        x = g->bc_buf;
    }
    cudaStream_t s = g->stream;
    const int S = g->pack_shift;
    double *inv = g->pr_inv, *y = g->pr_inv + n;
    pr_init_kernel<<<g->num_sms * 4, 256, 0, s>>>(g->R, g->Rt, n, x, inv, y, g->pr_acc, g->qv[0], g->qr[0],
                                                   g->qo[0], g->pr_cnt, S);
    int launches = 1, it = 0;
    const double base = (1.0 - damping) / (double)n;
    // When the filter has emptied the frontier, one more sweep over EVERY
    // vertex checks convergence (a frozen vertex's in-neighbours may have kept
    // moving): only an empty frontier after a full sweep ends the run, so at
    // the end one Jacobi step moved no rank by more than tol * rank.
    bool full = true;  // the current frontier is all vertices
    for (it = 0; it < max_iter; ++it) {
        unsigned long long qp = 0;
        GR_CUDA(cudaMemcpyAsync(&qp, g->pr_cnt + (it & 1), sizeof(qp), cudaMemcpyDeviceToHost, s));
        GR_CUDA(cudaStreamSynchronize(s));
        int64_t f = (int64_t)(qp & ((1ull << S) - 1)), mf = (int64_t)(qp >> S);
        if (f == 0) {
            if (full) break;  // the last full sweep kept nothing: converged
            pr_refill_kernel<<<g->num_sms * 4, 256, 0, s>>>(g->Rt, n, g->qv[it & 1], g->qr[it & 1], g->qo[it & 1],
                                                             g->pr_cnt + (it & 1), S);
            ++launches;
            f = n;
            mf = g->m;  // the CSC holds the same m edges
            full = true;
        } else {
            full = full && it == 0;
        }
        const int c = it & 1;
        PrAccOp op{y, g->pr_acc};
        if (mf > 0)
            pr_advance_kernel<<<g->num_sms * 8, kPrBlock, 0, s>>>(g->Ct, g->qv[c], g->qo[c], g->qr[c], f, mf, op);
        GR_CUDA(cudaMemsetAsync(g->pr_cnt + (c ^ 1), 0, sizeof(unsigned long long), s));
        PrAppender app;
        app.cnt = 0; app.S = S; app.cap = 2 * n;
        app.overflow = g->pr_cnt + 2;
        app.qv = g->qv[c ^ 1]; app.qo = g->qo[c ^ 1]; app.qr = g->qr[c ^ 1];
        app.counter = g->pr_cnt + (c ^ 1);
        const int64_t blocks = (f + kPrBlock - 1) / kPrBlock;
        pr_filter_kernel<<<(int)(blocks < g->num_sms * 8 ? blocks : g->num_sms * 8), kPrBlock, 0, s>>>(
            g->Rt, g->qv[c], f, x, inv, y, g->pr_acc, base, damping, tol, app);
        launches += 2;
    }
    if (!dev_out) GR_CUDA(cudaMemcpyAsync(rank_out, x, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    GR_CUDA(cudaGetLastError());
    GR_CUDA(cudaStreamSynchronize(s));
    count_launch(launches);
    if (iterations) *iterations = it;
    g->last_launches = launches;
    g->stats_levels = it;
    g->stats_records = -1;
    return GR_OK;
}

}  // extern "C"
