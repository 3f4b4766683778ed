// graph.cu -- device graph store (a1 of SURVEY §8(a)): CSR ingest, optional
// validation, reverse graph (CSC) for pull on directed inputs, degree stats,
// per-run scratch. P:237-244 (graph definition), P:267-278 (SOA + CSR),
// P:821-825 (bitmaps), S:31-34 / S:45 (CSR invariants, error naming the index).
#include <cub/cub.cuh>

#include "gr_internal.cuh"

namespace gr {

gr_status dev_alloc(Graph *g, void **p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        set_error("cudaMalloc of %zu bytes failed (out of device memory)", bytes);
        return GR_ERR_OUT_OF_MEMORY;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc", __FILE__, __LINE__);
    g->bytes += (int64_t)bytes;
    return GR_OK;
}

void dev_free_all(Graph *g) {
    void *ptrs[] = {g->R, g->C, g->W, (g->Rt != g->R) ? g->Rt : nullptr,
                    (g->Ct != g->C) ? g->Ct : nullptr, g->visited, g->noin, g->fbuf[0], g->fbuf[1], g->fbuf[2],
                    g->qv[0], g->qv[1], g->qo[0], g->qo[1], g->qr[0], g->qr[1], g->depth_buf, g->pred_buf,
                    g->dist_buf, g->dp, g->stamp, g->farq[0], g->farq[1], g->ctl, g->stats_dev,
                    g->sent, g->ps_best, g->ps_sstamp, g->bc_vert, g->bc_sig, g->bc_delta, g->bc_buf, g->bc_cnt,
                    g->cc_ctl, g->cc_list[0], g->cc_list[1], g->pr_inv, g->pr_acc, g->pr_cnt, g->ph, g->ps_ship, g->CW, g->CWt, g->ell, g->ellw};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (g->stats_host) cudaFreeHost(g->stats_host);
}

// ---------------------------------------------------------------- run totals
// Vertices reached by the last run and the directed edges leaving them (the
// TEPS numerator m_reached, reading A-14), from the run's internal state: the
// visited bitmap of a BFS (every discovery sets its bit; in-degree-0 vertices
// are pre-set from `noin` and only count if they are the source) or the
// packed dist|pred array of an SSSP (dist != UINT32_MAX). Launched by
// gr_get_run_stats, outside any timed region.
__global__ void reached_kernel(int kind, const uint32_t *visited, const uint32_t *noin,
                               const unsigned long long *dp, const int64_t *R, int64_t n, int32_t src,
                               unsigned long long *out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    unsigned long long cnt = 0, edges = 0;
    for (int64_t v = tid; v < n; v += nt) {
        bool r;
        if (kind == 1) {
            const uint32_t bit = 1u << (v & 31);
            r = (visited[v >> 5] & bit) && (!(noin[v >> 5] & bit) || v == src);
        } else {
            r = (dp[v] >> 32) != 0xFFFFFFFFull;
        }
        if (r) { ++cnt; edges += (unsigned long long)(R[v + 1] - R[v]); }
    }
    cnt = warp_sum(cnt);
    edges = warp_sum(edges);
    if ((threadIdx.x & 31) == 0 && (cnt || edges)) {
        atomicAdd(out, cnt);
        atomicAdd(out + 1, edges);
    }
}

gr_status count_reached(Graph *g, int64_t *reached, int64_t *reached_edges) {
    *reached = -1;
    *reached_edges = -1;
    if (g->last_kind == 0) return GR_OK;
    if (g->last_kind == 2 && !g->dp) return GR_OK;
    unsigned long long *d = nullptr;
    GR_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
    GR_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), g->stream));
    const int64_t blocks = (g->n + 255) / 256 < 4096 ? (g->n + 255) / 256 : 4096;
    reached_kernel<<<(unsigned)blocks, 256, 0, g->stream>>>(g->last_kind, g->visited, g->noin, g->dp, g->R,
                                                             g->n, g->last_src, d);
    unsigned long long h[2] = {0, 0};
    GR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    cudaFree(d);
    *reached = (int64_t)h[0];
    *reached_edges = (int64_t)h[1];
    return GR_OK;
}

// ---------------------------------------------------------------- validation
// err[0] = first bad row-offset index (or INT64_MAX), err[1] = first bad edge.
__global__ void validate_kernel(const int64_t *R, const int32_t *C, int64_t n, int64_t m,
                                int64_t ncols, unsigned long long *err) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i <= n; i += nt) {
        bool bad = (i == 0) ? (R[0] != 0) : (R[i] < R[i - 1]);
        if (i == n && R[n] != m) bad = true;
        if (bad) atomicMin(err, (unsigned long long)i);
    }
    for (int64_t e = tid; e < m; e += nt) {
        int32_t c = C[e];
        if (c < 0 || c >= ncols) atomicMin(err + 1, (unsigned long long)e);
    }
}

__global__ void degree_stats_kernel(const int64_t *R, const int64_t *Rt, int64_t n,
                                    unsigned long long *maxdeg, unsigned long long *noniso) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    unsigned long long mx = 0, cnt = 0;
    for (int64_t v = tid; v < n; v += nt) {
        unsigned long long d = (unsigned long long)(R[v + 1] - R[v]);
        mx = d > mx ? d : mx;
        cnt += (Rt[v + 1] > Rt[v]) ? 1 : 0;
    }
    for (int s = 16; s > 0; s >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, s);
        mx = o > mx ? o : mx;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxdeg, mx);
        atomicAdd(noniso, cnt);
    }
}

__global__ void max_weight_kernel(const uint32_t *W, int64_t m, unsigned int *out) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    unsigned int mx = 0;
    for (int64_t e = tid; e < m; e += nt) mx = max(mx, W[e]);
    for (int s = 16; s > 0; s >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// reverse graph: in-degree count, scan, scatter (order within a list is free)
__global__ void indeg_kernel(const int32_t *C, int64_t m, unsigned long long *cnt) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = tid; e < m; e += nt) atomicAdd(cnt + C[e], 1ull);
}

__global__ void csc_scatter_kernel(const int64_t *R, const int32_t *C, int64_t n,
                                   unsigned long long *cursor, int32_t *Ct) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = tid; u < n; u += nt)
        for (int64_t e = R[u]; e < R[u + 1]; ++e) {
            unsigned long long p = atomicAdd(cursor + C[e], 1ull);
            Ct[p] = (int32_t)u;
        }
}

// bitmap of vertices with no in-edge (never discoverable by a traversal)
__global__ void noin_kernel(const int64_t *Rt, int64_t n, uint32_t *noin) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    int64_t nw = (n + 31) / 32;
    for (int64_t w = tid; w < nw; w += nt) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            int64_t v = w * 32 + b;
            if (v < n && Rt[v + 1] == Rt[v]) bits |= 1u << b;
        }
        noin[w] = bits;
    }
}

// ---------------------------------------------------------------- list ordering
__global__ void nbr_key_kernel(const int32_t *L, const int64_t *R, const int32_t *deg, int64_t m, uint32_t *key,
                               int32_t *idx) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = tid; e < m; e += nt) {
        const int32_t u = L[e];
        const int64_t d = deg ? (int64_t)(uint32_t)deg[u] : R[u + 1] - R[u];
        key[e] = 0xFFFFFFFFu - (uint32_t)(d > 0xFFFFFFFFll ? 0xFFFFFFFFll : d);
        idx[e] = (int32_t)e;
    }
}
__global__ void gather_i32_kernel(const int32_t *src, const int32_t *perm, int64_t m, int32_t *dst) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = tid; e < m; e += nt) dst[e] = src[perm[e]];
}

// Sorts each pull list (Ct; C itself when symmetric, W permuted alongside) by
// neighbour out-degree, descending (segmented radix sort, one segment per row).
// deg: optional DEVICE out-degree array indexed by column id (a partition's
// columns are global ids, so its own R cannot give the neighbour's degree).
gr_status sort_lists_by_degree(Graph *g, cudaStream_t s, int blocks, const int32_t *deg) {
    const int64_t m = g->m, n = g->n;
    int32_t *L = g->Ct;
    uint32_t *k0 = nullptr, *k1 = nullptr;
    int32_t *v0 = nullptr, *v1 = nullptr;
    void *tbuf = nullptr;
    size_t tb = 0;
    gr_status st = GR_OK;
    auto fail = [&](cudaError_t e, const char *what) {
        st = cuda_fail(e, what, __FILE__, __LINE__);
        return st;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&k0, m * 4)) || (e = cudaMalloc(&k1, m * 4)) || (e = cudaMalloc(&v0, m * 4)) ||
        (e = cudaMalloc(&v1, m * 4))) {
        fail(e, "cudaMalloc (list sort)");
        goto done;
    }
    nbr_key_kernel<<<blocks, 256, 0, s>>>(L, g->R, deg, m, k0, v0);
    count_launch();
    if ((e = cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, k0, k1, v0, v1, m, n, g->Rt, g->Rt + 1, s))) {
        fail(e, "segmented sort (size)");
        goto done;
    }
    if ((e = cudaMalloc(&tbuf, tb))) { fail(e, "cudaMalloc (sort temp)"); goto done; }
    if ((e = cub::DeviceSegmentedSort::StableSortPairs(tbuf, tb, k0, k1, v0, v1, m, n, g->Rt, g->Rt + 1, s))) {
        fail(e, "segmented sort");
        goto done;
    }
    // permute: L and, for a symmetric graph (L == C), the weights
    gather_i32_kernel<<<blocks, 256, 0, s>>>(L, v1, m, (int32_t *)k0);
    if ((e = cudaMemcpyAsync(L, k0, m * 4, cudaMemcpyDeviceToDevice, s))) { fail(e, "copy"); goto done; }
    if (g->W && L == g->C) {
        gather_i32_kernel<<<blocks, 256, 0, s>>>((const int32_t *)g->W, v1, m, (int32_t *)k0);
        if ((e = cudaMemcpyAsync(g->W, k0, m * 4, cudaMemcpyDeviceToDevice, s))) { fail(e, "copy"); goto done; }
        count_launch();
    }
    count_launch();
    if ((e = cudaStreamSynchronize(s))) fail(e, "sync (list sort)");
done:
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tbuf);
    return st;
}

// Bounded-degree adjacency (gr_internal.cuh Graph::ell / ellw): every
// out-degree <= 4, ids < 2^28. Slot k of vertex v: (C[R[v]+k] << 3) | deg(C[R[v]+k]).
__global__ void build_ell_kernel(const int64_t *R, const int32_t *C, const uint32_t *W, int64_t n,
                                 int4 *ell, int4 *ellw) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nt) {
        const int64_t r0 = R[v];
        const int d = (int)(R[v + 1] - r0);
        int s[4], id[4], wt[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            s[k] = -1; id[k] = -1; wt[k] = 0;
            if (k < d) {
                const int32_t w = C[r0 + k];
                const int dw = (int)(R[w + 1] - R[w]);
                s[k] = (w << 3) | dw;
                id[k] = w;
                wt[k] = W ? (int)((W[r0 + k] << 3) | (uint32_t)dw) : 0;
            }
        }
        ell[v] = make_int4(s[0], s[1], s[2], s[3]);
        if (ellw) {
            ellw[2 * v] = make_int4(id[0], id[1], id[2], id[3]);
            ellw[2 * v + 1] = make_int4(wt[0], wt[1], wt[2], wt[3]);
        }
    }
}

// Packed SSSP edge stream: CW[e] = (C[e] << 7) | W[e] (sssp.cu RelaxOpT<true>).
__global__ void pack_cw_kernel(const int32_t *C, const uint32_t *W, int64_t m, uint32_t *CW) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = tid; e < m; e += nt) CW[e] = ((uint32_t)C[e] << 7) | W[e];
}

// Weighted in-lists for pull SSSP steps (sssp.cu): CWt[Rt[v] ..) holds
// (u << 7) | w(u, v) for every edge (u, v) -- the transpose of CW, so it is
// right for any weights (a symmetric structure need not carry symmetric
// weights). One warp per source row; the order inside an in-list is free.
__global__ void scatter_cwt_kernel(const int64_t *R, const uint32_t *CW, int64_t n,
                                   unsigned long long *cursor, uint32_t *CWt) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned l = threadIdx.x & 31;
    for (int64_t u = gw; u < n; u += nw)
        for (int64_t e = R[u] + l; e < R[u + 1]; e += 32) {
            const uint32_t x = CW[e];
            const unsigned long long p = atomicAdd(cursor + (x >> 7), 1ull);
            CWt[p] = ((uint32_t)u << 7) | (x & 127u);
        }
}

gr_status build_pull_weights(Graph *g) {
    if (g->CWt || !g->CW) return GR_OK;  // no packed edge stream: no pull SSSP
    gr_status st = dev_alloc(g, (void **)&g->CWt, g->m * sizeof(uint32_t) + 16);
    if (st != GR_OK) return st;
    unsigned long long *cur = nullptr;
    GR_CUDA(cudaMalloc((void **)&cur, (g->n + 1) * sizeof(unsigned long long)));
    GR_CUDA(cudaMemcpyAsync(cur, g->Rt, g->n * sizeof(int64_t), cudaMemcpyDeviceToDevice, g->stream));
    scatter_cwt_kernel<<<g->num_sms * 8, 256, 0, g->stream>>>(g->R, g->CW, g->n, cur, g->CWt);
    count_launch();
    cudaError_t e = cudaStreamSynchronize(g->stream);
    cudaFree(cur);
    if (e != cudaSuccess) return cuda_fail(e, "scatter_cwt_kernel", __FILE__, __LINE__);
    return GR_OK;
}

// Pull head (pull.cuh): per vertex its first in-list entry -- the highest-
// degree in-neighbour once lists are ordered -- and its in-degree, so a pull
// step resolves most candidates with one 8-byte load per vertex instead of
// a row-offset load followed by a dependent random load into Ct.
__global__ void pull_head_kernel(const int64_t *Rt, const int32_t *Ct, int64_t n, int2 *ph) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) {
        const int64_t b = Rt[v], d = Rt[v + 1] - b;
        ph[v] = make_int2(d > 0 ? Ct[b] : -1, (int)d);
    }
}

gr_status build_pull_head(Graph *g) {
    if (g->m >= (1ll << 31)) return GR_OK;  // a degree might not fit the int32 field: no head
    if (!g->ph) {
        gr_status st = dev_alloc(g, (void **)&g->ph, g->n * sizeof(int2));
        if (st != GR_OK) return st;
    }
    pull_head_kernel<<<g->num_sms * 8, 256, 0, g->stream>>>(g->Rt, g->Ct, g->n, g->ph);
    count_launch();
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

static bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static int bits_for(int64_t x) {  // smallest S with x < 2^S
    int s = 1;
    while (s < 62 && (x >> s) != 0) ++s;
    return s;
}

gr_status graph_create(int64_t n, int64_t m, const int64_t *R, const int32_t *C, const uint32_t *W,
                       uint32_t flags, int device, void *stream, Graph **out, int64_t ncols) {
    if (!out) { set_error("out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    *out = nullptr;
    if (n <= 0 || n > 0x7fffffffLL) { set_error("n=%lld must be in [1, 2^31-1]", (long long)n); return GR_ERR_INVALID_ARGUMENT; }
    if (ncols < 0) ncols = n;  // partitions: columns are global ids in [0, n_global)
    if (ncols != n) flags |= GR_SYMMETRIC;  // no CSC for a partition (push only)
    if (m < 0) { set_error("m=%lld < 0", (long long)m); return GR_ERR_INVALID_ARGUMENT; }
    if (!R || (m > 0 && !C)) { set_error("row_offsets / col_indices is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    GR_CUDA(cudaSetDevice(device));
    Graph *g = new Graph();
    g->device = device;
    g->stream = (cudaStream_t)stream;
    g->n = n; g->m = m;
    g->symmetric = (flags & GR_SYMMETRIC) != 0;
    g->has_w = (W != nullptr) || m == 0;  // m = 0: no weight is ever read
    GR_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
    gr_status st;
#define TRY(x) do { st = (x); if (st != GR_OK) { dev_free_all(g); delete g; return st; } } while (0)
#define TRYC(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { st = cuda_fail(e_, #x, __FILE__, __LINE__); dev_free_all(g); delete g; return st; } } while (0)
    cudaStream_t s = g->stream;
    TRY(dev_alloc(g, (void **)&g->R, (n + 1) * sizeof(int64_t)));
    // +16 B: the 16-byte cp.async chunks of the advance may read up to 12 B past
    // the last list (values unused)
    TRY(dev_alloc(g, (void **)&g->C, m * sizeof(int32_t) + 16));
    TRYC(cudaMemcpyAsync(g->R, R, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, s));
    if (m) TRYC(cudaMemcpyAsync(g->C, C, m * sizeof(int32_t), cudaMemcpyDefault, s));
    if (W) {
        TRY(dev_alloc(g, (void **)&g->W, m * sizeof(uint32_t) + 16));
        if (m) TRYC(cudaMemcpyAsync(g->W, W, m * sizeof(uint32_t), cudaMemcpyDefault, s));
    }
    unsigned long long *tmp = nullptr;  // 4 scratch words
    TRY(dev_alloc(g, (void **)&tmp, 8 * sizeof(unsigned long long)));
    g->bytes -= 8 * sizeof(unsigned long long);
    const int blocks = g->num_sms * 8;
    if (flags & GR_VALIDATE) {
        unsigned long long init[2] = {~0ull, ~0ull}, res[2];
        TRYC(cudaMemcpyAsync(tmp, init, sizeof(init), cudaMemcpyHostToDevice, s));
        validate_kernel<<<blocks, 256, 0, s>>>(g->R, g->C, n, m, ncols, tmp);
        count_launch();
        TRYC(cudaMemcpyAsync(res, tmp, sizeof(res), cudaMemcpyDeviceToHost, s));
        TRYC(cudaStreamSynchronize(s));
        if (res[0] != ~0ull || res[1] != ~0ull) {
            int64_t hv[2] = {0, 0};
            if (res[0] != ~0ull) {
                int64_t i = (int64_t)res[0];
                TRYC(cudaMemcpy(hv, g->R + (i > 0 ? i - 1 : 0), (i > 0 ? 2 : 1) * sizeof(int64_t),
                                cudaMemcpyDeviceToHost));
                if (i == 0) set_error("R[0]=%lld != 0", (long long)hv[0]);
                else if (hv[1] < hv[0]) set_error("R[%lld]=%lld < R[%lld]=%lld", (long long)i, (long long)hv[1], (long long)(i - 1), (long long)hv[0]);
                else set_error("R[%lld]=%lld != m=%lld", (long long)i, (long long)hv[1], (long long)m);
            } else {
                int32_t c;
                TRYC(cudaMemcpy(&c, g->C + res[1], sizeof(int32_t), cudaMemcpyDeviceToHost));
                set_error("C[%llu]=%d not in [0, n=%lld)", res[1], c, (long long)ncols);
            }
            cudaFree(tmp);
            dev_free_all(g);
            delete g;
            return GR_ERR_INVALID_GRAPH;
        }
    }
    if (g->symmetric) {
        g->Rt = g->R;
        g->Ct = g->C;
    } else {
        TRY(dev_alloc(g, (void **)&g->Rt, (n + 1) * sizeof(int64_t)));
        TRY(dev_alloc(g, (void **)&g->Ct, m * sizeof(int32_t)));
        unsigned long long *cnt = nullptr;
        TRY(dev_alloc(g, (void **)&cnt, (n + 1) * sizeof(unsigned long long)));
        g->bytes -= (n + 1) * sizeof(unsigned long long);
        TRYC(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(unsigned long long), s));
        indeg_kernel<<<blocks, 256, 0, s>>>(g->C, m, cnt + 1);
        count_launch();
        size_t tb = 0;
        TRYC(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt + 1, (unsigned long long *)g->Rt + 1, (int)n, s));
        void *tbuf = nullptr;
        TRYC(cudaMalloc(&tbuf, tb));
        TRYC(cub::DeviceScan::InclusiveSum(tbuf, tb, cnt + 1, (unsigned long long *)g->Rt + 1, (int)n, s));
        TRYC(cudaMemsetAsync(g->Rt, 0, sizeof(int64_t), s));
        TRYC(cudaMemcpyAsync(cnt, g->Rt, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        csc_scatter_kernel<<<blocks, 256, 0, s>>>(g->R, g->C, n, cnt, g->Ct);
        count_launch(2);
        TRYC(cudaStreamSynchronize(s));
        cudaFree(tbuf);
        cudaFree(cnt);
    }
    if (!(flags & GR_KEEP_ORDER) && ncols == n && m > 0 && m < (1ll << 31)) {
        // Symmetric graph: the pull lists get their own copy (Ct != C), so the
        // push lists keep the caller's order -- usually ascending neighbour id,
        // which makes the 32 culling probes of one warp into a long list share
        // a few bitmap lines (a hub's sorted neighbours are dense in id space).
        if (g->Ct == g->C && env_int("GR_SPLIT_ORDER", 1)) {
            TRY(dev_alloc(g, (void **)&g->Ct, m * sizeof(int32_t)));
            TRYC(cudaMemcpyAsync(g->Ct, g->C, m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        }
        // Order every in-list (the lists a pull step scans) by the out-degree of
        // the neighbour, descending: the early exit of the bottom-up sweep finds
        // a frontier parent sooner (measured: C3 -20%, C5 -19% per BFS). Any
        // order is a valid CSR; results are unchanged.
        st = sort_lists_by_degree(g, s, blocks, nullptr);
        if (st != GR_OK) { dev_free_all(g); delete g; return st; }
    }
    {
        unsigned long long zero[4] = {0, 0, 0, 0}, res[4];
        TRYC(cudaMemcpyAsync(tmp, zero, sizeof(zero), cudaMemcpyHostToDevice, s));
        degree_stats_kernel<<<blocks, 256, 0, s>>>(g->R, g->Rt, n, tmp, tmp + 1);
        count_launch();
        if (W && m) {
            max_weight_kernel<<<blocks, 256, 0, s>>>(g->W, m, (unsigned int *)(tmp + 2));
            count_launch();
        }
        TRYC(cudaMemcpyAsync(res, tmp, sizeof(res), cudaMemcpyDeviceToHost, s));
        TRYC(cudaStreamSynchronize(s));
        g->max_deg = (int64_t)res[0];
        g->nonisolated = (int64_t)res[1];
        g->max_w = (uint32_t)(res[2] & 0xffffffffu);
    }
    cudaFree(tmp);

    // per-run scratch for BFS (SSSP scratch is allocated on first use)
    const int64_t nw = (n + 31) / 32;
    TRY(dev_alloc(g, (void **)&g->visited, nw * sizeof(uint32_t)));
    TRY(dev_alloc(g, (void **)&g->noin, nw * sizeof(uint32_t)));
    noin_kernel<<<blocks, 256, 0, s>>>(g->Rt, n, g->noin);
    count_launch();
    TRYC(cudaGetLastError());
    for (int i = 0; i < 3; ++i) TRY(dev_alloc(g, (void **)&g->fbuf[i], nw * sizeof(uint32_t)));
    for (int i = 0; i < 2; ++i) {
        // 2n: room for the duplicates of idempotent (atomic-free) discovery
        TRY(dev_alloc(g, (void **)&g->qv[i], 2 * n * sizeof(int32_t)));
        TRY(dev_alloc(g, (void **)&g->qo[i], 2 * n * sizeof(int64_t)));
        TRY(dev_alloc(g, (void **)&g->qr[i], 2 * n * sizeof(int64_t)));
    }
    if (ncols == n) TRY(build_pull_head(g));  // partitions: after the global list order (pbfs.cu)
    // SSSP edge stream with the weight packed into the column word (4 bytes per
    // relaxed edge instead of 8): ids below 2^25 and weights <= 127 (the
    // paper's are integers 1..64)
    if (W && m > 0 && ncols < (1ll << 25) && g->max_w <= 127 && env_int("GR_PACK_W", 1)) {
        TRY(dev_alloc(g, (void **)&g->CW, m * sizeof(uint32_t) + 16));
        pack_cw_kernel<<<blocks, 256, 0, s>>>(g->C, g->W, m, g->CW);
        count_launch();
        TRYC(cudaGetLastError());
    }
    // Bounded-degree adjacency for high-diameter, low-degree graphs (C4): a
    // push step then costs one aligned 16-B load per frontier vertex and no
    // row-offset lookup per discovered vertex.
    if (ncols == n && m > 0 && g->max_deg <= 4 && n < (1ll << 28) && env_int("GR_ELL", 1)) {
        TRY(dev_alloc(g, (void **)&g->ell, n * sizeof(int4)));
        if (W && g->max_w < (1u << 28)) TRY(dev_alloc(g, (void **)&g->ellw, 2 * n * sizeof(int4)));
        build_ell_kernel<<<blocks, 256, 0, s>>>(g->R, g->C, W ? g->W : nullptr, n, g->ell, g->ellw);
        count_launch();
        TRYC(cudaGetLastError());
    }
    g->pack_shift = bits_for(2 * n + 1);
    TRY(dev_alloc(g, (void **)&g->ctl, sizeof(Ctl)));
    TRYC(cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), s));
    TRY(dev_alloc(g, (void **)&g->stats_dev, kMaxStatRecords * sizeof(gr_level_stats)));
    TRYC(cudaMallocHost((void **)&g->stats_host, kMaxStatRecords * sizeof(gr_level_stats)));
    TRYC(cudaStreamSynchronize(s));
#undef TRY
#undef TRYC
    *out = g;
    return GR_OK;
}

bool ptr_on_device(const void *p) { return is_device_ptr(p); }

}  // namespace gr
