// cc.cu -- connected components by hooking + pointer jumping on an edge
// frontier (paper §5.4).
//
// Paper: "Gunrock uses a filter operator on an edge frontier to implement
// hooking. The frontier starts with all edges and during each iteration, one
// end vertex of each edge in the frontier tries to assign its component ID to
// the other vertex, and the filter step removes the edge whose two end
// vertices have the same component ID ... then proceed to pointer-jumping,
// where a filter operator on vertices assigns the component ID of each vertex
// to its parent's component ID until it reaches the root".
//
// Reading A-22: hooking always points the larger root at the
// smaller one (atomicMin), instead of Soman's alternating direction
// (P:1001-1003): every pointer then decreases, the forest is acyclic by
// construction and the converged root of a component is its SMALLEST vertex
// id -- a canonical labelling, so parity with the oracle is bit-exact.
// Iteration: hook over the edge frontier (survivors: endpoints with different
// roots) -> full pointer jumping (every vertex to its root) -> repeat until
// no edge survives. The first two hooking passes read the CSR directly
// through the merge-path advance (no edge list is materialised while almost
// every edge still survives); later passes stream the compacted int2 list.
// Directed input: edges are taken as undirected (weak components).
#include "frontier.cuh"

namespace gr {

bool ptr_on_device(const void *p);

constexpr int kCcBlock = 256;

// Every vertex as a frontier: entry j = vertex j, degree prefix = R itself.
struct AllVertexFrontier {
    const int64_t *R;
    int64_t F, E;
    __device__ __forceinline__ int64_t off(int64_t i) const { return __ldg(R + i); }
    __device__ __forceinline__ void load(int64_t j, int32_t &v, int64_t &o, int64_t &rs, int64_t &end) const {
        v = (int32_t)j;
        o = __ldg(R + j);
        rs = o;
        end = (j + 1 < F) ? __ldg(R + j + 1) : E;
    }
};

// Hook one edge: roots a = comp[u], b = comp[v]; if different, the larger
// root is pointed at the smaller one. Returns true if the edge survives the
// filter (its endpoints were in different trees when it was read).
__device__ __forceinline__ bool cc_hook_ab(int32_t *comp, int32_t a, int32_t b) {
    if (a == b) return false;
    atomicMin(comp + (a > b ? a : b), a > b ? b : a);
    return true;
}
__device__ __forceinline__ bool cc_hook(int32_t *comp, int32_t u, int32_t v) {
    return cc_hook_ab(comp, __ldcg(comp + u), __ldcg(comp + v));
}

// warp-aggregated append of surviving edges (filter output)
__device__ __forceinline__ void cc_append(bool keep, int32_t u, int32_t v, int2 *out, unsigned long long *cnt,
                                          unsigned long long *changed, int64_t cap) {
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (!mask) return;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if ((int)lane_id() == leader) {
        if (out) base = atomicAdd(cnt, (unsigned long long)__popc(mask));
        *changed = 1ull;
    }
    if (!out) return;
    base = __shfl_sync(0xffffffffu, base, leader);
    const unsigned long long pos = base + __popc(mask & lanemask_lt());
    if (keep && pos < (unsigned long long)cap) out[pos] = make_int2(u, v);
    else if (keep) changed[2] = 1ull;  // list overflow: a GR_SYMMETRIC graph that is not symmetric
}

struct CcHookOp {
    int32_t *comp;
    int2 *out;                   // null: hook only, no edge list
    unsigned long long *cnt;
    unsigned long long *changed;
    bool half;                   // symmetric graph: each undirected edge once (u < v)
    int64_t cap;                 // edge-list capacity

    // comp[u] of the list's source, loaded once per window (it may be hooked
    // during the pass: a stale label is still a vertex of u's tree, and the
    // edge then survives and is hooked again next pass)
    __device__ __forceinline__ unsigned long long entry(int32_t v) { return (uint32_t)__ldcg(comp + v); }

    template <int U, class T5>
    __device__ __forceinline__ void edges(const bool *ok, const int32_t *src, const unsigned long long *pay,
                                          const int32_t *dst, const T5 *) {
        int32_t b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = (ok[u] && (!half || src[u] < dst[u])) ? __ldcg(comp + dst[u]) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool keep = b[u] >= 0 && cc_hook_ab(comp, (int32_t)pay[u], b[u]);
            cc_append(keep, src[u], dst[u], out, cnt, changed, cap);
        }
    }
};

__global__ void cc_init_kernel(int32_t *comp, int64_t n) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) comp[v] = (int32_t)v;
}

__global__ void __launch_bounds__(kCcBlock) cc_hook_csr_kernel(const int64_t *R, const int32_t *C, int64_t n,
                                                               int64_t m, CcHookOp op) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    AllVertexFrontier fr{R, n, m};
    expand_lb(fr, C, gw, nw, op);
}

__global__ void __launch_bounds__(kCcBlock) cc_hook_list_kernel(int32_t *comp, const int2 *in, int64_t k, int2 *out,
                                                                unsigned long long *cnt,
                                                                unsigned long long *changed, int64_t cap) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = tid - lane_id(); base < k; base += nt) {  // warp-uniform trip count
        const int64_t j = base + lane_id();
        int2 e = make_int2(0, 0);
        bool keep = false;
        if (j < k) {
            e = __ldcs(in + j);
            keep = cc_hook(comp, e.x, e.y);
        }
        cc_append(keep, e.x, e.y, out, cnt, changed, cap);
    }
}

// pointer jumping: every vertex to its root (filter on vertices)
__global__ void cc_jump_kernel(int32_t *comp, int64_t n) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < n; v += nt) {
        int32_t c = comp[v];
        for (;;) {
            const int32_t p = __ldcg(comp + c);
            if (p == c) break;
            c = p;
        }
        comp[v] = c;
    }
}

__global__ void cc_count_kernel(const int32_t *comp, int64_t n, unsigned long long *count) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    unsigned long long k = 0;
    for (int64_t v = tid; v < n; v += nt) k += comp[v] == (int32_t)v;
    k = warp_sum<unsigned long long>(k);
    if (lane_id() == 0 && k) atomicAdd(count, k);
}

}  // namespace gr

using namespace gr;

extern "C" {

gr_status gr_cc(gr_graph *h, int32_t *comp_out, int64_t *num_components) {
    Graph *g = (Graph *)h;
    if (!g || !comp_out) { set_error("graph or comp_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    if (g->part) { set_error("gr_cc needs a whole (unpartitioned) graph"); return GR_ERR_INVALID_ARGUMENT; }
    GR_CUDA(cudaSetDevice(g->device));
    if (g->pending && gr_graph_sync(h) != GR_OK) return GR_ERR_OVERFLOW;
    gr_status st;
    const int64_t n = g->n, m = g->m;
    const bool half = g->symmetric;
    const int64_t cap = half ? m / 2 + 1 : m + 1;  // edges a pass can keep
    if (!g->cc_ctl) {
        if ((st = dev_alloc(g, (void **)&g->cc_ctl, 4 * sizeof(unsigned long long))) != GR_OK) return st;
    }
    const bool dev_out = ptr_on_device(comp_out);
    int32_t *comp = comp_out;
    if (!dev_out) {
        if (!g->depth_buf && (st = dev_alloc(g, (void **)&g->depth_buf, n * sizeof(int32_t))) != GR_OK) return st;
        comp = g->depth_buf;
    }
    cudaStream_t s = g->stream;
    const int grid = g->num_sms * 8;
    unsigned long long *cnt = g->cc_ctl, *changed = g->cc_ctl + 1, *count = g->cc_ctl + 2;
    int launches = 0;
    cc_init_kernel<<<g->num_sms * 4, 256, 0, s>>>(comp, n);
    ++launches;
    int2 *list[2] = {nullptr, nullptr};
    int64_t k = -1;      // edges in the current list (-1: hook from the CSR)
    int cur = 0, passes = 0;
    for (;;) {
        GR_CUDA(cudaMemsetAsync(g->cc_ctl, 0, 2 * sizeof(unsigned long long), s));
        if (passes == 0) GR_CUDA(cudaMemsetAsync(g->cc_ctl + 3, 0, sizeof(unsigned long long), s));
        if (k < 0) {
            // CSR passes: the first hooks only; the second also writes the survivors
            int2 *out = nullptr;
            if (passes >= 1) {
                if (!g->cc_list[0]) {
                    if ((st = dev_alloc(g, (void **)&g->cc_list[0], cap * sizeof(int2))) != GR_OK ||
                        (st = dev_alloc(g, (void **)&g->cc_list[1], cap * sizeof(int2))) != GR_OK)
                        return st;
                }
                list[0] = g->cc_list[0];
                list[1] = g->cc_list[1];
                out = list[cur];
            }
            CcHookOp op{comp, out, cnt, changed, half, cap};
            cc_hook_csr_kernel<<<grid, kCcBlock, 0, s>>>(g->R, g->C, n, m, op);
        } else {
            cc_hook_list_kernel<<<grid, kCcBlock, 0, s>>>(comp, list[cur], k, list[cur ^ 1], cnt, changed, cap);
            cur ^= 1;
        }
        cc_jump_kernel<<<g->num_sms * 8, 256, 0, s>>>(comp, n);
        launches += 2;
        unsigned long long hc[4] = {0, 0, 0, 0};
        GR_CUDA(cudaMemcpyAsync(hc, g->cc_ctl, sizeof(hc), cudaMemcpyDeviceToHost, s));
        GR_CUDA(cudaStreamSynchronize(s));
        ++passes;
        if (hc[3]) {
            set_error("edge frontier overflow: the graph was created GR_SYMMETRIC but is not symmetric");
            return GR_ERR_INVALID_GRAPH;
        }
        if (!hc[1]) break;                 // no edge crossed two trees: converged
        if (passes >= 2) k = (int64_t)hc[0];
        if (k == 0) break;
    }
    if (num_components) {
        GR_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
        cc_count_kernel<<<g->num_sms * 4, 256, 0, s>>>(comp, n, count);
        ++launches;
        unsigned long long c = 0;
        GR_CUDA(cudaMemcpyAsync(&c, count, sizeof(c), cudaMemcpyDeviceToHost, s));
        GR_CUDA(cudaStreamSynchronize(s));
        *num_components = (int64_t)c;
    }
    if (!dev_out) GR_CUDA(cudaMemcpyAsync(comp_out, comp, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    GR_CUDA(cudaGetLastError());
    GR_CUDA(cudaStreamSynchronize(s));
    count_launch(launches);
    g->last_launches = launches;
    g->stats_levels = passes;
    g->stats_records = -1;
    return GR_OK;
}

}  // extern "C"
