// abi.cu -- the extern "C" boundary declared in include/gr.h.
// Argument checking, host/device output handling, scratch allocation and the
// per-run bookkeeping live here; every step of the path runs in the kernels
// of bfs.cu / sssp.cu.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>

#include "gr_internal.cuh"

namespace gr {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

gr_status cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error("CUDA error %d (%s: %s) in %s at %s:%d", (int)e, cudaGetErrorName(e),
              cudaGetErrorString(e), what, file, line);
    return e == cudaErrorMemoryAllocation ? GR_ERR_OUT_OF_MEMORY : GR_ERR_CUDA;
}

void count_launch(int k) { g_launches.fetch_add((unsigned long long)k); }

int64_t env_int(const char *name, int64_t dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoll(v) : dflt;
}

gr_status graph_create(int64_t n, int64_t m, const int64_t *R, const int32_t *C, const uint32_t *W,
                       uint32_t flags, int device, void *stream, Graph **out, int64_t ncols = -1);
bool ptr_on_device(const void *p);
gr_status run_bfs(Graph *g, int32_t src, int32_t *depth, int32_t *pred, const gr_bfs_opts &o,
                  int *launches);
gr_status run_sssp(Graph *g, int32_t src, uint32_t *dist, int32_t *pred, uint64_t delta, int32_t direction,
                   double alpha, int *launches);
gr_status pbfs_collective(Graph *g, int64_t src, int32_t *depth_out, int32_t *pred_out, const gr_bfs_opts &o);
gr_status psssp_collective(Graph *g, int64_t src, uint32_t *dist_out, int32_t *pred_out, uint32_t delta);

static gr_status finish_run(Graph *g) {
    GR_CUDA(cudaGetLastError());
    unsigned long long levels = 0, overflow = 0;
    GR_CUDA(cudaMemcpyAsync(&levels, &g->ctl->levels, sizeof(levels), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemcpyAsync(&overflow, &g->ctl->overflow, sizeof(overflow), cudaMemcpyDeviceToHost, g->stream));
    GR_CUDA(cudaMemsetAsync(&g->ctl->sticky, 0, sizeof(unsigned long long), g->stream));
    GR_CUDA(cudaStreamSynchronize(g->stream));
    g->stats_levels = (int)levels;
    g->stats_records = (int)(levels < (unsigned long long)kMaxStatRecords ? levels : kMaxStatRecords);
    g->stats_records = -1 - g->stats_records;  // lazily copied by gr_get_run_stats
    if (overflow) {
        set_error("a frontier queue exceeded its capacity");
        return GR_ERR_OVERFLOW;
    }
    return GR_OK;
}

static gr_status ensure(Graph *g, void **p, size_t bytes) {
    if (*p) return GR_OK;
    return dev_alloc(g, p, bytes);
}

}  // namespace gr

using namespace gr;

extern "C" {

// debug only (not in gr.h): the raw overflow word of the last run (low byte =
// which queue: 1 frontier/near, 2 far; bits 8.. = the slot count requested)
unsigned long long gr_debug_overflow(gr_graph *h) {
    unsigned long long v = 0;
    cudaMemcpy(&v, &((Graph *)h)->ctl->overflow, sizeof(v), cudaMemcpyDeviceToHost);
    return v;
}

const char *gr_last_error(void) { return g_err; }

uint64_t gr_kernel_launch_count(void) { return g_launches.load(); }

const char *gr_version(void) { return "gr_b200 0.1 sm_100a"; }


gr_status gr_graph_create(int64_t n, int64_t m, const int64_t *row_offsets, const int32_t *col_indices,
                          const uint32_t *weights, uint32_t flags, int device, void *cuda_stream,
                          gr_graph **out) {
    g_err[0] = 0;
    Graph *g = nullptr;
    gr_status st = graph_create(n, m, row_offsets, col_indices, weights, flags, device, cuda_stream, &g);
    if (out) *out = (gr_graph *)g;
    return st;
}

gr_status gr_graph_destroy(gr_graph *h) {
    if (!h) return GR_OK;
    Graph *g = (Graph *)h;
    cudaSetDevice(g->device);
    cudaStreamSynchronize(g->stream);
    if (g->comm) {
        if (g->comm->group && g->comm->group->graphs[g->comm->rank] == g) g->comm->group->graphs[g->comm->rank] = nullptr;
        comm_sym_free(g);
    }
    dev_free_all(g);
    delete g;
    return GR_OK;
}

gr_status gr_graph_set_stream(gr_graph *h, void *stream) {
    if (!h) { set_error("graph is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    ((Graph *)h)->stream = (cudaStream_t)stream;
    return GR_OK;
}

gr_status gr_graph_info_get(const gr_graph *h, gr_graph_info *out) {
    if (!h || !out) { set_error("NULL argument"); return GR_ERR_INVALID_ARGUMENT; }
    const Graph *g = (const Graph *)h;
    out->n = g->n; out->m = g->m; out->max_degree = g->max_deg; out->nonisolated = g->nonisolated;
    out->symmetric = g->symmetric; out->has_weights = g->has_w; out->max_weight = g->max_w;
    out->device = g->device; out->device_bytes = g->bytes;
    out->packed_weights = g->CW != nullptr;
    out->bounded_degree = g->ell != nullptr;
    return GR_OK;
}

static gr_status check_bfs_opts(const gr_bfs_opts &o) {
    if (o.direction < 0 || o.direction > 2 || o.strategy < 0 || o.strategy > 2 || o.switch_rule < 0 ||
        o.switch_rule > 1 || o.idempotent < 0 || o.idempotent > 1 || o.alpha < 0 || o.beta < 0) {
        set_error("invalid gr_bfs_opts");
        return GR_ERR_INVALID_ARGUMENT;
    }
    return GR_OK;
}

// gr_bfs on a graph of gr_graph_create_partitioned: src is a GLOBAL id, the
// outputs cover the owned block; collective over the comm's ranks (pbfs.cu)
static gr_status pbfs_entry(Graph *g, int32_t src, int32_t *depth_out, int32_t *pred_out, const gr_bfs_opts *opts) {
    if (!depth_out) { set_error("depth_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    if (src < 0 || src >= g->n_global) {
        set_error("src=%d not in [0, n=%lld)", src, (long long)g->n_global);
        return GR_ERR_OUT_OF_RANGE;
    }
    gr_bfs_opts o = opts ? *opts : gr_bfs_opts{};
    gr_status st = check_bfs_opts(o);
    if (st != GR_OK) return st;
    return pbfs_collective(g, src, depth_out, pred_out, o);
}

static gr_status bfs_args(gr_graph *h, int32_t src, const int32_t *depth_out, const gr_bfs_opts *opts,
                          gr_bfs_opts *o) {
    if (!h || !depth_out) { set_error("graph or depth_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    Graph *g = (Graph *)h;
    if (src < 0 || src >= g->n) {
        set_error("src=%d not in [0, n=%lld)", src, (long long)g->n);
        return GR_ERR_OUT_OF_RANGE;
    }
    *o = gr_bfs_opts{};
    if (opts) *o = *opts;
    if (o->direction < 0 || o->direction > 2 || o->strategy < 0 || o->strategy > 2 || o->switch_rule < 0 ||
        o->switch_rule > 1 || o->idempotent < 0 || o->idempotent > 1 || o->alpha < 0 || o->beta < 0) {
        set_error("invalid gr_bfs_opts");
        return GR_ERR_INVALID_ARGUMENT;
    }
    GR_CUDA(cudaSetDevice(g->device));
    return GR_OK;
}

gr_status gr_graph_sync(gr_graph *h);

gr_status gr_bfs(gr_graph *h, int32_t src, int32_t *depth_out, int32_t *pred_out, const gr_bfs_opts *opts) {
    g_err[0] = 0;
    gr_bfs_opts o;
    if (h && ((Graph *)h)->comm) return pbfs_entry((Graph *)h, src, depth_out, pred_out, opts);
    gr_status st = bfs_args(h, src, depth_out, opts, &o);
    if (st != GR_OK) return st;
    Graph *g = (Graph *)h;
    if (g->pending && (st = gr_graph_sync(h)) != GR_OK) return st;
    const bool dev_depth = ptr_on_device(depth_out);
    const bool dev_pred = pred_out && ptr_on_device(pred_out);
    int32_t *depth = depth_out, *pred = pred_out;
    if (!dev_depth) {
        if ((st = ensure(g, (void **)&g->depth_buf, g->n * sizeof(int32_t))) != GR_OK) return st;
        depth = g->depth_buf;
    }
    if (pred_out && !dev_pred) {
        if ((st = ensure(g, (void **)&g->pred_buf, g->n * sizeof(int32_t))) != GR_OK) return st;
        pred = g->pred_buf;
    }
    int launches = 0;
    if ((st = run_bfs(g, src, depth, pred, o, &launches)) != GR_OK) return st;
    if (!dev_depth)
        GR_CUDA(cudaMemcpyAsync(depth_out, depth, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    if (pred_out && !dev_pred)
        GR_CUDA(cudaMemcpyAsync(pred_out, pred, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    g->last_launches = launches;
    g->last_delta = 0;
    g->last_kind = 1; g->last_src = src; g->reached = -2;
    st = finish_run(g);
    if (st == GR_ERR_OVERFLOW && o.idempotent) {
        // the idempotent queue outgrew its capacity: redo with exactly-once claims
        o.idempotent = 0;
        if ((st = run_bfs(g, src, depth, pred, o, &launches)) != GR_OK) return st;
        if (!dev_depth)
            GR_CUDA(cudaMemcpyAsync(depth_out, depth, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        if (pred_out && !dev_pred)
            GR_CUDA(cudaMemcpyAsync(pred_out, pred, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        g->last_launches += launches;
        st = finish_run(g);
    }
    return st;
}

gr_status gr_bfs_async(gr_graph *h, int32_t src, int32_t *depth_out, int32_t *pred_out,
                       const gr_bfs_opts *opts) {
    g_err[0] = 0;
    if (h && ((Graph *)h)->comm) {
        set_error("gr_bfs_async: a partitioned graph runs collective synchronous gr_bfs calls");
        return GR_ERR_INVALID_ARGUMENT;
    }
    gr_bfs_opts o;
    gr_status st = bfs_args(h, src, depth_out, opts, &o);
    if (st != GR_OK) return st;
    Graph *g = (Graph *)h;
    if (!ptr_on_device(depth_out) || (pred_out && !ptr_on_device(pred_out))) {
        set_error("gr_bfs_async needs device output buffers");
        return GR_ERR_INVALID_ARGUMENT;
    }
    int launches = 0;
    if ((st = run_bfs(g, src, depth_out, pred_out, o, &launches)) != GR_OK) return st;
    GR_CUDA(cudaGetLastError());
    g->last_launches = launches;
    g->last_delta = 0;
    g->last_kind = 1; g->last_src = src; g->reached = -2;
    g->pending++;
    g->pending_kind = 1;
    g->pending_src = src;
    g->pending_out[0] = depth_out;
    g->pending_out[1] = pred_out;
    g->pending_bopts = o;
    return GR_OK;
}

static gr_status sssp_args(gr_graph *h, int32_t src, const uint32_t *dist_out, const gr_sssp_opts *opts,
                           uint64_t *delta_out, gr_sssp_opts *o_out) {
    if (!h || !dist_out) { set_error("graph or dist_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    Graph *g = (Graph *)h;
    if (!g->has_w) { set_error("graph was created without weights"); return GR_ERR_NO_WEIGHTS; }
    if (src < 0 || src >= g->n) {
        set_error("src=%d not in [0, n=%lld)", src, (long long)g->n);
        return GR_ERR_OUT_OF_RANGE;
    }
    if ((unsigned long long)g->max_w * (unsigned long long)(g->n - 1) >= 0xFFFFFFFFull) {
        set_error("max_w=%u * (n-1)=%lld may overflow uint32 distances", g->max_w, (long long)(g->n - 1));
        return GR_ERR_OVERFLOW;
    }
    gr_sssp_opts o{};
    if (opts) o = *opts;
    if (o.strategy < 0 || o.strategy > 2 || o.direction < 0 || o.direction > 2 || o.alpha < 0) {
        set_error("invalid gr_sssp_opts");
        return GR_ERR_INVALID_ARGUMENT;
    }
    *o_out = o;
    uint64_t delta = o.delta;
    if (delta == 0) {
        // auto delta (reading A-10): dense low-diameter graphs want narrow
        // bands (little re-relaxation); sparse high-diameter graphs want wide
        // bands (fewer bulk-synchronous iterations).
        double avg = g->n ? (double)g->m / (double)g->n : 0.0;
        uint64_t mw = g->max_w ? g->max_w : 1;
        // swept on B200: C3 (avg deg 76, w<=64) best at 3 of {1,2,3,4,8,16,32};
        // C4 (avg deg 2.4) best at 2048 of {256..16384}
        delta = avg >= 8.0 ? (mw + 10) / 21 : mw * 32;
        if (delta == 0) delta = 1;
    }
    *delta_out = delta;
    GR_CUDA(cudaSetDevice(g->device));
    gr_status st;
    if ((st = ensure(g, (void **)&g->dp, g->n * sizeof(unsigned long long))) != GR_OK) return st;
    if ((st = ensure(g, (void **)&g->stamp, g->n * sizeof(int32_t))) != GR_OK) return st;
    if (!g->farq[0]) {
        g->far_cap = 2 * g->m + g->n + 1024;
        if ((st = dev_alloc(g, (void **)&g->farq[0], g->far_cap * sizeof(int32_t))) != GR_OK) return st;
        if ((st = dev_alloc(g, (void **)&g->farq[1], g->far_cap * sizeof(int32_t))) != GR_OK) return st;
    }
    return GR_OK;
}

gr_status gr_sssp(gr_graph *h, int32_t src, uint32_t *dist_out, int32_t *pred_out, const gr_sssp_opts *opts) {
    g_err[0] = 0;
    if (h && ((Graph *)h)->comm) {  // partitioned graph: collective over the comm's ranks (psssp.cu)
        Graph *g = (Graph *)h;
        if (!dist_out) { set_error("dist_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
        if (src < 0 || src >= g->n_global) {
            set_error("src=%d not in [0, n=%lld)", src, (long long)g->n_global);
            return GR_ERR_OUT_OF_RANGE;
        }
        gr_sssp_opts o = opts ? *opts : gr_sssp_opts{};
        if (o.strategy < 0 || o.strategy > 2) { set_error("invalid gr_sssp_opts"); return GR_ERR_INVALID_ARGUMENT; }
        return psssp_collective(g, src, dist_out, pred_out, o.delta);
    }
    uint64_t delta = 0;
    gr_sssp_opts so{};
    gr_status st = sssp_args(h, src, dist_out, opts, &delta, &so);
    if (st != GR_OK) return st;
    Graph *g = (Graph *)h;
    if (g->pending && (st = gr_graph_sync(h)) != GR_OK) return st;
    const bool dev_dist = ptr_on_device(dist_out);
    const bool dev_pred = pred_out && ptr_on_device(pred_out);
    uint32_t *dist = dist_out;
    int32_t *pred = pred_out;
    if (!dev_dist) {
        if ((st = ensure(g, (void **)&g->dist_buf, g->n * sizeof(uint32_t))) != GR_OK) return st;
        dist = g->dist_buf;
    }
    if (pred_out && !dev_pred) {
        if ((st = ensure(g, (void **)&g->pred_buf, g->n * sizeof(int32_t))) != GR_OK) return st;
        pred = g->pred_buf;
    }
    int launches = 0;
    if ((st = run_sssp(g, src, dist, pred, delta, so.direction, so.alpha, &launches)) != GR_OK) return st;
    if (!dev_dist)
        GR_CUDA(cudaMemcpyAsync(dist_out, dist, g->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, g->stream));
    if (pred_out && !dev_pred)
        GR_CUDA(cudaMemcpyAsync(pred_out, pred, g->n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    g->last_launches = launches;
    g->last_delta = (uint32_t)(delta > 0xFFFFFFFFull ? 0xFFFFFFFFull : delta);
    g->last_kind = 2; g->last_src = src; g->reached = -2;
    return finish_run(g);
}

gr_status gr_sssp_async(gr_graph *h, int32_t src, uint32_t *dist_out, int32_t *pred_out,
                        const gr_sssp_opts *opts) {
    g_err[0] = 0;
    if (h && ((Graph *)h)->comm) {
        set_error("gr_sssp_async: a partitioned graph runs collective synchronous gr_sssp calls");
        return GR_ERR_INVALID_ARGUMENT;
    }
    uint64_t delta = 0;
    gr_sssp_opts so{};
    gr_status st = sssp_args(h, src, dist_out, opts, &delta, &so);
    if (st != GR_OK) return st;
    Graph *g = (Graph *)h;
    if (!ptr_on_device(dist_out) || (pred_out && !ptr_on_device(pred_out))) {
        set_error("gr_sssp_async needs device output buffers");
        return GR_ERR_INVALID_ARGUMENT;
    }
    int launches = 0;
    if ((st = run_sssp(g, src, dist_out, pred_out, delta, so.direction, so.alpha, &launches)) != GR_OK) return st;
    GR_CUDA(cudaGetLastError());
    g->last_launches = launches;
    g->last_delta = (uint32_t)(delta > 0xFFFFFFFFull ? 0xFFFFFFFFull : delta);
    g->last_kind = 2; g->last_src = src; g->reached = -2;
    g->pending++;
    g->pending_kind = 2;
    g->pending_src = src;
    g->pending_out[0] = dist_out;
    g->pending_out[1] = pred_out;
    return GR_OK;
}

gr_status gr_graph_sync(gr_graph *h) {
    if (!h) { set_error("graph is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    Graph *g = (Graph *)h;
    GR_CUDA(cudaSetDevice(g->device));
    unsigned long long sticky = 0;
    GR_CUDA(cudaMemcpyAsync(&sticky, &g->ctl->sticky, sizeof(sticky), cudaMemcpyDeviceToHost, g->stream));
    const int np = g->pending;
    g->pending = 0;
    gr_status st = finish_run(g);  // synchronises; stats of the last run; clears sticky
    if (np == 0) return GR_OK;
    if (st == GR_OK && sticky) {
        set_error("a frontier queue exceeded its capacity in one of %d asynchronous runs", np);
        st = GR_ERR_OVERFLOW;
    }
    if (st == GR_ERR_OVERFLOW && np == 1 && g->pending_kind == 1 && g->pending_bopts.idempotent) {
        // the one pending idempotent BFS overflowed: redo it with exactly-once claims
        gr_bfs_opts o = g->pending_bopts;
        o.idempotent = 0;
        int launches = 0;
        if ((st = run_bfs(g, g->pending_src, (int32_t *)g->pending_out[0], (int32_t *)g->pending_out[1], o,
                          &launches)) != GR_OK)
            return st;
        g->last_launches += launches;
        st = finish_run(g);
    }
    return st;
}

gr_status gr_get_run_stats(gr_graph *h, gr_run_stats *out) {
    if (!h || !out) { set_error("NULL argument"); return GR_ERR_INVALID_ARGUMENT; }
    Graph *g = (Graph *)h;
    if (g->stats_records < 0) {
        int rec = -1 - g->stats_records;
        if (rec > 0) {
            GR_CUDA(cudaMemcpyAsync(g->stats_host, g->stats_dev, rec * sizeof(gr_level_stats),
                                    cudaMemcpyDeviceToHost, g->stream));
            GR_CUDA(cudaStreamSynchronize(g->stream));
        }
        g->stats_records = rec;
    }
    out->num_levels = g->stats_levels;
    out->num_records = g->stats_records;
    out->levels = g->stats_host;
    if (g->reached == -2) {  // first query since the run: count from the run's state
        gr_status st = count_reached(g, &g->reached, &g->reached_edges);
        if (st != GR_OK) return st;
    }
    out->reached = g->reached;
    out->reached_edges = g->reached_edges;
    out->delta = g->last_delta;
    out->kernel_launches = g->last_launches;
    return GR_OK;
}

}  // extern "C"
