/*
 * gr.h -- C ABI of the B200-native frontier library (BFS / SSSP hot path of
 * Gunrock, Wang et al., PPoPP'16, arXiv 1501.05387).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n;
 * "A-k" = a reading of the paper listed in DESIGN.md "Readings".
 *
 * Conventions for every entry point
 *  - C99, no C++ types, no torch types. Status codes only; no exception
 *    crosses the boundary. On failure gr_last_error() returns a message
 *    (thread-local, valid until the next call on that thread) and outputs are
 *    unspecified.
 *  - Pointers may be host or device memory; the library detects which with
 *    cudaPointerGetAttributes. Device outputs (e.g. a torch tensor's
 *    data_ptr()) are written in place; host outputs are filled by a
 *    device->host copy at the end of the call.
 *  - Every call is synchronous with respect to the host. All device work is
 *    enqueued on the stream given to gr_graph_create (or gr_graph_set_stream).
 *  - One traversal at a time per gr_graph (the scratch space is per graph,
 *    cf. S:177 "A single traversal run is not reentrant"). Distinct graphs are
 *    independent. The library never retains a caller pointer after returning.
 */
#ifndef GR_H_
#define GR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GR_OK = 0,
    GR_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, n <= 0, bad option value        */
    GR_ERR_INVALID_GRAPH = 2,    /* CSR invariant broken; message names the index  */
    GR_ERR_OUT_OF_RANGE = 3,     /* src not in [0, n)                     */
    GR_ERR_NO_WEIGHTS = 4,       /* gr_sssp on a graph created without weights */
    GR_ERR_OVERFLOW = 5,         /* a distance could exceed UINT32_MAX-1 (A-19), or
                                    a queue capacity would be exceeded             */
    GR_ERR_OUT_OF_MEMORY = 6,
    GR_ERR_CUDA = 7,             /* a CUDA runtime error; message has the detail   */
    GR_ERR_NCCL = 8
} gr_status;

typedef struct gr_graph gr_graph; /* opaque; immutable topology after create */

/* gr_graph_create flags */
enum {
    GR_SYMMETRIC = 1u << 0, /* caller asserts (u,v) in E <=> (v,u) in E (the paper's
                               undirected inputs); pull then
                               reads the CSR as its own CSC. Without it the library
                               builds the reverse graph (CSC) on the device (A-18). */
    GR_VALIDATE = 1u << 2,  /* O(n+m) CSR checks on the device:
                               R[0]=0, R non-decreasing, R[n]=m, 0<=C[e]<n.       */
    GR_KEEP_ORDER = 1u << 3 /* keep the caller's neighbour order. By default every
                               in-list is reordered by neighbour degree (descending)
                               so pull steps exit early sooner; for a GR_SYMMETRIC
                               graph that reordered copy is separate (4m bytes more)
                               and the out-lists keep the caller's order (ascending
                               ids make a warp's culling probes share bitmap lines).
                               Results (depth, dist) are unaffected, the parent
                               picked may differ. */
};

/*
 * gr_graph_create -- build the device graph G=(V,E,w_e) from a CSR
 * (§3 "A graph is an ordered pair G=(V,E,w_e,w_v)"
 * "CSR uses a column-indices array, C, ... and a row-offsets array, R").
 *   n            number of vertices, >= 1 (n <= 2^31-1)
 *   m            number of directed edges, >= 0
 *   row_offsets  int64[n+1]: neighbours of v are col_indices[R[v] .. R[v+1])
 *   col_indices  int32[m], each in [0, n). Self-loops and parallel edges are
 *                allowed (BFS ignores them; SSSP takes the minimum weight).
 *   weights      uint32[m] non-negative edge weights w_e, or NULL
 *                for a BFS-only graph (with m = 0 the graph counts as
 *                weighted: no weight is ever read).
 *   flags        GR_SYMMETRIC | GR_VALIDATE
 *   device       CUDA device ordinal the graph lives on
 *   cuda_stream  cudaStream_t to enqueue all work on (NULL = legacy stream)
 *   out          receives the handle
 * All inputs are copied; the caller may free them on return. Graph creation is
 * outside the timed region of every benchmark ("All results
 * ignore transfer time").
 * Errors: GR_ERR_INVALID_ARGUMENT, GR_ERR_INVALID_GRAPH (first bad index named,
 * e.g. "R[17]=5 < R[16]=9" or "C[1234]=70000 >= n"), GR_ERR_OUT_OF_MEMORY,
 * GR_ERR_CUDA.
 */
gr_status gr_graph_create(int64_t n, int64_t m, const int64_t *row_offsets,
                          const int32_t *col_indices, const uint32_t *weights,
                          uint32_t flags, int device, void *cuda_stream,
                          gr_graph **out);

/* Frees all device memory owned by g. NULL is a no-op. */
gr_status gr_graph_destroy(gr_graph *g);

/* Re-targets subsequent work of g to another stream on the same device. */
gr_status gr_graph_set_stream(gr_graph *g, void *cuda_stream);

typedef struct {
    int64_t n, m;
    int64_t max_degree;      /* max out-degree                                  */
    int64_t nonisolated;     /* vertices with in-degree > 0 (pull candidates)   */
    int32_t symmetric;       /* 1 if created with GR_SYMMETRIC                  */
    int32_t has_weights;
    uint32_t max_weight;
    int32_t device;
    int64_t device_bytes;    /* device memory currently owned by the graph      */
    int32_t packed_weights;  /* 1: SSSP streams the packed (C << 7) | W array
                                (n < 2^25, weights <= 127; 4 B per edge)         */
    int32_t bounded_degree;  /* 1: every out-degree <= 4 and n < 2^28: push and
                                relax steps read a 16-B (BFS) / 32-B (SSSP, if
                                weighted) per-vertex adjacency record instead of
                                R + C (road-like graphs)           */
} gr_graph_info;

gr_status gr_graph_info_get(const gr_graph *g, gr_graph_info *out);

/*
 * gr_bfs -- breadth-first search from src (§5.1: "BFS initializes
 * its vertex frontier with a single source vertex. On each iteration, it
 * generates a new frontier of vertices with all unvisited neighbor vertices
 * in the current frontier, setting their depths"). Each level is one
 * bulk-synchronous step: a fused advance+filter
 * (push) or a pull advance over in-edges.
 *   src        source vertex in [0, n)
 *   depth_out  int32[n]: hop distance from src following out-edges, -1 when
 *              unreached (A-2). Deterministic.
 *   pred_out   int32[n] or NULL: a valid BFS parent (pred[v] -> v is an edge
 *              and depth[pred[v]] = depth[v]-1), pred[src] = src (A-1), -1 when
 *              unreached. Which valid parent is nondeterministic.
 *   opts       NULL = defaults (all zero fields = defaults)
 * Errors: GR_ERR_OUT_OF_RANGE for src outside [0,n); GR_ERR_INVALID_ARGUMENT.
 */
typedef struct {
    int32_t direction;   /* 0 auto (direction-optimizing), 1 push only, 2 pull only */
    int32_t strategy;    /* 0 auto, 1 thread/warp/CTA (node-granular), 2 merge-path LB
                            over edges (threshold reading A-4)            */
    int32_t idempotent;  /* 0 = exactly-once claim (atomicOr on the visited bitmap,
                            P:800-802); 1 = atomic-free idempotent discovery with
                            culling heuristics (A-5, A-6)    */
    int32_t switch_rule; /* 0 Beamer alpha/beta (default), 1 paper-literal
                            "unvisited < frontier" (A-3)                */
    double alpha, beta;  /* Beamer parameters; 0 = 20, 24 (single GPU; 14, 24 partitioned) */
    int64_t lb_threshold;/* frontier size at which auto strategy switches from
                            node-granular to edge-granular balancing; 0 = default
                            65536 (swept on B200, scripts/lb_sweep.py; auto also
                            needs short lists: m_f <= 16 f, max degree <= 4096) */
} gr_bfs_opts;

gr_status gr_bfs(gr_graph *g, int32_t src, int32_t *depth_out, int32_t *pred_out,
                 const gr_bfs_opts *opts);

/*
 * gr_sssp -- single-source shortest paths with non-negative integer weights,
 * delta-stepping with Gunrock's two-level near/far priority queue
 * (Alg. 1; §5.2; priority queue P:838-857).
 *   dist_out  uint32[n]: exact shortest distance, UINT32_MAX when unreached
 *             (A-2). Deterministic.
 *   pred_out  int32[n] or NULL: a tight parent (dist[pred[v]] + w = dist[v]),
 *             pred[src] = src, -1 when unreached (A-9).
 *   opts      NULL = defaults; delta = 0 picks a delta from graph statistics.
 * Errors: GR_ERR_NO_WEIGHTS, GR_ERR_OUT_OF_RANGE, GR_ERR_OVERFLOW (if
 * max_w*(n-1) >= UINT32_MAX, A-19), GR_ERR_INVALID_ARGUMENT.
 */
typedef struct {
    uint32_t delta;      /* near/far band width; 0 = auto; UINT32_MAX = one band
                            (Bellman-Ford-like)                                    */
    int32_t strategy;    /* as gr_bfs_opts.strategy                                */
    int32_t direction;   /* near iterations: 0 auto, 1 push (relax the frontier's
                            out-edges), 2 pull (every vertex takes the minimum over
                            its in-edges from the frontier, named for
                            SSSP in P:832-834; reading A-24). Pull needs the packed
                            edge stream (gr_graph_info.packed_weights); otherwise
                            push runs. Partitioned graphs: push.               */
    double alpha;        /* auto: pull when frontier edges * alpha > m; 0 = 2     */
} gr_sssp_opts;

gr_status gr_sssp(gr_graph *g, int32_t src, uint32_t *dist_out, int32_t *pred_out,
                  const gr_sssp_opts *opts);

/*
 * Asynchronous variants: the same traversal (same arguments, same results,
 * same errors for bad arguments) is only ENQUEUED on g's stream; the call
 * returns without waiting, so back-to-back runs and the caller's own stream
 * work (events, copies) run on the device without host round trips between
 * them (SURVEY §8(d) timing: the CUDA-event time of the call's GPU work).
 *   depth_out / dist_out / pred_out must be DEVICE memory (else
 *   GR_ERR_INVALID_ARGUMENT); they are valid once the stream reaches the end
 *   of the run (gr_graph_sync, or any later stream-ordered consumer).
 * gr_graph_sync waits for every run enqueued on g, makes the per-level stats
 * of the last one available (gr_get_run_stats) and reports a queue overflow
 * of any of them: if exactly one idempotent BFS was pending it is re-run with
 * exactly-once claims (as gr_bfs does), otherwise GR_ERR_OVERFLOW. gr_bfs /
 * gr_sssp call gr_graph_sync first when runs are pending.
 */
gr_status gr_bfs_async(gr_graph *g, int32_t src, int32_t *depth_out, int32_t *pred_out,
                       const gr_bfs_opts *opts);
gr_status gr_sssp_async(gr_graph *g, int32_t src, uint32_t *dist_out, int32_t *pred_out,
                        const gr_sssp_opts *opts);
gr_status gr_graph_sync(gr_graph *g);

/* Per-level records of the last gr_bfs / gr_sssp on g (SURVEY §5 tracing). */
typedef struct {
    int32_t level;           /* BFS level or SSSP iteration                        */
    int32_t direction;       /* 1 push, 2 pull, 3 SSSP relax, 4 SSSP far re-split  */
    int64_t frontier;        /* |frontier| (queue entries)                         */
    int64_t frontier_edges;  /* sum of out-degrees of the frontier                 */
    int64_t discovered;      /* vertices discovered / improved-and-queued          */
    int64_t inspected_edges; /* edges actually read (push: frontier_edges; pull:
                                up to the first frontier hit, early exit)          */
    int64_t aux;             /* SSSP: far-queue size; BFS: unvisited (heuristic u) */
    int64_t ns;              /* device time of the step (%globaltimer, ns)         */
} gr_level_stats;

typedef struct {
    int32_t num_levels;            /* levels executed (may exceed records kept)    */
    int32_t num_records;           /* records available in levels[]                */
    const gr_level_stats *levels;  /* valid until the next run / destroy           */
    int64_t reached;               /* vertices reached (depth >= 0 / dist < inf),
                                      counted on the device at the first query    */
    uint32_t delta;                /* SSSP: delta used                             */
    int32_t kernel_launches;       /* kernels launched by the last run            */
    int64_t reached_edges;         /* directed edges whose source is reached: the
                                      TEPS numerator m_reached (reading A-14; the
                                      paper's Table 3 MTEPS = |E| / t) */
} gr_run_stats;

gr_status gr_get_run_stats(gr_graph *g, gr_run_stats *out);

/* Message for the last failure on the calling thread ("" if none). */
const char *gr_last_error(void);

/* Kernels this process has launched through the library (all graphs). */
uint64_t gr_kernel_launch_count(void);

/* Library version string, e.g. "gr_b200 0.1 sm_100a". */
const char *gr_version(void);

/* ===========================================================================
 * Betweenness centrality (paper §5.3: Brandes's
 * formulation, "a forward BFS pass to accumulate sigma values for each node,
 * and a backward BFS pass to compute centrality values").
 *   bc_out[v] = sum over s in sources of delta_s(v),
 *   delta_s(v) = sum over t != s, v of sigma_st(v) / sigma_st
 * (shortest = fewest edges along CSR out-edges; sigma_st = number of shortest
 * s->t paths, sigma_st(v) = those through v; delta_s(s) = 0). No halving:
 * for an undirected (symmetric) graph and sources = all vertices, Brandes's
 * betweenness (each unordered pair once) is bc_out / 2.
 * sources: HOST int32[nsrc], each in [0, n) (GR_ERR_OUT_OF_RANGE otherwise).
 * bc_out: double[n], host or device (overwritten). sigma_out: double[n] or
 * NULL: sigma_s of the LAST source (host or device). fp64 throughout; path
 * counts beyond ~1e308 (very high-diameter meshes) overflow to inf.
 * Synchronous: one host read per BFS level of each source.
 * =========================================================================== */
gr_status gr_bc(gr_graph *g, const int32_t *sources, int64_t nsrc, double *bc_out, double *sigma_out);

/* gr_bc with options: the direction of each forward level (the paper names
 * pull as the next step for BC): push = the advance over the
 * level queue above; pull = every undiscovered vertex sums sigma over its
 * in-neighbours at the current depth (no atomics, no early exit). Auto picks
 * pull when the frontier's edges exceed the undiscovered vertices' edges /
 * alpha (reading A-24). Results are identical in every mode.
 * gr_get_run_stats after a gr_bc: per-level records (direction, frontier,
 * frontier edges; aux = undiscovered edges) of the LAST source's forward pass. */
typedef struct {
    int32_t direction;   /* 0 auto, 1 push only, 2 pull only                           */
    double alpha;        /* auto: pull when m_f > m_u / alpha; 0 = 2                 */
} gr_bc_opts;
gr_status gr_bc_ex(gr_graph *g, const int32_t *sources, int64_t nsrc, double *bc_out, double *sigma_out,
                   const gr_bc_opts *opts);

/* ===========================================================================
 * Connected components (paper §5.4: hooking on
 * an edge frontier with a filter removing edges whose endpoints share a
 * component ID, then pointer jumping "until it reaches the root").
 *   comp_out[v] = the smallest vertex id of v's connected component (edges
 *   taken as undirected: weak components of a directed CSR). The canonical
 *   min-id label is reading A-22 (hooking always points the larger root at
 *   the smaller).
 * comp_out: int32[n], host or device (overwritten). num_components: host
 * int64 or NULL. Synchronous (one host read per hooking pass).
 * =========================================================================== */
gr_status gr_cc(gr_graph *g, int32_t *comp_out, int64_t *num_components);

/* ===========================================================================
 * PageRank (paper §5.5: a frontier of all
 * vertices, one advance computing PageRank on the frontier, one filter
 * removing converged vertices, AtomicAdd accumulation). Reading A-23:
 *   PR(v) = (1 - damping)/n + damping * sum over in-edges (u,v) of PR(u)/outdeg(u)
 * from PR = 1/n, no dangling-mass redistribution; a vertex leaves the
 * frontier when |PR_new(v) - PR_old(v)| <= tol * PR_new(v); stops when the
 * frontier is empty or after max_iter steps.
 * damping in [0,1), tol >= 0, max_iter >= 1 (GR_ERR_INVALID_ARGUMENT).
 * rank_out: double[n], host or device. iterations: host int32 or NULL.
 * In-edges come from the CSC (the CSR itself for GR_SYMMETRIC graphs).
 * =========================================================================== */
gr_status gr_pagerank(gr_graph *g, double damping, double tol, int32_t max_iter, double *rank_out,
                      int32_t *iterations);

/* ===========================================================================
 * Multi-GPU group + partitioned graph. The paper is
 * single-GPU and names multi-GPU as future work ("to multiple GPUs on a
 * single node"); the method per partition is the single-GPU
 * one above.
 *
 * gr_comm is one rank of a group of nranks <= 8 GPUs of one node, one process
 * per GPU. The caller bootstraps the group: rank 0 calls
 * gr_comm_get_unique_id, broadcasts the 128 bytes (e.g. torch.distributed),
 * then every rank calls gr_comm_create with its rank and CUDA device. The
 * library owns the ncclComm_t (NCCL of the calling process, libnccl.so.2) and
 * uses it for the collective set-up steps; every traversal step, including
 * the exchange between ranks, runs inside the library's kernels over peer
 * memory (CUDA IPC mappings of each rank's symmetric region, NVLink).
 *   gr_comm_get_unique_id  id_out: 128 writable bytes (ncclUniqueId).
 *   gr_comm_create         collective over the nranks processes; errors:
 *                          GR_ERR_INVALID_ARGUMENT (rank/nranks), GR_ERR_NCCL.
 *   gr_comm_create_loopback  nranks VIRTUAL ranks in this process on one GPU
 *                          (out: gr_comm*[nranks]). Collective calls on their
 *                          graphs (gr_bfs) are joined: every rank's call is
 *                          recorded and the call of the last rank runs all
 *                          ranks in ONE launch, writes every rank's outputs and
 *                          returns; the earlier calls return GR_OK at once with
 *                          their outputs pending. For testing the multi-rank
 *                          path on one GPU.
 *   gr_comm_destroy        frees the handle (after the graphs using it).
 *   gr_comm_info           rank, nranks, loopback flag (any output may be NULL).
 * =========================================================================== */
typedef struct gr_comm gr_comm;
gr_status gr_comm_get_unique_id(void *id_out);
gr_status gr_comm_create(int rank, int nranks, const void *nccl_unique_id, int device, gr_comm **out);
gr_status gr_comm_create_loopback(int nranks, int device, gr_comm **out);
gr_status gr_comm_destroy(gr_comm *c);
gr_status gr_comm_info(const gr_comm *c, int32_t *rank, int32_t *nranks, int32_t *loopback);

/*
 * gr_graph_create_partitioned -- this rank's part of a symmetric graph with
 * n_global vertices under a 1D vertex partition: rank q owns the block
 * [q*B, min(n_global, (q+1)*B)), B = 32*ceil(n_global/(32*nranks)) (a multiple
 * of 32 so bitmap shards concatenate), and stores the out-lists of its
 * vertices with GLOBAL column ids (which double as in-lists for pull steps,
 * hence GR_SYMMETRIC is required: "converted all datasets to
 * undirected graphs").
 *   v_begin, v_end  the owned block (checked against the formula above)
 *   m_local         edges of the owned rows
 *   row_offsets     int64[v_end - v_begin + 1], local rows, R[0] = 0
 *   col_indices     int32[m_local], GLOBAL ids in [0, n_global)
 *   weights         uint32[m_local] or NULL (reserved for a partitioned SSSP)
 *   flags           GR_SYMMETRIC (required) | GR_VALIDATE | GR_KEEP_ORDER
 *   cuda_stream     stream of this rank's work; the device is the comm's
 * Copies its inputs. Collective for real ranks (the symmetric regions are
 * mapped between the ranks here). Errors as gr_graph_create, plus
 * GR_ERR_INVALID_ARGUMENT for a wrong block, a non-symmetric flag or a second
 * graph on one loopback rank, GR_ERR_NCCL.
 *
 * gr_bfs(g, src, depth_out, pred_out, opts) on such a graph is COLLECTIVE
 * (every rank calls it with the same GLOBAL src and opts): one persistent
 * kernel per rank runs every level -- push levels ship remote discoveries
 * straight into the owner's inbox, pull levels all-gather the frontier-bitmap
 * shards with peer stores, and the per-level counters are exchanged the same
 * way, so every rank takes the same direction decision (A-3) and stops at the
 * same level; no host round trip per level. depth_out / pred_out: int32
 * [v_end - v_begin] (host or device) for the OWNED block; pred holds GLOBAL
 * ids. opts.strategy and opts.idempotent are ignored (merge-path advance,
 * exactly-once claims). gr_get_run_stats: global per-level counters; `aux` of
 * a level = bytes the level sent between ranks (push: 8 per shipped pair;
 * pull: the shards); reached / reached_edges count the owned block.
 * gr_bfs_async is not available for partitioned graphs.
 */
gr_status gr_graph_create_partitioned(gr_comm *c, int64_t n_global, int64_t v_begin, int64_t v_end,
                                      int64_t m_local, const int64_t *row_offsets, const int32_t *col_indices,
                                      const uint32_t *weights, uint32_t flags, void *cuda_stream, gr_graph **out);

#ifdef __cplusplus
}
#endif

#endif /* GR_H_ */
