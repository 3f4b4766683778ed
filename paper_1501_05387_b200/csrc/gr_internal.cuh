// gr_internal.cuh -- shared device/host internals of the B200 frontier library.
// Not part of the ABI (include/gr.h is). Citations: P:n = PAPER.md line n.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gr.h"

namespace gr {

namespace cg = cooperative_groups;

constexpr int kWarp = 32;
#ifndef GR_BLOCK
#define GR_BLOCK 512   // 512 x 2 CTAs/SM measured best of {1024x1, 512x2, 256x4} (C2, C4)
#endif
constexpr int kBlock = GR_BLOCK;         // threads per CTA of the persistent kernels
#ifndef GR_MINB
#define GR_MINB 2
#endif
constexpr int kMinBlocks = GR_MINB;      // resident CTAs per SM the kernels are built for
constexpr int kWarpsPerBlock = kBlock / kWarp;
#ifndef GR_STAGE_CAP
#define GR_STAGE_CAP 128   // 128 vs 64: half the flushes on the one grid-wide queue counter (C3 discovery-heavy push step 402 -> 269 us)
#endif
constexpr int kStageCap = GR_STAGE_CAP;  // per-warp smem staging of appended vertices
constexpr int kMaxStatRecords = 1 << 16; // per-level records kept for gr_get_run_stats
constexpr int kSlots = 4;                // rotating per-level control slots
constexpr int kMaxRanks = 8;             // one NVSwitch box: 1/2/4/8 GPUs (north star)

// ---------------------------------------------------------------- error plumbing
void set_error(const char *fmt, ...);
gr_status cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define GR_CUDA(call)                                                             \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) return ::gr::cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

void count_launch(int k = 1);
int64_t env_int(const char *name, int64_t dflt);  // tuning knobs

// ---------------------------------------------------------------- control block
// One slot per in-flight level (rotating, kSlots). Level L reads the frontier
// descriptor of slot L%4, writes that of slot (L+1)%4, and resets slot
// (L+2)%4 (which no block reads or writes during level L).
struct Slot {
    unsigned long long qpack;   // frontier queue: (sum of degrees << S) | count
    unsigned long long ndisc;   // vertices discovered / queued in this step
    unsigned long long fpack;   // SSSP far appends (count) during this step
    unsigned long long work;    // dynamic work counter
    unsigned long long minfar;  // SSSP re-split: min far distance
    unsigned long long insp;    // edges inspected in this step
    unsigned long long dmax;    // max out-degree appended to this frontier (upper bound)
    unsigned long long pad[1];
};

struct Ctl {
    Slot slot[kSlots];
    unsigned long long overflow;   // set when a queue capacity would be exceeded
    unsigned long long levels;     // levels executed by the last run
    unsigned long long reached;    // psssp.cu: length of the current step's ship list
    unsigned long long far_count[2];
    long long bstate[8];           // small-mode handoff of the traversal state
    unsigned long long sticky;     // some run since the last gr_graph_sync overflowed
    unsigned long long epoch;      // partitioned runs: cross-rank barrier epochs used so far
    unsigned int gbar;             // GridBar arrival word (any initial value; never reset)
    unsigned int pad_gbar;
    unsigned long long handoff;    // bounded-degree BFS: 1 the cluster kernel handed the traversal
                                   // to the grid kernel (state in bstate), 2 it finished it
};

// Grid-wide barrier of the persistent kernels (replaces cg::grid_group::sync):
// the same arrive (atom.add.release, the master's addend flips bit 31 once all
// CTAs arrived) and acquire poll as cooperative groups, but the poll backs off
// with __nanosleep. cg's tight poll keeps one load per CTA in flight on the
// barrier word's L2 slice for the whole level; on narrow levels (C4: ~20 of
// 296 CTAs work, the rest wait) that traffic delayed the working CTAs'
// accesses to the same slice (measured per-level time).
struct GridBar {
    unsigned int *bar;
    int max_ns;   // backoff cap (0: tight poll)
    __device__ __forceinline__ void sync() const {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned int nb = (blockIdx.x == 0) ? 0x80000000u - (gridDim.x - 1) : 1u;
            unsigned int old, cur;
            asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
            int ns = 16;
            for (;;) {
                asm volatile("ld.acquire.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
                if ((old ^ cur) & 0x80000000u) break;
                if (max_ns > 0) {
                    __nanosleep(ns);
                    ns = ns * 2 > max_ns ? max_ns : ns * 2;
                }
            }
        }
        __syncthreads();
    }
};

struct Graph;
struct LoopGroup;
// gr_comm: one rank of a multi-GPU group (comm.cu). Either a real rank (one
// process per GPU, the library's own ncclComm_t used for the collective
// set-up steps: IPC handle and degree all-gathers) or one virtual rank of a
// loopback group (all ranks in one process on one GPU; the partitioned kernel
// then hosts every rank in one cooperative launch -- the test harness for the
// multi-rank logic on a single GPU).
struct Comm {
    int rank = 0, nranks = 1, device = 0;
    void *nccl = nullptr;          // ncclComm_t (real ranks)
    LoopGroup *group = nullptr;    // loopback ranks
};
struct LoopGroup {
    int P = 0, device = 0, alive = 0;
    Comm *ranks[kMaxRanks] = {};
    Graph *graphs[kMaxRanks] = {};
    // a collective call (gr_bfs / gr_sssp) joined by some ranks, launched when all have
    int joined = 0;                // bitmask of ranks that joined
    int kind = 0;                  // 1 BFS, 2 SSSP
    int64_t src = 0;
    void *out0[kMaxRanks] = {}, *out1[kMaxRanks] = {};
    gr_bfs_opts bopts{};
    gr_sssp_opts sopts{};
};
gr_status nccl_fail(int res, const char *what);
gr_status comm_allgather_bytes(Comm *c, const void *dsend, void *drecv, size_t bytes, cudaStream_t s);
gr_status comm_sym_alloc(Comm *c, Graph *g, size_t bytes);
void comm_sym_free(Graph *g);

// ---------------------------------------------------------------- graph object
struct Graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t n = 0, m = 0;
    bool symmetric = false;
    bool has_w = false;
    uint32_t max_w = 0;
    int64_t max_deg = 0, nonisolated = 0;
    int pack_shift = 32;          // S: bits of the count field in Slot::qpack

    // topology (device)
    int64_t *R = nullptr;         // [n+1]
    int32_t *C = nullptr;         // [m]
    uint32_t *W = nullptr;        // [m] or null
    uint32_t *CW = nullptr;       // [m] packed (C << 7) | W for SSSP, or null (graph.cu)
    uint32_t *CWt = nullptr;      // [m] packed in-lists (u << 7) | w(u,v) at Rt: pull SSSP (lazy)
    int64_t *Rt = nullptr;        // CSC (== R when symmetric)
    int32_t *Ct = nullptr;
    int2 *ph = nullptr;           // pull head: {Ct[Rt[v]] or -1, in-degree} (pull steps, pull.cuh)
    // Bounded-degree ("ELL") adjacency, built when every out-degree is <= 4
    // (road-like graphs, C4): one 16-B record per vertex whose slot k holds
    // (k-th neighbour w << 3) | out-degree(w), or -1. A push step reads a
    // frontier vertex's whole list with one aligned load and learns each
    // discovered vertex's degree without touching R (graph.cu, frontier.cuh).
    int4 *ell = nullptr;
    // SSSP companion: 32 B per vertex, ellw[2v] = the four neighbour ids (-1),
    // ellw[2v+1] = (w(v, nbr) << 3) | out-degree(nbr) per slot.
    int4 *ellw = nullptr;

    // per-run scratch (device)
    uint32_t *visited = nullptr;  // [nwords] visited bitmap (P:793-799 culling)
    uint32_t *noin = nullptr;     // [nwords] vertices with in-degree 0 (never discoverable)
    uint32_t *fbuf[3] = {nullptr, nullptr, nullptr}; // rotating frontier bitmaps
    int32_t *qv[2] = {nullptr, nullptr};    // frontier queues (vertex ids)
    int64_t *qo[2] = {nullptr, nullptr};    // exclusive prefix of degrees
    int64_t *qr[2] = {nullptr, nullptr};    // row start R[v] of each queue entry
    int32_t *depth_buf = nullptr; // internal outputs when caller passes host memory
    int32_t *pred_buf = nullptr;
    uint32_t *dist_buf = nullptr;
    // SSSP scratch
    unsigned long long *dp = nullptr; // packed (dist << 32) | pred  (A-9)
    int32_t *stamp = nullptr;         // RemoveRedundant stamp (A-7)
    int32_t *farq[2] = {nullptr, nullptr};
    int64_t far_cap = 0;

    Ctl *ctl = nullptr;
    gr_level_stats *stats_dev = nullptr;
    gr_level_stats *stats_host = nullptr;
    int stats_levels = 0, stats_records = 0;
    int64_t reached = -1, reached_edges = -1;  // totals of the last run (lazy, gr_get_run_stats)
    int last_kind = 0;             // 1 BFS, 2 SSSP: the kind of the last single-GPU run
    int32_t last_src = 0;
    uint32_t last_delta = 0;
    int last_launches = 0;
    int64_t bytes = 0;

    // asynchronous runs (gr_bfs_async / gr_sssp_async) not yet synchronised
    int pending = 0;               // runs enqueued since the last sync
    int pending_kind = 0;          // 1 BFS, 2 SSSP (the last one enqueued)
    int32_t pending_src = 0;
    void *pending_out[2] = {nullptr, nullptr};
    gr_bfs_opts pending_bopts{};

    int num_sms = 148;
    int nwords() const { return (int)((n + 31) / 32); }

    // 1D partition (gr_graph_create_partitioned); n = owned vertices, columns global
    bool part = false;
    int64_t n_global = 0, v_begin = 0, v_end = 0, block = 0;
    int nparts = 1, rank = 0;
    uint32_t *sent = nullptr;          // [ceil(n_global/32)] remote vertices already shipped (pbfs.cu)
    // partitioned graph of a gr_comm (gr_graph_create_partitioned; pbfs.cu)
    Comm *comm = nullptr;
    char *sym = nullptr;               // symmetric region (same layout on every rank)
    size_t sym_bytes = 0;
    char *sym_peer[kMaxRanks] = {};    // every rank's region, mapped here (sym_peer[rank] = sym)
    bool sym_ipc[kMaxRanks] = {};      // sym_peer[q] was opened with cudaIpcOpenMemHandle
    bool prepared = false;             // peers mapped, pull lists ordered by global degree
    bool flags_keep_order = false;     // GR_KEEP_ORDER: keep the caller's pull-list order
    void *pbfs_ranks = nullptr;        // device table of the ranks a launch hosts (pbfs.cu PRank)
    int64_t m_global = 0, nonisolated_global = 0;
    uint32_t maxw_global = 0;
    int32_t *ps_ship = nullptr;             // [n_global] vertices shipped in the current step (psssp.cu)
    // partitioned SSSP (psssp.cu)
    unsigned long long *ps_best = nullptr;  // [n_global] best (dist<<32|pred) shipped per remote vertex
    int32_t *ps_sstamp = nullptr;           // [n_global] step of the last shipment (one per step)
    // betweenness centrality (bc.cu)
    void *bc_vert = nullptr;                // [n] 16-B (sigma|coef, depth) records (bc.cu BcVert)
    double *bc_sig = nullptr, *bc_delta = nullptr, *bc_buf = nullptr;
    unsigned long long *bc_cnt = nullptr;   // [n + 3] per-level packed counters
    // connected components (cc.cu)
    unsigned long long *cc_ctl = nullptr;   // survivors, changed, count
    int2 *cc_list[2] = {nullptr, nullptr};  // edge frontier ping-pong
    // PageRank (pagerank.cu)
    double *pr_inv = nullptr, *pr_acc = nullptr;
    unsigned long long *pr_cnt = nullptr;
};

gr_status dev_alloc(Graph *g, void **p, size_t bytes);
gr_status count_reached(Graph *g, int64_t *reached, int64_t *reached_edges);
gr_status build_pull_weights(Graph *g);
void dev_free_all(Graph *g);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// L2-coherent load (bypasses L1): used for state that other SMs update
// within the same step (visited bitmap, distances).
__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long *p) {
    return __ldcg(p);
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    return *(volatile const unsigned long long *)p;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, d);
        if ((int)lane_id() >= d) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
    return x;
}

}  // namespace gr
