// comm.cu -- gr_comm: the multi-GPU group of a 1D-partitioned graph
// (SURVEY §8(b) "gr_comm_create(rank, nranks, ncclUniqueId, device)", §8(e)).
// The paper is single-GPU; multi-GPU is its future work.
//
// Two kinds of rank:
//  * real: one process per GPU. The library owns an ncclComm_t created from a
//    128-byte ncclUniqueId that the caller broadcasts (torch.distributed only
//    bootstraps that id). NCCL runs the collective set-up steps (all-gather
//    of the CUDA IPC handles of every rank's symmetric region, all-gather of
//    the vertex degrees); the traversal itself exchanges data with plain
//    loads / stores / atomics on the peers' regions over NVLink inside one
//    persistent kernel per rank (pbfs.cu).
//  * loopback: nranks virtual ranks in one process on one GPU; every region is
//    local device memory and ONE cooperative launch hosts all ranks. This is
//    how the multi-rank logic (remote inbox atomics, peer stores, barriers,
//    shard all-gather) is exercised on a single GPU.
#include <nccl.h>

#include "gr_internal.cuh"

namespace gr {

gr_status nccl_fail(int res, const char *what) {
    set_error("NCCL error %d (%s) in %s", res, ncclGetErrorString((ncclResult_t)res), what);
    return GR_ERR_NCCL;
}

#define GR_NCCL(call)                                             \
    do {                                                          \
        ncclResult_t r_ = (call);                                 \
        if (r_ != ncclSuccess) return ::gr::nccl_fail((int)r_, #call); \
    } while (0)

// All-gather of `bytes` per rank (device buffers; drecv holds nranks*bytes,
// rank order). Synchronises the stream. Loopback ranks never call it.
gr_status comm_allgather_bytes(Comm *c, const void *dsend, void *drecv, size_t bytes, cudaStream_t s) {
    if (c->nranks == 1 || !c->nccl) {
        GR_CUDA(cudaMemcpyAsync(drecv, dsend, bytes, cudaMemcpyDeviceToDevice, s));
    } else {
        GR_NCCL(ncclAllGather(dsend, drecv, bytes, ncclUint8, (ncclComm_t)c->nccl, s));
    }
    GR_CUDA(cudaStreamSynchronize(s));
    return GR_OK;
}

// Symmetric region of a partitioned graph: `bytes` of device memory on every
// rank, same layout, each rank's region mapped into every other rank's
// address space (CUDA IPC over NVLink for real ranks; plain pointers in a
// loopback group, filled in when the group's last rank is created).
gr_status comm_sym_alloc(Comm *c, Graph *g, size_t bytes) {
    GR_CUDA(cudaMalloc((void **)&g->sym, bytes));
    GR_CUDA(cudaMemsetAsync(g->sym, 0, bytes, g->stream));
    g->sym_bytes = bytes;
    g->bytes += (int64_t)bytes;
    for (int q = 0; q < kMaxRanks; ++q) { g->sym_peer[q] = nullptr; g->sym_ipc[q] = false; }
    g->sym_peer[c->rank] = g->sym;
    if (c->group || c->nranks == 1) {
        GR_CUDA(cudaStreamSynchronize(g->stream));
        return GR_OK;
    }
    cudaIpcMemHandle_t h;
    GR_CUDA(cudaIpcGetMemHandle(&h, g->sym));
    char *dbuf = nullptr;
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    GR_CUDA(cudaMalloc((void **)&dbuf, hb * (c->nranks + 1)));
    GR_CUDA(cudaMemcpyAsync(dbuf, &h, hb, cudaMemcpyHostToDevice, g->stream));
    gr_status st = comm_allgather_bytes(c, dbuf, dbuf + hb, hb, g->stream);
    if (st != GR_OK) { cudaFree(dbuf); return st; }
    cudaIpcMemHandle_t all[kMaxRanks];
    GR_CUDA(cudaMemcpy(all, dbuf + hb, hb * c->nranks, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    for (int q = 0; q < c->nranks; ++q) {
        if (q == c->rank) continue;
        void *p = nullptr;
        GR_CUDA(cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess));
        g->sym_peer[q] = (char *)p;
        g->sym_ipc[q] = true;
    }
    return GR_OK;
}

void comm_sym_free(Graph *g) {
    for (int q = 0; q < kMaxRanks; ++q) {
        if (g->sym_ipc[q] && g->sym_peer[q]) cudaIpcCloseMemHandle(g->sym_peer[q]);
        g->sym_peer[q] = nullptr;
        g->sym_ipc[q] = false;
    }
    if (g->sym) cudaFree(g->sym);
    g->sym = nullptr;
}

}  // namespace gr

using namespace gr;

extern "C" {

gr_status gr_comm_get_unique_id(void *id_out) {
    if (!id_out) { set_error("id_out is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    ncclUniqueId id;
    GR_NCCL(ncclGetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return GR_OK;
}

gr_status gr_comm_create(int rank, int nranks, const void *nccl_unique_id, int device, gr_comm **out) {
    if (!out || !nccl_unique_id || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) {
        set_error("invalid gr_comm_create arguments (rank=%d nranks=%d, at most %d ranks)", rank, nranks, kMaxRanks);
        return GR_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    GR_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t nc = nullptr;
    GR_NCCL(ncclCommInitRank(&nc, nranks, id, rank));
    Comm *c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    c->nccl = nc;
    *out = (gr_comm *)c;
    return GR_OK;
}

gr_status gr_comm_create_loopback(int nranks, int device, gr_comm **out) {
    if (!out || nranks < 1 || nranks > kMaxRanks) {
        set_error("invalid gr_comm_create_loopback arguments (nranks=%d, at most %d)", nranks, kMaxRanks);
        return GR_ERR_INVALID_ARGUMENT;
    }
    GR_CUDA(cudaSetDevice(device));
    LoopGroup *grp = new LoopGroup();
    grp->P = nranks;
    grp->device = device;
    grp->alive = nranks;
    for (int r = 0; r < nranks; ++r) {
        Comm *c = new Comm();
        c->rank = r;
        c->nranks = nranks;
        c->device = device;
        c->group = grp;
        grp->ranks[r] = c;
        out[r] = (gr_comm *)c;
    }
    return GR_OK;
}

gr_status gr_comm_destroy(gr_comm *h) {
    if (!h) return GR_OK;
    Comm *c = (Comm *)h;
    gr_status st = GR_OK;
    if (c->nccl) {
        ncclResult_t r = ncclCommDestroy((ncclComm_t)c->nccl);
        if (r != ncclSuccess) st = nccl_fail((int)r, "ncclCommDestroy");
    }
    if (c->group) {
        LoopGroup *grp = c->group;
        grp->ranks[c->rank] = nullptr;
        if (--grp->alive == 0) delete grp;
    }
    delete c;
    return st;
}

gr_status gr_comm_info(const gr_comm *h, int32_t *rank, int32_t *nranks, int32_t *loopback) {
    if (!h) { set_error("comm is NULL"); return GR_ERR_INVALID_ARGUMENT; }
    const Comm *c = (const Comm *)h;
    if (rank) *rank = c->rank;
    if (nranks) *nranks = c->nranks;
    if (loopback) *loopback = c->group != nullptr;
    return GR_OK;
}

}  // extern "C"
