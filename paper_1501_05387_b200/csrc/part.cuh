// part.cuh -- pieces shared by the partitioned persistent kernels (pbfs.cu,
// psssp.cu): the symmetric region every rank maps from every other rank, the
// published-counter table, and the system-scope flag primitives of the
// cross-process barrier. SURVEY §8(b), §8(e); multi-GPU is the paper's future
// work.
#pragma once

#include "gr_internal.cuh"

namespace gr {

// ---------------------------------------------------------------- symmetric region
// Same layout on every rank; peers address it through Graph::sym_peer.
struct SymHdr {
    unsigned long long flag[kMaxRanks];       // barrier: flag[q] = epoch of rank q's last arrival here
    unsigned long long inbox_count;           // BFS: (vertex, parent) pairs stored into this rank's inbox this run
    unsigned long long sin_count[2];          // SSSP: triples stored into this rank's inbox, by step parity
    unsigned long long pad0[5];
    unsigned long long st[2][kMaxRanks][8];   // per publish parity, per sender rank: published counters
};
// st fields (the next local frontier of the sender, after its level):
enum { kStF = 0, kStMf = 1, kStDisc = 2, kStOvf = 3, kStInsp = 4, kStShip = 5, kStDmax = 6, kStAux = 7 };
// level-0 table: kStInsp = m_local, kStAux = non-isolated local vertices
constexpr size_t kSymHdrBytes = 4096;
static_assert(sizeof(SymHdr) <= kSymHdrBytes, "symmetric header");

struct SymLayout {
    size_t gfront[2];    // BFS: global frontier bitmaps (all-gathered shards), by pull-level parity
    size_t inbox;        // BFS: int2 (vertex, parent) pairs shipped to this rank
    int64_t inbox_cap;   // pairs / triples: (P-1) * block (a peer ships a vertex at most once per
                         // BFS run / per SSSP step)
    size_t sinbox[2];    // SSSP (weighted graphs): int4 (vertex, dist, parent, -) by step parity
    int64_t gwords;      // words of a global bitmap (P * block / 32)
    size_t bytes;
};

static inline SymLayout sym_layout(int P, int64_t block, bool weighted) {
    SymLayout L;
    L.gwords = (int64_t)P * block / 32;
    const size_t gb = ((size_t)L.gwords * 4 + 255) & ~(size_t)255;
    L.gfront[0] = kSymHdrBytes;
    L.gfront[1] = L.gfront[0] + gb;
    L.inbox = L.gfront[1] + gb;
    L.inbox_cap = P > 1 ? (int64_t)(P - 1) * block : 1;
    L.sinbox[0] = (L.inbox + (size_t)L.inbox_cap * 8 + 255) & ~(size_t)255;
    L.sinbox[1] = L.sinbox[0] + (weighted ? (size_t)L.inbox_cap * 16 : 0);
    L.bytes = L.sinbox[1] + (weighted ? (size_t)L.inbox_cap * 16 : 0);
    return L;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long pgtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}


// Cross-rank group state every CTA of a rank keeps identically (registers):
// the barrier epoch and the device pointers of every rank's symmetric header.
// All threads of the rank's CTAs call bar()/publish() together.
struct RankSync {
    const cg::grid_group *grid;
    char *const *sym;          // sym[q]: rank q's region as mapped here
    int rank, nranks, multiproc, bid;
    Ctl *ctl;
    unsigned long long ep;

    __device__ __forceinline__ SymHdr *hdr(int q) const { return reinterpret_cast<SymHdr *>(sym[q]); }

    // cross-process half of a barrier, between two grid barriers: thread q of
    // the rank's first CTA announces this rank's arrival to rank q and waits
    // for rank q's (a dead peer ends the wait after 20 s with overflow = 3)
    __device__ __forceinline__ void peer_flags() {
        ++ep;
        if (bid == 0 && (int)threadIdx.x < nranks) {
            const int q = threadIdx.x;
            __threadfence_system();
            st_release_sys(&hdr(q)->flag[rank], ep);
            const long long t0 = pgtimer();
            while (ld_acquire_sys(&hdr(rank)->flag[q]) < ep) {
                if (pgtimer() - t0 > 20000000000ll) { atomicExch(&ctl->overflow, 3ull); break; }
            }
        }
    }
    // barrier of every rank of the group
    __device__ __forceinline__ void bar() {
        grid->sync();
        if (multiproc) {
            peer_flags();
            grid->sync();
        }
    }
    // the rank's first thread writes vals[8] into every rank's table `par`,
    // then barrier: afterwards every rank reads the same table
    __device__ __forceinline__ void publish(int par, const unsigned long long *vals) {
        if (bid == 0 && threadIdx.x == 0)
            for (int q = 0; q < nranks; ++q)
                for (int k = 0; k < 8; ++k) hdr(q)->st[par][rank][k] = vals[k];
        if (multiproc) {
            __syncthreads();
            peer_flags();
        }
        grid->sync();
    }
    // table `par` reduced over ranks (thread-local; sum, except max / or per field)
    __device__ __forceinline__ void read(int par, unsigned long long *t, int max_field, int or_field,
                                         int min_field = -1) const {
        for (int k = 0; k < 8; ++k) t[k] = (k == min_field) ? ~0ull : 0ull;
        for (int q = 0; q < nranks; ++q) {
            const unsigned long long *row = hdr(rank)->st[par][q];
            for (int k = 0; k < 8; ++k) {
                const unsigned long long x = __ldcg(row + k);
                if (k == or_field) t[k] |= x;
                else if (k == max_field) t[k] = max(t[k], x);
                else if (k == min_field) t[k] = min(t[k], x);
                else t[k] += x;
            }
        }
    }
};

}  // namespace gr
