// Throughput of random 4-B bitmap probes (the push step's culling test) on
// the whole GPU: through L1 (ld.ca), L2 (ld.cg), shared memory (each CTA
// holds the whole 256 KB... too big: 128 KB half), and distributed shared
// memory in 2-CTA clusters (each CTA holds half of a 256 KB bitmap).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hsh(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
constexpr unsigned kWords = 65536;   // 256 KB bitmap (C2: 2^21 vertices)
template <int MODE>
__global__ void probe(const unsigned *bm, int iters, unsigned *sink) {
    extern __shared__ unsigned sh[];
    const unsigned half = kWords / 2;
    unsigned rank = 0;
    if (MODE >= 2) {
        if (MODE == 3) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        const unsigned base = (MODE == 3) ? rank * half : 0;
        for (unsigned i = threadIdx.x; i < half; i += blockDim.x) sh[i] = bm[base + i];
        __syncthreads();
        if (MODE == 3) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    unsigned acc = 0, x = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sh);
    for (int i = 0; i < iters; ++i) {
        unsigned wv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x = hsh(x + k);
            const unsigned w = x & (kWords - 1);
            if (MODE == 4) { wv[k] = atomicOr((unsigned *)bm + w, 1u << (x & 31)); }
            else if (MODE == 5) { atomicOr((unsigned *)bm + w, 1u << (x & 31)); wv[k] = 0; }
            else if (MODE == 6) { ((volatile unsigned *)bm)[w] = x; wv[k] = 0; }
            else if (MODE == 0) { unsigned r; asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(r) : "l"(bm + w)); wv[k] = r; }
            else if (MODE == 1) wv[k] = __ldcg(bm + w);
            else if (MODE == 2) { unsigned r; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(sbase + 4u * (w & (half - 1)))); wv[k] = r; }
            else {
                const unsigned owner = w / half, a = sbase + 4u * (w & (half - 1));
                unsigned ra, r;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(owner));
                asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(r) : "r"(ra));
                wv[k] = r;
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += wv[k];
    }
    if (MODE == 3) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (acc == 0x12345678u) *sink = acc;
}
int main() {
    unsigned *bm, *sink; cudaMalloc(&bm, kWords * 4); cudaMalloc(&sink, 4); cudaMemset(bm, 0x5a, kWords * 4);
    const int iters = 256, threads = 1024, ctas = 148;  // 1 CTA per SM
    const double probes = (double)iters * 8 * threads * ctas;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[] = {"L1 (ld.ca)", "L2 (ld.cg)", "smem (half bitmap)", "DSMEM cluster-2 (whole bitmap)",
                           "atomicOr with return", "RED.OR (no return)", "plain 4-B store"};
    for (int mode = 0; mode < 7; ++mode) {
        size_t smem = mode >= 2 ? kWords / 2 * 4 : 0;
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = mode == 3 ? 1 : 0;
        void (*k)(const unsigned *, int, unsigned *) = mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2>
                                                      : mode == 3 ? probe<3> : mode == 4 ? probe<4> : mode == 5 ? probe<5> : probe<6>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, k, (const unsigned *)bm, iters, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-32s %8.3f ms  %7.1f G probes/s  (%s)\n", names[mode], ms, probes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
}
