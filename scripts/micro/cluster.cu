// Cluster feasibility on B200: max active clusters of 16 x 1024-thread CTAs
// with ~200 KB smem, barrier.cluster round time, DSMEM load latency.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(1, 1, 1) dummy() {}
__global__ void kern(long long *out, int iters) {
    extern __shared__ unsigned sm[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank(), csize = cl.num_blocks();
    if (threadIdx.x == 0) sm[0] = rank * 7 + 1;
    cl.sync();
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    long long c1 = clock64();
    // DSMEM dependent chain: read peer (rank+1)%csize's sm[0] repeatedly
    unsigned v = 0;
    long long c2 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            unsigned *peer = cl.map_shared_rank(sm, (rank + 1 + (v & 0)) % csize);
            v += *(volatile unsigned *)peer;
        }
    }
    long long c3 = clock64();
    cl.sync();
    if (threadIdx.x == 0 && rank == 0) { out[0] = (c1 - c0) / iters; out[1] = (c3 - c2) / iters; out[2] = v; out[3] = csize; }
}
int main() {
    long long *out; cudaMalloc(&out, 64);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {8, 16}) for (int smem : {64 << 10, 200 << 10}) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int ncl = -1;
        cudaError_t e1 = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
        cudaError_t e2 = cudaLaunchKernelEx(&cfg, kern, out, 1000);
        cudaError_t e3 = cudaDeviceSynchronize();
        long long h[4] = {0}; cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        printf("cluster %2d smem %3d KB: maxActiveClusters %d (%s) launch %s sync %s | barrier.cluster %lld cyc, DSMEM dep load %lld cyc, size %lld\n",
               cs, smem >> 10, ncl, cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3), h[0], h[1], h[3]);
    }
}
