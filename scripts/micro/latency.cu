// Latency microbenchmark (one thread, dependent chains): L2-hit load, DRAM
// load, global atomicOr with return, across a 3 MB bitmap and a 384 MB array;
// also the same with 512 CTAs x 1 warp issuing concurrently (low load).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory"); return t; }

__global__ void chase(const uint32_t *next, int steps, long long *out, uint32_t start) {
    uint32_t p = start;
    long long c0 = clock64(), t0 = gt();
    for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
    long long c1 = clock64(), t1 = gt();
    out[0] = (c1 - c0) / steps; out[1] = (t1 - t0) / steps; out[2] = p;
}
__global__ void chase_atom(uint32_t *next, int steps, long long *out, uint32_t start) {
    uint32_t p = start;
    long long c0 = clock64(), t0 = gt();
    for (int i = 0; i < steps; ++i) p = atomicOr(next + p, 0u);
    long long c1 = clock64(), t1 = gt();
    out[0] = (c1 - c0) / steps; out[1] = (t1 - t0) / steps; out[2] = p;
}
__global__ void chase_many(uint32_t *next, int steps, long long *out, uint32_t n, int atom) {
    uint32_t p = (blockIdx.x * 7919u + threadIdx.x * 104729u) % n;
    long long t0 = gt();
    for (int i = 0; i < steps; ++i) p = atom ? atomicOr(next + p, 0u) : __ldcg(next + p);
    long long t1 = gt();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = (t1 - t0) / steps; out[1] = p; }
    if (p == 0xffffffffu) out[2] = 1;
}
__global__ void perm_init(uint32_t *a, uint32_t n, uint32_t stride) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        a[i] = (uint32_t)(((uint64_t)i + stride) % n);
}
int main() {
    long long *out; cudaMalloc(&out, 64);
    long long h[3];
    struct { const char *name; size_t n; } cfg[] = {{"3MB (L2)", 3u << 18}, {"384MB (DRAM)", 96u << 20}};
    for (auto &c : cfg) {
        uint32_t *a; cudaMalloc(&a, c.n * 4);
        perm_init<<<1024, 256>>>(a, (uint32_t)c.n, 7919 * 64 + 1);  // jump ~500 KB each step
        chase<<<1, 1>>>(a, 2000, out, 0); cudaDeviceSynchronize();
        chase<<<1, 1>>>(a, 2000, out, 0); cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
        printf("%-14s load   : %lld cycles, %lld ns per dependent access\n", c.name, h[0], h[1]);
        chase_atom<<<1, 1>>>(a, 2000, out, 0); cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
        printf("%-14s atomic : %lld cycles, %lld ns per dependent access\n", c.name, h[0], h[1]);
        for (int atom = 0; atom < 2; ++atom) {
            chase_many<<<296, 32>>>(a, 500, out, (uint32_t)c.n, atom); cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            printf("%-14s %s x 296 warps concurrent: %lld ns per dependent access\n", c.name, atom ? "atomic" : "load  ", h[0]);
        }
        cudaFree(a);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
