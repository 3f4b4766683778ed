// Does an L2 prefetch make a later dependent load an L2 hit? Chase 2000
// random 16-B records over a 384 MB array (one thread), after: nothing (cold),
// prefetch.global.L2 of every record, cp.async.bulk.prefetch.L2 of every
// record, or a previous chase (warm).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void build(unsigned *arr, unsigned n, int steps, unsigned seed, unsigned *addr) {
    if (blockIdx.x || threadIdx.x) return;
    unsigned p = seed % n;
    for (int i = 0; i < steps; ++i) {
        unsigned q = (unsigned)(((unsigned long long)(p + 1) * 2654435761ull + seed) % n) & ~3u;
        arr[p] = q; addr[i] = p; p = q;
    }
    addr[steps] = p;
}
__global__ void pf(const unsigned *arr, const unsigned *addr, int steps, int mode) {
    for (int i = threadIdx.x; i < steps; i += blockDim.x) {
        const unsigned *p = arr + addr[i];
        if (mode == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        if (mode == 2) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 16;" ::"l"(p) : "memory");
        if (mode == 3) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
    }
}
__global__ void chase(const unsigned *arr, unsigned start, int steps, long long *out) {
    unsigned p = start;
    long long c0 = clock64();
    for (int i = 0; i < steps; ++i) p = __ldcg(arr + p);
    long long c1 = clock64();
    out[0] = (c1 - c0) / steps; out[1] = p;
}
int main() {
    const unsigned n = 96u << 20;  // 384 MB of uint32
    const int steps = 2000;
    unsigned *arr, *addr; long long *out; long long h[2];
    cudaMalloc(&arr, (size_t)n * 4); cudaMalloc(&addr, (steps + 1) * 4); cudaMalloc(&out, 16);
    unsigned *flush; cudaMalloc(&flush, 512u << 20);
    const char *names[] = {"cold (no prefetch)", "prefetch.global.L2", "cp.async.bulk.prefetch.L2", "prefetch.L2::evict_last", "warm (second chase)"};
    for (int mode = 0; mode < 5; ++mode) {
        unsigned seed = 12345u + 7919u * mode;
        build<<<1, 1>>>(arr, n, steps, seed, addr);
        cudaMemset(flush, mode, 512u << 20);  // evict L2
        unsigned start; cudaMemcpy(&start, addr, 4, cudaMemcpyDeviceToHost);
        if (mode >= 1 && mode <= 3) pf<<<1, 256>>>(arr, addr, steps, mode);
        if (mode == 4) chase<<<1, 1>>>(arr, start, steps, out);
        cudaDeviceSynchronize();
        chase<<<1, 1>>>(arr, start, steps, out);
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("%-28s %5lld cycles per dependent 4-B load\n", names[mode], h[0]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
