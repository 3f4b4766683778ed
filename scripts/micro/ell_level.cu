// Microbenchmark of one bounded-degree BFS level's dependent chain, outside
// the BFS kernel: 18 warps (one per CTA of 296) each take 32 frontier entries,
// load the 16-B adjacency record, then issue 4 claims (atomicOr with return)
// on a 3 MB bitmap. Per-phase globaltimer stamps of lane 0 of warp 0.
// Variants: claims as atomicOr / as plain loads; bitmap warm (L2) or cold.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory"); return t; }
__device__ __forceinline__ int4 ldnc(const int4 *p) { int4 r; asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w) : "l"(p)); return r; }
__global__ void level(const int *qv, int f, const int4 *ell, unsigned *vis, long long *out, int mode) {
    const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    const int j = gw * 32 + (threadIdx.x & 31);
    if (gw * 32 >= f) return;
    long long t0 = gt();
    int v = j < f ? qv[j] : 0;
    volatile int d0 = v; (void)d0;
    long long t1 = gt();
    int4 s = ldnc(ell + v);
    volatile int d1 = s.x; (void)d1;
    long long t2 = gt();
    int sl[4] = {s.x, s.y, s.z, s.w};
    unsigned o[4];
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < 4; ++k) {
        unsigned *p = vis + ((unsigned)sl[k] >> 5);
        if (mode == 3) p = vis + (((unsigned)sl[0] >> 5) & ~31u) + lane + 32 * k;   // coalesced
        o[k] = 0;
        if (mode == 2 && k > 0) continue;
        if (mode == 4 && lane != 0) continue;
        o[k] = mode == 0 ? atomicOr(p, 1u << (sl[k] & 31)) : __ldcg(p);
    }
    volatile unsigned d2 = o[0] + o[1] + o[2] + o[3]; (void)d2;
    long long t3 = gt();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] += t1 - t0; out[1] += t2 - t1; out[2] += t3 - t2; out[3] += 1; }
}
__global__ void init(int *qv, int f, int4 *ell, int n, unsigned seed) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        ell[i] = make_int4((h * 7) % n, (h * 13 + 1) % n, (h * 31 + 7) % n, (h * 61 + 3) % n);
        if (i < f) qv[i] = (h * 97 + 11) % n;
    }
}
__global__ void newq(int *qv, int f, int n, unsigned seed) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < f) qv[i] = (int)((((unsigned)i * 2654435761u) ^ seed) * 97u % (unsigned)n);
}
__global__ void touch(const unsigned *vis, int words, unsigned *sink) {
    unsigned acc = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x) acc += __ldcg(vis + i);
    if (acc == 0x12345) *sink = acc;
}
int main() {
    const int n = 24000000, f = 560, words = (n + 31) / 32;
    int *qv; int4 *ell; unsigned *vis, *sink; long long *out;
    cudaMalloc(&qv, f * 4); cudaMalloc(&ell, (size_t)n * 16); cudaMalloc(&vis, words * 4); cudaMalloc(&sink, 4); cudaMalloc(&out, 64);
    for (int mode = 0; mode < 5; ++mode) for (int warm = 1; warm < 2; ++warm) {
        cudaMemset(out, 0, 64); cudaMemset(vis, 0, words * 4);
        for (int it = 0; it < 200; ++it) {
            if (it == 0) init<<<1024, 256>>>(qv, f, ell, n, 0x9e37u);
            newq<<<4, 256>>>(qv, f, n, 0x9e37u * (it + 1));  // fresh random queue each round
            if (warm) touch<<<296, 512>>>(vis, words, sink);
            level<<<296, 512>>>(qv, f, ell, vis, out, mode);
        }
        long long h[4]; cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        const char *names[] = {"4 atomics  ", "4 loads    ", "1 load     ", "4 coalesced", "lane0 only "};
        printf("%s %s: qv %.0f ns, record %.0f ns, 4 claims %.0f ns\n", names[mode], warm ? "warm bitmap" : "cold bitmap",
               (double)h[0] / h[3], (double)h[1] / h[3], (double)h[2] / h[3]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
