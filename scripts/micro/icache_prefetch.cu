// Can a kernel prefetch its own code into L2?  After the 256 MiB flush the code lines of a
// kernel come from HBM one miss at a time (icache_cold.cu: ~36 ns per 128-B line).  Here the
// body is a __noinline__ device function; its address (a device function pointer) is used as a
// global address: (1) a load from it is compared with the SASS encoding, (2) the body's lines
// are requested into L2 (cp.async.bulk.prefetch.L2) by warp 0 at kernel start, before the
// body runs.  Time with and without the prefetch.
#include <cstdio>
#include <cuda_runtime.h>
#ifndef THREADS
#define THREADS 1024
#endif
template <int N>
__device__ __noinline__ unsigned body(unsigned a, unsigned b, unsigned c, unsigned d) {
#pragma unroll
    for (int i = 0; i < N; i++) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(b) : "r"(c));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(c) : "r"(d));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(d) : "r"(a));
    }
    return a + b + c + d;
}
template <int N>
__global__ void k_run(unsigned* out, unsigned x, int pf, int mode) {
    if (pf && threadIdx.x < 32) {
        unsigned (*fp)(unsigned, unsigned, unsigned, unsigned) = body<N>;
        const unsigned long long a0 = (unsigned long long)fp & ~127ull;
        const unsigned bytes = (N * 64 + 1024 + 127) & ~127u;
        if (mode == 0) {  // bulk prefetch, 32 KB pieces spread over the lanes
            for (unsigned o = threadIdx.x * 4096u; o < bytes; o += 32u * 4096u) {
                const unsigned n = bytes - o < 4096u ? bytes - o : 4096u;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0 + o), "r"(n) : "memory");
            }
        } else {  // per-line prefetch
            for (unsigned o = threadIdx.x * 128u; o < bytes; o += 32u * 128u)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a0 + o));
        }
    }
    const unsigned a = threadIdx.x ^ x;
    const unsigned r = body<N>(a, a * 3u, a + 7u, a ^ 0x55u);
    if (r == 0x12345u) out[threadIdx.x] = r;
}
__global__ void k_probe(unsigned long long* out) {
    unsigned (*fp)(unsigned, unsigned, unsigned, unsigned) = body<16>;
    const unsigned long long a = (unsigned long long)fp;
    out[0] = a;
    unsigned long long v0 = 0, v1 = 0;
    asm volatile("ld.global.u64 %0, [%1];" : "=l"(v0) : "l"(a));
    asm volatile("ld.global.u64 %0, [%1+8];" : "=l"(v1) : "l"(a));
    out[1] = v0;
    out[2] = v1;
}
template <int N>
void run(void* flush, int pf, int mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0; int n = 40;
    for (int i = 0; i < n + 5; i++) {
        cudaMemsetAsync(flush, i, 256 << 20);
        cudaEventRecord(e0);
        k_run<N><<<148, THREADS>>>(nullptr, i, pf, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) tot += ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("N=%5d (%6d B of code) prefetch %d mode %d: %.2f us  (%s)\n", N, N * 64, pf, mode, 1e3 * tot / n,
           cudaGetErrorString(e));
}
int main(int argc, char** argv) {
    if (argc > 1) {  // probe: does a load from the function address return the code?
        unsigned long long* d; cudaMalloc(&d, 64);
        k_probe<<<1, 1>>>(d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[3] = {0};
        cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        printf("probe: err %s addr 0x%llx words 0x%016llx 0x%016llx\n", cudaGetErrorString(e), h[0], h[1], h[2]);
        return 0;
    }
    void* flush; cudaMalloc(&flush, 256 << 20);
    for (int pf = 0; pf < 3; pf++) {
        const int p = pf ? 1 : 0, m = pf == 2 ? 1 : 0;
        run<256>(flush, p, m);
        run<1024>(flush, p, m);
        run<4096>(flush, p, m);
    }
    return 0;
}
