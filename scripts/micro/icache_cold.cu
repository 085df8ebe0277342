// Cost of executing straight-line code once when the L2 was just flushed (the kernel's code
// lines come from HBM): one 1024-thread CTA runs a body of N dependent-free integer ops
// (N * 16 B of SASS), after a 256 MiB memset vs after a tiny one.  Separates instruction
// fetch from launch cost (compare with N = 0).
#include <cstdio>
#include <cuda_runtime.h>
#ifndef THREADS
#define THREADS 1024
#endif
template <int N>
__global__ void k_body(unsigned* out, unsigned x) {
    unsigned a = threadIdx.x ^ x, b = a * 3u, c = a + 7u, d = a ^ 0x55u;
#pragma unroll
    for (int i = 0; i < N; i++) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(b) : "r"(c));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(c) : "r"(d));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(d) : "r"(a));
    }
    if (a + b + c + d == 0x12345u) out[threadIdx.x] = a;
}
template <int N>
void run(void* flush, bool big) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0; int n = 40;
    for (int i = 0; i < n + 5; i++) {
        cudaMemsetAsync(flush, i, big ? (256 << 20) : 4096);
        cudaEventRecord(e0);
        k_body<N><<<1, THREADS>>>(nullptr, i);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) tot += ms;
    }
    printf("N=%5d (%6d B of code) %s flush: %.2f us\n", N, N * 4 * 16, big ? "256 MiB" : "tiny   ", 1e3 * tot / n);
}
int main() {
    void* flush; cudaMalloc(&flush, 256 << 20);
    run<1>(flush, true); run<1>(flush, false);
    run<256>(flush, true); run<256>(flush, false);
    run<1024>(flush, true); run<1024>(flush, false);
    run<4096>(flush, true); run<4096>(flush, false);
    return 0;
}
