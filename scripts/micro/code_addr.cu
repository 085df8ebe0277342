// Can a kernel see its own code through a device function pointer?  Reads the first words at
// the address of a __noinline__ device function (compare with cuobjdump's encoding) and the
// address of the kernel relative to it.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __noinline__ int marker(int x) { return x * 3 + 1; }
__global__ void k(unsigned long long* out, int x) {
    int (*fp)(int) = marker;
    const unsigned long long a = (unsigned long long)fp;
    out[0] = a;
    unsigned long long v = 0;
    asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(a));
    out[1] = v;
    asm volatile("ld.global.u64 %0, [%1+8];" : "=l"(v) : "l"(a));
    out[2] = v;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    out[3] = fp(x);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 64);
    k<<<1, 1>>>(d, 5);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[4] = {0};
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("err %s addr 0x%llx words 0x%016llx 0x%016llx ret %llu\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
    return 0;
}
