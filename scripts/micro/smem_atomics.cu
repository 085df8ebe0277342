// Microbenchmark: shared-memory counting throughput on B200, 1024-thread CTA per SM,
// random 14-bit bins: atomicAdd with return, atomicAdd result unused (RED), and
// conflict-free plain LDS/STS for reference.  Reports SM cycles per key.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, int iters, uint32_t seed) {
    __shared__ uint32_t cnt[8192];
    for (int i = threadIdx.x; i < 8192; i += 1024) cnt[i] = 0;
    __syncthreads();
    uint32_t x = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 97u);
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        x = x * 1664525u + 1013904223u;
        uint32_t d = x >> 19;
        if (MODE == 0) acc += atomicAdd(&cnt[d], 1u);
        else if (MODE == 1) atomicAdd(&cnt[d], 1u);
        else if (MODE == 2) { acc += cnt[(threadIdx.x + i * 32) & 8191]; }
        else { cnt[(threadIdx.x * 16 + i) & 8191] += 1; }  // private column RMW (conflict-prone layout)
    }
    __syncthreads();
    out[blockIdx.x * 1024 + threadIdx.x] = acc + cnt[threadIdx.x];
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* o; cudaMalloc(&o, sms * 1024 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    const char* names[] = {"atomicAdd+ret", "atomicAdd(RED)", "LDS (ref)", "RMW col"};
    for (int mode = 0; mode < 4; mode++) {
        float ms = 0;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<sms, 1024>>>(o, iters, rep);
            else if (mode == 1) k<1><<<sms, 1024>>>(o, iters, rep);
            else if (mode == 2) k<2><<<sms, 1024>>>(o, iters, rep);
            else k<3><<<sms, 1024>>>(o, iters, rep);
            cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("%-16s %.3f ms  %.2f SM-cycles per key\n", names[mode], ms, ms * 1e-3 * 1.965e9 / (iters * 1024.0));
    }
    return 0;
}
