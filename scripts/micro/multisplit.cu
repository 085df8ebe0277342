// Microbenchmark: cost of a stable warp multisplit peer mask for 8-bit digits,
// __match_any_sync vs 9 ballots, at full occupancy of 1024-thread CTAs on every SM.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t peers_ballot(uint32_t d) {
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) { uint32_t on = (d >> b) & 1u; uint32_t bb = __ballot_sync(~0u, on); m &= on ? bb : ~bb; }
    return m;
}
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x = seed ^ (threadIdx.x * 2654435761u) ^ blockIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        x = x * 1664525u + 1013904223u;
        uint32_t d = x >> 24;
        uint32_t p = MODE == 0 ? __match_any_sync(~0u, d) : peers_ballot(d);
        acc += __popc(p & ((1u << (threadIdx.x & 31)) - 1u));
    }
    out[blockIdx.x * 1024 + threadIdx.x] = acc;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* o; cudaMalloc(&o, sms * 1024 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    for (int mode = 0; mode < 2; mode++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<sms, 1024>>>(o, iters, rep); else k<1><<<sms, 1024>>>(o, iters, rep);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double per_warp_op = ms * 1e-3 * 1.965e9 / (iters * 32.0);  // SM cycles per warp-op (32 warps/SM)
            if (rep == 2) printf("%s: %.3f ms, %.1f SM-cycles per warp multisplit (32 warps/SM)\n",
                                 mode == 0 ? "match_any" : "ballot x8", ms, per_warp_op);
        }
    }
    return 0;
}
