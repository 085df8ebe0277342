// kernels_ingest.cu -- predictor ingest and error injection.
//
// k_predict turns one truth record per thread into a predicted segment:
// bin -> tokens (10 b + 5) and the paper's Gaussian error injection
// predicted = max(0, m + N(0, p m)) with an integer,
// counter-based normal draw (reading R27, include/lamps.h lamps_noise):
// 17 splitmix64 words per (record, field); the popcount of 16 of them is
// Binomial(1024, 1/2), the 17th adds a uniform dither of one binomial step.
// All integer: the same draw on any device or host.
#include "lamps_internal.h"

namespace lamps {

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// output number n (1-based) of splitmix64 seeded with `seed`
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t n) {
    uint64_t z = seed + n * kGolden;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Z = (X - 512) 2^16 + dither, z = Z / 2^20 ~ N(0, 1)
__device__ __forceinline__ long long normal_q20(uint64_t seed, uint64_t key, uint32_t field) {
    const uint64_t n0 = (key * 4u + field) * 32u + 1u;
    int x = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) x += __popcll(splitmix_at(seed, n0 + (uint64_t)k));
    const long long u = (long long)(splitmix_at(seed, n0 + 16u) >> 48);
    return (long long)(x - 512) * 65536ll + u - 32768ll;
}

// m + round-half-away(ppm * m * Z / (1e6 * 2^20)), clamped to [0, hi]
__device__ __forceinline__ uint32_t perturb(uint32_t m, uint32_t ppm, long long Z, uint64_t hi) {
    if (ppm == 0u || m == 0u) return m;
    const unsigned __int128 den = (unsigned __int128)1000000u << 20;
    const unsigned __int128 mag = (unsigned __int128)((uint64_t)ppm * m) * (uint64_t)(Z < 0 ? -Z : Z);
    const uint64_t e = (uint64_t)((mag + den / 2u) / den);  // |error| < 2^42 (ppm <= 1e7, |Z| < 2^26)
    long long v = (long long)m + (Z < 0 ? -(long long)e : (long long)e);
    if (v < 0) v = 0;
    return (uint64_t)v > hi ? (uint32_t)hi : (uint32_t)v;
}

__global__ void k_predict(const TruthRec* __restrict__ in, PredRec* __restrict__ out, uint32_t n, uint64_t seed,
                          uint32_t len_ppm, uint32_t api_ppm) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const TruthRec t = in[i];
    const uint32_t pre_m = t.pre_bin == 0xffffffffu ? t.pre : t.pre_bin * 10u + 5u;
    PredRec r;
    r.pre = len_ppm ? perturb(pre_m, len_ppm, normal_q20(seed, t.key, 0u), 1ull << 24) : pre_m;
    r.resp = t.has ? t.resp : 0u;
    r.post = 0u;
    r.api = 0u;
    if (t.has) {
        r.post = len_ppm ? perturb(t.post, len_ppm, normal_q20(seed, t.key, 1u), 1ull << 24) : t.post;
        r.api = api_ppm ? perturb(t.api, api_ppm, normal_q20(seed, t.key, 2u), 0xffffffffull) : t.api;
    }
    out[i] = r;
}

}  // namespace

cudaError_t launch_predict(const TruthRec* d_in, PredRec* d_out, uint32_t n, uint64_t seed, uint32_t len_ppm,
                           uint32_t api_ppm, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_predict<<<(n + 255) / 256, 256, 0, s>>>(d_in, d_out, n, seed, len_ppm, api_ppm);
    return cudaGetLastError();
}

}  // namespace lamps
