// kernels_sort.cu -- A4: onesweep LSD radix sort of the unique 64-bit keys
// (ascending = ranked order, Alg.1).  sm_100a.
//
// One kernel launch per 8-bit digit pass that does work (the K1 plan skips
// digit positions whose value is the same for every key).  Per pass, each CTA
// takes a tile of 2048 keys by a dynamic tile id (forward progress), ranks its
// keys by digit with a warp multisplit (__match_any_sync, stable), publishes
// its per-digit counts, resolves its global per-digit offsets by decoupled
// look-back over the preceding tiles, stages the keys digit-sorted in shared
// memory and scatters them in coalesced runs.  The global digit histograms were
// computed by K1, so every pass reads and writes each key exactly once.
#include "lamps_internal.h"

namespace lamps {

namespace {

constexpr uint32_t kFlagAgg = 1u, kFlagInc = 2u;
constexpr int kWarps = kSortThreads / 32;

__device__ __forceinline__ unsigned long long pack_status(uint32_t epoch, uint32_t flag,
                                                          uint32_t cnt) {
    return ((unsigned long long)epoch << 32) | ((unsigned long long)flag << 30) | cnt;
}

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(Bufs b, uint32_t pass, uint32_t epoch) {
    __shared__ uint32_t sh_whist[kWarps][kBins];     // per-warp digit counts -> warp prefix
    __shared__ uint32_t sh_tile_excl[kBins];         // tile-local digit offsets
    __shared__ uint32_t sh_gdst[kBins];              // global destination base per digit
    __shared__ uint32_t sh_scan[kWarps];
    __shared__ uint32_t sh_tile;
    __shared__ uint64_t sh_keys[kSortTile];          // digit-sorted staging

    Ctl* ctl = b.ctl;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t n_passes = __ldcg(&ctl->n_passes);
    if (pass >= n_passes) return;
    const uint32_t n = __ldcg(&ctl->n_elig);
    const uint32_t ntiles = (n + kSortTile - 1) / kSortTile;
    if (tid == 0) sh_tile = atomicAdd(&ctl->tile_ctr[pass], 1u);
    for (uint32_t i = tid; i < kWarps * kBins; i += kSortThreads) (&sh_whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = sh_tile;
    if (tile >= ntiles) return;
    const uint32_t shift = __ldcg(&ctl->shift[pass]);
    const uint64_t* __restrict__ in = b.keys[pass & 1u];
    uint64_t* __restrict__ out = b.keys[(pass + 1u) & 1u];
    const uint32_t base = tile * kSortTile;
    const uint32_t tn = min((uint32_t)kSortTile, n - base);

    // ---- load: warp-striped (warp w owns [w*256, w*256+256), item j at j*32+lane)
    uint64_t key[kSortItems];
    uint32_t dig[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t li = warp * (32 * kSortItems) + j * 32 + lane;
        key[j] = li < tn ? __ldcg(in + base + li) : ~0ull;
        dig[j] = li < tn ? (uint32_t)(key[j] >> shift) & 0xffu : 256u;
    }

    // ---- warp multisplit: stable rank of each key among same-digit keys of its warp
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t rank[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t d = dig[j];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t leader = __ffs(peers) - 1u;
        uint32_t prior = 0;
        if (d < 256u && lane == leader) {
            prior = sh_whist[warp][d];
            sh_whist[warp][d] = prior + __popc(peers);
        }
        prior = __shfl_sync(0xffffffffu, prior, leader);
        rank[j] = prior + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();

    // ---- per digit (thread = digit): exclusive prefix over warps, tile count
    const uint32_t d = tid;  // kSortThreads == kBins
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; w++) {
        const uint32_t v = sh_whist[w][d];
        sh_whist[w][d] = cnt;
        cnt += v;
    }
    // publish this tile's aggregate (tile 0 publishes its inclusive prefix)
    unsigned long long* st = b.status + (size_t)tile * kBins + d;
    st_status(st, pack_status(epoch, tile == 0 ? kFlagInc : kFlagAgg, cnt));

    // tile-local exclusive scan over digits
    {
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) sh_scan[warp] = x;
        __syncthreads();
        uint32_t before = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++)
            if ((uint32_t)w < warp) before += sh_scan[w];
        sh_tile_excl[d] = before + x - cnt;
    }

    // decoupled look-back for digit d
    uint32_t excl = 0;
    if (tile > 0) {
        int t = (int)tile - 1;
        while (true) {
            unsigned long long v;
            const unsigned long long* p = b.status + (size_t)t * kBins + d;
            while (true) {
                v = ld_status(p);
                if ((uint32_t)(v >> 32) == epoch && ((v >> 30) & 3u) != 0) break;
                __nanosleep(32);
            }
            excl += (uint32_t)(v & 0x3fffffffu);
            if (((v >> 30) & 3u) == kFlagInc) break;
            --t;
        }
        st_status(st, pack_status(epoch, kFlagInc, excl + cnt));
    }
    const uint32_t gbase = __ldg(&b.offs[pass * kBins + d]) + excl;
    sh_gdst[d] = gbase - sh_tile_excl[d];
    __syncthreads();

    // ---- stage digit-sorted in shared memory
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t dj = dig[j];
        if (dj < 256u) sh_keys[sh_tile_excl[dj] + sh_whist[warp][dj] + rank[j]] = key[j];
    }
    __syncthreads();

    // ---- scatter: consecutive staging positions of one digit go to consecutive addresses
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t i = j * kSortThreads + tid;
        if (i < tn) {
            const uint64_t k = sh_keys[i];
            const uint32_t dk = (uint32_t)(k >> shift) & 0xffu;
            out[sh_gdst[dk] + i] = k;
        }
    }
}

}  // namespace

cudaError_t launch_sort(const Bufs& b, const Cost& c, const StepArgs& a, uint32_t cap,
                        cudaStream_t s, cudaEvent_t* mid_events) {
    (void)c;
    (void)mid_events;
    const uint32_t grid = (cap + kSortTile - 1) / kSortTile;
    for (uint32_t pass = 0; pass < (uint32_t)kDigits; pass++) {
        k_sort_pass<<<grid, kSortThreads, 0, s>>>(b, pass, a.epoch + pass);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace lamps
