// kernels_sort.cu -- A4: LSD radix sort of the unique 64-bit keys, ascending
// (= ranked order, Alg.1).  sm_100a.
//
// One persistent cooperative launch does every pass.  The grid is exactly the
// set of CTAs that can be resident (one 1024-thread CTA per SM), so the whole
// key set is processed by a single wave and CTAs can synchronise:
//
//   per pass (8-bit digit, only digit positions whose bits vary -- from the
//   per-block key OR/AND that K1 produced):
//     A  each CTA loads its tile(s) (warp-striped, 8 keys/thread) and ranks
//        every key among the same-digit keys of its warp with a stable warp
//        multisplit (__match_any_sync); per-digit counts of its keys go to
//        global memory
//     -- grid barrier --
//     B  each CTA reads the counts of the CTAs before it (its global per-digit
//        offsets) and of all CTAs (digit totals -> digit bases)
//     C  keys are staged digit-sorted in shared memory and written to their
//        final positions in coalesced runs
//     -- grid barrier --
//
// This replaces the per-tile decoupled look-back of a classic onesweep pass:
// measured on B200 (profiles/r01/ncu_v0_lookback.txt) the look-back over ~450
// concurrently started tiles serialised (25 us per pass); with one resident
// wave a grid-synchronous exchange of per-CTA counts is shorter and exact.
#include <cooperative_groups.h>

#include "lamps_internal.h"

namespace lamps {

namespace {

constexpr int kWarps = kSortThreads / 32;  // 32

struct SortSmem {
    uint64_t stage[kSortTile];                       // 64 KB: digit-sorted staging
    uint32_t whist[kWarps][kBins];                   // 32 KB: per-warp digit counts -> prefix
    uint32_t tcnt[kSortMaxTilesPerCta][kBins];       // own tiles' digit counts
    uint32_t tbase[kSortMaxTilesPerCta][kBins];      // own tiles' global digit bases
    uint32_t texcl[kBins];                           // tile-local exclusive digit offsets
    uint32_t part[4][kBins];                         // phase B partial sums
    uint32_t scan[kWarps];
    uint32_t pass_shift[kDigits];
    uint32_t n_pass;
};

__device__ __forceinline__ void grid_barrier(Ctl* ctl, uint32_t nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t* gen = &ctl->bar_gen;
        const uint32_t g = *gen;
        __threadfence();
        if (atomicAdd(&ctl->bar_count, 1u) == nblocks - 1) {
            ctl->bar_count = 0;
            __threadfence();
            atomicAdd(&ctl->bar_gen, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// Stable rank of each key of one tile among the same-digit keys of its warp.
// Keys are warp-striped: warp w owns tile positions [w*256, w*256+256); item j
// of lane l is position w*256 + j*32 + l, so (j, lane) order is tile order.
__device__ __forceinline__ void rank_tile(const uint64_t* __restrict__ in, uint32_t lo, uint32_t tn,
                                          uint32_t shift, SortSmem& sm, uint64_t (&key)[kSortItems],
                                          uint32_t (&dig)[kSortItems], uint32_t (&rank)[kSortItems]) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint32_t i = tid; i < kWarps * kBins; i += kSortThreads) (&sm.whist[0][0])[i] = 0;
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t li = warp * (32 * kSortItems) + j * 32 + lane;
        key[j] = li < tn ? __ldcg(in + lo + li) : ~0ull;
        dig[j] = li < tn ? (uint32_t)(key[j] >> shift) & 0xffu : 256u;
    }
    __syncthreads();
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t d = dig[j];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t leader = __ffs(peers) - 1u;
        uint32_t prior = 0;
        if (d < 256u && lane == leader) {
            prior = sm.whist[warp][d];
            sm.whist[warp][d] = prior + __popc(peers);
        }
        prior = __shfl_sync(0xffffffffu, prior, leader);
        rank[j] = prior + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();
}

// per digit d (threads 0..255): warp counts -> exclusive prefix over warps; returns the tile count
__device__ __forceinline__ uint32_t warp_prefix(SortSmem& sm, uint32_t d) {
    uint32_t cnt = 0;
#pragma unroll 8
    for (int w = 0; w < kWarps; w++) {
        const uint32_t v = sm.whist[w][d];
        sm.whist[w][d] = cnt;
        cnt += v;
    }
    return cnt;
}

// exclusive scan over the 256 digits held by threads 0..255 (all threads must call)
__device__ __forceinline__ uint32_t digit_excl_scan(SortSmem& sm, uint32_t v) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (tid < kBins && lane == 31) sm.scan[warp] = x;
    __syncthreads();
    uint32_t before = 0;
    if (tid < kBins)
        for (uint32_t w = 0; w < warp; w++) before += sm.scan[w];
    __syncthreads();
    return before + x - v;
}

__device__ __forceinline__ void scatter_tile(uint64_t* __restrict__ out, uint32_t tn, uint32_t shift,
                                             SortSmem& sm, const uint32_t* gbase,
                                             const uint64_t (&key)[kSortItems],
                                             const uint32_t (&dig)[kSortItems],
                                             const uint32_t (&rank)[kSortItems]) {
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t d = dig[j];
        if (d < 256u) sm.stage[sm.texcl[d] + sm.whist[warp][d] + rank[j]] = key[j];
    }
    __syncthreads();
    for (uint32_t i = tid; i < tn; i += kSortThreads) {
        const uint64_t k = sm.stage[i];
        const uint32_t d = (uint32_t)(k >> shift) & 0xffu;
        out[gbase[d] - sm.texcl[d] + i] = k;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSortThreads, 1) k_sort(Bufs b) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
    Ctl* ctl = b.ctl;
    const uint32_t tid = threadIdx.x;
    const uint32_t G = gridDim.x, bid = blockIdx.x;
    const uint32_t n = __ldcg(&ctl->n_elig);

    // ---- digit positions whose bits vary across the keys (from K1's OR/AND)
    if (tid < 32) {
        unsigned long long o = 0, a = ~0ull;
        for (uint32_t i = tid; i < b.score_grid; i += 32) {
            o |= __ldcg(&b.kmask[i]);
            a &= __ldcg(&b.kmask[b.score_grid + i]);
        }
#pragma unroll
        for (int s = 16; s; s >>= 1) {
            o |= __shfl_xor_sync(0xffffffffu, o, s);
            a &= __shfl_xor_sync(0xffffffffu, a, s);
        }
        if (tid == 0) {
            const unsigned long long vary = n ? (o ^ a) : 0ull;
            uint32_t np = 0;
            for (int d = 0; d < kDigits; d++)
                if ((vary >> (8 * d)) & 0xffull) sm.pass_shift[np++] = 8u * d;
            sm.n_pass = np;
            if (bid == 0) ctl->n_passes = np;
        }
    }
    __syncthreads();
    const uint32_t n_pass = sm.n_pass;
    if (n_pass == 0) return;

    // ---- this CTA's tiles: keys [bid*per, (bid+1)*per) in tiles of <= kSortTile
    const uint32_t per = (n + G - 1) / G;
    const uint32_t lo_cta = min(n, bid * per), hi_cta = min(n, lo_cta + per);
    const uint32_t ntile = (hi_cta - lo_cta + kSortTile - 1) / kSortTile;  // <= kSortMaxTilesPerCta

    uint64_t key[kSortItems];
    uint32_t dig[kSortItems], rank[kSortItems];

    for (uint32_t p = 0; p < n_pass; p++) {
        const uint32_t shift = sm.pass_shift[p];
        const uint64_t* __restrict__ in = b.keys[p & 1u];
        uint64_t* __restrict__ out = b.keys[(p + 1u) & 1u];
        uint32_t* bsum = b.blocksum + (size_t)(p & 1u) * b.sort_grid * kBins;

        // ---- A: per-tile digit counts (tile 0's ranking is kept in registers)
        uint32_t own = 0;  // this CTA's count of digit tid
        for (uint32_t t = 0; t < ntile; t++) {
            const uint32_t lo = lo_cta + t * kSortTile, tn = min((uint32_t)kSortTile, hi_cta - lo);
            rank_tile(in, lo, tn, shift, sm, key, dig, rank);
            if (tid < kBins) {
                const uint32_t c = warp_prefix(sm, tid);
                sm.tcnt[t][tid] = c;
                own += c;
            }
            __syncthreads();
        }
        if (tid < kBins) bsum[(size_t)bid * kBins + tid] = own;
        grid_barrier(ctl, G);

        // ---- B: global base of each digit for this CTA = digit base + counts of earlier CTAs
        {
            const uint32_t d = tid & (kBins - 1), q = tid >> 8;  // 4 partial sums per digit
            uint32_t before = 0, total = 0;
            for (uint32_t c = q; c < G; c += 4) {
                const uint32_t v = __ldcg(&bsum[(size_t)c * kBins + d]);
                total += v;
                if (c < bid) before += v;
            }
            sm.part[q][d] = before;
            __syncthreads();
            uint32_t tot_d = 0, bef_d = 0;
            if (tid < kBins) bef_d = sm.part[0][d] + sm.part[1][d] + sm.part[2][d] + sm.part[3][d];
            __syncthreads();
            sm.part[q][d] = total;
            __syncthreads();
            if (tid < kBins) tot_d = sm.part[0][d] + sm.part[1][d] + sm.part[2][d] + sm.part[3][d];
            const uint32_t dbase = digit_excl_scan(sm, tid < kBins ? tot_d : 0u);
            if (tid < kBins) {
                uint32_t run = dbase + bef_d;
                for (uint32_t t = 0; t < ntile; t++) {
                    sm.tbase[t][tid] = run;
                    run += sm.tcnt[t][tid];
                }
            }
            __syncthreads();
        }

        // ---- C: stage digit-sorted, scatter in coalesced runs
        for (uint32_t t = 0; t < ntile; t++) {
            const uint32_t lo = lo_cta + t * kSortTile, tn = min((uint32_t)kSortTile, hi_cta - lo);
            if (ntile > 1) {  // re-rank (registers hold only the last tile)
                rank_tile(in, lo, tn, shift, sm, key, dig, rank);
                if (tid < kBins) (void)warp_prefix(sm, tid);
                __syncthreads();
            }
            const uint32_t e = digit_excl_scan(sm, tid < kBins ? sm.tcnt[t][tid] : 0u);
            if (tid < kBins) sm.texcl[tid] = e;
            __syncthreads();
            scatter_tile(out, tn, shift, sm, sm.tbase[t], key, dig, rank);
        }
        if (p + 1 < n_pass) grid_barrier(ctl, G);
    }
}

}  // namespace

int sort_blocks_per_sm() {
    int nb = 0;
    cudaFuncSetAttribute(k_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sort, kSortThreads, sizeof(SortSmem));
    return nb;
}

cudaError_t launch_sort(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s) {
    (void)c;
    (void)a;
    Bufs bb = b;
    void* args[] = {&bb};
    return cudaLaunchCooperativeKernel((const void*)k_sort, dim3(b.sort_grid), dim3(kSortThreads), args,
                                       sizeof(SortSmem), s);
}

}  // namespace lamps
