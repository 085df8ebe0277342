// sort_dev.cuh -- grid-synchronous LSD radix sort of 64-bit keys in global memory
// (device function, used by the standalone sort kernel of the multi-kernel path
// and as the fallback of the fused step kernel), and the grid barrier.
#pragma once
#include "lamps_internal.h"

namespace lamps {

constexpr int kSortWarps = kSortThreads / 32;  // 32

struct SortSmem {
    uint64_t stage[kSortTile];                       // 64 KB: digit-sorted staging
    uint32_t whist[kSortWarps][kBins];               // 32 KB: per-warp digit counts -> prefix
    uint32_t tcnt[kSortMaxTilesPerCta][kBins];       // own tiles' digit counts
    uint32_t tbase[kSortMaxTilesPerCta][kBins];      // own tiles' global digit bases
    uint32_t texcl[kBins];                           // tile-local exclusive digit offsets
    uint32_t part[4][kBins];                         // count-exchange partial sums
    uint32_t scan[kSortWarps];
    uint32_t pass_shift[kDigits];
    uint32_t n_pass;
};

// Grid barrier for a cooperative launch (all CTAs resident), flat: thread 0 of
// every CTA adds 1 to a 64-bit counter that only grows (acq_rel atomic); the
// arrivals of one barrier are G consecutive counter values, so the CTA whose add
// returned `old` waits until the counter reaches (old / G + 1) * G (acquire
// polls).  The counter is a multiple of G between barriers; kernels with
// different grid sizes use different counter lines (G mod 16).  Measured on B200
// with 148 x 1024 threads: 1.16 us per barrier, vs 2.57 us for a two-level tree
// (scripts/micro/barrier.cu).  `value` is unused (kept for the call sites'
// bookkeeping of barriers per step).
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t nblocks, uint32_t value) {
    (void)value;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(bar + 32u * (1u + (nblocks & 15u)));
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
        const unsigned long long target = (old / nblocks + 1ull) * nblocks;
        if (old + 1ull != target) {
            unsigned long long cur;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(cnt) : "memory");
            } while (cur < target);
        }
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
    for (uint32_t i = tid; i < kSortWarps * kBins; i += kSortThreads) (&sm.whist[0][0])[i] = 0;
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
        const uint32_t peers = digit_peers(d);
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
    for (int w = 0; w < kSortWarps; w++) {
        const uint32_t v = sm.whist[w][d];
        sm.whist[w][d] = cnt;
        cnt += v;
    }
    return cnt;
}

// exclusive scan over the 256 digits held by threads 0..255 (all threads must call)
__device__ __forceinline__ uint32_t digit_excl_scan(uint32_t* scan_ws, uint32_t v) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (tid < kBins && lane == 31) scan_ws[warp] = x;
    __syncthreads();
    uint32_t before = 0;
    if (tid < kBins)
        for (uint32_t w = 0; w < warp; w++) before += scan_ws[w];
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

// LSD sort of b.keys[0][0..n) over the 8-bit digit positions whose bits vary
// (OR / AND of the keys from nmask per-block partials at kmask[0..nmask) and
// kmask[nmask..2*nmask)).  Every CTA of the cooperative grid calls it.
// Passes alternate keys[0] -> keys[1] -> ...; returns the number of passes
// (the result is in keys[passes & 1]).
//
// per pass: A  each CTA ranks its tile(s) with a stable warp multisplit
// (__match_any_sync) and publishes its per-digit counts;  grid barrier;
// B  each CTA reads the counts of all CTAs (digit totals) and of the CTAs
// before it (its offsets);  C  keys are staged digit-sorted in shared memory
// and written in coalesced runs;  grid barrier.
__device__ __forceinline__ uint32_t lsd_sort_global(const Bufs& b, uint32_t n,
                                                    const unsigned long long* kmask, uint32_t nmask,
                                                    SortSmem& sm, uint32_t& bar) {
    const uint32_t tid = threadIdx.x;
    const uint32_t G = gridDim.x, bid = blockIdx.x;

    if (tid < 32) {
        unsigned long long o = 0, a = ~0ull;
        for (uint32_t i = tid; i < nmask; i += 32) {
            o |= __ldcg(&kmask[i]);
            a &= __ldcg(&kmask[nmask + i]);
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
        }
    }
    __syncthreads();
    const uint32_t n_pass = sm.n_pass;
    if (n_pass == 0) return 0;

    const uint32_t per = (n + G - 1) / G;
    const uint32_t lo_cta = min(n, bid * per), hi_cta = min(n, lo_cta + per);
    const uint32_t ntile = (hi_cta - lo_cta + kSortTile - 1) / kSortTile;  // <= kSortMaxTilesPerCta

    uint64_t key[kSortItems];
    uint32_t dig[kSortItems], rank[kSortItems];

    for (uint32_t p = 0; p < n_pass; p++) {
        const uint32_t shift = sm.pass_shift[p];
        const uint64_t* __restrict__ in = b.keys[p & 1u];
        uint64_t* __restrict__ out = b.keys[(p + 1u) & 1u];
        uint32_t* bsum = b.blocksum + (size_t)(p & 1u) * G * kBins;

        // ---- A
        uint32_t own = 0;
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
        grid_barrier(b.flags, G, ++bar);

        // ---- B: digit base + counts of the CTAs before this one (4 partials per digit,
        //         loads batched 8 at a time to keep them in flight)
        {
            const uint32_t d = tid & (kBins - 1), q = tid >> 8;
            uint32_t before = 0, total = 0;
            for (uint32_t c0 = q; c0 < G; c0 += 32) {
                uint32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const uint32_t c = c0 + 4u * u;
                    v[u] = c < G ? __ldcg(&bsum[(size_t)c * kBins + d]) : 0u;
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const uint32_t c = c0 + 4u * u;
                    total += v[u];
                    before += c < bid ? v[u] : 0u;
                }
            }
            sm.part[q][d] = before;
            __syncthreads();
            uint32_t tot_d = 0, bef_d = 0;
            if (tid < kBins) bef_d = sm.part[0][d] + sm.part[1][d] + sm.part[2][d] + sm.part[3][d];
            __syncthreads();
            sm.part[q][d] = total;
            __syncthreads();
            if (tid < kBins) tot_d = sm.part[0][d] + sm.part[1][d] + sm.part[2][d] + sm.part[3][d];
            const uint32_t dbase = digit_excl_scan(sm.scan, tid < kBins ? tot_d : 0u);
            if (tid < kBins) {
                uint32_t run = dbase + bef_d;
                for (uint32_t t = 0; t < ntile; t++) {
                    sm.tbase[t][tid] = run;
                    run += sm.tcnt[t][tid];
                }
            }
            __syncthreads();
        }

        // ---- C
        for (uint32_t t = 0; t < ntile; t++) {
            const uint32_t lo = lo_cta + t * kSortTile, tn = min((uint32_t)kSortTile, hi_cta - lo);
            if (ntile > 1) {  // registers hold only the last tile's ranking
                rank_tile(in, lo, tn, shift, sm, key, dig, rank);
                if (tid < kBins) (void)warp_prefix(sm, tid);
                __syncthreads();
            }
            const uint32_t e = digit_excl_scan(sm.scan, tid < kBins ? sm.tcnt[t][tid] : 0u);
            if (tid < kBins) sm.texcl[tid] = e;
            __syncthreads();
            scatter_tile(out, tn, shift, sm, sm.tbase[t], key, dig, rank);
        }
        if (p + 1 < n_pass) grid_barrier(b.flags, G, ++bar);
    }
    return n_pass;
}

}  // namespace lamps
