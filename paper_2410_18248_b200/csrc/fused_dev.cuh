#pragma once
// fused_dev.cuh -- device pieces of the fused step kernel (kernels_fused.cu) and the one-CTA
// small-pool kernel (kernels_small.cu): shared-memory layouts, bucket tables, the on-chip range
// sorts, the local LSD.  (Included by both translation units; anonymous namespace.)
//
// The whole scheduling step (A0 default update .. A5) as
// ONE cooperative kernel, one 1024-thread CTA per SM, for pools whose per-SM
// share of keys fits in shared memory (capacity <= #SM * kKcap).
//
//   S  score: each CTA scores its contiguous range of slots (A0 fused, A1, A2,
//      A3, key) and keeps its keys in shared memory, with a histogram over
//      "float-like" buckets of the key, (starving, bit length of the score, next
//      kBucketM score bits): an exact monotone function of the key
//   H  the CTA adds its bucket counts to the step's global totals with atomics;
//      the returned old values are its offsets inside the buckets
//   -- barrier --
//   X  bucket starts (scan of the totals) and scatter of the keys into bucket
//      order in global memory; every CTA derives the bucket-aligned key range
//      it will sort
//   -- barrier --
//   L  each CTA sorts its range (<= kKcap keys) on chip: keys in registers, one
//      counting pass by a per-bucket digit, rank-by-comparison inside the
//      sub-buckets (range_sort).  If any range exceeds kKcap (a huge bucket of
//      near-equal scores) every CTA runs the grid-synchronous global LSD sort
//      instead (sort_dev.cuh).
//   A  CTA 0 admits (A5) as soon as the head of the order it needs is sorted.
#include <algorithm>

#include "merge_dev.cuh"
#include "sort_dev.cuh"
#include "step_dev.cuh"

namespace lamps {

namespace {

constexpr int kFT = 1024;                   // threads per CTA
constexpr int kFW = kFT / 32;               // warps
constexpr int kKcap = kFusedKcap;           // keys per CTA in shared memory
constexpr int kMaxBuckets = 14848;          // bucket table capacity (bucket_t, bt_update)
constexpr int kTabW = 136;                  // bucket table: [0, 130) octave entries, [130] bucket count
constexpr uint32_t kTabNB = 130;
constexpr int kLocalItems = kKcap / kFT;    // 10
constexpr int kMaxCtas = 256;               // range weights: grid size limit
// splitters in shared memory: entry i at i + i / 16 (no bank conflicts in the binary search,
// whose steps read the odd multiples of 128, 64, ... -- same banks without the padding)
constexpr int kSplPad = kMaxCtas + 1 + (kMaxCtas + 1) / 16 + 1;
__host__ __device__ constexpr uint32_t spl_pos(uint32_t i) { return i + (i >> 4); }
// Global splitter grid per parity (written by each step for the next): fine[f], f = 0 .. 16 G;
// range r = keys in [fine[16 r], fine[16 r + 16]), the 15 entries between are its quantiles
// (the range sort's piecewise-linear digit); fine[16 G] = the largest key
constexpr int kSeg = 16;
constexpr int kSplG = kSeg * kMaxCtas + 16;

struct PhaseS {                  // S, H, X (cold), R
    uint64_t kbuf[kKcap];        // 80 KB: this CTA's keys (compacted, in no particular order)
    uint32_t cnt[kMaxBuckets];   // 58 KB: bucket counts (cold); R: with start, the keys sorted by range
    uint32_t start[kMaxBuckets]; // 58 KB: bucket totals -> bucket start positions (cold)
    uint32_t w32[kFW + 1];
    unsigned long long red[3][kFW];
    uint32_t nk, base;
    uint32_t vmask[kKcap / 32];  // S: which kbuf positions hold keys
    float ccost[kMaxCtas];       // range-sort cycles per key of each CTA (previous steps)
    uint32_t rb[kMaxCtas + 1], jb[kMaxCtas + 1];  // X: key / bucket boundaries of the ranges
    float wx[kMaxCtas + 1];      // X: exclusive prefix of the range weights
    alignas(16) unsigned long long spl[kSplPad];  // R: range r = keys in [spl[P(r)], spl[P(r + 1)]), P = spl_pos
    uint32_t lcnt[kMaxCtas + 1], lst[kMaxCtas + 1], gbase[kMaxCtas];  // R: this CTA's run per range
    uint32_t novf, nmiss;        // binned R: keys in the overflow list, hint misses queued
    alignas(8) unsigned long long hbar;  // binned R: the range hints' copy (mbarrier)
};
// Binned R: byte layout over sm.s.cnt + start (free in warm steps): range hints / ranges by
// position (the copy starts at the 16-B boundary below the CTA's first slot), G bins of kBinCap
// keys, the overflow list (position | index in the run << 14, every key of the CTA fits), the
// queue of hint misses.
constexpr uint32_t kBinCap = 56;
constexpr uint32_t kRbBins = (kKcap + 32u + 63u) & ~63u;
constexpr uint32_t kRbBinsMax = 148u * kBinCap * 8u;
constexpr uint32_t kRbOvl = kRbBins + kRbBinsMax;
constexpr uint32_t kRbMiss = kRbOvl + 4u * kKcap;
constexpr uint32_t kMissCap = (sizeof(uint32_t) * 2u * kMaxBuckets - kRbMiss) / 2u;
static_assert(kMissCap >= 512u, "binned R: the miss queue is too small");
__host__ __device__ constexpr bool bins_fit(uint32_t G) { return G <= 148u; }
// thread 0 at kernel start: the hints of slots [s_lo, s_hi) (16-B aligned around them) -> dst
__device__ __forceinline__ void range_hint_issue(unsigned long long& bar, uint8_t* dst, const uint8_t* hint,
                                                 uint32_t s_lo, uint32_t s_hi) {
    const uint32_t a0 = s_lo & ~15u, a1 = (s_hi + 15u) & ~15u;
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(a1 - a0) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)), "l"(hint + a0), "r"(a1 - a0), "r"(mb) : "memory");
}
__device__ __forceinline__ void range_hint_wait(unsigned long long& bar) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(mb) : "memory");
}
constexpr int kSubBits = 13;                // local MSD digit
constexpr int kSubBuckets = 1 << kSubBits;
constexpr uint32_t kMaxRankM = 32;          // largest group ranked by comparison
constexpr int kChunk = 1024;                // score phase: slots per cp.async chunk
constexpr int kMaxBig = 1024;               // groups per refinement list (else full LSD)
constexpr int kMaxLevels = 6;               // refinement passes before the LSD fallback
struct PhaseL {                  // L
    uint64_t a[kKcap];           // 96 KB
    uint64_t b[kKcap];           // 96 KB
    union {
        struct {                         // local LSD (fallback)
            uint16_t whist[kFW][kBins];  // 16 KB
            uint32_t part[4][kBins];     // 4 KB
            uint32_t texcl[kBins];
            uint32_t scan[kFW];
        };
        struct {                         // local MSD + rank
            uint32_t pos[kKcap > kSubBuckets ? kKcap : kSubBuckets];  // 40 KB: counts -> starts; sbi
            uint32_t w32[kFW + 1];
            uint32_t nbig;
        };
    };
    unsigned long long red[2][kFW];
    AdmitSmem adm;                                // admission scratch (CTA 0, keys stay in a[])
    uint32_t rsz[kMaxCtas], rpre[kMaxCtas];       // every range's size and position in the order
    unsigned long long fine[kSeg + 1], fcode[kSeg + 1];  // this range's grid entries, their key codes
    uint32_t shs[kSeg];                                  // range sort: per segment, the digit's shift
    uint32_t shr[kSeg];                                  // range_sort_tma: per segment, the raw-key shift (or 255)
    alignas(8) unsigned long long mbar;                  // range_sort_tma: the staging copy's mbarrier
    uint32_t gf[2];                                      // the next step's grid entries [gf0, gf1) in this range
};
struct FusedSmem {
    union {
        PhaseS s;
        PhaseL l;
        SortSmem g;
    };
    alignas(16) uint32_t btab[kTabW];  // this step's bucket table (bucket_t), every phase
    unsigned long long pin_all;        // CTA 0: A5's pinned total (summed right after the grid barrier)
};
// After the union, untouched by every phase: the peer-memory exchange's state (peer
// buffer pointers, prefetched at kernel start) and the in-kernel merge's small structures.
struct SmemTail {
    MergeRec* xp[32];
    AdmitSmem adm;
    uint32_t nv[32];
    unsigned long long hsum[2];
};
constexpr size_t kFusedSmemBytes = sizeof(FusedSmem) + ((sizeof(SmemTail) + 127) & ~(size_t)127);

// Bucket of a key: (starving flag, bit length e of v = the key's score|id bits, the
// next m_e bits of v) -- a float-like, exact monotone function of the key whose
// resolution m_e per octave (ns, e) comes from a table: entry ns*65+e = base | s << 16 |
// m << 24 (s = e-1-m: the low bits of v the bucket leaves free), bucket = base + the m
// bits of v below its leading one.  Over v rather than the score alone, so keys whose
// scores are equal or small (FCFS: all 0) still spread by id.  The table adapts to the
// key distribution: every step writes the next step's table from its own octave counts
// (bt_update), so buckets hold about the same number of keys; any valid table gives the
// same order (only the balance of the ranges depends on it).
__device__ __forceinline__ uint32_t bucket_t(uint64_t key, const uint32_t* tab, uint32_t vb, uint32_t& sv) {
    const uint32_t ns = (uint32_t)(key >> vb) & 1u;
    const uint64_t v = key & ((1ull << vb) - 1ull);
    const uint32_t e = 64u - (uint32_t)__clzll((long long)v);  // bit length
    const uint32_t t = tab[ns * 65u + e];
    sv = (t >> 16) & 63u;
    return (t & 0xffffu) + ((uint32_t)(v >> sv) & ((1u << (t >> 24)) - 1u));
}

// Next step's table from this step's bucket starts (exclusive scan `start` over the NB
// buckets of the current table `tab`, n keys): octave o gets 2^m' buckets with
// m' = floor(log2(n_o * kTabTarget / n)) (at least 1 bucket, at most 2^min(14, e-1)),
// empty octaves 2 buckets; bases are the prefix of the spans in (ns, e) order.  The
// total stays <= kTabTarget + 2 * 130 <= kMaxBuckets.  One warp.
constexpr uint32_t kTabTarget = 12288;
__device__ __forceinline__ void bt_update(const uint32_t* tab, const uint32_t* start, uint32_t n, uint32_t vb,
                                          uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t NB = tab[kTabNB];
    uint32_t carry = 0;
    for (uint32_t o0 = 0; o0 < kTabNB; o0 += 32) {
        const uint32_t o = o0 + lane;
        const uint32_t e = o % 65u;
        const bool valid = o < kTabNB && e <= vb;
        uint32_t span = 0, mq = 0;
        if (valid) {
            const uint32_t t = tab[o], base = t & 0xffffu, sp0 = 1u << (t >> 24);
            const uint32_t s0 = base < NB ? start[base] : n, s1 = base + sp0 < NB ? start[base + sp0] : n;
            const uint32_t no = s1 - s0, cap_m = e >= 1u ? min(14u, e - 1u) : 0u;
            if (no == 0) {
                mq = min(cap_m, 1u);
            } else {
                const uint64_t want = (uint64_t)no * kTabTarget / (n ? n : 1u);
                mq = want <= 1 ? 0u : min(cap_m, 63u - (uint32_t)__clzll((long long)want));
            }
            span = 1u << mq;
        }
        uint32_t x = span;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= (uint32_t)d) x += y;
        }
        const uint32_t base = carry + x - span;
        if (o < kTabNB) out[o] = valid ? (base | ((e >= 1u ? e - 1u - mq : 0u) << 16) | (mq << 24)) : base;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) out[kTabNB] = carry;
}

// Stable LSD sort of the n (<= kKcap) keys at src[0..n) in shared memory over the
// 8-bit digit positions where `vary` has bits, ping-ponging with dst[0..n);
// returns the buffer holding the result.  Keys are spread evenly over the 32
// warps: warp w owns the contiguous segment [w*32*ipt, (w+1)*32*ipt), item j of
// lane l is position w*32*ipt + j*32 + l, so (warp, j, lane) order is array
// order (stability).  Ranks come from a ballot multisplit (digit_peers).
__device__ __forceinline__ uint64_t* local_lsd(PhaseL& sm, uint64_t* src, uint64_t* dst, uint32_t n,
                                               unsigned long long vary) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t ipt = (n + kFT - 1) / kFT;  // items per lane, <= kLocalItems
    const uint32_t seg = 32u * ipt;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int dpos = 0; dpos < kDigits; dpos++) {
        if (!((vary >> (8 * dpos)) & 0xffull)) continue;
        const uint32_t shift = 8u * dpos;
        for (uint32_t i = tid; i < kFW * kBins; i += kFT) (&sm.whist[0][0])[i] = 0;
        __syncthreads();
        uint32_t pk[kLocalItems];  // digit << 16 | rank within the warp (digit 256 = empty)
#pragma unroll
        for (int j = 0; j < kLocalItems; j++) {
            pk[j] = 256u << 16;
            if ((uint32_t)j < ipt) {  // warp-uniform
                const uint32_t li = warp * seg + j * 32 + lane;
                const uint32_t d = li < n ? (uint32_t)(src[li] >> shift) & 0xffu : 256u;
                const uint32_t peers = digit_peers(d);
                const uint32_t leader = __ffs(peers) - 1u;
                uint32_t prior = 0;
                if (d < 256u && lane == leader) {
                    prior = sm.whist[warp][d];
                    sm.whist[warp][d] = (uint16_t)(prior + __popc(peers));
                }
                prior = __shfl_sync(0xffffffffu, prior, leader);
                pk[j] = (d << 16) | (prior + __popc(peers & lt_mask));
                __syncwarp();
            }
        }
        __syncthreads();
        {   // per digit: exclusive prefix over the 32 warps, 4 threads per digit (8 warps each)
            const uint32_t d = tid & 255u, q = tid >> 8;
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kFW / 4; w++) run += sm.whist[q * (kFW / 4) + w][d];
            sm.part[q][d] = run;
            __syncthreads();
            uint32_t before = 0, tot = 0;
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
                const uint32_t v = sm.part[qq][d];
                before += (uint32_t)qq < q ? v : 0u;
                tot += v;
            }
#pragma unroll
            for (int w = 0; w < kFW / 4; w++) {
                uint16_t& h = sm.whist[q * (kFW / 4) + w][d];
                const uint32_t v = h;
                h = (uint16_t)before;
                before += v;
            }
            const uint32_t e = digit_excl_scan(sm.scan, tid < kBins ? tot : 0u);
            if (tid < kBins) sm.texcl[tid] = e;
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < kLocalItems; j++) {
            const uint32_t d = pk[j] >> 16;
            if (d < 256u) {
                const uint32_t li = warp * seg + j * 32 + lane;
                dst[sm.texcl[d] + sm.whist[warp][d] + (pk[j] & 0xffffu)] = src[li];
            }
        }
        __syncthreads();
        uint64_t* t = src; src = dst; dst = t;
    }
    return src;
}

__device__ __forceinline__ void block_or_and(PhaseL& sm, const uint64_t* x, uint32_t n,
                                             unsigned long long& o, unsigned long long& an) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    o = 0; an = ~0ull;
    for (uint32_t i = tid; i < n; i += kFT) { o |= x[i]; an &= x[i]; }
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        an &= __shfl_xor_sync(0xffffffffu, an, s);
    }
    if (lane == 0) { sm.red[0][warp] = o; sm.red[1][warp] = an; }
    __syncthreads();
    o = 0; an = ~0ull;
    for (int w = 0; w < kFW; w++) { o |= sm.red[0][w]; an &= sm.red[1][w]; }
    __syncthreads();
}

constexpr uint32_t kHeadPre = 2560;
constexpr uint32_t kHeadMargin = 128;   // the head range: max_batch + this many keys of the previous order
// range_sort ranks sub-buckets of up to this many keys by comparison (one thread per
// key, O(size) shared-memory reads): cheaper than a refinement pass for the few
// sub-buckets of near-equal keys (e.g. saturated scores) a range may hold
#ifndef LAMPS_RANK_M  // A/B builds: scripts/build_variant.sh out.so -DLAMPS_RANK_M=...
#define LAMPS_RANK_M 256
#endif
constexpr uint32_t kRangeRankM = LAMPS_RANK_M;
constexpr uint32_t kHeadTC = 2 * kKcap / 2, kHeadTW = kHeadTC + kHeadPre;  // by initial position
constexpr uint32_t kHeadD = kHeadTW + kHeadPre, kHeadW = kHeadD + kHeadPre;  // sorted demand / state
static_assert(kHeadW + kHeadPre <= 2 * kKcap, "head arrays exceed sm.b");
// Sort of a CTA's key range (rn <= kKcap keys at src, global) into sm.a with one counting
// pass on a LINEAR digit of the key, d = (k - kmin) >> sh, over 2^ceil(log2 rn) counters
// spanning [kmin, kmax] of the range's own keys: a range between two quantiles of the order
// holds keys of about one octave, spread about evenly, so a counter holds ~1 key.  Keys of a
// counter are ranked by comparison (<= kRangeRankM keys; unique keys: rank = number of
// smaller keys), bigger groups are refined (refine_groups), an LSD of the range is the last
// resort -- any key distribution gives the exact order.  Keys stay in registers (NI per thread).
// Code space of the linear digit: the key's (starving flag, bit length e of v, the 40 bits of v
// below its leading one) -- monotone in the key, linear in v inside an octave, so a range
// spanning several octaves (or the starving / not-starving boundary) still spreads evenly.
__device__ __forceinline__ unsigned long long key_code(uint64_t k, uint32_t vb) {
    const uint64_t v = k & ((1ull << vb) - 1ull);
    const uint32_t e = 64u - (uint32_t)__clzll((long long)v);
    const uint64_t mant = e ? ((v << (64u - e)) << 1) >> 24 : 0ull;
    return ((unsigned long long)(((uint32_t)(k >> vb) << 6) | e) << 40) | mant;
}
// Sort of a CTA's key range (rn <= kKcap keys at src, global, L2-resident) straight into its
// place in the ranked order (out, global), in compact loops (this code runs once per step and
// is fetched cold, so no per-thread item arrays).  One counting pass on a piecewise-linear
// digit: the range's 16 segments between its grid entries sm.fine[0..16] (quantiles of the
// previous step's order, so each segment holds ~1/16 of the keys) get W counters each, a key's
// counter is seg * W + (code(k) - code(fine[seg])) >> shift(seg), clamped -- monotone in the
// key, ~2 counters per key whatever the density inside the range.  Placement by digit into
// sm.a, then each key's rank inside its counter by comparison (<= kRangeRankM keys; unique keys:
// the number of smaller keys) gives its final position.  Returns false if a counter held more
// keys: sm.a then holds the range (placed by digit) and the caller sorts it otherwise.
// CTA 0 (pool != nullptr, head staging): the admission's per-key loads (ctx for the demand
// blk(ctx + 1), the state word) are issued in the rank pass and land in dsm / wsm (shared
// memory) by final position, and the ranked keys stay in sm.b: A5 then needs no global round
// trip for its head.
__device__ __forceinline__ bool range_sort_loop(PhaseL& sm, const uint64_t* __restrict__ src, uint32_t rn,
                                                uint64_t* __restrict__ out, uint32_t vb, unsigned long long* tr,
                                                const Pool* pool = nullptr, uint32_t id_base_mod = 0,
                                                const Cost* cc = nullptr, uint32_t* dsm = nullptr,
                                                uint32_t* wsm = nullptr, const uint32_t* __restrict__ pd_src = nullptr,
                                                const uint32_t* __restrict__ pw_src = nullptr) {
#define LTRACE(k) do { if (tr && threadIdx.x == 0) tr[k] = clock64(); } while (0)
    const uint32_t tid = threadIdx.x;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(sm.b);                      // <= 2^13 + 1 counters
    uint16_t* dp = reinterpret_cast<uint16_t*>(sm.b) + 2u * ((1u << 13) + 4u);  // per position: digit
    uint32_t* dv = sm.pos;                                                   // per key: digit | order << 13
    uint64_t* A = sm.a;
    LTRACE(0);
    const uint32_t cb = max(min(rn > 1u ? 33u - (uint32_t)__clz(rn - 1u) : 0u, 13u), 4u);  // ~2-4 counters per key
    const uint32_t lw = cb - 4u, W = 1u << lw, ncnt = (uint32_t)kSeg * W;  // W counters per segment
    uint32_t* shs = sm.shs;  // per segment: shift of the code difference
    if (tid < (uint32_t)kSeg) {
        const unsigned long long d = sm.fcode[tid + 1] > sm.fcode[tid] ? sm.fcode[tid + 1] - sm.fcode[tid] : 0ull;
        const uint32_t nb = 64u - (uint32_t)__clzll((long long)d);
        shs[tid] = nb > lw ? nb - lw : 0u;
    }
    for (uint32_t i = tid; i <= ncnt; i += kFT) cnt[i] = 0u;
    __syncthreads();
    auto digit = [&](uint64_t k) -> uint32_t {
        uint32_t sg = 0;
#pragma unroll
        for (uint32_t st = kSeg / 2; st; st >>= 1) sg = k >= sm.fine[sg + st] ? sg + st : sg;
        const unsigned long long c = key_code(k, vb), c0 = sm.fcode[sg];
        const unsigned long long d = (c > c0 ? c - c0 : 0ull) >> shs[sg];
        return sg * W + (uint32_t)min(d, (unsigned long long)(W - 1u));
    };
    LTRACE(1);
    for (uint32_t i0 = tid; i0 < rn; i0 += 4u * kFT) {  // four loads in flight per thread
        uint64_t kk[4];
#pragma unroll
        for (int u = 0; u < 4; u++) kk[u] = i0 + (uint32_t)u * kFT < rn ? __ldcg(src + i0 + (uint32_t)u * kFT) : 0ull;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t i = i0 + (uint32_t)u * kFT;
            if (i < rn) {
                const uint32_t d = digit(kk[u]);
                dv[i] = d | (atomicAdd(&cnt[d], 1u) << 13);
            }
        }
    }
    __syncthreads();
    LTRACE(2);
    (void)smem_excl_scan<kFT, (1 << 13) / kFT + 1>(cnt, ncnt, sm.w32);
    if (tid == 0) cnt[ncnt] = rn;
    LTRACE(3);
    // CTA 0 with the head's payload (pd_src / pw_src beside the keys): placed with the keys
    uint32_t* const Pd = sm.pos + 3u * kHeadPre;                         // [kHeadPre] by placed position
    uint32_t* const Pw = reinterpret_cast<uint32_t*>(sm.b) + 14336u;     // [kHeadPre], past cnt / dp
    if (pd_src) {  // rn <= kHeadPre: all loads in flight at once
        constexpr int kPU = (kHeadPre + kFT - 1) / kFT;
        uint32_t pdv[kPU], pwv[kPU];
#pragma unroll
        for (int u = 0; u < kPU; u++) {
            const uint32_t i = tid + (uint32_t)u * kFT;
            pdv[u] = i < rn ? __ldcg(pd_src + i) : 0u;
            pwv[u] = i < rn ? __ldcg(pw_src + i) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPU; u++) {
            const uint32_t i = tid + (uint32_t)u * kFT;
            if (i < rn) {
                const uint32_t v = dv[i], p = cnt[v & 0x1fffu] + (v >> 13);
                Pd[p] = pdv[u];
                Pw[p] = pwv[u];
            }
        }
    }
    for (uint32_t i0 = tid; i0 < rn; i0 += 4u * kFT) {
        uint64_t kk[4];
#pragma unroll
        for (int u = 0; u < 4; u++) kk[u] = i0 + (uint32_t)u * kFT < rn ? __ldcg(src + i0 + (uint32_t)u * kFT) : 0ull;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t i = i0 + (uint32_t)u * kFT;
            if (i < rn) {
                const uint32_t v = dv[i], d = v & 0x1fffu, p = cnt[d] + (v >> 13);
                A[p] = kk[u];
                dp[p] = (uint16_t)d;
            }
        }
    }
    __syncthreads();
    LTRACE(4);
    bool big = false;
    for (uint32_t p = tid; p < rn; p += kFT) {
        const uint64_t k = A[p];
        const uint32_t d = dp[p], st = cnt[d], m2 = cnt[d + 1] - st;
        uint32_t r = 0;
        if (m2 <= 4u) {  // the common case: straight-line, predicated compares
            if (m2 > 1u) {
                r += A[st] < k ? 1u : 0u;
                r += A[st + 1] < k ? 1u : 0u;
                if (m2 > 2u) r += A[st + 2] < k ? 1u : 0u;
                if (m2 > 3u) r += A[st + 3] < k ? 1u : 0u;
            }
        } else if (m2 <= kRangeRankM) {
            for (uint32_t q = 0; q < m2; q++) r += A[st + q] < k ? 1u : 0u;
        } else {
            big = true;
            continue;
        }
        dv[p] = st + r;  // final position (dv is free after the placement)
        if (pd_src) {
            dsm[st + r] = Pd[p];
            wsm[st + r] = Pw[p];
        }
    }
    LTRACE(5);
    if (__syncthreads_or(big)) return false;
    // the ranked keys gathered in shared memory (sm.b: the counters are dead), then written out
    // whole lines at a time (scattered 8-byte stores to lines not in L2 stall the store path)
    uint64_t* B2 = sm.b;
    for (uint32_t p = tid; p < rn; p += kFT) B2[dv[p]] = A[p];
    __syncthreads();
    if (dsm && !pd_src) {  // CTA 0 without payload: the admission's loads (L2 hits), all in flight at once
        for (uint32_t i0 = tid; i0 < rn; i0 += 4u * kFT) {
            uint32_t cx[4], w[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t i = i0 + (uint32_t)u * kFT;
                const uint32_t slot = i < rn ? (id_base_mod + (uint32_t)(B2[i] & cc->cap_mask)) & cc->cap_mask : 0u;
                cx[u] = i < rn ? __ldcg(&pool->ctx[slot]) : 0u;
                w[u] = i < rn ? __ldcg(&pool->sfc[slot]) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t i = i0 + (uint32_t)u * kFT;
                if (i < rn) {
                    dsm[i] = (uint32_t)blk((uint64_t)cx[u] + 1u, *cc);
                    wsm[i] = w[u];
                }
            }
        }
        __syncthreads();
    }
    for (uint32_t i = tid; i < rn; i += kFT) out[i] = B2[i];
    LTRACE(6);
#undef LTRACE
    return true;
}

// ---- The range sort staged by TMA (rn <= kTmaMax keys; every CTA, the head's too, runs this
// same code, so its lines are fetched once for all SMs).  After the grid barrier one thread
// requests the range's keys (the region the runs of all CTAs were stored into) into shared
// memory with ONE bulk copy (cp.async.bulk, completion on an mbarrier; CTA 0 with the head's
// payload: two more, the demand and state words R stored beside the head's keys).  Then the
// counting pass on the piecewise-linear digit as in range_sort_loop, every pass over shared
// memory, and the rank pass stores each key straight to its place in the output (a warp's
// consecutive placed positions go to a few consecutive lines: the placement is the order up to
// a counter's keys); with `keep` (CTA 0) also into shared memory for the admission, with the
// payload by sorted position.
// Layout (bytes): sm.a: A (placed keys) [0, 8 kTmaMax) | dp (u16 counter per placed position);
// head payload placed: Pd [8 kHeadPre, 12 kHeadPre), Pw [12 kHeadPre, 16 kHeadPre) (rn <= kHeadPre).
// From sm.b on (sm.b and the union after it): S (staged keys) [0, 8 kTmaMax) | cnt | dv;
// head payload staged at [8 kHeadPre, 16 kHeadPre) of S's space; after the place pass the sorted
// head goes to [0, 8 rn) (kept keys) and its payload to the staged payload's places (dsm / wsm).
// Position of the next step's grid entry f (0 .. 16 G) in this step's order of n keys: range 0's
// 16 segments over [0, q1), the other ranges' over [q1, n) evenly (past the last key: the last key).
// (in double precision: the products stay below 2^53 and the quotients' fractional parts are
// at least 2^-44 relative away from an integer, so the correctly rounded division floors /
// ceils exactly -- cheaper than a 64-bit integer division)
__device__ __forceinline__ uint32_t grid_q(uint32_t f, uint32_t q1, uint32_t n, uint32_t G) {
    if (!n) return 0u;
    const uint32_t p = f <= (uint32_t)kSeg
                           ? (uint32_t)(((uint64_t)q1 * f) >> 4)
                           : q1 + (uint32_t)floor((double)((uint64_t)(f - kSeg) * (uint64_t)(n - q1)) /
                                                  (double)((uint64_t)kSeg * (G - 1u)));
    return min(p, n - 1u);
}
static_assert(kSeg == 16, "grid_q divides by 16 with a shift");
// The first f with grid_q(f) >= q (16 G + 1 if none), in closed form: for q <= q1 the head's
// floor(q1 f / 16) >= q <=> f >= ceil(16 q / q1); past the head floor((f - 16) D / M) >= q - q1 <=>
// f - 16 >= ceil((q - q1) M / D) (D = n - q1, M = 16 (G - 1)); the clamp at n - 1 only bites q >= n.
__device__ __forceinline__ uint32_t grid_f(uint32_t q, uint32_t q1, uint32_t n, uint32_t G) {
    if (q == 0u) return 0u;
    if (q >= n) return (uint32_t)kSeg * G + 1u;
    if (q <= q1) return (uint32_t)ceil((double)q * kSeg / (double)q1);
    const double num = (double)((uint64_t)(q - q1) * kSeg * (G - 1u)), D = (double)(n - q1);
    return kSeg + (uint32_t)ceil(num / D);
}
constexpr uint32_t kTmaMax = 7167;  // (the kept keys sit one key later when the range starts at an odd position)
constexpr uint32_t kTsCnt = 8u * (kTmaMax + 1u);                         // byte offsets from sm.b
constexpr uint32_t kTsDv = (kTsCnt + 4u * ((1u << 13) + 1u) + 15u) & ~15u;
constexpr uint32_t kTsHd = 8u * kHeadPre, kTsHw = 12u * kHeadPre;        // head payload (sm.b / sm.a)
static_assert(kTsHw + 4u * kHeadPre <= kTsCnt, "TMA range sort: head payload overlaps cnt");
static_assert(kTsDv + 4u * kTmaMax <= 8u * kKcap + 4u * kKcap, "TMA range sort: S/cnt/dv exceed sm.b + sm.pos");
static_assert(kTsCnt % 16u == 0u && kTsHd % 16u == 0u && kTsHw % 16u == 0u, "TMA staging offsets: 16-B aligned");
static_assert(offsetof(PhaseL, b) + 8u * kKcap == offsetof(PhaseL, pos), "sm.pos must follow sm.b");
static_assert(offsetof(PhaseL, w32) >= offsetof(PhaseL, b) + kTsDv + 4u * kTmaMax, "TMA range sort overlaps sm.w32");
static_assert(8u * kTmaMax + 2u * kTmaMax <= 8u * kKcap, "TMA range sort: A + dp exceed sm.a");
static_assert(kTsHw + 4u * kHeadPre <= 8u * kTmaMax, "TMA range sort: placed head payload overlaps dp");

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mb) : "memory");
}
// one thread, after the grid barrier: the range's keys [src, src + rn) -> sm.b, and (hd != null)
// the head's demand / state words -> their staging places (16-B multiples: a few words past rn
// may be copied, inside the regions)
__device__ __forceinline__ void range_stage_issue(PhaseL& sm, const uint64_t* src, uint32_t rn,
                                                  const uint32_t* hd = nullptr, const uint32_t* hw = nullptr) {
    const uint32_t kb = ((rn + 1u) & ~1u) * 8u, pb = ((rn + 3u) & ~3u) * 4u;
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm.b);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the region was written by other CTAs' generic stores (ordered by the barrier's acquire),
    // shared memory by this CTA's generic stores: both before the async proxy's copy
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(kb + (hd ? 2u * pb : 0u)) : "memory");
    bulk_g2s(dst, src, kb, mb);
    if (hd) {
        bulk_g2s(dst + kTsHd, hd, pb, mb);
        bulk_g2s(dst + kTsHw, hw, pb, mb);
    }
}
// every thread (after a __syncthreads that follows range_stage_issue): the copies have landed
__device__ __forceinline__ void range_stage_wait(PhaseL& sm) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(mb) : "memory");
}
// the kept head (keep): sorted keys at sm.b, demand / state words by sorted position
__device__ __forceinline__ uint32_t* tma_head_dem(PhaseL& sm) { return reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(sm.b) + kTsHd); }
__device__ __forceinline__ uint32_t* tma_head_st(PhaseL& sm) { return reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(sm.b) + kTsHw); }

// The sorted keys go to shared memory, sm.b + (o = the output position's parity) -- so that key i
// and out[i] share their alignment -- and thread 0 stores them to out with one bulk copy (TMA,
// its bulk group left open: the caller waits before the CTA exits or anyone reads out); the key
// before the first and after the last 16-B pair of out by plain stores.  pay: the head payload
// was staged; its words go to their sorted positions.  Returns false if a counter held more than
// kRangeRankM keys (nothing stored): sm.a then holds the range placed by digit (the caller sorts
// it otherwise).
__device__ __forceinline__ bool range_sort_tma(PhaseL& sm, uint32_t rn, uint64_t* __restrict__ out, uint32_t o,
                                               uint32_t vb, unsigned long long* tr, bool pay, bool staged = true,
                                               bool bulk = true) {
#define LTRACE(k) do { if (tr && threadIdx.x == 0) tr[k] = clock64(); } while (0)
    const uint32_t tid = threadIdx.x;
    unsigned char* fb = reinterpret_cast<unsigned char*>(sm.b);
    uint64_t* S = sm.b;                                          // staged keys, then (keep) the sorted head
    uint32_t* cnt = reinterpret_cast<uint32_t*>(fb + kTsCnt);    // <= 2^13 + 1 counters
    uint32_t* dv = reinterpret_cast<uint32_t*>(fb + kTsDv);      // per staged key: digit | order << 13
    uint32_t* Hd = reinterpret_cast<uint32_t*>(fb + kTsHd);      // head payload staged, then by sorted position
    uint32_t* Hw = reinterpret_cast<uint32_t*>(fb + kTsHw);
    uint64_t* A = sm.a;                                          // placed keys
    uint16_t* dp = reinterpret_cast<uint16_t*>(sm.a + kTmaMax);  // per placed position: its counter
    uint32_t* Pd = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(sm.a) + kTsHd);  // payload placed
    uint32_t* Pw = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(sm.a) + kTsHw);
    LTRACE(0);
    const uint32_t cb = max(min(rn > 1u ? 33u - (uint32_t)__clz(rn - 1u) : 0u, 13u), 4u);  // ~2-4 counters per key
    const uint32_t lw = cb - 4u, W = 1u << lw, ncnt = (uint32_t)kSeg * W;
    uint32_t* shs = sm.shs;
    if (tid < (uint32_t)kSeg) {
        const unsigned long long d = sm.fcode[tid + 1] > sm.fcode[tid] ? sm.fcode[tid + 1] - sm.fcode[tid] : 0ull;
        const uint32_t nb = 64u - (uint32_t)__clzll((long long)d);
        shs[tid] = nb > lw ? nb - lw : 0u;
        // a segment whose ends share the starving flag and whose key parts differ in bit length
        // by at most one holds keys of about one density: its digit is linear in the raw key
        // (one subtract and shift); others take the code (bit length, mantissa) of the key
        const unsigned long long f0 = sm.fine[tid], f1 = sm.fine[tid + 1], vm = (1ull << vb) - 1ull;
        const uint32_t e0 = 64u - (uint32_t)__clzll((long long)(f0 & vm)), e1 = 64u - (uint32_t)__clzll((long long)(f1 & vm));
        const unsigned long long dr = f1 > f0 ? f1 - f0 : 0ull;
        const uint32_t nr = 64u - (uint32_t)__clzll((long long)dr);
        sm.shr[tid] = ((f0 >> vb) == (f1 >> vb) && e1 <= e0 + 1u) ? (nr > lw ? nr - lw : 0u) : 255u;
    }
    for (uint32_t i = tid; i <= ncnt; i += kFT) cnt[i] = 0u;
    if (staged) range_stage_wait(sm);  // (else the caller wrote S / the payload itself)
    __syncthreads();
    // any digit monotone inside each segment gives the exact order (segments own disjoint
    // counter ranges; ties of a counter are ranked by comparison)
    auto digit = [&](uint64_t k) -> uint32_t {
        uint32_t sg = 0;
#pragma unroll
        for (uint32_t st = kSeg / 2; st; st >>= 1) sg = k >= sm.fine[sg + st] ? sg + st : sg;
        const uint32_t sr = sm.shr[sg];
        unsigned long long d;
        if (sr != 255u) {
            const unsigned long long f0 = sm.fine[sg];
            d = (k > f0 ? k - f0 : 0ull) >> sr;
        } else {
            const unsigned long long c = key_code(k, vb), c0 = sm.fcode[sg];
            d = (c > c0 ? c - c0 : 0ull) >> shs[sg];
        }
        return sg * W + (uint32_t)min(d, (unsigned long long)(W - 1u));
    };
    LTRACE(1);
    for (uint32_t i0 = tid; i0 < rn; i0 += 4u * kFT) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t i = i0 + (uint32_t)u * kFT;
            if (i < rn) {
                const uint32_t d = digit(S[i]);
                dv[i] = d | (atomicAdd(&cnt[d], 1u) << 13);
            }
        }
    }
    __syncthreads();
    LTRACE(2);
    (void)smem_excl_scan<kFT, (1 << 13) / kFT + 1>(cnt, ncnt, sm.w32);
    if (tid == 0) cnt[ncnt] = rn;
    LTRACE(3);
    for (uint32_t i0 = tid; i0 < rn; i0 += 4u * kFT) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t i = i0 + (uint32_t)u * kFT;
            if (i < rn) {
                const uint32_t v = dv[i], d = v & 0x1fffu, p = cnt[d] + (v >> 13);
                A[p] = S[i];
                dp[p] = (uint16_t)d;
                if (pay) {
                    Pd[p] = Hd[i];
                    Pw[p] = Hw[i];
                }
            }
        }
    }
    __syncthreads();
    LTRACE(4);
    bool big = false;
    for (uint32_t p = tid; p < rn; p += kFT) {
        const uint64_t k = A[p];
        const uint32_t d = dp[p], st = cnt[d], m2 = cnt[d + 1] - st;
        uint32_t r = 0;
        if (m2 <= 4u) {
            if (m2 > 1u) {
                r += A[st] < k ? 1u : 0u;
                r += A[st + 1] < k ? 1u : 0u;
                if (m2 > 2u) r += A[st + 2] < k ? 1u : 0u;
                if (m2 > 3u) r += A[st + 3] < k ? 1u : 0u;
            }
        } else if (m2 <= kRangeRankM) {
            for (uint32_t q = 0; q < m2; q++) r += A[st + q] < k ? 1u : 0u;
        } else {
            big = true;
            continue;
        }
        S[o + st + r] = k;
        if (pay) {
            Hd[st + r] = Pd[p];
            Hw[st + r] = Pw[p];
        }
    }
    LTRACE(5);
    if (__syncthreads_or(big)) return false;
    const uint64_t* K = S + o;  // K[i] = the key of out[i]
    if (!bulk) {  // (one-CTA kernel: plain coalesced stores, nothing outstanding at its end)
        for (uint32_t i = tid; i < rn; i += kFT) out[i] = K[i];
        LTRACE(6);
        return true;
    }
    const uint32_t i0 = o, i1 = o + ((rn - min(o, rn)) & ~1u);  // out[i0, i1): whole 16-B pairs
    if (tid == 0 && i1 > i0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the rank pass's stores, then the copy
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\ncp.async.bulk.commit_group;" ::"l"(out + i0),
                     "r"((uint32_t)__cvta_generic_to_shared(K + i0)), "r"((i1 - i0) * 8u) : "memory");
    }
    if (tid == 32u && i0 > 0u && rn) out[0] = K[0];
    if (tid == 64u && i1 < rn) out[rn - 1u] = K[rn - 1u];
    LTRACE(6);
#undef LTRACE
    return true;
}
// the issuing thread: the bulk store has read shared memory (before the CTA exits) / is complete
// and visible to generic loads (before another CTA or a later phase reads out)
__device__ __forceinline__ void bulk_store_read_wait() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_store_done() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// (Measured and not kept: range_sort_lean -- one L2 load, the digit recomputed
// per pass -- and range_sort_cp -- cp.async staging, single-key loops: less code, but the
// rank-by-comparison of clustered counters needs the unrolled loop; 53.2 / 56.1 vs 52.4 us.)
#define LAMPS_RANGE_SORT range_sort_loop
constexpr bool kSortedInA = false;  // where a successful range sort leaves the sorted keys (sm.b)

// A small range (rn <= kSmallSort keys): ranked by comparison against all its keys (the
// keys are unique, so the rank is the count of smaller keys; the few hundred keys are read
// as shared-memory broadcasts), no bucket table.  A small pool's head range can span
// thousands of sparse buckets (starving keys first, over the whole score range), where
// the table dominates.  HEAD (CTA 0): the admission's per-key loads by sorted position into
// the staged head arrays, prefetched to L2 while ranking.
constexpr uint32_t kSmallSort = 384;
template <bool HEAD>
__device__ __forceinline__ void small_sort(PhaseL& sm, const uint64_t* __restrict__ src, uint32_t rn, const Cost& c,
                                           const Pool* pool, uint32_t id_base_mod) {
    const uint32_t tid = threadIdx.x;
    uint64_t* A = sm.a;
    uint64_t* Bq = sm.b;  // scratch [0, rn): below the staged head arrays
    uint64_t k = 0;
    if (tid < rn) {
        k = __ldcg(src + tid);
        A[tid] = k;
        if (HEAD) {
            const uint32_t slot = (id_base_mod + (uint32_t)(k & c.cap_mask)) & c.cap_mask;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pool->ctx + slot));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pool->sfc + slot));
        }
    }
    __syncthreads();
    if (tid < rn) {
        uint32_t r = 0;
#pragma unroll 8
        for (uint32_t q = 0; q < rn; q++) r += A[q] < k ? 1u : 0u;
        Bq[r] = k;
    }
    __syncthreads();
    if (tid < rn) {
        const uint64_t x = Bq[tid];
        A[tid] = x;
        if (HEAD) {
            uint32_t* b32 = reinterpret_cast<uint32_t*>(sm.b);
            const uint32_t slot = (id_base_mod + (uint32_t)(x & c.cap_mask)) & c.cap_mask;
            b32[kHeadD + tid] = (uint32_t)blk((uint64_t)__ldcg(&pool->ctx[slot]) + 1u, c);
            b32[kHeadW + tid] = __ldcg(&pool->sfc[slot]);
        }
    }
    __syncthreads();
}


}  // namespace
}  // namespace lamps
