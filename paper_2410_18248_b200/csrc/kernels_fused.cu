// kernels_fused.cu -- the whole scheduling step (A0 default update .. A5) as
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
};
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
    // group refinement: lists of groups still to split (ping-pong), and per group of the
    // current batch: key offset (prefix of sizes), digit shift / bits, counter base, OR / AND
    uint16_t gl_lo[2][kMaxBig], gl_n[2][kMaxBig];
    uint32_t ngl[2];
    uint16_t gcum[kMaxBig], gbase[kMaxBig];
    uint8_t gsh[kMaxBig], gdb[kMaxBig];
    unsigned long long gor[kMaxBig / 4], gand[kMaxBig / 4];
    unsigned long long red[2][kFW];
    AdmitSmem adm;                                // admission scratch (CTA 0, keys stay in a[])
    uint32_t rsz[kMaxCtas], rpre[kMaxCtas];       // every range's size and position in the order
    unsigned long long fine[kSeg + 1], fcode[kSeg + 1];  // this range's grid entries, their key codes
    uint32_t shs[kSeg];                                  // range sort: per segment, the digit's shift
};
struct FusedSmem {
    union {
        PhaseS s;
        PhaseL l;
        SortSmem g;
    };
    alignas(16) uint32_t btab[kTabW];  // this step's bucket table (bucket_t), every phase
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

// Refinement of the groups listed in sm.gl_lo[0] / gl_n[0] (sm.ngl[0] of them; keys
// at A[lo, lo+n), Bf scratch at the same offsets) until every group is <= kMaxRankM
// keys and ranked.  Each pass: per group a digit of its own top varying bits (db =
// ceil(log2 size) bits, from the group's OR/AND), counted with shared-memory atomics
// into a counter block of its own; one scan over the blocks of a batch gives
// positions; sub-groups still bigger than kMaxRankM go to the next pass.  Returns
// true if the lists overflowed or kMaxLevels passes did not finish (the caller
// then sorts the whole part by LSD).
__device__ __forceinline__ bool refine_groups(PhaseL& sm, uint64_t* A, uint64_t* Bf, unsigned long long* xtr) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint32_t cur = 0;
    bool full_lsd = false;
    for (int level = 0; !full_lsd && level < kMaxLevels; level++) {
        const uint32_t ng = sm.ngl[cur];
        if (xtr && tid == 0) { xtr[2 * level] = clock64(); xtr[2 * level + 1] = ng; }
        if (ng == 0) break;
        if (ng > (uint32_t)kMaxBig) { full_lsd = true; break; }
        const uint32_t nxt = cur ^ 1u;
        if (tid == 0) sm.ngl[nxt] = 0;
        if (warp == 0) {  // key offsets: exclusive prefix of the group sizes
            uint32_t cum = 0;
            for (uint32_t g0 = 0; g0 < ng; g0 += 32) {
                const uint32_t g = g0 + lane, mm = g < ng ? sm.gl_n[cur][g] : 0u;
                uint32_t x = mm;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                if (g < ng) sm.gcum[g] = (uint16_t)(cum + x - mm);
                cum += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) sm.w32[kFW] = cum;
        }
        __syncthreads();
        const uint32_t K = sm.w32[kFW];
        auto group_of = [&](uint32_t f, uint32_t g0, uint32_t g1) {
            uint32_t lo_ = g0, hi_ = g1;
            while (hi_ - lo_ > 1) {
                const uint32_t mid = (lo_ + hi_) >> 1;
                if (sm.gcum[mid] <= f) lo_ = mid; else hi_ = mid;
            }
            return lo_;
        };
        for (uint32_t gb = 0; gb < ng;) {  // batches: OR/AND slots and counter blocks must fit
            const uint32_t ge = min(ng, gb + (uint32_t)(kMaxBig / 4));
            // OR / AND of each group's keys: one warp per group, shuffle reduction (64-bit
            // shared-memory atomicOr/And would be CAS loops on a handful of addresses)
            for (uint32_t g = gb + warp; g < ge; g += kFW) {
                const uint32_t lo_g = sm.gl_lo[cur][g], m = sm.gl_n[cur][g];
                unsigned long long o = 0, an = ~0ull;
                for (uint32_t i = lane; i < m; i += 32) {
                    const uint64_t k = A[lo_g + i];
                    o |= k;
                    an &= k;
                }
#pragma unroll
                for (int sh = 16; sh; sh >>= 1) {
                    o |= __shfl_xor_sync(0xffffffffu, o, sh);
                    an &= __shfl_xor_sync(0xffffffffu, an, sh);
                }
                if (lane == 0) { sm.gor[g - gb] = o; sm.gand[g - gb] = an; }
            }
            const uint32_t f0 = sm.gcum[gb];
            __syncthreads();
            if (xtr && tid == 0 && level == 0 && gb == 0) xtr[16] = clock64();
            if (warp == 0) {  // digit shift / bits, counter bases; cut the batch at kSubBuckets
                uint32_t base = 0, cut = ge;
                for (uint32_t g0 = gb; g0 < ge; g0 += 32) {
                    const uint32_t g = g0 + lane;
                    uint32_t sz = 0;
                    if (g < ge) {
                        const unsigned long long v = sm.gor[g - gb] ^ sm.gand[g - gb];  // != 0: unique keys
                        const int h = 63 - __clzll((long long)v);
                        uint32_t db = 32u - (uint32_t)__clz((uint32_t)sm.gl_n[cur][g] - 1u);  // ceil(log2 m)
                        db = db > (uint32_t)kSubBits ? (uint32_t)kSubBits : db;
                        sm.gsh[g] = (uint8_t)(h + 1 >= (int)db ? h + 1 - (int)db : 0);
                        sm.gdb[g] = (uint8_t)db;
                        sz = 1u << db;
                    }
                    uint32_t x = sz;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= (uint32_t)o) x += y;
                    }
                    if (g < ge) sm.gbase[g] = (uint16_t)min(base + x - sz, 65535u);
                    const uint32_t ob = __ballot_sync(0xffffffffu, g < ge && base + x > (uint32_t)kSubBuckets);
                    if (ob && cut == ge) cut = g0 + __ffs(ob) - 1;
                    base += __shfl_sync(0xffffffffu, x, 31);
                }
                if (lane == 0) sm.w32[kFW - 1] = cut > gb ? cut : gb + 1;
            }
            __syncthreads();
            const uint32_t gcut = sm.w32[kFW - 1];
            const uint32_t fc = gcut < ng ? (uint32_t)sm.gcum[gcut] : K;
            const uint32_t ncnt = (uint32_t)sm.gbase[gcut - 1] + (1u << sm.gdb[gcut - 1]);
            for (uint32_t i = tid; i < ncnt; i += kFT) sm.pos[i] = 0;
            __syncthreads();
#define GDIGIT(k, g) (sm.gbase[g] + ((uint32_t)((k) >> sm.gsh[g]) & ((1u << sm.gdb[g]) - 1u)))
            for (uint32_t f = f0 + tid; f < fc; f += kFT) {
                const uint32_t g = group_of(f, gb, gcut);
                atomicAdd(&sm.pos[GDIGIT(A[sm.gl_lo[cur][g] + (f - sm.gcum[g])], g)], 1u);
            }
            __syncthreads();
            if (xtr && tid == 0 && level == 0 && gb == 0) xtr[17] = clock64();
            (void)smem_excl_scan<kFT, kSubBuckets / kFT + 1>(sm.pos, ncnt, sm.w32);
            if (xtr && tid == 0 && level == 0 && gb == 0) xtr[18] = clock64();
            // group g's keys occupy [gcum_g - f0, gcum_g - f0 + m_g) of the batch's scan space
            for (uint32_t f = f0 + tid; f < fc; f += kFT) {
                const uint32_t g = group_of(f, gb, gcut);
                const uint32_t lo_g = sm.gl_lo[cur][g], gz = sm.gcum[g] - f0;
                const uint64_t k = A[lo_g + (f - sm.gcum[g])];
                Bf[lo_g + atomicAdd(&sm.pos[GDIGIT(k, g)], 1u) - gz] = k;
            }
            __syncthreads();
            if (xtr && tid == 0 && level == 0 && gb == 0) xtr[19] = clock64();
            for (uint32_t f = f0 + tid; f < fc; f += kFT) {  // finish small sub-groups, list big ones
                const uint32_t g = group_of(f, gb, gcut);
                const uint32_t lo_g = sm.gl_lo[cur][g], gz = sm.gcum[g] - f0;
                const uint32_t i = f - sm.gcum[g];
                const uint64_t k = Bf[lo_g + i];
                const uint32_t d = GDIGIT(k, g);
                const uint32_t e = sm.pos[d] - gz;
                const uint32_t st = (d > sm.gbase[g] ? sm.pos[d - 1] : sm.gcum[g] - f0 + gz * 0u) - gz;
                const uint32_t stc = d > sm.gbase[g] ? st : 0u;
                const uint32_t m2 = e - stc;
                if (m2 > kMaxRankM) {
                    A[lo_g + i] = k;
                    if (i == stc) {
                        const uint32_t t = atomicAdd(&sm.ngl[nxt], 1u);
                        if (t < (uint32_t)kMaxBig) {
                            sm.gl_lo[nxt][t] = (uint16_t)(lo_g + stc);
                            sm.gl_n[nxt][t] = (uint16_t)m2;
                        }
                    }
                    continue;
                }
                uint32_t r = 0;
#pragma unroll 8
                for (uint32_t q = stc; q < e; q++) r += Bf[lo_g + q] < k ? 1u : 0u;
                A[lo_g + stc + r] = k;
            }
#undef GDIGIT
            __syncthreads();
            if (xtr && tid == 0 && level == 0 && gb == 0) { xtr[20] = clock64(); xtr[21] = gcut; xtr[22] = fc - f0; }
            gb = gcut;
        }
        cur = nxt;
        if (level + 1 == kMaxLevels && sm.ngl[cur]) full_lsd = true;
    }
    return full_lsd;
}

// Sort of the n keys at A[0..n) of one part of a range (same starving flag) in
// shared memory; result in A, Bf is scratch.  The part arrives in global-bucket
// order and its buckets [j0, j1) are known, so the buckets are the first-level
// groups (sizes = the global totals T[j]; a bucket lies entirely in one range).
// Groups of <= kMaxRankM keys are finished by rank-by-comparison (keys are
// unique).  Bigger groups are refined in flat passes over all their keys: per
// group a digit of its own top varying bits (db = ceil(log2 size) bits, from the
// group's OR/AND), counted with shared-memory atomics into a counter block of
// its own; one scan over the blocks of a batch gives positions; sub-groups
// still bigger than kMaxRankM go to the next pass.  After kMaxLevels passes (or
// if the group tables overflow) the stable LSD finishes the part.
__device__ __forceinline__ void local_sort(PhaseL& sm, uint64_t* A, uint64_t* Bf, uint32_t n,
                                           const uint32_t* T, uint32_t j0, uint32_t j1,
                                           unsigned long long* tr, unsigned long long* xtr = nullptr) {
#define LTRACE(k) do { if (tr && threadIdx.x == 0) tr[k] = clock64(); } while (0)
    const uint32_t tid = threadIdx.x;
    if (n <= 1) return;
    LTRACE(0);
    bool full_lsd = false;
    // ---- level 1: bucket runs.  pos[0..nb] = starts of the part's buckets.
    const uint32_t nb = j1 - j0;
    if (nb + 1 > (uint32_t)kSubBuckets) {
        full_lsd = true;
    } else {
        for (uint32_t j = tid; j < nb; j += kFT) sm.pos[j] = __ldcg(&T[j0 + j]);
        if (tid == 0) { sm.ngl[0] = 0; sm.ngl[1] = 0; }
        for (uint32_t i = tid; i < n; i += kFT) Bf[i] = A[i];
        __syncthreads();
        (void)smem_excl_scan<kFT, kSubBuckets / kFT + 1>(sm.pos, nb, sm.w32);
        if (tid == 0) sm.pos[nb] = n;
        __syncthreads();
        LTRACE(1);
        for (uint32_t i = tid; i < n; i += kFT) {
            uint32_t lo_ = 0, hi_ = nb;  // last bucket with start <= i
            while (hi_ - lo_ > 1) {
                const uint32_t mid = (lo_ + hi_) >> 1;
                if (sm.pos[mid] <= i) lo_ = mid; else hi_ = mid;
            }
            const uint32_t st = sm.pos[lo_], e = sm.pos[lo_ + 1], m = e - st;
            const uint64_t k = Bf[i];
            if (m > kMaxRankM) {
                if (i == st) {
                    const uint32_t t = atomicAdd(&sm.ngl[0], 1u);
                    if (t < (uint32_t)kMaxBig) { sm.gl_lo[0][t] = (uint16_t)st; sm.gl_n[0][t] = (uint16_t)m; }
                }
                continue;  // A[i] == k already
            }
            uint32_t r = 0;
#pragma unroll 8
            for (uint32_t q = st; q < e; q++) r += Bf[q] < k ? 1u : 0u;
            A[st + r] = k;
        }
        __syncthreads();
        LTRACE(2);
    }
    // ---- refinement passes over the big groups
    if (!full_lsd) full_lsd = refine_groups(sm, A, Bf, xtr);
    LTRACE(3);
    if (xtr && tid == 0) xtr[14] = clock64();
    if (full_lsd) {  // pathological distributions: stable LSD of the whole part
        unsigned long long o, an;
        block_or_and(sm, A, n, o, an);
        const uint64_t* r = local_lsd(sm, A, Bf, n, o ^ an);
        if (r != A)
            for (uint32_t i = tid; i < n; i += kFT) A[i] = r[i];
        __syncthreads();
    }
    if (tr && tid == 0) tr[5] = full_lsd ? 1000u : sm.ngl[0];
    LTRACE(4);
#undef LTRACE
}

// Digit of key k inside its bucket: the top db bits of the sv low bits of v the bucket
// leaves free (sv from bucket_t), i.e. (low score bits, id offset).  The id offset
// (id - id_base, the key's low IB bits) is < cap = 2^lg_cap, so it is packed into lg_cap
// bits (not IB) and its top bits carry information.  Monotone in the key within a
// bucket, so (bucket, digit) order is key order.
__device__ __forceinline__ uint32_t sub_digit_t(uint64_t k, uint32_t sv, uint32_t db, const Cost& c,
                                                uint32_t lg_cap) {
    const uint64_t idoff = k & (uint64_t)c.cap_mask;
    uint64_t v;
    uint32_t wv;
    if (sv > c.IB) {  // varying score bits, then the id offset packed into lg_cap bits
        v = (((k >> c.IB) & ((1ull << (sv - c.IB)) - 1ull)) << lg_cap) | idoff;
        wv = sv - c.IB + lg_cap;
    } else {          // id bits only; those above lg_cap are always 0
        wv = sv < lg_cap ? sv : lg_cap;
        v = idoff & ((1ull << wv) - 1ull);
    }
    return wv >= db ? (uint32_t)(v >> (wv - db)) : (uint32_t)(v << (db - wv));
}

// Sort of a CTA's key range (rn <= kKcap keys in global src, buckets [j_lo, j_hi),
// j_hi - j_lo < kSubBuckets) into sm.a.  Keys stay in registers (<= kLocalItems per
// thread).  One counting pass: each bucket of m keys gets 2^ceil(log2 m) counters
// (the bucket's exact size is the global total T[j]: a bucket lies entirely in one
// range) indexed by sub_digit, so the sub-buckets hold ~1 key; keys of sub-buckets
// of <= kMaxRankM keys are ranked by comparison, bigger ones (many near-equal keys)
// go to refine_groups, and an LSD of the whole range is the last resort.
//
// Head range (pool != nullptr, rn <= kHeadPre): the admission's per-key loads (ctx for
// the demand blk(ctx+1), the state word) are issued with the key loads and land in
// shared memory in sorted order (kHeadD / kHeadW words of sm.b), so A5 needs no
// dependent global round trip.  Returns whether those arrays are valid (not after a
// refinement pass, which moves keys).
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
// NI = keys per thread (kLocalItems; 3 for the head range, whose loads for the
// admission stay in flight in registers for the whole sort)
template <int NI, bool HEAD>
__device__ __forceinline__ bool range_sort(PhaseL& sm, const uint64_t* __restrict__ src, uint32_t rn,
                                           uint32_t j_lo, uint32_t j_hi, const Cost& c,
                                           const uint32_t* tab, unsigned long long* tr, const Pool* pool = nullptr,
                                           uint32_t id_base_mod = 0) {
#define LTRACE(k) do { if (tr && threadIdx.x == 0) tr[k] = clock64(); } while (0)
    const uint32_t tid = threadIdx.x;
    const uint32_t nb = j_hi - j_lo;
    const uint32_t lg_cap = 31u - (uint32_t)__clz(c.cap);
    uint32_t* P = sm.pos;                                  // per bucket: start | counter base << 14
    uint32_t* cnt = reinterpret_cast<uint32_t*>(sm.b);     // <= 2 * kKcap counters
    uint64_t* A = sm.a;
    LTRACE(0);
    static_assert(!HEAD || NI * kFT >= (int)kHeadPre, "head items");
    uint64_t k[NI];
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        k[u] = i < rn ? __ldcg(src + i) : 0ull;
    }
    uint32_t* b32 = reinterpret_cast<uint32_t*>(sm.b);
    constexpr int kHU = HEAD ? NI : 1;
    if (HEAD) {  // L2 prefetch of what the admission reads (no registers held in flight)
#pragma unroll
        for (int u = 0; u < kHU; u++) {
            const uint32_t i = tid + (uint32_t)u * kFT;
            if (i < rn) {
                const uint32_t slot = (id_base_mod + (uint32_t)(k[u] & c.cap_mask)) & c.cap_mask;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pool->ctx + slot));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pool->sfc + slot));
            }
        }
    }
    // the bucket of every key (kept in registers: J - j_lo | sv << 16) and the range's own
    // bucket counts (a bucket may straddle two ranges)
    for (uint32_t j = tid; j <= nb; j += kFT) P[j] = 0;
    if (tid == 0) sm.ngl[0] = 0;
    __syncthreads();
    uint32_t jv[NI];
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        jv[u] = 0;
        if (i < rn) {
            uint32_t sv;
            const uint32_t J = bucket_t(k[u], tab, c.SB + c.IB, sv) - j_lo;
            jv[u] = J | (sv << 16);
            atomicAdd(&P[J], 1u);
        }
    }
    __syncthreads();
    for (uint32_t j = tid; j < nb; j += kFT) {
        const uint32_t m = P[j];
        const uint32_t db = m > 1u ? 32u - (uint32_t)__clz(m - 1u) : 0u;
        P[j] = m | ((m ? 1u << db : 0u) << 14);  // empty buckets take no counters: ncnt < 2 rn
    }
    __syncthreads();
    const uint32_t ptot = smem_excl_scan<kFT, kSubBuckets / kFT + 1>(P, nb, sm.w32);
    const uint32_t ncnt = ptot >> 14;
    if (tid == 0) P[nb] = ptot;
    for (uint32_t i = tid; i < ncnt; i += kFT) cnt[i] = 0;
    __syncthreads();
    LTRACE(1);
    uint32_t it[NI];  // counter index | order within the sub-bucket << 15
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        it[u] = 0;
        if (i < rn) {
            const uint32_t J = jv[u] & 0xffffu, sv = jv[u] >> 16;
            const uint32_t p0 = P[J], p1 = P[J + 1];
            const uint32_t m = (p1 & 0x3fffu) - (p0 & 0x3fffu);
            const uint32_t db = m > 1u ? 32u - (uint32_t)__clz(m - 1u) : 0u;
            const uint32_t idx = (p0 >> 14) + sub_digit_t(k[u], sv, db, c, lg_cap);
            it[u] = idx | (atomicAdd(&cnt[idx], 1u) << 15);
        }
    }
    __syncthreads();
    (void)smem_excl_scan<kFT, 2 * NI + 1>(cnt, ncnt, sm.w32);
    LTRACE(2);
    // initial placement: sub-bucket start + arrival order; per position its sub-bucket's
    // (start, size) in sbi (P is dead after the count pass)
    uint32_t* sbi = sm.pos;
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        if (i < rn) {
            const uint32_t idx = it[u] & 0x7fffu;
            const uint32_t st = cnt[idx], e = idx + 1u < ncnt ? cnt[idx + 1] : rn;
            const uint32_t p = st + (it[u] >> 15);
            A[p] = k[u];
            sbi[p] = st | ((e - st) << 14);
            if (HEAD) {  // the admission's loads (L2 hits by now), by position
                const uint32_t slot = (id_base_mod + (uint32_t)(k[u] & c.cap_mask)) & c.cap_mask;
                b32[kHeadTC + p] = __ldcg(&pool->ctx[slot]);
                b32[kHeadTW + p] = __ldcg(&pool->sfc[slot]);
            }
        }
    }
    __syncthreads();
    // rank inside sub-buckets of <= kRangeRankM keys by comparison; list the bigger ones.
    // Thread t takes positions t + u*kFT: a sub-bucket's keys are contiguous, so the lanes
    // of a warp mostly share a sub-bucket and the loop trip counts agree
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t p = tid + (uint32_t)u * kFT;
        it[u] = 0;
        if (p < rn) {
            k[u] = A[p];
            const uint32_t inf = sbi[p];
            const uint32_t st = inf & 0x3fffu, m2 = inf >> 14;
            if (m2 <= kRangeRankM) {
                uint32_t r = 0;
#pragma unroll 4
                for (uint32_t q = 0; q < m2; q++) r += A[st + q] < k[u] ? 1u : 0u;
                it[u] = (st + r) | 0x80000000u;
            } else if (p == st) {
                const uint32_t t = atomicAdd(&sm.ngl[0], 1u);
                if (t < (uint32_t)kMaxBig) { sm.gl_lo[0][t] = (uint16_t)st; sm.gl_n[0][t] = (uint16_t)m2; }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t p = tid + (uint32_t)u * kFT;
        if (p < rn && (it[u] >> 31)) {
            const uint32_t pos = it[u] & 0x7fffffffu;
            A[pos] = k[u];
            if (HEAD) {
                b32[kHeadD + pos] = (uint32_t)blk((uint64_t)b32[kHeadTC + p] + 1u, c);
                b32[kHeadW + pos] = b32[kHeadTW + p];
            }
        }
    }
    __syncthreads();
    LTRACE(3);
    bool full_lsd = false;
    if (sm.ngl[0]) full_lsd = refine_groups(sm, A, sm.b, nullptr);
    if (full_lsd) {
        unsigned long long o, an;
        block_or_and(sm, A, rn, o, an);
        const uint64_t* r = local_lsd(sm, A, sm.b, rn, o ^ an);
        if (r != A)
            for (uint32_t i = tid; i < rn; i += kFT) A[i] = r[i];
        __syncthreads();
    }
    const bool dw_ok = HEAD && sm.ngl[0] == 0;
    if (tr && tid == 0) { tr[5] = full_lsd ? 1000u : sm.ngl[0]; }
    LTRACE(4);
#undef LTRACE
    return dw_ok;
}

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
                                                uint32_t* wsm = nullptr) {
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
    }
    LTRACE(5);
    if (__syncthreads_or(big)) return false;
    // the ranked keys gathered in shared memory (sm.b: the counters are dead), then written out
    // whole lines at a time (scattered 8-byte stores to lines not in L2 stall the store path)
    uint64_t* B2 = sm.b;
    for (uint32_t p = tid; p < rn; p += kFT) B2[dv[p]] = A[p];
    __syncthreads();
    if (dsm) {  // CTA 0: the admission's loads (L2 hits: the score phase read them), all in flight at once
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

// CTA 0's head range when its buckets are sparse (nb > 2 rn: the head's starving keys span
// a wide score range): a counting sort over the OCCUPIED buckets only -- a bitmap of the
// keys' buckets, their compact index by popcount prefix -- then rank by comparison inside
// each bucket (a bucket holds ~1 key here), then the admission's per-key loads by sorted
// position (prefetched to L2 at the start).  No bucket table over the whole interval.
// Returns false (nothing written) if a bucket holds more than kRangeRankM keys; the caller
// then uses range_sort.
__device__ __forceinline__ bool head_sparse_sort(PhaseL& sm, const uint64_t* __restrict__ src, uint32_t rn,
                                                 const Cost& c, const uint32_t* tab, uint32_t j_lo, uint32_t nb,
                                                 const Pool& pool, uint32_t id_base_mod) {
    constexpr int NI = (kHeadPre + kFT - 1) / kFT;  // 3
    const uint32_t tid = threadIdx.x;
    uint32_t* bm = sm.pos;            // bucket bitmap, nw <= 1024 words
    uint32_t* wp = sm.pos + 1024;     // exclusive popcount prefix per word
    uint32_t* cnt = sm.pos + 2048;    // per occupied bucket: count -> start
    uint32_t* sbi = sm.pos + 4608;    // per position: bucket start | size << 14
    uint64_t* A = sm.a;
    uint64_t* Bq = sm.b;              // [0, rn): below the staged head arrays
    const uint32_t nw = (nb + 31u) >> 5;
    for (uint32_t w = tid; w < nw; w += kFT) bm[w] = 0u;
    __syncthreads();
    uint64_t k[NI];
    uint32_t J[NI], ci[NI];
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        k[u] = 0;
        J[u] = 0;
        if (i < rn) {
            k[u] = __ldcg(src + i);
            uint32_t sv;
            J[u] = bucket_t(k[u], tab, c.SB + c.IB, sv) - j_lo;
            atomicOr(&bm[J[u] >> 5], 1u << (J[u] & 31u));
            const uint32_t slot = (id_base_mod + (uint32_t)(k[u] & c.cap_mask)) & c.cap_mask;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pool.ctx + slot));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pool.sfc + slot));
        }
    }
    __syncthreads();
    for (uint32_t w = tid; w < nw; w += kFT) wp[w] = __popc(bm[w]);
    __syncthreads();
    const uint32_t nocc = smem_excl_scan<kFT, 1>(wp, nw, sm.w32);
    for (uint32_t q = tid; q < nocc; q += kFT) cnt[q] = 0u;
    __syncthreads();
    uint32_t ord[NI];
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        ci[u] = 0;
        ord[u] = 0;
        if (i < rn) {
            const uint32_t w = J[u] >> 5;
            ci[u] = wp[w] + __popc(bm[w] & ((1u << (J[u] & 31u)) - 1u));
            ord[u] = atomicAdd(&cnt[ci[u]], 1u);
        }
    }
    __syncthreads();
    uint32_t big = 0;
    for (uint32_t q = tid; q < nocc; q += kFT) big |= cnt[q] > kRangeRankM ? 1u : 0u;
    if (__syncthreads_or(big)) return false;
    (void)smem_excl_scan<kFT, 3>(cnt, nocc, sm.w32);
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t i = tid + (uint32_t)u * kFT;
        if (i < rn) {
            const uint32_t st = cnt[ci[u]], e = ci[u] + 1u < nocc ? cnt[ci[u] + 1u] : rn;
            const uint32_t p = st + ord[u];
            A[p] = k[u];
            sbi[p] = st | ((e - st) << 14);
        }
    }
    __syncthreads();
    uint32_t* b32 = reinterpret_cast<uint32_t*>(sm.b);
#pragma unroll
    for (int u = 0; u < NI; u++) {
        const uint32_t p = tid + (uint32_t)u * kFT;
        if (p < rn) {
            const uint64_t x = A[p];
            const uint32_t inf = sbi[p], st = inf & 0x3fffu, m = inf >> 14;
            uint32_t r = 0;
            for (uint32_t q = 0; q < m; q++) r += A[st + q] < x ? 1u : 0u;
            const uint32_t fp = st + r;
            Bq[fp] = x;
            const uint32_t slot = (id_base_mod + (uint32_t)(x & c.cap_mask)) & c.cap_mask;
            b32[kHeadD + fp] = (uint32_t)blk((uint64_t)__ldcg(&pool.ctx[slot]) + 1u, c);
            b32[kHeadW + fp] = __ldcg(&pool.sfc[slot]);
        }
    }
    __syncthreads();
    for (uint32_t p = tid; p < rn; p += kFT) A[p] = Bq[p];
    __syncthreads();
    return true;
}

#define TRACE(k)                                                                         \
    do {                                                                                 \
        if (b.trace && threadIdx.x == 0) b.trace[blockIdx.x * kTraceSlots + (k)] = clock64(); \
    } while (0)

// P2P: the peer-memory exchange + in-kernel merge instance (its code and shared-memory
// tail are left out of the plain instance)
template <bool DBG, bool P2P>
__global__ void __launch_bounds__(kFT, 1) k_fused(const __grid_constant__ Bufs b, const __grid_constant__ Cost c, StepArgs a,
                                                  const __grid_constant__ InlineStage inl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FusedSmem& sm = *reinterpret_cast<FusedSmem*>(smem_raw);
    Ctl* ctl = b.ctl;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t G = gridDim.x, bid = blockIdx.x;
    const uint32_t vb = c.SB + c.IB;  // buckets over the key's score|id bits (bucket_t)
    // this CTA's slots; all of their SoA words are requested into L2 at once (bulk
    // prefetches, no shared memory), so the score phase's double-buffered TMA copies below
    // hit L2 and HBM sees the whole pool's reads in flight
    const uint32_t ngroups = (c.cap + 3u) >> 2;
    const uint32_t gpc = (ngroups + G - 1) / G;
    const uint32_t s_lo = 4u * min(ngroups, bid * gpc), s_hi = 4u * min(ngroups, bid * gpc + gpc);
    if (warp == 0) {
        const uint32_t npf = 7u * ((s_hi - s_lo + kChunk - 1) / kChunk);
        for (uint32_t q = lane; q < npf; q += 32u) {
            const uint32_t ai = q % 7u, base = s_lo + (q / 7u) * kChunk;
            const uint32_t bytes = min((uint32_t)kChunk, s_hi - base) * 4u;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b.pool.sfc + (size_t)ai * b.pool.stride + base),
                         "r"(bytes) : "memory");
        }
    }
    uint32_t* T = b.btot + (a.parity ? kMaxBuckets : 0);  // [NB] bucket totals of this step (cold steps)
    {   // the other parity's totals are zeroed for the next step (whose table may be larger)
        uint4* Tn = reinterpret_cast<uint4*>(b.btot + (a.parity ? 0 : kMaxBuckets));
        for (uint32_t j = bid * kFT + tid; j < (uint32_t)kMaxBuckets / 4u; j += G * kFT) Tn[j] = make_uint4(0, 0, 0, 0);
    }
    uint32_t* rcur = b.rcur + (a.parity ? kMaxCtas : 0);  // [G] keys written to each range
    if (bid == 0 && tid < (uint32_t)kMaxCtas) b.rcur[(a.parity ? 0 : kMaxCtas) + tid] = 0u;  // the next step's
    // the bucket table and (warm steps) the splitters the previous step wrote -> shared memory
    // by cp.async: read only after the score phase, so their latency hides behind it
    if (tid < (uint32_t)kTabW / 4u) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.btab[4 * tid]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\ncp.async.commit_group;" ::"r"(dst),
                     "l"(b.btab + (size_t)a.parity * kTabW + 4 * tid) : "memory");
    }
    if (!a.cold && tid <= (uint32_t)kMaxCtas) {  // the range splitters fine[16 r] (r < G), the largest key
        if (tid < G || tid == (uint32_t)kMaxCtas) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.s.spl[spl_pos(tid)]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\ncp.async.commit_group;" ::"r"(dst),
                         "l"(b.spl + (size_t)a.parity * kSplG + kSeg * min(tid, G)) : "memory");
        } else {
            sm.s.spl[spl_pos(tid)] = ~0ull;
        }
    }

    TRACE(0);
    SmemTail& tail = *reinterpret_cast<SmemTail*>(smem_raw + sizeof(FusedSmem));
    if (P2P && tid < a.world) {  // the peers' exchange buffers
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tail.xp[tid]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\ncp.async.commit_group;" ::"r"(dst),
                     "l"(b.xpeers + tid) : "memory");
    }
    // cold steps: the CTAs' measured range-sort costs (previous steps) weight the key ranges (X)
    if (a.cold && tid < G && tid < (uint32_t)kMaxCtas) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.s.ccost[tid]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\ncp.async.commit_group;" ::"r"(dst),
                     "l"(b.cta_cost + tid) : "memory");
    }
    if (a.n_ev | a.n_ret | a.n_sub) {  // API returns, arrivals and A0 for the engine's events on
                                       // this CTA's slots, before they are scored (the three touch
                                       // disjoint slots: PAUSED, FREE, admitted last step)
        const ReturnRec* rets = a.inl ? reinterpret_cast<const ReturnRec*>(inl.bytes)
                                      : static_cast<const ReturnRec*>(b.returns);
        const SubmitRec* subs = a.inl ? reinterpret_cast<const SubmitRec*>(inl.bytes) + a.n_ret
                                      : static_cast<const SubmitRec*>(b.arrivals);
        const DevEvent* evs = a.inl ? reinterpret_cast<const DevEvent*>(reinterpret_cast<const SubmitRec*>(inl.bytes) +
                                                                        a.n_ret + a.n_sub)
                                    : static_cast<const DevEvent*>(b.events);
        for (uint32_t e = tid; e < a.n_ret; e += kFT) {
            const ReturnRec R = rets[e];
            if (R.slot >= s_lo && R.slot < s_hi) apply_return(b.pool, c, R);
        }
        for (uint32_t e = tid; e < a.n_sub; e += kFT) {
            const SubmitRec R = subs[e];
            if (R.slot >= s_lo && R.slot < s_hi) apply_submit(b.pool, c, R);
        }
        for (uint32_t e = tid; e < a.n_ev; e += kFT) {
            const DevEvent E = evs[e];
            const uint32_t s = (uint32_t)E.id & c.cap_mask;
            if (s >= s_lo && s < s_hi) apply_event(b.pool, c, E);
        }
        __syncthreads();
    }
    if (tid < (uint32_t)kMaxCtas) sm.s.lcnt[tid] = 0u;  // R's per-range counts
    if (a.cold) {
        for (uint32_t i = tid; i < (uint32_t)kMaxBuckets / 4u; i += kFT)
            reinterpret_cast<uint4*>(sm.s.cnt)[i] = make_uint4(0, 0, 0, 0);
        asm volatile("cp.async.wait_all;" ::: "memory");  // the bucket table (histogram below)
    }
    __syncthreads();
    // ---------------- S: score this CTA's slots, two per thread per round (64-bit loads of the
    // seven SoA words, L2 hits after the bulk prefetch above); keys compacted into kbuf (warp-
    // aggregated: one shared-memory atomic per warp); cold steps also count the keys' buckets
    uint32_t pinned = 0, nmine = 0;  // this thread's pinned blocks (< 2^32: <= 8 slots of < 2^16) and keys
    const bool fixed16 = c.SH == 16u && c.lgB == 4u;  // the workloads' profiles (gen/configs.py)
    auto score1 = [&](uint32_t slot, uint32_t w, uint32_t ctx, uint32_t pre, uint32_t api, uint32_t resp,
                      uint32_t post, uint32_t pend, uint64_t& key) -> bool {
        if (w & SFC_RAN) {  // A0: the previous batch generated one token
            ctx += 1u;
            pre = pre ? pre - 1u : 0u;
            pend = 0u;
            b.pool.ctx[slot] = ctx;
            b.pool.pre[slot] = pre;
            b.pool.pend[slot] = 0u;
        }
        const uint32_t st = sfc_state(w);
        pinned += st == ST_PP ? (ctx + c.B - 1u) >> c.lgB : 0u;
        if (st != ST_READY) return false;
        const uint32_t has = sfc_has(w), rp = has ? resp : 0u, pp = has ? post : 0u;
        // fast check: all four below 2^18, so their sum is below 2^20 (kFastCtxLimit)
        if (c.lean && (ctx | pre | rp | pp) < (1u << 18)) {
            // A1 + A2 (score_lean; SH = 16, B = 16 with immediate shifts), A3: starvation, counter, key
            uint64_t sc, wp, wd, ws;
            const uint32_t strat = fixed16 ? score_lean<16, 4>(ctx, pre, api, rp, pp, pend, has, c, sc, wp, wd, ws)
                                           : score_lean(ctx, pre, api, rp, pp, pend, has, c, sc, wp, wd, ws);
            const uint32_t cnt = sfc_cnt(w);
            const uint32_t starv = sfc_starv(w) | (cnt >= c.T ? 1u : 0u);
            w = sfc_pack(ST_READY, has, starv, strat, cnt < 65535u ? cnt + 1u : 65535u);
            key = (starv ? 0ull : c.nsbit) | (sc << c.IB) | ((slot - a.id_base_mod) & c.cap_mask);
            if (DBG) {
                unsigned long long* d = b.dbg + 4ull * slot;
                d[0] = wp; d[1] = wd; d[2] = ws; d[3] = sc;
            }
        } else {
            const ColdOut o = score_slot_cold<DBG>(b.pool, c, a.id_base_mod, b.dbg, slot, w, ctx, pre, api, resp,
                                                   post, pend);
            key = o.key;
            w = o.w;
        }
        b.pool.sfc[slot] = w;
        nmine++;
        return true;
    };
    // keys stay at their slot's position in kbuf (position = slot - s_lo); which positions hold
    // keys: one ballot word per warp and slot parity (vmask[2 * (q >> 5) + j], q = pair index)
    {
        const uint32_t p_lo = s_lo >> 1, p_hi = s_hi >> 1;  // slot pairs
        const uint2* S2 = reinterpret_cast<const uint2*>(b.pool.sfc);
        const uint32_t st2 = b.pool.stride >> 1;
        for (uint32_t p0 = p_lo + (tid & ~31u); p0 < p_hi; p0 += kFT) {  // warp-uniform bound
            const uint32_t pr = p0 + lane;
            uint64_t k0 = 0, k1 = 0;
            bool h0 = false, h1 = false;
            if (pr < p_hi) {
                const uint2 w = __ldcg(S2 + pr), cx = __ldcg(S2 + st2 + pr), pe = __ldcg(S2 + 2 * st2 + pr),
                            ap = __ldcg(S2 + 3 * st2 + pr), rs = __ldcg(S2 + 4 * st2 + pr),
                            po = __ldcg(S2 + 5 * st2 + pr), pd = __ldcg(S2 + 6 * st2 + pr);
                h0 = score1(2u * pr, w.x, cx.x, pe.x, ap.x, rs.x, po.x, pd.x, k0);
                h1 = score1(2u * pr + 1u, w.y, cx.y, pe.y, ap.y, rs.y, po.y, pd.y, k1);
                reinterpret_cast<ulonglong2*>(sm.s.kbuf)[pr - p_lo] = make_ulonglong2(k0, k1);
                if (a.cold) {
                    uint32_t sv;
                    if (h0) atomicAdd(&sm.s.cnt[bucket_t(k0, sm.btab, vb, sv)], 1u);
                    if (h1) atomicAdd(&sm.s.cnt[bucket_t(k1, sm.btab, vb, sv)], 1u);
                }
            }
            const uint32_t m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
            if (lane == 0) {
                const uint32_t wq = (p0 - p_lo) >> 5;
                sm.s.vmask[2 * wq] = m0;
                sm.s.vmask[2 * wq + 1] = m1;
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // table, splitters, costs, peer pointers
    const uint32_t npos = s_hi - s_lo;  // kbuf positions (slots of this CTA)
    const uint32_t NB = sm.btab[kTabNB];  // buckets of this step's table
    unsigned long long pin64 = pinned;
    uint32_t nk_cta = nmine;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        pin64 += __shfl_xor_sync(0xffffffffu, pin64, o);
        nk_cta += __shfl_xor_sync(0xffffffffu, nk_cta, o);
    }
    if (lane == 0) { sm.s.red[0][warp] = pin64; sm.s.red[1][warp] = nk_cta; }
    __syncthreads();
    {
        uint32_t t = 0;
#pragma unroll 8
        for (int w = 0; w < kFW; w++) t += (uint32_t)sm.s.red[1][w];
        nk_cta = t;  // keys of this CTA
    }
    if (tid == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kFW; w++) t += sm.s.red[0][w];
        b.pin_part[bid] = t;
        b.nk_part[bid] = nk_cta;
    }
    TRACE(1);
    uint32_t bar = a.step * kBarPerStep;
    const bool head_mode = (a.flags & kStepHeadOnly) != 0;
    if (a.cold) {
        // ---------------- cold step (no splitters from a previous step): bucket histogram ->
        // totals -> bucket-aligned key ranges -> splitters = the ranges' lowest bucket keys
        {   // H: this CTA's bucket counts into the totals
            constexpr int kU = 8;
            for (uint32_t j0 = 0; j0 < NB; j0 += kU * kFT) {
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    const uint32_t j = j0 + (uint32_t)u * kFT + tid;
                    const uint32_t v = j < NB ? sm.s.cnt[j] : 0u;
                    if (v) atomicAdd(&T[j], v);
                }
            }
        }
        TRACE(2);
        grid_barrier(b.flags, G, ++bar);
        TRACE(3);
        {   // X: bucket starts (the totals loaded coalesced, scanned in place by raking)
            constexpr int kPer4 = (kMaxBuckets / 4 + kFT - 1) / kFT;  // 4
            uint4 tv[kPer4];
            const uint32_t nb4 = (NB + 3u) / 4u;
#pragma unroll
            for (int u = 0; u < kPer4; u++) {
                const uint32_t j = tid + (uint32_t)u * kFT;
                tv[u] = j < nb4 ? __ldcg(reinterpret_cast<const uint4*>(T) + j) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kPer4; u++) {
                const uint32_t j = tid + (uint32_t)u * kFT;
                if (j < nb4) reinterpret_cast<uint4*>(sm.s.start)[j] = tv[u];
            }
        }
        __syncthreads();
        TRACE(10);
        {
            const uint32_t tot = smem_excl_scan<kFT, (kMaxBuckets + kFT - 1) / kFT>(sm.s.start, NB, sm.s.w32);
            if (tid == 0) sm.s.base = tot;  // total number of keys
        }
        __syncthreads();
        TRACE(11);
        const uint32_t n0 = sm.s.base;
        // the next step's bucket table from this step's octave counts (one warp of the last CTA)
        if (bid == G - 1u && warp == kFW - 1) bt_update(sm.btab, sm.s.start, n0, vb, b.btab + (size_t)(a.parity ^ 1u) * kTabW);
        // CTA 0 sorts only the head (the max_batch keys the admission may take, to the end of
        // their bucket) so it can start the admission early; the other CTAs share the rest in
        // proportion to their measured speed (cycles per key of the previous steps' range
        // sorts), weight mean/cost capped at 1.25; below 0.4 the CTA gets no range (G <= 255)
        const uint32_t kRW = (G + 1u + 31u) / 32u;
        if (warp < kRW) {
            float* wx = sm.s.wx;  // [G + 1] exclusive weight prefix
            if (warp == 0) {
                constexpr int kW = kMaxCtas / 32;
                float cst[kW];
                float ksum = 0.f, kcnt = 0.f;
#pragma unroll
                for (int u = 0; u < kW; u++) {
                    const uint32_t r = lane * kW + (uint32_t)u;
                    cst[u] = (r >= 1 && r < G) ? sm.s.ccost[r] : 0.f;
                    if (cst[u] > 0.f) { ksum += cst[u]; kcnt += 1.f; }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
                    kcnt += __shfl_xor_sync(0xffffffffu, kcnt, o);
                }
                const float mean = kcnt > 0.f ? __fdividef(ksum, kcnt) : 1.f;
                float w[kW], run = 0.f;
#pragma unroll
                for (int u = 0; u < kW; u++) {
                    const uint32_t r = lane * kW + (uint32_t)u;
                    w[u] = 0.f;
                    if (r >= 1 && r < G) {
                        const float rel = cst[u] > 0.f ? __fdividef(mean, cst[u]) : 1.f;
                        w[u] = rel < 0.4f ? 0.f : fminf(rel, (a.tune & 8u) ? 1.f : 1.25f);
                        if (a.tune & 1u) w[u] = 1.f;
                    }
                    run += w[u];
                }
                float x = run;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                float e = x - run;
#pragma unroll
                for (int u = 0; u < kW; u++) {
                    const uint32_t r = lane * kW + (uint32_t)u;
                    if (r <= G) wx[r] = e;  // r = G: the total
                    e += w[u];
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kRW * 32u) : "memory");  // the kRW warps only
            if (tid <= G) {
                const uint32_t head = min(n0, a.max_batch + 32u);
                const float wt = wx[G];
                const float f = tid == 0 ? 0.f : (wt > 0.f ? fminf(__fdividef(wx[tid], wt), 1.f) : 0.f);
                const uint32_t q = tid == 0 ? 0u : head + min(n0 - head, (uint32_t)(f * (float)(n0 - head)));
                uint32_t lo = 0, hi = NB;  // first j with start(j) >= q
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (sm.s.start[mid] >= q) hi = mid; else lo = mid + 1;
                }
                sm.s.jb[tid] = tid == G ? NB : lo;
            }
        }
        __syncthreads();
        // splitter r = the lowest key of bucket jb[r] (octave (ns, e) found by binary search
        // over the table's bases; key = ns | (2^m + mantissa) << s); none past the last bucket.
        // Entry kMaxCtas: the largest key's bound (the last nonempty bucket's highest key).
        auto bucket_key = [&](uint32_t j, bool high) -> unsigned long long {
            uint32_t lo = 0, hi = kTabNB - 1u;  // last octave with base <= j and a nonzero span
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1u) >> 1;
                if ((sm.btab[mid] & 0xffffu) <= j) lo = mid; else hi = mid - 1u;
            }
            while (lo > 0 && (sm.btab[lo] & 0xffffu) == (lo + 1u < kTabNB ? sm.btab[lo + 1] & 0xffffu : NB)) lo--;
            const uint32_t t = sm.btab[lo], e = lo % 65u, ns = lo / 65u;
            const uint32_t sv = (t >> 16) & 63u, m = t >> 24, mm = j - (t & 0xffffu);
            unsigned long long v = e == 0u ? 0ull : ((unsigned long long)((1u << m) | mm) << sv);
            if (high) v |= (1ull << sv) - 1ull;
            return ((unsigned long long)ns << vb) | v;
        };
        if (tid < (uint32_t)kMaxCtas + 1u) {
            unsigned long long sk = ~0ull;
            if (tid == 0) {
                sk = 0ull;
            } else if (tid < G && sm.s.jb[tid] < NB) {
                sk = bucket_key(sm.s.jb[tid], false);
            } else if (tid == (uint32_t)kMaxCtas && n0) {
                uint32_t lo = 0, hi = NB;  // first j with start(j) >= n0; the last nonempty is before it
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (sm.s.start[mid] >= n0) hi = mid; else lo = mid + 1;
                }
                sk = bucket_key(lo - 1u, true);
            }
            sm.s.spl[spl_pos(tid)] = sk;
        }
        __syncthreads();
        // this step's grid (every CTA: its own range's quantiles are read back after the
        // barrier; head-only steps keep the grid): splitters, and between two of them
        // entries interpolated linearly in key space (no quantiles known yet)
        for (uint32_t f = bid * kFT + tid; f <= kSeg * G; f += G * kFT) {
            const uint32_t r = f / kSeg, j = f % kSeg;
            const unsigned long long lo = sm.s.spl[spl_pos(r == G ? kMaxCtas : r)];
            unsigned long long v = lo;
            if (r < G && j) {
                const unsigned long long hi = r + 1u < G ? sm.s.spl[spl_pos(r + 1u)] : sm.s.spl[spl_pos(kMaxCtas)];
                const unsigned long long h2 = hi == ~0ull ? sm.s.spl[spl_pos(kMaxCtas)] : hi;
                v = h2 > lo ? lo + (h2 - lo) / kSeg * j : lo;
            }
            b.spl[(size_t)a.parity * kSplG + f] = v;
        }
    }
    else if (bid == G - 1u && tid < (uint32_t)kTabW) {
        b.btab[(size_t)(a.parity ^ 1u) * kTabW + tid] = sm.btab[tid];  // warm step: the table carries over
    }
    // ---------------- R: every key to its range, range r = keys in [spl[r], spl[r+1]) (a
    // binary search over the splitters), written into the range's region keys0[r * kKcap ...]:
    // per range this CTA's keys form one run (a local counting sort), whose offset inside
    // the region one global atomic per range gives, so the stores are contiguous
    // (compact loops, no per-thread item arrays: the kernel runs once per step and its code is
    // fetched cold -- straight-line unrolled code costs more in instruction fetch than it saves)
    uint32_t* const kr = reinterpret_cast<uint32_t*>(sm.s.cnt);          // scratch over cnt + start
    uint64_t* const kb2 = reinterpret_cast<uint64_t*>(kr);                 // [kKcap] keys by range
    uint8_t* const rr = reinterpret_cast<uint8_t*>(kr) + 8u * kKcap;       // [kKcap] their range
    uint8_t* const rv = rr + kKcap;                                        // [kKcap] range by position
    {
        const unsigned long long* spl = sm.s.spl;
        for (uint32_t i0 = tid; i0 < npos; i0 += 2u * kFT) {  // two searches advanced together
            uint64_t k[2];
            bool ok[2];
            uint32_t r[2];
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const uint32_t i = i0 + (uint32_t)u * kFT, q = i >> 1;
                ok[u] = i < npos && ((sm.s.vmask[2u * (q >> 5) + (i & 1u)] >> (q & 31u)) & 1u);
                k[u] = ok[u] ? sm.s.kbuf[i] : 0ull;
                r[u] = 0;
            }
#pragma unroll
            for (uint32_t st = kMaxCtas / 2u; st; st >>= 1) {
#pragma unroll
                for (int u = 0; u < 2; u++) r[u] = k[u] >= spl[spl_pos(r[u] + st)] ? r[u] + st : r[u];
            }
#pragma unroll
            for (int u = 0; u < 2; u++) {
                if (!ok[u]) continue;
                const uint32_t rg = min(r[u], G - 1u);
                rv[i0 + (uint32_t)u * kFT] = (uint8_t)rg;
                atomicAdd(&sm.s.lcnt[rg], 1u);
            }
        }
    }
    __syncthreads();
    TRACE(4);
    if (tid < G) {
        const uint32_t m = sm.s.lcnt[tid];
        sm.s.gbase[tid] = m ? atomicAdd(&rcur[tid], m) : 0u;
    }
    if (tid < (uint32_t)kMaxCtas) sm.s.lst[tid] = sm.s.lcnt[tid];
    __syncthreads();
    (void)smem_excl_scan<kFT, 1>(sm.s.lst, kMaxCtas, sm.s.w32);
    if (tid < (uint32_t)kMaxCtas) sm.s.lcnt[tid] = sm.s.lst[tid];  // run cursors
    __syncthreads();
    TRACE(5);
    for (uint32_t i = tid; i < npos; i += kFT) {
        const uint32_t q = i >> 1;
        if (!((sm.s.vmask[2u * (q >> 5) + (i & 1u)] >> (q & 31u)) & 1u)) continue;
        const uint32_t r = rv[i], lp = atomicAdd(&sm.s.lcnt[r], 1u);  // order within a run is free
        kb2[lp] = sm.s.kbuf[i];
        rr[lp] = (uint8_t)r;
    }
    __syncthreads();
    TRACE(12);
    for (uint32_t i = tid; i < nk_cta; i += kFT) {
        const uint32_t r = rr[i], pos = sm.s.gbase[r] + (i - sm.s.lst[r]);
        if (pos < (uint32_t)kKcap) b.keys[0][(size_t)r * kKcap + pos] = kb2[i];  // else: overflow -> fallback
    }
    TRACE(6);
    grid_barrier(b.flags, G, ++bar);
    TRACE(7);
    // ranges' sizes (prefix: where each sorted range goes) and the CTAs' key counts (n)
    uint32_t rsz = 0, rpre = 0, n = 0;
    bool fallback = (a.flags & kStepForceFallback) != 0;
    if (warp == 0) {  // one round trip: 8 ranges and 8 CTAs per lane, a warp scan
        uint32_t v[kMaxCtas / 32], tot = 0, nq = 0, big = 0;
#pragma unroll
        for (int j = 0; j < kMaxCtas / 32; j++) {
            const uint32_t r = lane * (kMaxCtas / 32) + (uint32_t)j;
            v[j] = r < G ? __ldcg(&rcur[r]) : 0u;
            nq += r < G ? __ldcg(&b.nk_part[r]) : 0u;
        }
#pragma unroll
        for (int j = 0; j < kMaxCtas / 32; j++) { tot += v[j]; big |= v[j] > (uint32_t)kKcap ? 1u : 0u; }
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        uint32_t run = x - tot;
#pragma unroll
        for (int j = 0; j < kMaxCtas / 32; j++) {
            const uint32_t r = lane * (kMaxCtas / 32) + (uint32_t)j;
            sm.l.rsz[r] = v[j];
            sm.l.rpre[r] = run;
            run += v[j];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) nq += __shfl_xor_sync(0xffffffffu, nq, o);
        big = __any_sync(0xffffffffu, big != 0u) ? 1u : 0u;
        if (lane == 0) { sm.l.w32[0] = nq; sm.l.w32[1] = big; }
    }
    __syncthreads();
    n = sm.l.w32[0];
    fallback = fallback || sm.l.w32[1] != 0u;
    rsz = sm.l.rsz[bid];
    rpre = sm.l.rpre[bid];
    const uint32_t r_end0 = sm.l.rsz[0];
    // head-only mode (F3): CTA 0 ranks the head; the others stop here, unless the head range
    // does not hold the keys the admission needs (then every range is sorted)
    const bool head_only = head_mode && !fallback && r_end0 >= min(n, a.max_batch + 32u);
    // positions of the next step's splitters in this step's order: the head (range 0) ends
    // at max_batch + kHeadMargin keys, the other ranges share the rest evenly
    const uint32_t q1 = G > 1u ? min(n, a.max_batch + kHeadMargin) : n;
    // position of grid entry f (0 .. 16 G) in this step's order: range 0's 16 segments over
    // [0, q1), the other ranges' over [q1, n) evenly (past the last key: the last key)
    auto qf = [&](uint32_t f) -> uint32_t {
        const uint64_t p = f <= (uint32_t)kSeg
                               ? (uint64_t)q1 * f / kSeg
                               : q1 + (uint64_t)(f - kSeg) * (uint64_t)(n - q1) / ((uint64_t)kSeg * (G - 1u));
        return n ? (uint32_t)min(p, (uint64_t)(n - 1u)) : 0u;
    };
    unsigned long long* spl_next = b.spl + (size_t)(a.parity ^ 1u) * kSplG;
    if (head_only && bid == G - 1u)  // the grid is kept: the other ranges were not sorted
        for (uint32_t f = tid; f <= kSeg * G; f += kFT) spl_next[f] = __ldcg(&b.spl[(size_t)a.parity * kSplG + f]);
    // this range's grid entries fine[16 bid .. 16 bid + 16]: key codes and per-segment shifts of
    // the range sort's piecewise-linear digit (segment j: keys in [fine[j], fine[j + 1]))
    if (warp == 1 && lane <= (uint32_t)kSeg) {
        const unsigned long long fk = __ldcg(&b.spl[(size_t)a.parity * kSplG + kSeg * bid + lane]);
        sm.l.fine[lane] = fk;
        sm.l.fcode[lane] = key_code(fk, vb);
    }

    __syncthreads();  // the grid entries
    // ---------------- L: sort the key ranges
    uint32_t final_buf, passes;
    bool head_dw = false;  // CTA 0: demands / state words of its head in sm.l.b (sorted order)
    bool written = false;  // the range sort wrote the sorted range to keys1 itself
    bool head_loop = false;  // CTA 0: head keys in sm.l.b, demands / states in sm.l.pos (range_sort_loop)
    if (!fallback && (!head_only || bid == 0)) {
        const uint32_t rn = rsz;
        const uint64_t* src = b.keys[0] + (size_t)bid * kKcap;
        const long long l_t0 = clock64();
        unsigned long long g_t0 = 0;
        if (b.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t0));
        unsigned long long* tr = b.trace ? b.trace + (size_t)bid * kTraceSlots : nullptr;
        if (tr && tid == 0) {
            tr[30] = rn; tr[31] = 0;
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            tr[28] = smid;  // diagnostics: SM of this CTA
            for (int q = 32; q < 64; q++) tr[q] = 0;
        }
        if (rn <= kSmallSort && !(a.tune & 4u)) {
            TRACE(13);
            if (bid == 0) {
                small_sort<true>(sm.l, src, rn, c, &b.pool, a.id_base_mod);
                head_dw = true;
            } else {
                small_sort<false>(sm.l, src, rn, c, nullptr, 0u);
            }
        } else {  // linear-digit counting sort, straight to the output (CTA 0: the head)
            TRACE(13);
            // CTA 0 (single shard): head + admission loads on chip
            const bool stage = bid == 0 && rn <= kHeadPre && !(a.flags & kStepMerge);
            written = range_sort_loop(sm.l, src, rn, b.keys[1] + rpre, vb, tr ? tr + 32 : nullptr, &b.pool,
                                      a.id_base_mod, &c, stage ? sm.l.pos + kHeadPre : nullptr,
                                      stage ? sm.l.pos + 2u * kHeadPre : nullptr);
            head_loop = stage && written;
            if (!written) {  // a counter held too many keys: sort the placed range by LSD
                unsigned long long o, an;
                block_or_and(sm.l, sm.l.a, rn, o, an);
                const uint64_t* r = local_lsd(sm.l, sm.l.a, sm.l.b, rn, o ^ an);
                if (r != sm.l.a)
                    for (uint32_t i = tid; i < rn; i += kFT) sm.l.a[i] = r[i];
                __syncthreads();
            }
        }
        TRACE(14);
        if (b.trace && tid == 0) {
            unsigned long long g_t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t1));
            b.trace[(size_t)bid * kTraceSlots + 26] = g_t0;
            b.trace[(size_t)bid * kTraceSlots + 27] = g_t1;
        }
        if (tid == 0 && bid != 0 && rn >= 1024u) {
            // this CTA's range-sort cycles per key, for the cold steps' range weights (EMA;
            // the CTA -> SM placement of the cooperative launch is stable in practice)
            const float cst = __fdividef((float)(clock64() - l_t0), (float)rn);
            const float old = b.cta_cost[bid];
            b.cta_cost[bid] = old > 0.f ? 0.75f * old + 0.25f * cst : cst;
        }
        if (!written)
            for (uint32_t i = tid; i < rn; i += kFT) b.keys[1][rpre + i] = sm.l.a[i];
        __syncthreads();  // the range's keys are in place (visible to this CTA's threads)
        // the next step's grid entries that fall in this range
        if (!head_only && rn)
            for (uint32_t f = tid; f <= kSeg * G; f += kFT) {
                const uint32_t q = qf(f);
                if (q >= rpre && q < rpre + rn) spl_next[f] = __ldcg(&b.keys[1][q]);
            }
        final_buf = 1;
        passes = 1;
    } else if (fallback) {
        {   // the keys compacted into keys0 (this CTA's at the prefix of the CTAs' key counts)
            uint32_t off = 0;
            {
                const uint32_t q = tid < bid ? __ldcg(&b.nk_part[tid]) : 0u;
                uint32_t tot;
                (void)block_excl_scan_u32<kFT>(q, sm.l.w32, &tot);
                off = tot;
            }
            // kb2 (this CTA's keys, compacted by R) is intact: since the barrier only PhaseL's
            // small arrays past sm.l.b (w32, rsz, rpre) were written
            for (uint32_t i = tid; i < nk_cta; i += kFT) b.keys[0][off + i] = kb2[i];
            grid_barrier(b.flags, G, ++bar);
        }
        {   // OR / AND of the keys (the LSD skips digit positions that never vary)
            unsigned long long o = 0, an = ~0ull;
            for (uint32_t i = bid * kFT + tid; i < n; i += G * kFT) {
                const uint64_t k = __ldcg(&b.keys[0][i]);
                o |= k;
                an &= k;
            }
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                o |= __shfl_xor_sync(0xffffffffu, o, s);
                an &= __shfl_xor_sync(0xffffffffu, an, s);
            }
            if (lane == 0) { sm.s.red[1][warp] = o; sm.s.red[2][warp] = an; }
            __syncthreads();
            if (tid == 0) {
                for (int w = 0; w < kFW; w++) { o |= sm.s.red[1][w]; an &= sm.s.red[2][w]; }
                b.kmask[bid] = o;
                b.kmask[G + bid] = an;
            }
            grid_barrier(b.flags, G, ++bar);
        }
        passes = lsd_sort_global(b, n, b.kmask, G, sm.g, bar);
        final_buf = passes & 1u;
    } else {
        final_buf = 1;  // head-only: CTA 0 ranked the head; this CTA is done
        passes = 1;
    }
    // the next step's splitters past the last key, and (after the LSD) all of them
    if (bid == 0 && !head_only && n == 0)  // no keys: an empty grid
        for (uint32_t f = tid; f <= kSeg * G; f += kFT) spl_next[f] = 0ull;
    unsigned long long pinned_all = 0;
    if (bid == 0 && warp == 0) {  // A5's budget: the pinned total
        for (uint32_t r = lane; r < G; r += 32) pinned_all += __ldcg(&b.pin_part[r]);
#pragma unroll
        for (int o = 16; o; o >>= 1) pinned_all += __shfl_xor_sync(0xffffffffu, pinned_all, o);
    }

    TRACE(8);
    // ---------------- A: admission by CTA 0
    // CTA 0 may start as soon as the head it needs is sorted: without the fallback
    // the keys [0, rsz[0]) are sorted by CTA 0 itself.
    const uint32_t need = min(n, a.max_batch);  // the admission (or the merge records) reads keys [0, need)
    const bool wait = fallback || r_end0 < need;
    if (wait) grid_barrier(b.flags, G, ++bar);
    if (fallback && bid == 0 && n)
        for (uint32_t f = tid; f <= kSeg * G; f += kFT) spl_next[f] = __ldcg(&b.keys[final_buf][qf(f)]);
    if (bid != 0) return;
    if (tid == 0) sm.l.adm.w64[0] = pinned_all;
    __syncthreads();
    pinned_all = sm.l.adm.w64[0];
    __syncthreads();
    if (tid == 0) {
        ctl->n_passes = passes;
        ctl->final_buf = final_buf;
        if (fallback) atomicAdd(&ctl->fallbacks, 1u);  // a reduction, no load on the path
        ctl->n_ranked = head_only ? r_end0 : n;  // head-only: keys [0, hb_r) are ranked
    }
    TRACE(15);
    // CTA 0 holds [0, need) in shared memory unless it waited (or its range sort wrote them out)
    const bool hl = head_loop && !wait;  // head keys in sm.l.b, demands / states in sm.l.pos
    const uint64_t* head = wait ? b.keys[final_buf]
                                : (hl ? reinterpret_cast<const uint64_t*>(sm.l.b) : (written ? b.keys[final_buf] : sm.l.a));
    const bool dw = head_dw && !wait;
    if (a.flags & kStepMerge) {
        // multi-GPU: publish this rank's head as exchange records instead of admitting
        const uint32_t K = a.max_batch, nv = min(n, K);
        const uint64_t idmask = (1ull << c.IB) - 1ull;
        constexpr bool p2p = P2P;
        const uint32_t W = a.world, par = a.xseq & 1u;
        // peer-memory transport: record i of this rank goes to every peer's receive area
        // [par][rank] by NVLink stores (the one-shot all-gather), then flags, then the merge
        const size_t slot0 = ((size_t)par * W + a.rank) * (K + 1);
        for (uint32_t i = tid; i <= nv; i += kFT) {
            MergeRec r;
            if (i == 0) {
                MergeHdr* h = reinterpret_cast<MergeHdr*>(&r);
                h->pinned = pinned_all;
                h->kv_total = a.kv_total;
                h->n_valid = nv;
                h->n_local = n;
                h->pad = 0;
            } else {
                const uint64_t k = head[i - 1];
                const uint64_t lid = a.id_base + (k & idmask);
                const uint32_t slot = (uint32_t)(lid & c.cap_mask);
                r.sk = k >> c.IB;
                r.gid = lid * a.world + a.rank;
                r.demand = dw ? reinterpret_cast<const uint32_t*>(sm.l.b)[kHeadD + i - 1]
                              : (uint32_t)blk((uint64_t)b.pool.ctx[slot] + 1u, c);
                r.slot = slot;
                r.pad = 0;
            }
            if (p2p) {
                for (uint32_t p = 0; p < W; p++) tail.xp[p][slot0 + i] = r;
            } else {
                b.xsend[i] = r;
            }
        }
        if (!p2p) {
            TRACE(9);
            return;
        }
        unsigned long long* xtr = b.trace ? b.trace + 48 : nullptr;  // CTA 0's slots 48..55
        if (xtr && tid == 0) xtr[0] = clock64();
        __syncthreads();
        const size_t nrec = p2p_rec_count(W, K);
        // the CTA's records (ordered before by the barrier) before the flags: system scope
        // when the peers are other GPUs, device scope when every rank shares this device
        const bool sys = (a.flags & kStepP2PSys) != 0;
        if (tid == 0) {
            if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
            else asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (uint32_t p = 0; p < W; p++) {
                uint32_t* pf = reinterpret_cast<uint32_t*>(tail.xp[p] + nrec) + par * 32u + a.rank;
                if (sys) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(pf), "r"(a.xseq) : "memory");
                else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(pf), "r"(a.xseq) : "memory");
            }
            if (xtr) xtr[1] = clock64();
        }
        bool late = false;  // bounded wait: a peer that never steps must not hang the GPU
        if (tid < W) {
            const uint32_t* of = reinterpret_cast<const uint32_t*>(b.xown + nrec) + par * 32u + tid;
            unsigned long long t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            const unsigned long long lim = (unsigned long long)a.xtimeout_ms * 1000000ull;
            for (uint32_t it = 1;; it++) {
                uint32_t v;
                if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(of) : "memory");
                else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(of) : "memory");
                if (v == a.xseq) break;
                if (!(it & 255u)) {
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t - t0 > lim) {
                        late = true;
                        break;
                    }
                }
            }
        }
        late = __syncthreads_or(late);
        if (tid == 0) b.hres->xfail = late ? 1u : 0u;
        if (late) {
            TRACE(9);
            return;
        }
        TRACE(15);
        // merge scratch over sm.l.a (the head keys are no longer needed there: the admission
        // reads this rank's keys from b.keys), small structures at the end of shared memory.
        // While the scratch stays inside sm.l.a the admission keeps the preempted-check hash
        // table (start of sm.l.b) and, below the staged head arrays, their demand / state words
        const size_t mb = merge_smem_bytes(W, K);
        AdmitSmem& madm = tail.adm;
        uint32_t* mnv = tail.nv;
        unsigned long long* mhs = tail.hsum;
        uint32_t hs = 1024;
        while (hs < 2u * K) hs <<= 1;
        const bool in_a = mb <= sizeof(sm.l.a) && !wait;
        const bool use_h = in_a && hs <= kHeadTC;
        const bool use_d = dw && mb <= (size_t)kHeadD * 4u + sizeof(sm.l.a);
        uint32_t* b32 = reinterpret_cast<uint32_t*>(sm.l.b);
        merge_admit_cta(b, c, a, b.xown + (size_t)par * W * (K + 1), smem_raw, madm, mnv, mhs,
                        use_h ? b32 : nullptr, use_h ? hs : 0u, use_d ? b32 + kHeadD : nullptr,
                        use_d ? b32 + kHeadW : nullptr, xtr ? xtr + 2 : nullptr);
        TRACE(9);
        return;
    }
    // the preempted check probes a hash table of the admitted slots in shared memory
    // (sm.l.b is free once the range is sorted); very large batches stamp P.stamp
    uint32_t hs = 1024;
    while (hs < 2u * a.max_batch) hs <<= 1;
    const bool use_h = !wait && hs <= kHeadTC;
    const uint32_t* b32 = reinterpret_cast<const uint32_t*>(sm.l.b);
    uint32_t* htab = hl ? reinterpret_cast<uint32_t*>(sm.l.a) : reinterpret_cast<uint32_t*>(sm.l.b);
    admit_cta(b, c, a, head, n, pinned_all, sm.l.adm, use_h ? htab : nullptr, use_h ? hs : 0u,
              b.trace ? b.trace + 40 : nullptr,
              hl ? sm.l.pos + kHeadPre : (dw ? b32 + kHeadD : nullptr),
              hl ? sm.l.pos + 2u * kHeadPre : (dw ? b32 + kHeadW : nullptr));
    TRACE(9);
}

// ---------------------------------------------------------------------------
// Small pools (capacity <= kSmallCap, BASELINE C1-C3): the whole step in ONE 1024-thread
// CTA, a plain (non-cooperative) launch -- no grid barriers, no bucket tables, no
// exchange of keys between CTAs.  The same device functions as the fused kernel:
//   prologue  API returns, arrivals, A0 for the engine's events (apply_return /
//             apply_submit / apply_event), then A0's default update and A1-A3 per slot
//             (score_slot: strategy, score, starvation, key), keys compacted to keys[0]
//   sort      range_sort_loop over all keys: one counting pass on a piecewise-linear digit
//             over 16 segments whose ends are the previous step's quantiles (this step's
//             smallest / largest key at the ends; cold steps: interpolated), rank by
//             comparison inside counters, a local LSD as the last resort
//   A5        admit_cta from the sorted keys on chip (demand / state staged by the sort)
// The quantiles of this step's order are written for the next step.
constexpr uint32_t kSmallCap = 4096;
constexpr int kSmallPer = kSmallCap / kFT;  // slots per thread
template <bool DBG>
__global__ void __launch_bounds__(kFT, 1) k_small(const __grid_constant__ Bufs b, const __grid_constant__ Cost c,
                                                  StepArgs a, const __grid_constant__ InlineStage inl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FusedSmem& sm = *reinterpret_cast<FusedSmem*>(smem_raw);
    Ctl* ctl = b.ctl;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t vb = c.SB + c.IB;
    const uint32_t cap = c.cap;
    if (b.trace && tid == 0) b.trace[0] = clock64();
    // the previous step's quantiles (warm steps), consumed after scoring
    unsigned long long fk = 0;
    if (!a.cold && tid <= (uint32_t)kSeg) fk = __ldcg(&b.spl[(size_t)a.parity * kSplG + tid]);
    if (a.n_ev | a.n_ret | a.n_sub) {  // prologue, as the fused kernel's (disjoint slots)
        const ReturnRec* rets = a.inl ? reinterpret_cast<const ReturnRec*>(inl.bytes)
                                      : static_cast<const ReturnRec*>(b.returns);
        const SubmitRec* subs = a.inl ? reinterpret_cast<const SubmitRec*>(inl.bytes) + a.n_ret
                                      : static_cast<const SubmitRec*>(b.arrivals);
        const DevEvent* evs = a.inl ? reinterpret_cast<const DevEvent*>(reinterpret_cast<const SubmitRec*>(inl.bytes) +
                                                                        a.n_ret + a.n_sub)
                                    : static_cast<const DevEvent*>(b.events);
        for (uint32_t e = tid; e < a.n_ret; e += kFT) apply_return(b.pool, c, rets[e]);
        for (uint32_t e = tid; e < a.n_sub; e += kFT) apply_submit(b.pool, c, subs[e]);
        for (uint32_t e = tid; e < a.n_ev; e += kFT) apply_event(b.pool, c, evs[e]);
        __syncthreads();
    }
    // ---- A0 default update, A1-A3 for this thread's slots (tid + u * kFT), keys in registers
    const Pool& P = b.pool;
    uint64_t key[kSmallPer];
    uint32_t nk = 0, pinned = 0;
    unsigned long long kmin = ~0ull, kmax = 0ull;
#pragma unroll
    for (int u = 0; u < kSmallPer; u++) {
        const uint32_t slot = tid + (uint32_t)u * kFT;
        key[u] = 0;
        if (slot >= cap) continue;
        // the seven SoA words in one round trip
        uint32_t w = P.sfc[slot], ctx = P.ctx[slot], pre = P.pre[slot], pend = P.pend[slot];
        const uint32_t api = P.api[slot], resp = P.resp[slot], post = P.post[slot];
        if (w & SFC_RAN) {  // A0: the previous batch generated one token
            ctx += 1u;
            pre = pre ? pre - 1u : 0u;
            pend = 0u;
            P.ctx[slot] = ctx;
            P.pre[slot] = pre;
            P.pend[slot] = 0u;
        }
        const uint32_t st = sfc_state(w);
        if (st == ST_PP) pinned += (ctx + c.B - 1u) >> c.lgB;
        if (st != ST_READY) continue;
        uint64_t k;
        (void)score_slot<DBG>(P, c, a.id_base_mod, b.dbg, slot, w, ctx, pre, api, resp, post, pend, k);
        P.sfc[slot] = w;
#pragma unroll
        for (int q = 0; q < kSmallPer; q++)  // packed to the front (no dynamic register index)
            if (q == (int)nk) key[q] = k;
        nk++;
        kmin = min(kmin, (unsigned long long)k);
        kmax = max(kmax, (unsigned long long)k);
    }
    // ---- compaction into keys[0] (block scan), the pinned total, this step's key bounds
    uint32_t n;
    const uint32_t pos = block_excl_scan_u32<kFT>(nk, sm.l.w32, &n);
#pragma unroll
    for (int q = 0; q < kSmallPer; q++)
        if ((uint32_t)q < nk) b.keys[0][pos + q] = key[q];
    unsigned long long pin64 = pinned;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        pin64 += __shfl_xor_sync(0xffffffffu, pin64, o);
        kmin = min(kmin, (unsigned long long)__shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, (unsigned long long)__shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) { sm.l.red[0][warp] = kmin; sm.l.red[1][warp] = kmax; sm.l.adm.w64[warp] = pin64; }
    __syncthreads();  // also orders the key stores before the sort's loads (same CTA)
    if (warp == 0) {
        unsigned long long lo = sm.l.red[0][lane], hi = sm.l.red[1][lane], pn = sm.l.adm.w64[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lo = min(lo, (unsigned long long)__shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, (unsigned long long)__shfl_xor_sync(0xffffffffu, hi, o));
            pn += __shfl_xor_sync(0xffffffffu, pn, o);
        }
        if (lane == 0) { sm.l.red[0][0] = lo; sm.l.red[1][0] = hi; sm.l.red[0][1] = pn; }
    }
    __syncthreads();
    const unsigned long long lo = sm.l.red[0][0], hi = sm.l.red[1][0];
    const unsigned long long pinned_all = sm.l.red[0][1];
    if (b.trace && tid == 0) b.trace[1] = clock64();
    // ---- the digit's grid: ends = this step's bounds, inside = the previous step's quantiles
    // clamped to them (cold steps: interpolated linearly in key space)
    if (tid <= (uint32_t)kSeg) {
        unsigned long long g;
        if (tid == 0) g = lo;
        else if (tid == (uint32_t)kSeg) g = hi;
        else if (!a.cold) g = min(max((unsigned long long)fk, lo), hi);
        else g = lo + (hi - lo) / kSeg * tid;
        sm.l.fine[tid] = g;
        sm.l.fcode[tid] = key_code(g, vb);
    }
    __syncthreads();
    // ---- A4: sort (stages the admission's demand / state words when the keys fit the arrays)
    const bool stage = n <= kHeadPre;
    uint32_t* dsm = stage ? sm.l.pos + kHeadPre : nullptr;
    uint32_t* wsm = stage ? sm.l.pos + 2u * kHeadPre : nullptr;
    bool written = false, tiny = false;
    if (n > 1u && n <= kSmallSort && !(a.flags & kStepForceFallback)) {
        // a few hundred keys: rank of each by comparison against all (unique keys), the
        // admission's per-key loads staged by sorted position (small_sort)
        small_sort<true>(sm.l, b.keys[0], n, c, &b.pool, a.id_base_mod);
        for (uint32_t i = tid; i < n; i += kFT) b.keys[1][i] = sm.l.a[i];
        tiny = true;
    } else if (n > 1u && !(a.flags & kStepForceFallback)) {
        written = range_sort_loop(sm.l, b.keys[0], n, b.keys[1], vb, nullptr, &b.pool, a.id_base_mod, &c, dsm, wsm);
    }
    if (!written && !tiny) {  // a counter held too many keys (or the forced fallback): LSD of the whole pool
        if (n <= 1u || (a.flags & kStepForceFallback))
            for (uint32_t i = tid; i < n; i += kFT) sm.l.a[i] = __ldcg(&b.keys[0][i]);
        __syncthreads();
        if (n > 1u) {
            unsigned long long o, an;
            block_or_and(sm.l, sm.l.a, n, o, an);
            const uint64_t* r = local_lsd(sm.l, sm.l.a, sm.l.b, n, o ^ an);
            if (r != sm.l.a)
                for (uint32_t i = tid; i < n; i += kFT) sm.l.a[i] = r[i];
            __syncthreads();
        }
        for (uint32_t i = tid; i < n; i += kFT) b.keys[1][i] = sm.l.a[i];
    }
    const uint64_t* srt = written ? reinterpret_cast<const uint64_t*>(sm.l.b) : sm.l.a;
    // the next step's grid: the quantiles of this order
    if (n && tid <= (uint32_t)kSeg) b.spl[(size_t)(a.parity ^ 1u) * kSplG + tid] = srt[min((uint32_t)((uint64_t)n * tid / kSeg), n - 1u)];
    if (b.trace && tid == 0) b.trace[2] = clock64();
    if (tid == 0) {
        ctl->n_passes = 1;
        ctl->final_buf = 1;
        if (!written && !tiny && n > 1u) atomicAdd(&ctl->fallbacks, 1u);
        ctl->n_ranked = n;
    }
    __syncthreads();
    // ---- A5: admission from the sorted keys on chip; the preempted check's hash table in the
    // other key buffer
    uint32_t hs = 1024;
    while (hs < 2u * a.max_batch) hs <<= 1;
    const bool use_h = hs <= kHeadTC;
    uint32_t* htab = written ? reinterpret_cast<uint32_t*>(sm.l.a) : reinterpret_cast<uint32_t*>(sm.l.b);
    const bool dw = written && stage;
    const uint32_t* b32 = reinterpret_cast<const uint32_t*>(sm.l.b);  // small_sort's staged arrays
    static_assert(kHeadTC <= kHeadD, "small_sort's staged arrays lie past the hash table");
    admit_cta(b, c, a, srt, n, pinned_all, sm.l.adm, use_h ? htab : nullptr, use_h ? hs : 0u, nullptr,
              dw ? dsm : (tiny ? b32 + kHeadD : nullptr), dw ? wsm : (tiny ? b32 + kHeadW : nullptr));
    if (b.trace && tid == 0) b.trace[3] = clock64();
}

}  // namespace

static_assert(kFusedSmemBytes <= 232448, "fused kernel shared memory exceeds 227 KB");
size_t fused_smem_bytes() { return offsetof(FusedSmem, btab); }  // the union (in-kernel merge scratch limit)

int fused_blocks_per_sm() {
    int nb = 0;
    cudaFuncSetAttribute(k_fused<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FusedSmem));
    cudaFuncSetAttribute(k_fused<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FusedSmem));
    cudaFuncSetAttribute(k_fused<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedSmemBytes);
    cudaFuncSetAttribute(k_fused<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedSmemBytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fused<false, true>, kFT, kFusedSmemBytes);
    return nb;
}

uint32_t fused_max_buckets() { return kMaxBuckets; }
uint32_t small_max_cap() { return kSmallCap; }

cudaError_t launch_small(const Bufs& b, const Cost& c, const StepArgs& a, const InlineStage* inl, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FusedSmem));
        cudaFuncSetAttribute(k_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FusedSmem));
        attr = true;
    }
    static const InlineStage kNone{};
    if (b.dbg)
        k_small<true><<<1, kFT, sizeof(FusedSmem), s>>>(b, c, a, inl ? *inl : kNone);
    else
        k_small<false><<<1, kFT, sizeof(FusedSmem), s>>>(b, c, a, inl ? *inl : kNone);
    return cudaGetLastError();
}

// The initial bucket table (before any step has measured the key distribution): every
// octave (ns, e) of v's bit length gets 2^min(7, e-1) buckets -- the fixed float-like
// buckets of 7 mantissa bits.  bt_update replaces it after the first step.
void fused_default_table(uint32_t vb, uint32_t* out) {
    uint32_t base = 0;
    for (uint32_t o = 0; o < kTabNB; o++) {
        const uint32_t e = o % 65u;
        if (e > vb) { out[o] = base; continue; }
        const uint32_t m = e >= 1u ? std::min(7u, e - 1u) : 0u;
        out[o] = base | ((e >= 1u ? e - 1u - m : 0u) << 16) | (m << 24);
        base += 1u << m;
    }
    out[kTabNB] = base;
    for (uint32_t o = kTabNB + 1; o < (uint32_t)kTabW; o++) out[o] = 0;
}

cudaError_t launch_fused(const Bufs& b, const Cost& c, const StepArgs& a, const InlineStage* inl, uint32_t grid,
                         cudaStream_t s) {
    static const InlineStage kNone{};
    Bufs bb = b;
    Cost cc = c;
    StepArgs aa = a;
    void* args[] = {&bb, &cc, &aa, const_cast<InlineStage*>(inl ? inl : &kNone)};
    const bool p2p = (a.flags & kStepP2P) != 0;
    const void* fn = p2p ? (b.dbg ? (const void*)k_fused<true, true> : (const void*)k_fused<false, true>)
                         : (b.dbg ? (const void*)k_fused<true, false> : (const void*)k_fused<false, false>);
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kFT), args, p2p ? kFusedSmemBytes : sizeof(FusedSmem), s);
}

}  // namespace lamps
