// lamps_dev.cuh -- device-side arithmetic of the LAMPS pass (sm_100a).
//
// Integer only.  Every quantity is exact: 64x64->128-bit products, sums kept
// in 128 bits, clamps at the end.  These functions are the GPU path's own
// implementation (closed forms, no loops); the CPU oracle under oracle/ is an
// independent transcription with explicit summation.
#pragma once
#include <cstdint>

namespace lamps {

typedef unsigned __int128 u128;

// Packed per-slot state word `sfc` (one u32 per slot in the SoA):
//   bits 0..2  state (FREE, READY, PAUSED_P, PAUSED_D, PAUSED_S)
//   bit  3     has_api     bit 4 starving (sticky)
//   bits 5..6  strategy    (label of the last pass / frozen at API entry)
//   bits 16..31 cnt        (StarvationCnt, Alg.1, saturating)
enum : uint32_t { ST_FREE = 0, ST_READY = 1, ST_PP = 2, ST_PD = 3, ST_PS = 4 };
enum : uint32_t { STR_P = 0, STR_D = 1, STR_S = 2, STR_NONE = 3 };
enum : uint32_t { EV_API_CALL = 1, EV_FINISHED = 2 };

__host__ __device__ __forceinline__ uint32_t sfc_state(uint32_t w) { return w & 7u; }
__host__ __device__ __forceinline__ uint32_t sfc_has(uint32_t w) { return (w >> 3) & 1u; }
__host__ __device__ __forceinline__ uint32_t sfc_starv(uint32_t w) { return (w >> 4) & 1u; }
__host__ __device__ __forceinline__ uint32_t sfc_strat(uint32_t w) { return (w >> 5) & 3u; }
__host__ __device__ __forceinline__ uint32_t sfc_cnt(uint32_t w) { return w >> 16; }
__host__ __device__ __forceinline__ uint32_t sfc_pack(uint32_t st, uint32_t has, uint32_t starv,
                                                      uint32_t strat, uint32_t cnt) {
    return st | (has << 3) | (starv << 4) | (strat << 5) | (cnt << 16);
}

constexpr uint32_t SFC_RAN = 1u << 7;  // admitted by the previous step (A0 pending)
// selective score update (R26): steps since the cached score was computed, and
// "segment changed" (set by submit / API return)
constexpr uint32_t SFC_AGE_SHIFT = 8, SFC_AGE_MASK = 0x7fu << SFC_AGE_SHIFT;
constexpr uint32_t SFC_DIRTY = 1u << 15;
constexpr uint32_t SFC_META = SFC_AGE_MASK | SFC_DIRTY;
__host__ __device__ __forceinline__ uint32_t sfc_age(uint32_t w) { return (w >> SFC_AGE_SHIFT) & 0x7fu; }
// rank policies (R25)
constexpr uint32_t POL_LAMPS = 0, POL_FCFS = 1, POL_SJF = 2, POL_SJF_TOTAL = 3;

// Per-handle constants, passed by value as a kernel parameter (constant bank).
struct Cost {
    uint64_t tau, A1, A2, S0, S1, c_other;
    uint64_t score_max;  // 2^SB - 1
    uint64_t nsbit;      // 1 << (SB + IB): the key's "not starving" bit
    uint32_t SH, lgB, B, T;
    uint32_t SB, IB, cap_mask, cap;
    uint32_t fast;       // constants satisfy the 64-bit fast-path bounds (host-checked)
    uint32_t policy;     // POL_* (R25)
    uint32_t interval;   // selective score update interval (R26)
    uint32_t cache;      // policy == LAMPS && interval > 1: the score cache is in use
    uint32_t lean;       // fast && B >= 2 && LAMPS policy && !cache: score_lean applies (per-slot check)
};

// Per-slot bound of the fast path (see strategy_score_fast): ctx+pre+resp+post < 2^20.
constexpr uint64_t kFastCtxLimit = 1ull << 20;

// Pool SoA (device pointers into the workspace), 16-byte aligned, padded.
struct Pool {
    uint32_t *sfc, *ctx, *pre, *api, *resp, *post, *pend;
    uint32_t* stamp;  // step number at which the slot was last admitted
    uint32_t *sclo, *schi;  // cached score (R26), low / high word
    uint32_t stride;  // words between consecutive SoA arrays (ctx == sfc + stride, ...)
};

__device__ __forceinline__ uint64_t sat64(u128 x) {
    return (uint64_t)(x >> 64) ? ~0ull : (uint64_t)x;
}

// ceil(n / B), B = 2^lgB (n < 2^40 so no overflow)
__device__ __forceinline__ uint64_t blk(uint64_t n, const Cost& c) {
    return (n + c.B - 1) >> c.lgB;
}

// T_fwd(x) = (A1 x + A2 x^2) >> SH  (R1; prefill shape k1 n^2 d)
__device__ __forceinline__ uint64_t t_fwd(uint64_t x, const Cost& c) {
    u128 sq = (u128)x * x;
    u128 v = (u128)c.A1 * x + (u128)c.A2 * sq;
    return sat64(v >> c.SH);
}

// T_swap(x) = x ? (S0 + S1 x) >> SH : 0  (R2)
__device__ __forceinline__ uint64_t t_swap(uint64_t x, const Cost& c) {
    if (x == 0) return 0;
    return sat64(((u128)c.S0 + (u128)c.S1 * x) >> c.SH);
}

// Eq. (1)-(3), M dropped (R5); C_i = ctx + pre,
// C_batch = C_i + C_other (R4).  Returns the first-min strategy in P, D, S order.
__device__ __forceinline__ uint32_t strategy_of(uint64_t ctx, uint64_t pre, uint64_t api,
                                                const Cost& c, uint64_t* wp_o = nullptr,
                                                uint64_t* wd_o = nullptr,
                                                uint64_t* ws_o = nullptr) {
    const uint64_t ci = ctx + pre;
    const uint64_t cb = ci + c.c_other;
    const uint64_t wp = sat64((u128)api * ci);
    const uint64_t wd = sat64((u128)t_fwd(ci, c) * cb);
    const uint64_t ws = sat64(((u128)t_swap(ci, c) * cb) << 1);
    if (wp_o) { *wp_o = wp; *wd_o = wd; *ws_o = ws; }
    return (wp <= wd && wp <= ws) ? STR_P : (wd <= ws ? STR_D : STR_S);
}

// F(n) = sum_{j=1..n} ceil(j/B) = B Q(Q+1)/2 + R(Q+1), n = Q B + R (closed form)
__device__ __forceinline__ u128 ramp_prefix(uint64_t n, const Cost& c) {
    const uint64_t Q = n >> c.lgB, R = n & (c.B - 1);
    const u128 q = (u128)Q * (Q + 1);
    return ((q >> 1) << c.lgB) + (u128)R * (Q + 1);
}

// Memory-over-time score, readings R7-R10:
// pending rectangle + pre-API ramp + API phase by strategy + post-API ramp,
// in KV blocks x ticks, clamped at 2^SB - 1.
__device__ __forceinline__ uint64_t score_of(uint64_t ctx, uint64_t pre, uint64_t api,
                                             uint64_t resp, uint64_t post, uint64_t pend,
                                             uint32_t has, uint32_t strat, const Cost& c) {
    const uint64_t ci = ctx + pre;
    u128 s = (u128)blk(ctx, c) * pend;
    s += (u128)c.tau * (ramp_prefix(ci, c) - ramp_prefix(ctx, c));
    if (has) {
        const uint64_t cr = ci + resp;
        if (strat == STR_P) {
            s += (u128)blk(ci, c) * api;
        } else if (strat == STR_D) {
            s += (u128)blk(cr, c) * t_fwd(cr, c);
        } else if (strat == STR_S) {
            s += ((u128)blk(ci, c) * t_swap(ci, c)) << 1;
        }
        s += (u128)c.tau * (ramp_prefix(cr + post, c) - ramp_prefix(cr, c));
    }
    return s > (u128)c.score_max ? c.score_max : (uint64_t)s;
}

// ---------------------------------------------------------------------------
// Fast path: 32x32->64 products, no overflow checks.  The host sets
// Cost::fast only when A1, A2, S0, S1, tau < 2^32, c_other < 2^26 and, for every
// context value c < kFastCtxLimit (2^20 tokens), it has proven with exact
// 128-bit arithmetic that every product and every sum below stays < 2^63 (see
// fast_bounds_ok in lamps_api.cu); the kernel
// takes this path for a slot iff ctx + pre + resp + post < 2^20.  Under those
// bounds the results equal the exact ones (no clamp can trigger except the
// final min with 2^SB - 1, which is applied).
// ---------------------------------------------------------------------------
// (fast path: A1, A2, S0, S1, tau < 2^32 and every context value x < 2^20, host-checked)
__device__ __forceinline__ uint64_t wide32(uint32_t a, uint32_t b) { return (uint64_t)a * b; }
// 32-bit a times a 64-bit b < 2^40
__device__ __forceinline__ uint64_t mul32x40(uint32_t a, uint64_t b) {
    return wide32(a, (uint32_t)b) + (wide32(a, (uint32_t)(b >> 32)) << 32);
}
__device__ __forceinline__ uint64_t t_fwd_fast(uint32_t x, const Cost& c) {
    return (wide32((uint32_t)c.A1, x) + mul32x40((uint32_t)c.A2, wide32(x, x))) >> c.SH;
}
__device__ __forceinline__ uint64_t t_swap_fast(uint32_t x, const Cost& c) {
    return x ? (c.S0 + wide32((uint32_t)c.S1, x)) >> c.SH : 0ull;
}
// F(n) = sum_{j=1..n} ceil(j/B) = B Q(Q+1)/2 + R(Q+1), n = Q B + R
// = (Q+1)(QB + 2R)/2 = (Q+1)(n+R)/2 (the product is even: QB even for B >= 2, Q(Q+1) for B = 1)
__device__ __forceinline__ uint64_t ramp_fast(uint32_t n, const Cost& c) {
    const uint32_t Q = n >> c.lgB, R = n & (c.B - 1u);
    return wide32(Q + 1u, n + R) >> 1;
}

// strategy (A1) and score (A2) of one READY slot on the fast path
__device__ __forceinline__ uint32_t strategy_score_fast(uint32_t ctx, uint32_t pre, uint32_t api,
                                                        uint32_t resp, uint32_t post, uint32_t pend,
                                                        uint32_t has, const Cost& c, uint64_t* score,
                                                        uint64_t* wp_o, uint64_t* wd_o, uint64_t* ws_o) {
    const uint32_t tau = (uint32_t)c.tau;
    const uint32_t ci = ctx + pre;
    uint64_t s = wide32((ctx + c.B - 1u) >> c.lgB, pend) + mul32x40(tau, ramp_fast(ci, c) - ramp_fast(ctx, c));
    uint32_t strat = STR_NONE;
    uint64_t wp = 0, wd = 0, ws = 0;
    if (has) {
        const uint32_t cb = ci + (uint32_t)c.c_other;  // < 2^27
        const uint64_t tf = t_fwd_fast(ci, c), ts = t_swap_fast(ci, c);
        wp = wide32(api, ci);
        wd = tf * cb;
        ws = (ts * cb) << 1;
        strat = (wp <= wd && wp <= ws) ? STR_P : (wd <= ws ? STR_D : STR_S);
        const uint32_t bci = (ci + c.B - 1u) >> c.lgB;
        const uint32_t cr = ci + resp;
        uint64_t a;
        if (strat == STR_P) a = wide32(bci, api);
        else if (strat == STR_D) a = t_fwd_fast(cr, c) * ((cr + c.B - 1u) >> c.lgB);
        else a = (ts * bci) << 1;
        s += a + mul32x40(tau, ramp_fast(cr + post, c) - ramp_fast(cr, c));
    }
    *score = s > c.score_max ? c.score_max : s;
    *wp_o = wp; *wd_o = wd; *ws_o = ws;
    return strat;
}

// ---------------------------------------------------------------------------
// Lean fast path (the fused kernel's score phase): the same values as
// strategy_score_fast, computed branch-free with fewer instructions.  Valid
// when Cost::lean (fast bounds, B >= 2, LAMPS policy, no score cache) and the
// slot passes the per-slot fast check.  rp / pp = resp / post if has_api, else 0.
//   * F(n) = (Q+1)(n+R)/2 = (Q+1) * ((n+R) >> 1): n+R = QB+2R is even for even B
//   * the two ramps share one multiply by tau:
//       tau*(F(ci)-F(ctx)) + tau*(F(ce)-F(cr)) = tau*((F(ci)+F(ce)) - (F(ctx)+F(cr)))
//     (without an API rp = pp = 0, so ce = cr = ci and the second ramp vanishes)
//   * the three API-phase areas are all formed and the argmin selects one (no
//     divergence between lanes of different strategies); each is bounded by the
//     host's proof (fast_bounds_ok bounds the largest of the three)
// a*b for a < 2^32 and any b whose product stays < 2^64 (two IMADs)
__device__ __forceinline__ uint64_t mul32x64(uint32_t a, uint64_t b) {
    return wide32(a, (uint32_t)b) + (wide32(a, (uint32_t)(b >> 32)) << 32);
}
// SHC / LGC: the fixed-point shift SH and log2 B as compile-time constants (0: the runtime
// values); the fused kernel instantiates the common (16, 4) so the 64-bit shifts are immediate
template <uint32_t SHC = 0, uint32_t LGC = 0>
__device__ __forceinline__ uint32_t score_lean(uint32_t ctx, uint32_t pre, uint32_t api, uint32_t rp, uint32_t pp,
                                               uint32_t pend, uint32_t has, const Cost& c, uint64_t& sc,
                                               uint64_t& wp, uint64_t& wd, uint64_t& ws) {
    const uint32_t lg = LGC ? LGC : c.lgB, Bm1 = (1u << lg) - 1u;
    const uint32_t SHv = SHC ? SHC : c.SH;
    const uint32_t ci = ctx + pre, cr = ci + rp, ce = cr + pp;
    auto F = [&](uint32_t n) { return wide32((n >> lg) + 1u, (n + (n & Bm1)) >> 1); };
    const uint64_t D = (F(ci) + F(ce)) - (F(ctx) + F(cr));
    uint64_t s = wide32((ctx + Bm1) >> lg, pend) + mul32x64((uint32_t)c.tau, D);
    const uint32_t A1 = (uint32_t)c.A1, A2 = (uint32_t)c.A2;
    const uint64_t tf = (wide32(A1, ci) + mul32x64(A2, wide32(ci, ci))) >> SHv;   // T_fwd(C_i)
    const uint64_t ts = ci ? (c.S0 + wide32((uint32_t)c.S1, ci)) >> SHv : 0ull;  // T_swap(C_i)
    const uint32_t cb = ci + (uint32_t)c.c_other;
    wp = wide32(api, ci);           // Eq. (1)
    wd = mul32x64(cb, tf);          // Eq. (2)
    ws = mul32x64(cb, ts) << 1;     // Eq. (3)
    const uint32_t strat = (wp <= wd && wp <= ws) ? STR_P : (wd <= ws ? STR_D : STR_S);
    const uint32_t bci = (ci + Bm1) >> lg, bcr = (cr + Bm1) >> lg;
    const uint64_t tfr = (wide32(A1, cr) + mul32x64(A2, wide32(cr, cr))) >> SHv;  // T_fwd(C_i + resp)
    const uint64_t aP = wide32(bci, api), aD = mul32x64(bcr, tfr), aS = mul32x64(bci, ts) << 1;
    // branch-free selection (predicated moves, no divergence between strategies)
    uint64_t aX = strat == STR_D ? aD : aS;
    aX = strat == STR_P ? aP : aX;
    s += has ? aX : 0ull;
    sc = s > c.score_max ? c.score_max : s;
    if (!has) wp = wd = ws = 0;
    return has ? strat : STR_NONE;
}

// Lanes of the warp holding the same 8-bit digit d (0..255; 256 = empty lane),
// from 9 ballots: a multisplit that avoids __match_any_sync (measured as the
// dominant latency of the in-SM ranking on B200).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
    const bool valid = d < 256u;
    const uint32_t vm = __ballot_sync(0xffffffffu, valid);
    uint32_t m = valid ? vm : ~vm;
#pragma unroll
    for (int bit = 0; bit < 8; bit++) {
        const uint32_t on = (d >> bit) & 1u;
        const uint32_t bb = __ballot_sync(0xffffffffu, on);
        m &= on ? bb : ~bb;
    }
    return m;
}

}  // namespace lamps
