// step_dev.cuh -- device bodies shared by the multi-kernel path (K1, K3) and the
// fused cooperative step kernel: scoring of a group of four slots (A0 default
// update, A1, A2, A3 + key) and the single-CTA admission (A5).
#pragma once
#include "lamps_internal.h"

namespace lamps {

struct DevEvent {
    unsigned long long id;
    uint32_t kind, reserved;
};

// A0 for one engine event about a request admitted by the previous step (K0, or the
// fused kernel's prologue): API_CALL routes it to P/D/S by the label of the ranking pass
// (Alg.1) and resets its counter unless starving; FINISHED frees
// the slot.  The token of this iteration is counted (SFC_RAN).
__device__ __forceinline__ void apply_event(const Pool& P, const Cost& c, const DevEvent E) {
    const uint32_t s = (uint32_t)E.id & c.cap_mask;
    const uint32_t w = P.sfc[s];
    if (E.kind == EV_FINISHED) {
        P.sfc[s] = 0u;
        return;
    }
    const uint32_t ctx = P.ctx[s] + ((w & SFC_RAN) ? 1u : 0u);  // this iteration's token
    P.ctx[s] = ctx;
    P.pre[s] = 0u;
    P.pend[s] = 0u;
    // routed by the label of the ranking pass that admitted it (Alg.1, R11); a
    // request never ranked with an API ahead takes the argmin at C_i = ctx
    const uint32_t lab = sfc_strat(w);
    const uint32_t st = lab != STR_NONE ? lab : strategy_of(ctx, 0, P.api[s], c);
    const uint32_t starv = sfc_starv(w);
    P.sfc[s] = sfc_pack(ST_PP + st, sfc_has(w), starv, st, starv ? sfc_cnt(w) : 0u) | (w & SFC_META);
}

// Intake of one new request (Alg.1): READY, ctx = prompt, the prefill owed
// T_fwd(prompt), a new segment (k_submit, or the fused kernel's prologue).
__device__ __forceinline__ void apply_submit(const Pool& P, const Cost& c, const SubmitRec r) {
    const uint32_t s = r.slot;
    P.ctx[s] = r.ctx;
    P.pre[s] = r.pre;
    P.api[s] = r.api;
    P.resp[s] = r.resp;
    P.post[s] = r.post;
    const uint64_t f = t_fwd(r.ctx, c);  // prefill owed
    P.pend[s] = f > 0xffffffffull ? 0xffffffffu : (uint32_t)f;
    P.sfc[s] = sfc_pack(ST_READY, r.has, 0, STR_NONE, 0) | SFC_DIRTY;  // a new segment (R26)
}

// API return of one PAUSED request (Alg.1, R10): ctx grows by the actual
// response; the owed prefill / swap-in by its handling strategy; the next segment's
// predictions; READY (K_api_return, or the fused kernel's prologue).
__device__ __forceinline__ void apply_return(const Pool& P, const Cost& c, const ReturnRec r) {
    const uint32_t s = r.slot;
    const uint32_t w = P.sfc[s];
    const uint64_t ci = P.ctx[s];
    const uint64_t c1 = ci + r.actual;
    const uint64_t f1 = t_fwd(c1, c), f0 = t_fwd(ci, c);
    const uint64_t inc = f1 - f0;  // T_fwd is non-decreasing
    uint64_t owed;
    const uint32_t st = sfc_state(w);
    if (st == ST_PD) {
        owed = f1;  // discarded: recompute everything
    } else if (st == ST_PS) {
        const uint64_t sw = t_swap(ci, c);
        owed = sw + inc < sw ? ~0ull : sw + inc;  // swap-in + prefill of the response
    } else {
        owed = inc;  // preserved: prefill of the response
    }
    P.pend[s] = owed > 0xffffffffull ? 0xffffffffu : (uint32_t)owed;
    P.ctx[s] = (uint32_t)c1;
    P.pre[s] = r.pre;
    P.api[s] = r.api;
    P.resp[s] = r.resp;
    P.post[s] = r.post;
    // RAN clear; a new segment: its score is recomputed at the next step (R26)
    P.sfc[s] = sfc_pack(ST_READY, r.has, sfc_starv(w), sfc_strat(w), sfc_cnt(w)) | (w & SFC_AGE_MASK) | SFC_DIRTY;
}

// block-wide exclusive scans (all NT threads call; totals in *tot)
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* sh_warp, uint32_t* tot) {
    constexpr int NW = NT / 32;
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) sh_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < (unsigned)NW ? sh_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= (unsigned)o) t += y;
        }
        if (lane < (unsigned)NW) sh_warp[lane] = t;
    }
    __syncthreads();
    const uint32_t before = w ? sh_warp[w - 1] : 0u;
    *tot = sh_warp[NW - 1];
    __syncthreads();
    return before + x - v;
}

template <int NT>
__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v,
                                                                  unsigned long long* sh_warp,
                                                                  unsigned long long* tot) {
    constexpr int NW = NT / 32;
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) sh_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long t = lane < (unsigned)NW ? sh_warp[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= (unsigned)o) t += y;
        }
        if (lane < (unsigned)NW) sh_warp[lane] = t;
    }
    __syncthreads();
    const unsigned long long before = w ? sh_warp[w - 1] : 0ull;
    *tot = sh_warp[NW - 1];
    __syncthreads();
    return before + x - v;
}

// Exclusive scan of arr[0..L) in shared memory by all NT threads, L <= R*NT.
// Raking: thread t owns the R consecutive words [t*R, t*R+R) (R odd => the lanes
// of a warp hit distinct banks), sums them serially, one warp scan of the thread
// sums, one scan of the warp sums, then rewrites its words.  ~2R shared-memory
// accesses + 10 shuffles per thread.  Returns the total; `add` (optional)
// receives arr[j] + exclusive(j).
template <int NT, int R>
__device__ __forceinline__ uint32_t smem_excl_scan(uint32_t* arr, uint32_t L, uint32_t* w32,
                                                   uint32_t* add = nullptr) {
    // the R words are read twice from shared memory (sum, then rewrite) instead of being
    // held in registers: no spills for large R
    constexpr int NW = NT / 32;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t j0 = threadIdx.x * (uint32_t)R;
    const uint32_t jn = j0 < L ? min((uint32_t)R, L - j0) : 0u;  // words of this thread
    uint32_t s = 0;
#pragma unroll 4
    for (uint32_t r = 0; r < jn; r++) s += arr[j0 + r];
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) w32[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t t = lane < (uint32_t)NW ? w32[lane] : 0u;
        uint32_t y = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= (uint32_t)o) y += z;
        }
        if (lane < (uint32_t)NW) w32[lane] = y - t;
        if (lane == NW - 1) w32[NW] = y;
    }
    __syncthreads();
    uint32_t run = w32[warp] + x - s;
    const uint32_t total = w32[NW];
#pragma unroll 4
    for (uint32_t r = 0; r < jn; r++) {
        const uint32_t v = arr[j0 + r];
        arr[j0 + r] = run;
        if (add) add[j0 + r] += run;
        run += v;
    }
    __syncthreads();
    return total;
}

// Baseline rank keys (R25): FCFS 0 (order = id), SJF the remaining iterations of
// the segment (decode tokens + owed prefill / swap-in, ceil(pending / tau): "a
// post-API part of length 2 (including recomputation)"), SJF by total
// length + the API duration in iterations.
__device__ __forceinline__ uint64_t policy_score(const Cost& c, uint32_t has, uint32_t pre, uint32_t post,
                                                 uint32_t api, uint32_t pend) {
    uint64_t v = 0;
    if (c.policy == POL_SJF || c.policy == POL_SJF_TOTAL)
        v = (uint64_t)pre + (has ? post : 0u) + ((uint64_t)pend + c.tau - 1u) / c.tau;
    if (c.policy == POL_SJF_TOTAL && has) v += ((uint64_t)api + c.tau - 1u) / c.tau;
    return v < c.score_max ? v : c.score_max;
}

// A1 + A2 of one READY slot under the configured policy and the selective score
// update (R25, R26): a cached (strategy, score) is reused unless the segment
// changed or it is `interval` steps old.  meta = the slot's new age / dirty bits.
__device__ __forceinline__ uint32_t strategy_score(const Pool& P, const Cost& c, uint32_t slot, uint32_t w,
                                                   uint32_t ctx, uint32_t pre, uint32_t api, uint32_t resp,
                                                   uint32_t post, uint32_t pend, uint64_t& sc, uint64_t& wp,
                                                   uint64_t& wd, uint64_t& ws, uint32_t& meta) {
    if (c.cache) {
        const uint32_t age = sfc_age(w);
        if (!(w & SFC_DIRTY) && age + 1u < c.interval) {
            sc = ((uint64_t)P.schi[slot] << 32) | P.sclo[slot];
            wp = wd = ws = 0;
            meta = (age + 1u) << SFC_AGE_SHIFT;
            return sfc_strat(w);
        }
    }
    const uint32_t has = sfc_has(w);
    uint32_t strat;
    // fast path iff the slot's lengths sum below 2^20; checked in 32 bits: all four below
    // 2^18 (so the sum cannot wrap) and the sum below 2^20 (a rarer slot with one length in
    // [2^18, 2^20) takes the exact path, which gives the same result)
    const uint32_t rp = has ? resp : 0u, pp = has ? post : 0u;
    if (c.fast && (ctx | pre | rp | pp) < (1u << 18) && ctx + pre + rp + pp < (uint32_t)kFastCtxLimit) {
        strat = strategy_score_fast(ctx, pre, api, resp, post, pend, has, c, &sc, &wp, &wd, &ws);
    } else {
        wp = wd = ws = 0;
        strat = STR_NONE;
        if (has) strat = strategy_of(ctx, pre, api, c, &wp, &wd, &ws);
        sc = score_of(ctx, pre, api, resp, post, pend, has, strat, c);
    }
    if (c.policy != POL_LAMPS) sc = policy_score(c, has, pre, post, api, pend);
    if (c.cache) {
        P.sclo[slot] = (uint32_t)sc;
        P.schi[slot] = (uint32_t)(sc >> 32);
    }
    meta = 0;
    return strat;
}

// One group of four consecutive slots g*4..g*4+3 (128-bit loads of the SoA).
// A0 (fused): slots admitted by the previous step (SFC_RAN) generated one
// token: ctx += 1, pre_rem -= 1 (floor 0), pending = 0.
// A1 strategy argmin of Eq. (1)-(3), A2 score, A3 starvation, counter +1
// (reset by admission), 64-bit key.  Returns the number of keys written to key[].
template <bool DBG>
__device__ __forceinline__ uint32_t score_group(const Pool& P, const Cost& c, uint32_t id_base_mod,
                                                unsigned long long* dbg, uint32_t g, uint64_t (&key)[4],
                                                unsigned long long& pinned) {
    const uint4 w4 = __ldcs(reinterpret_cast<const uint4*>(P.sfc) + g);
    const uint4 cx = __ldcs(reinterpret_cast<const uint4*>(P.ctx) + g);
    const uint4 pr = __ldcs(reinterpret_cast<const uint4*>(P.pre) + g);
    const uint4 ap = __ldcs(reinterpret_cast<const uint4*>(P.api) + g);
    const uint4 rs = __ldcs(reinterpret_cast<const uint4*>(P.resp) + g);
    const uint4 po = __ldcs(reinterpret_cast<const uint4*>(P.post) + g);
    const uint4 pe = __ldcs(reinterpret_cast<const uint4*>(P.pend) + g);
    uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
    uint32_t cv[4] = {cx.x, cx.y, cx.z, cx.w};
    uint32_t prv[4] = {pr.x, pr.y, pr.z, pr.w};
    uint32_t pev[4] = {pe.x, pe.y, pe.z, pe.w};
    const uint32_t apv[4] = {ap.x, ap.y, ap.z, ap.w};
    const uint32_t rsv[4] = {rs.x, rs.y, rs.z, rs.w};
    const uint32_t pov[4] = {po.x, po.y, po.z, po.w};
    bool ran = false;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (wv[j] & SFC_RAN) {
            ran = true;
            cv[j] += 1u;
            prv[j] = prv[j] ? prv[j] - 1u : 0u;
            pev[j] = 0u;
        }
    }
    if (ran) {
        reinterpret_cast<uint4*>(P.ctx)[g] = make_uint4(cv[0], cv[1], cv[2], cv[3]);
        reinterpret_cast<uint4*>(P.pre)[g] = make_uint4(prv[0], prv[1], prv[2], prv[3]);
        reinterpret_cast<uint4*>(P.pend)[g] = make_uint4(pev[0], pev[1], pev[2], pev[3]);
    }
    const uint32_t key_top = c.SB + c.IB;
    uint32_t nk = 0;
    bool any_ready = false;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint32_t w = wv[j];
        const uint32_t st = sfc_state(w);
        if (st == ST_PP) pinned += blk(cv[j], c);
        key[j] = 0;
        if (st != ST_READY) continue;
        any_ready = true;
        const uint32_t has = sfc_has(w);
        const uint32_t slot = 4u * g + (uint32_t)j;
        uint64_t wp, wd, ws, sc;
        uint32_t meta;
        const uint32_t strat = strategy_score(P, c, slot, w, cv[j], prv[j], apv[j], rsv[j], pov[j], pev[j], sc,
                                              wp, wd, ws, meta);
        const uint32_t cnt = sfc_cnt(w);
        const uint32_t starv = sfc_starv(w) | (cnt >= c.T ? 1u : 0u);
        const uint32_t cnt2 = cnt < 65535u ? cnt + 1u : 65535u;
        wv[j] = sfc_pack(ST_READY, has, starv, strat, cnt2) | meta;
        const uint32_t idoff = (slot - id_base_mod) & c.cap_mask;
        // keys are packed to the front of key[] in slot order (predicated, no dynamic index)
        const uint64_t k = ((uint64_t)(starv ^ 1u) << key_top) | (sc << c.IB) | idoff;
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (q == (int)nk) key[q] = k;
        nk++;
        if (DBG) {
            unsigned long long* d = dbg + 4ull * slot;
            d[0] = wp; d[1] = wd; d[2] = ws; d[3] = sc;
        }
    }
    if (any_ready) reinterpret_cast<uint4*>(P.sfc)[g] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    return nk;
}

// One slot given its seven SoA words (A0 default update already applied by the
// caller).  Returns true and the key if the slot is READY; updates *w (sfc).
template <bool DBG>
__device__ __forceinline__ bool score_slot(const Pool& P, const Cost& c, uint32_t id_base_mod,
                                           unsigned long long* dbg, uint32_t slot, uint32_t& w, uint32_t ctx,
                                           uint32_t pre, uint32_t api, uint32_t resp, uint32_t post,
                                           uint32_t pend, uint64_t& key) {
    const uint32_t has = sfc_has(w);
    uint64_t wp, wd, ws, sc;
    uint32_t meta;
    const uint32_t strat = strategy_score(P, c, slot, w, ctx, pre, api, resp, post, pend, sc, wp, wd, ws, meta);
    const uint32_t cnt = sfc_cnt(w);
    const uint32_t starv = sfc_starv(w) | (cnt >= c.T ? 1u : 0u);
    w = sfc_pack(ST_READY, has, starv, strat, cnt < 65535u ? cnt + 1u : 65535u) | meta;
    key = (starv ? 0ull : c.nsbit) | (sc << c.IB) | ((slot - id_base_mod) & c.cap_mask);
    if (DBG) {
        unsigned long long* d = dbg + 4ull * slot;
        d[0] = wp; d[1] = wd; d[2] = ws; d[3] = sc;
    }
    return true;
}

// score_slot out of line: the fused kernel's score phase inlines only score_lean and
// calls this for the slots (or configurations) the lean path does not cover
// (exact 128-bit path, baseline policies, score cache).
struct ColdOut {
    unsigned long long key;
    uint32_t w;
};
template <bool DBG>
__device__ __noinline__ ColdOut score_slot_cold(const Pool& P, const Cost& c, uint32_t id_base_mod,
                                                unsigned long long* dbg, uint32_t slot, uint32_t w, uint32_t ctx,
                                                uint32_t pre, uint32_t api, uint32_t resp, uint32_t post,
                                                uint32_t pend) {
    uint64_t key = 0;
    (void)score_slot<DBG>(P, c, id_base_mod, dbg, slot, w, ctx, pre, api, resp, post, pend, key);
    return ColdOut{key, w};
}

// The step summary into mapped host memory (one thread, after the Ctl fields are final).
// (three 16-B stores: each store to mapped memory is its own transaction over the host link)
__device__ __forceinline__ void publish_host_result(const Bufs& b) {
    const Ctl* ctl = b.ctl;
    HostRes* r = b.hres;
    const unsigned long long bu = *(volatile const unsigned long long*)&ctl->budget_used;
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(&r->n_elig), "l"((unsigned long long)ctl->n_elig_out),
                 "l"((unsigned long long)ctl->pinned_out) : "memory");
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(&r->budget), "l"((unsigned long long)ctl->budget), "l"(bu)
                 : "memory");
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(&r->n_admitted), "r"(ctl->n_admitted),
                 "r"(ctl->n_preempted), "r"(ctl->blocked_head), "r"(ctl->final_buf) : "memory");
}
static_assert(offsetof(HostRes, pinned) == 8 && offsetof(HostRes, budget) == 16 && offsetof(HostRes, budget_used) == 24 &&
                  offsetof(HostRes, n_admitted) == 32 && offsetof(HostRes, final_buf) == 44,
              "publish_host_result's vector stores follow HostRes");

// A5 admission by one 1024-thread CTA over the ranked keys (see k_admit).
struct AdmitSmem {
    unsigned long long w64[32];
    uint32_t w32[32];
};

// htab (optional, shared memory, >= 2 * max_batch u32 entries, power of two hsize):
// admitted slots are inserted into an open-addressing table and the preempted check
// probes it, instead of stamping P.stamp and re-reading it from global memory.
__device__ __forceinline__ uint32_t slot_hash(uint32_t s, uint32_t mask) { return (s * 2654435761u >> 7) & mask; }

__device__ __forceinline__ void admit_cta(const Bufs& b, const Cost& c, const StepArgs& a,
                                          const uint64_t* keys, uint64_t n_elig, uint64_t pinned,
                                          AdmitSmem& sm, uint32_t* htab = nullptr, uint32_t hsize = 0,
                                          unsigned long long* tr = nullptr, const uint32_t* dsm = nullptr,
                                          const uint32_t* wsm = nullptr) {
#define ATRACE(k) do { if (tr && threadIdx.x == 0) tr[k] = clock64(); } while (0)
    constexpr int NT = 1024;
    constexpr uint32_t kEmpty = 0xffffffffu;
    Ctl* ctl = b.ctl;
    const Pool& P = b.pool;
    const uint32_t tid = threadIdx.x;
    const uint32_t n_prev = ctl->n_admitted;
    const uint64_t budget = a.kv_total > pinned ? a.kv_total - pinned : 0ull;
    uint64_t Wn = n_elig < a.max_batch ? n_elig : a.max_batch;
    if (budget < Wn) Wn = budget;
    const uint64_t idmask = (1ull << c.IB) - 1ull;
    const uint32_t par = a.parity, prev = par ^ 1u;
    const uint32_t hmask = hsize - 1u;
    ATRACE(0);
    if (htab)
        for (uint32_t i = tid; i < hsize; i += NT) htab[i] = kEmpty;

    // prefetch the previous admitted list (independent of the ranking)
    uint32_t pslot = 0, pw = 0;
    uint64_t pid = 0;
    if (tid < n_prev) {
        pslot = b.adm_slot[prev][tid];
        pid = b.adm_id[prev][tid];
        pw = P.sfc[pslot];
    }
    unsigned long long carry = 0;
    uint32_t cut = 0;
    for (uint32_t base = 0; base < Wn; base += NT) {
        const uint32_t k = base + tid;
        uint32_t slot = 0, w = 0;
        uint64_t idoff = 0;
        unsigned long long dem = 0;
        if (k < Wn) {
            idoff = keys[k] & idmask;
            slot = (uint32_t)((a.id_base + idoff) & c.cap_mask);
            if (dsm) {  // demand and state word staged on chip by the range sort
                dem = dsm[k];
                w = wsm[k];
            } else {
                const uint32_t ctx = P.ctx[slot];
                w = P.sfc[slot];
                dem = blk((uint64_t)ctx + 1u, c);
            }
        }
        if (base == 0) ATRACE(1);
        unsigned long long tot;
        const unsigned long long incl = carry + block_excl_scan_u64<NT>(dem, sm.w64, &tot) + dem;
        const bool fit = k < Wn && incl <= budget;
        const uint32_t nfit = (uint32_t)__syncthreads_count(fit);
        if (base == 0) ATRACE(2);
        if (fit) {
            b.adm_slot[par][k] = slot;
            b.adm_id[par][k] = a.id_base + idoff;
            b.adm_strat[par][k] = (uint8_t)sfc_strat(w);
#ifndef LAMPS_NO_HOSTRES  // (measurement-only build: the mapped host writes left out)
            b.h_adm_id[k] = a.id_base + idoff;  // the host's copy (mapped memory)
            b.h_adm_strat[k] = (uint8_t)sfc_strat(w);
#endif
            if (htab) {
                uint32_t h = slot_hash(slot, hmask);
                while (atomicCAS(&htab[h], kEmpty, slot) != kEmpty) h = (h + 1u) & hmask;
            } else {
                P.stamp[slot] = a.step;
            }
            P.sfc[slot] = (w & 0xffffu) | SFC_RAN;  // StarvationCnt <- 0; runs this iteration
            if (k == base + nfit - 1) ctl->budget_used = incl;
        }
        cut += nfit;
        carry += tot;
        const uint32_t chunk = (uint32_t)min((uint64_t)NT, Wn - base);
        if (nfit < chunk) break;
    }
    if (tid == 0 && cut == 0) ctl->budget_used = 0;
    __syncthreads();
    ATRACE(3);

    // preempted: admitted last step, still READY, not admitted now (previous rank order)
    uint32_t npre = 0;
    for (uint32_t base = 0; base < n_prev; base += NT) {
        const uint32_t k = base + tid;
        uint32_t f = 0;
        uint64_t id = 0;
        if (k < n_prev) {
            const uint32_t s = base ? b.adm_slot[prev][k] : pslot;
            const uint32_t w = base ? P.sfc[s] : pw;
            id = base ? b.adm_id[prev][k] : pid;
            bool now;
            if (htab) {
                uint32_t h = slot_hash(s, hmask), v;
                while ((v = htab[h]) != s && v != kEmpty) h = (h + 1u) & hmask;
                now = v == s;
            } else {
                now = P.stamp[s] == a.step;
            }
            f = (sfc_state(w) == ST_READY && !now) ? 1u : 0u;
        }
        uint32_t tot;
        const uint32_t pos = block_excl_scan_u32<NT>(f, sm.w32, &tot);
        if (f) {
            b.pre_id[npre + pos] = id;
#ifndef LAMPS_NO_HOSTRES
            b.h_pre_id[npre + pos] = id;
#endif
        }
        npre += tot;
    }
    if (tid == 0) {
        ctl->n_admitted = cut;
        ctl->n_preempted = npre;
        ctl->blocked_head = (n_elig > 0 && cut == 0) ? 1u : 0u;
        ctl->budget = budget;
        ctl->n_elig_out = n_elig;
        ctl->pinned_out = pinned;
        ctl->n_elig = 0;  // accumulators of the next step
        ctl->pinned = 0;
#ifndef LAMPS_NO_HOSTRES
        publish_host_result(b);
#endif
    }
    ATRACE(4);
#undef ATRACE
}

}  // namespace lamps
