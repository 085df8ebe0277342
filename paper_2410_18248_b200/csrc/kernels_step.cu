// kernels_step.cu -- A0 events (K0), A1-A3 strategy/score/key (K1),
// A5 admission (K3) and the ingest scatter kernels.  sm_100a, integer only.
#include "lamps_internal.h"

namespace lamps {

namespace {

struct DevEvent {
    unsigned long long id;
    uint32_t kind, reserved;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// block-wide exclusive scan of one u32 per thread (NT threads); returns total in *tot
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* sh_warp,
                                                        uint32_t* tot) {
    constexpr int NW = NT / 32;
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
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
        if (lane < (unsigned)NW) sh_warp[lane] = t;  // inclusive warp prefix
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
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
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

// ---------------------------------------------------------------------------
// A0 -- the previously admitted batch ran one iteration: every
// admitted slot carries SFC_RAN (set by K3).  Slots without an event get
// ctx += 1, pre_rem -= 1 (floor 0), pending = 0 inside K1 (fused, no extra pass
// over memory).  K0 handles only the engine's events and runs only when there
// are any: API_CALL routes the request to P/D/S by argmin waste at C_i = ctx
// (Alg.1) and resets its counter unless starving;
// FINISHED frees the slot.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_events(Bufs b, Cost c, StepArgs a) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.n_ev) return;
    const Pool& P = b.pool;
    const DevEvent E = static_cast<const DevEvent*>(b.events)[e];
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
    const uint32_t st = strategy_of(ctx, 0, P.api[s], c);
    const uint32_t starv = sfc_starv(w);
    P.sfc[s] = sfc_pack(ST_PP + st, sfc_has(w), starv, st, starv ? sfc_cnt(w) : 0u);
}

// ---------------------------------------------------------------------------
// K1: A0 default update (fused), A1 strategy, A2 score, A3 starvation + key,
// compaction of the eligible keys, the pinned Preserve sum and the per-block
// OR/AND of the keys (the sort skips digit positions that never vary).
// Four slots per thread through 128-bit loads of the SoA.
// ---------------------------------------------------------------------------
template <bool DBG>
__global__ void __launch_bounds__(kScoreThreads) k_score(Bufs b, Cost c, StepArgs a) {
    __shared__ uint32_t sh_warp[kScoreThreads / 32];
    __shared__ unsigned long long sh_red[3][kScoreThreads / 32];
    __shared__ uint32_t sh_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

    const Pool& P = b.pool;
    const uint32_t ngroups = (c.cap + 3u) >> 2;  // SoA arrays are padded to a multiple of 4
    const uint32_t key_top = c.SB + c.IB;
    unsigned long long pinned = 0, kor = 0, kand = ~0ull;

    for (uint32_t g0 = blockIdx.x * kScoreThreads; g0 < ngroups; g0 += gridDim.x * kScoreThreads) {
        const uint32_t g = g0 + tid;
        const bool in = g < ngroups;
        uint4 w4 = make_uint4(0, 0, 0, 0), cx = w4, pr = w4, ap = w4, rs = w4, po = w4, pe = w4;
        if (in) {
            w4 = __ldcs(reinterpret_cast<const uint4*>(P.sfc) + g);
            cx = __ldcs(reinterpret_cast<const uint4*>(P.ctx) + g);
            pr = __ldcs(reinterpret_cast<const uint4*>(P.pre) + g);
            ap = __ldcs(reinterpret_cast<const uint4*>(P.api) + g);
            rs = __ldcs(reinterpret_cast<const uint4*>(P.resp) + g);
            po = __ldcs(reinterpret_cast<const uint4*>(P.post) + g);
            pe = __ldcs(reinterpret_cast<const uint4*>(P.pend) + g);
        }
        uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
        uint32_t cv[4] = {cx.x, cx.y, cx.z, cx.w};
        uint32_t prv[4] = {pr.x, pr.y, pr.z, pr.w};
        uint32_t pev[4] = {pe.x, pe.y, pe.z, pe.w};
        const uint32_t apv[4] = {ap.x, ap.y, ap.z, ap.w};
        const uint32_t rsv[4] = {rs.x, rs.y, rs.z, rs.w};
        const uint32_t pov[4] = {po.x, po.y, po.z, po.w};
        // A0: the previous batch generated one token each
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
        uint64_t key[4];
        uint32_t nk = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t w = wv[j];
            const uint32_t st = sfc_state(w);
            if (st == ST_PP) pinned += blk(cv[j], c);
            if (st != ST_READY) continue;
            const uint32_t has = sfc_has(w);
            uint64_t wp, wd, ws, sc;
            uint32_t strat;
            const uint64_t span = (uint64_t)cv[j] + prv[j] + (has ? (uint64_t)rsv[j] + pov[j] : 0ull);
            if (c.fast && span < kFastCtxLimit) {
                strat = strategy_score64(cv[j], prv[j], apv[j], rsv[j], pov[j], pev[j], has, c, &sc,
                                         &wp, &wd, &ws);
            } else {
                wp = wd = ws = 0;
                strat = STR_NONE;
                if (has) strat = strategy_of(cv[j], prv[j], apv[j], c, &wp, &wd, &ws);
                sc = score_of(cv[j], prv[j], apv[j], rsv[j], pov[j], pev[j], has, strat, c);
            }
            const uint32_t cnt = sfc_cnt(w);
            const uint32_t starv = sfc_starv(w) | (cnt >= c.T ? 1u : 0u);
            const uint32_t cnt2 = cnt < 65535u ? cnt + 1u : 65535u;
            wv[j] = sfc_pack(ST_READY, has, starv, strat, cnt2);
            const uint32_t slot = 4u * g + (uint32_t)j;
            const uint32_t idoff = (slot - a.id_base_mod) & c.cap_mask;
            const uint64_t k = ((uint64_t)(starv ^ 1u) << key_top) | (sc << c.IB) | idoff;
            key[nk++] = k;
            kor |= k;
            kand &= k;
            if (DBG) {
                unsigned long long* d = b.dbg + 4ull * slot;
                d[0] = wp; d[1] = wd; d[2] = ws; d[3] = sc;
            }
        }
        if (in) reinterpret_cast<uint4*>(P.sfc)[g] = make_uint4(wv[0], wv[1], wv[2], wv[3]);

        // compaction: warp prefix by shuffles, one global atomic per CTA iteration
        uint32_t x = nk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) sh_warp[warp] = x;
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < kScoreThreads / 32; w++) {
                const uint32_t v = sh_warp[w];
                sh_warp[w] = t;
                t += v;
            }
            sh_base = t ? atomicAdd(&b.ctl->n_elig, t) : 0u;
        }
        __syncthreads();
        uint64_t* dst = b.keys[0] + sh_base + sh_warp[warp] + (x - nk);
        for (uint32_t j = 0; j < nk; j++) dst[j] = key[j];
        __syncthreads();
    }

    // block reductions: pinned sum, key OR / AND
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        pinned += __shfl_xor_sync(0xffffffffu, pinned, o);
        kor |= __shfl_xor_sync(0xffffffffu, kor, o);
        kand &= __shfl_xor_sync(0xffffffffu, kand, o);
    }
    if (lane == 0) {
        sh_red[0][warp] = pinned;
        sh_red[1][warp] = kor;
        sh_red[2][warp] = kand;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long t = 0, o = 0, n = ~0ull;
        for (int w = 0; w < kScoreThreads / 32; w++) {
            t += sh_red[0][w];
            o |= sh_red[1][w];
            n &= sh_red[2][w];
        }
        if (t) atomicAdd(&b.ctl->pinned, t);
        b.kmask[blockIdx.x] = o;
        b.kmask[b.score_grid + blockIdx.x] = n;
    }
}

// ---------------------------------------------------------------------------
// K3: A5 admission.  One CTA.  budget = kv_total - pinned (R23); demand of the
// k-th ranked request = blk(ctx+1) (R19); exclusive prefix over the head window
// W = min(n_elig, max_batch, budget) (every demand is >= 1 block), in chunks of
// 1024 ranks, stopping at the first chunk that does not fit completely;
// cut = longest prefix with sum <= budget (Alg.1, R15).  Outputs,
// counter reset of the admitted (Alg.1), the preempted list, and the
// per-step accumulators reset for the next step.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kAdmitThreads) k_admit(Bufs b, Cost c, StepArgs a) {
    __shared__ unsigned long long sh_w64[kAdmitThreads / 32];
    __shared__ uint32_t sh_w32[kAdmitThreads / 32];
    Ctl* ctl = b.ctl;
    const Pool& P = b.pool;
    const uint32_t tid = threadIdx.x;
    const uint64_t n_elig = ctl->n_elig;
    const uint64_t pinned = ctl->pinned;
    const uint32_t n_prev = ctl->n_admitted;
    const uint64_t budget = a.kv_total > pinned ? a.kv_total - pinned : 0ull;
    uint64_t Wn = n_elig < a.max_batch ? n_elig : a.max_batch;
    if (budget < Wn) Wn = budget;
    const uint64_t* keys = b.keys[ctl->n_passes & 1u];
    const uint64_t idmask = (1ull << c.IB) - 1ull;
    const uint32_t par = a.parity;

    unsigned long long carry = 0;
    uint32_t cut = 0;
    for (uint32_t base = 0; base < Wn; base += kAdmitThreads) {
        const uint32_t k = base + tid;
        uint32_t slot = 0;
        uint64_t idoff = 0;
        unsigned long long dem = 0;
        if (k < Wn) {
            idoff = keys[k] & idmask;
            slot = (uint32_t)((a.id_base + idoff) & c.cap_mask);
            dem = blk((uint64_t)P.ctx[slot] + 1u, c);
        }
        unsigned long long tot;
        const unsigned long long incl = carry + block_excl_scan_u64<kAdmitThreads>(dem, sh_w64, &tot) + dem;
        const bool fit = k < Wn && incl <= budget;
        const uint32_t nfit = (uint32_t)__syncthreads_count(fit);
        if (fit) {
            const uint32_t w = P.sfc[slot];
            b.adm_slot[par][k] = slot;
            b.adm_id[par][k] = a.id_base + idoff;
            b.adm_strat[par][k] = (uint8_t)sfc_strat(w);
            P.stamp[slot] = a.step;
            P.sfc[slot] = (w & 0xffffu) | SFC_RAN;  // StarvationCnt <- 0; runs this iteration
            if (k == base + nfit - 1) ctl->budget_used = incl;
        }
        cut += nfit;
        carry += tot;
        const uint32_t chunk = (uint32_t)min((uint64_t)kAdmitThreads, Wn - base);
        if (nfit < chunk) break;
    }
    if (tid == 0 && cut == 0) ctl->budget_used = 0;
    __syncthreads();

    // preempted: admitted last step, still READY, not admitted now (in the previous rank order)
    const uint32_t prev = par ^ 1u;
    uint32_t npre = 0;
    for (uint32_t base = 0; base < n_prev; base += kAdmitThreads) {
        const uint32_t k = base + tid;
        uint32_t f = 0;
        if (k < n_prev) {
            const uint32_t s = b.adm_slot[prev][k];
            f = (sfc_state(P.sfc[s]) == ST_READY && P.stamp[s] != a.step) ? 1u : 0u;
        }
        uint32_t tot;
        const uint32_t pos = block_excl_scan_u32<kAdmitThreads>(f, sh_w32, &tot);
        if (f) b.pre_id[npre + pos] = b.adm_id[prev][k];
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
    }
}

// ---------------------------------------------------------------------------
// ingest scatter kernels (Alg.1 intake P:965-969 and API return P:971-975)
// ---------------------------------------------------------------------------
__global__ void k_submit(Pool P, Cost c, const SubmitRec* rec, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SubmitRec r = rec[i];
    const uint32_t s = r.slot;
    P.ctx[s] = r.ctx;
    P.pre[s] = r.pre;
    P.api[s] = r.api;
    P.resp[s] = r.resp;
    P.post[s] = r.post;
    const uint64_t f = t_fwd(r.ctx, c);  // prefill owed
    P.pend[s] = f > 0xffffffffull ? 0xffffffffu : (uint32_t)f;
    P.sfc[s] = sfc_pack(ST_READY, r.has, 0, STR_NONE, 0);
}

__global__ void k_api_return(Pool P, Cost c, const ReturnRec* rec, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const ReturnRec r = rec[i];
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
    P.sfc[s] = sfc_pack(ST_READY, r.has, sfc_starv(w), sfc_strat(w), sfc_cnt(w));  // RAN clear
}

__global__ void k_gather_u32(const uint32_t* src, const uint32_t* slots, uint32_t* out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[slots[i]];
}

}  // namespace

cudaError_t launch_gather_u32(const uint32_t* src, const uint32_t* d_slots, uint32_t* d_out,
                              uint32_t n, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_gather_u32<<<(n + 255) / 256, 256, 0, s>>>(src, d_slots, d_out, n);
    return cudaGetLastError();
}

cudaError_t launch_events(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s) {
    if (!a.n_ev) return cudaSuccess;
    k_events<<<(a.n_ev + 255) / 256, 256, 0, s>>>(b, c, a);
    return cudaGetLastError();
}

cudaError_t launch_score(const Bufs& b, const Cost& c, const StepArgs& a, int grid,
                         cudaStream_t s) {
    if (b.dbg)
        k_score<true><<<grid, kScoreThreads, 0, s>>>(b, c, a);
    else
        k_score<false><<<grid, kScoreThreads, 0, s>>>(b, c, a);
    return cudaGetLastError();
}

cudaError_t launch_admit(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s) {
    k_admit<<<1, kAdmitThreads, 0, s>>>(b, c, a);
    return cudaGetLastError();
}

cudaError_t launch_submit(const Pool& p, const Cost& c, const SubmitRec* d_rec, uint32_t n,
                          cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_submit<<<(n + 255) / 256, 256, 0, s>>>(p, c, d_rec, n);
    return cudaGetLastError();
}

cudaError_t launch_api_return(const Pool& p, const Cost& c, const ReturnRec* d_rec, uint32_t n,
                              cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_api_return<<<(n + 255) / 256, 256, 0, s>>>(p, c, d_rec, n);
    return cudaGetLastError();
}

}  // namespace lamps
