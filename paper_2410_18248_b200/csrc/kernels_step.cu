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
// K0: A0 -- the previously admitted batch ran one iteration; apply events.
// One CTA.  Also resets the per-step accumulators read by K1/K2.
// Paper: iteration-level semantics P:610-611; routing Alg.1 P:1014-1022;
// removal P:1004; counter reset on API entry unless starving P:1085.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_events(Bufs b, Cost c, StepArgs a) {
    Ctl* ctl = b.ctl;
    const uint32_t tid = threadIdx.x;
    const uint32_t n_prev = ctl->n_admitted;  // previous K3's result
    for (uint32_t i = tid; i < kDigits * kBins; i += blockDim.x) b.hist[i] = 0;
    const uint32_t prev = a.parity ^ 1u;
    const Pool& P = b.pool;
    for (uint32_t k = tid; k < n_prev; k += blockDim.x) {
        const uint32_t s = b.adm_slot[prev][k];
        if (sfc_state(P.sfc[s]) != ST_READY) continue;
        P.ctx[s] = P.ctx[s] + 1u;
        const uint32_t pr = P.pre[s];
        P.pre[s] = pr ? pr - 1u : 0u;
        P.pend[s] = 0u;
    }
    __syncthreads();
    const DevEvent* ev = static_cast<const DevEvent*>(b.events);
    for (uint32_t e = tid; e < a.n_ev; e += blockDim.x) {
        const DevEvent E = ev[e];
        const uint32_t s = (uint32_t)E.id & c.cap_mask;
        const uint32_t w = P.sfc[s];
        if (E.kind == EV_FINISHED) {
            P.sfc[s] = 0u;
        } else {
            P.pre[s] = 0u;
            const uint32_t st = strategy_of(P.ctx[s], 0, P.api[s], c);
            const uint32_t starv = sfc_starv(w);
            P.sfc[s] = sfc_pack(ST_PP + st, sfc_has(w), starv, st, starv ? sfc_cnt(w) : 0u);
        }
    }
    if (tid == 0) {
        ctl->n_prev = n_prev;
        ctl->n_elig = 0;
        ctl->k1_done = 0;
        ctl->pinned = 0;
        ctl->n_passes = 0;
#pragma unroll
        for (int d = 0; d < kDigits; d++) ctl->tile_ctr[d] = 0;
    }
}

// ---------------------------------------------------------------------------
// K1: A1 strategy, A2 score, A3 starvation + key, fused with the compaction of
// eligible keys, the eight digit histograms of the radix sort, the pinned
// Preserve sum and (last CTA) the sort plan.  Four slots per thread through
// 128-bit loads of the SoA.
// ---------------------------------------------------------------------------
template <bool DBG>
__global__ void __launch_bounds__(kScoreThreads) k_score(Bufs b, Cost c, StepArgs a) {
    __shared__ uint32_t sh_hist[kDigits * kBins];
    __shared__ uint32_t sh_warp[kScoreThreads / 32];
    __shared__ unsigned long long sh_pin[kScoreThreads / 32];
    __shared__ uint32_t sh_base;
    __shared__ bool sh_last;
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = tid; i < kDigits * kBins; i += kScoreThreads) sh_hist[i] = 0;
    __syncthreads();

    const Pool& P = b.pool;
    const uint32_t ngroups = (c.cap + 3u) >> 2;  // SoA arrays are padded to a multiple of 4
    const uint4* sfc4 = reinterpret_cast<const uint4*>(P.sfc);
    const uint4* ctx4 = reinterpret_cast<const uint4*>(P.ctx);
    const uint4* pre4 = reinterpret_cast<const uint4*>(P.pre);
    const uint4* api4 = reinterpret_cast<const uint4*>(P.api);
    const uint4* resp4 = reinterpret_cast<const uint4*>(P.resp);
    const uint4* post4 = reinterpret_cast<const uint4*>(P.post);
    const uint4* pend4 = reinterpret_cast<const uint4*>(P.pend);
    uint64_t* keys_out = b.keys[0];
    const uint32_t key_top = c.SB + c.IB;
    unsigned long long pinned = 0;

    for (uint32_t g0 = blockIdx.x * kScoreThreads; g0 < ngroups; g0 += gridDim.x * kScoreThreads) {
        const uint32_t g = g0 + tid;
        const bool in = g < ngroups;
        uint4 w4 = make_uint4(0, 0, 0, 0), cx = w4, pr = w4, ap = w4, rs = w4, po = w4, pe = w4;
        if (in) {
            w4 = sfc4[g]; cx = ctx4[g]; pr = pre4[g]; ap = api4[g];
            rs = resp4[g]; po = post4[g]; pe = pend4[g];
        }
        uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
        const uint32_t cv[4] = {cx.x, cx.y, cx.z, cx.w};
        const uint32_t prv[4] = {pr.x, pr.y, pr.z, pr.w};
        const uint32_t apv[4] = {ap.x, ap.y, ap.z, ap.w};
        const uint32_t rsv[4] = {rs.x, rs.y, rs.z, rs.w};
        const uint32_t pov[4] = {po.x, po.y, po.z, po.w};
        const uint32_t pev[4] = {pe.x, pe.y, pe.z, pe.w};
        uint64_t key[4];
        uint32_t nk = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t w = wv[j];
            const uint32_t st = sfc_state(w);
            if (st == ST_PP) pinned += blk(cv[j], c);
            if (st != ST_READY) continue;
            const uint32_t has = sfc_has(w);
            uint64_t wp = 0, wd = 0, ws = 0;
            uint32_t strat = STR_NONE;
            if (has) strat = strategy_of(cv[j], prv[j], apv[j], c, &wp, &wd, &ws);
            const uint64_t sc = score_of(cv[j], prv[j], apv[j], rsv[j], pov[j], pev[j], has, strat, c);
            const uint32_t cnt = sfc_cnt(w);
            const uint32_t starv = sfc_starv(w) | (cnt >= c.T ? 1u : 0u);
            const uint32_t cnt2 = cnt < 65535u ? cnt + 1u : 65535u;
            wv[j] = sfc_pack(ST_READY, has, starv, strat, cnt2);
            const uint32_t slot = 4u * g + (uint32_t)j;
            const uint32_t idoff = (slot - a.id_base_mod) & c.cap_mask;
            key[nk++] = ((uint64_t)(starv ^ 1u) << key_top) | (sc << c.IB) | idoff;
            if (DBG) {
                unsigned long long* d = b.dbg + 4ull * slot;
                d[0] = wp; d[1] = wd; d[2] = ws; d[3] = sc;
            }
        }
        if (in) reinterpret_cast<uint4*>(P.sfc)[g] = make_uint4(wv[0], wv[1], wv[2], wv[3]);

        // compaction: one atomic per CTA iteration
        uint32_t tot;
        const uint32_t off = block_excl_scan_u32<kScoreThreads>(nk, sh_warp, &tot);
        if (tid == 0) sh_base = tot ? atomicAdd(&b.ctl->n_elig, tot) : 0u;
        __syncthreads();
        const uint32_t base = sh_base + off;
        for (uint32_t j = 0; j < nk; j++) {
            const uint64_t k = key[j];
            keys_out[base + j] = k;
#pragma unroll
            for (int d = 0; d < kDigits; d++)
                atomicAdd(&sh_hist[d * kBins + (uint32_t)((k >> (8 * d)) & 0xffu)], 1u);
        }
        __syncthreads();
    }

    // flush histograms and the pinned sum
    for (uint32_t i = tid; i < kDigits * kBins; i += kScoreThreads) {
        const uint32_t v = sh_hist[i];
        if (v) atomicAdd(&b.hist[i], v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) pinned += __shfl_xor_sync(0xffffffffu, pinned, o);
    if (lane_id() == 0) sh_pin[tid >> 5] = pinned;
    __syncthreads();
    if (tid == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kScoreThreads / 32; w++) t += sh_pin[w];
        if (t) atomicAdd(&b.ctl->pinned, t);
    }

    // last CTA: build the sort plan (skip digit positions that are constant)
    __threadfence();
    __syncthreads();
    if (tid == 0) sh_last = atomicAdd(&b.ctl->k1_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!sh_last) return;
    __threadfence();
    const uint32_t n = __ldcg(&b.ctl->n_elig);
    uint32_t np = 0;
    for (int d = 0; d < kDigits; d++) {
        const uint32_t v = tid < kBins ? __ldcg(&b.hist[d * kBins + tid]) : 0u;
        const int constant = __syncthreads_or(n > 0 && v == n);
        if (n == 0 || constant) continue;
        uint32_t tot;
        const uint32_t ex = block_excl_scan_u32<kScoreThreads>(v, sh_warp, &tot);
        if (tid < kBins) b.offs[np * kBins + tid] = ex;
        if (tid == 0) b.ctl->shift[np] = 8u * d;
        np++;
    }
    if (tid == 0) b.ctl->n_passes = np;
}

// ---------------------------------------------------------------------------
// K3: A5 admission.  One CTA.  budget = kv_total - pinned (R23); demand of the
// k-th ranked request = blk(ctx+1) (R19); exclusive prefix sum over the head
// window W = min(n_elig, max_batch, budget) (every demand is >= 1 block);
// cut = longest prefix with sum <= budget (Alg.1, R15).  Then the
// outputs, counter reset of the admitted (Alg.1) and the preempted list.
// ---------------------------------------------------------------------------
constexpr int kAdmitItems = kMaxBatch / kAdmitThreads;  // 16

__global__ void __launch_bounds__(kAdmitThreads) k_admit(Bufs b, Cost c, StepArgs a) {
    __shared__ unsigned long long sh_w64[kAdmitThreads / 32];
    __shared__ uint32_t sh_w32[kAdmitThreads / 32];
    Ctl* ctl = b.ctl;
    const Pool& P = b.pool;
    const uint32_t tid = threadIdx.x;
    const uint64_t n_elig = ctl->n_elig;
    const uint64_t pinned = ctl->pinned;
    const uint64_t budget = a.kv_total > pinned ? a.kv_total - pinned : 0ull;
    uint64_t Wn = n_elig < a.max_batch ? n_elig : a.max_batch;
    if (budget < Wn) Wn = budget;
    const uint64_t* keys = b.keys[ctl->n_passes & 1u];
    const uint64_t idmask = (c.IB >= 64) ? ~0ull : ((1ull << c.IB) - 1ull);

    uint32_t slot[kAdmitItems];
    unsigned long long dem[kAdmitItems];
    uint64_t idoff[kAdmitItems];
    unsigned long long tsum = 0;
#pragma unroll
    for (int i = 0; i < kAdmitItems; i++) {
        const uint32_t k = tid * kAdmitItems + i;
        dem[i] = 0; slot[i] = 0; idoff[i] = 0;
        if (k < Wn) {
            idoff[i] = keys[k] & idmask;
            slot[i] = (uint32_t)((a.id_base + idoff[i]) & c.cap_mask);
            dem[i] = blk((uint64_t)P.ctx[slot[i]] + 1u, c);
        }
        tsum += dem[i];
    }
    unsigned long long total;
    unsigned long long run = block_excl_scan_u64<kAdmitThreads>(tsum, sh_w64, &total);
    uint32_t fit = 0;
    unsigned long long incl[kAdmitItems];
#pragma unroll
    for (int i = 0; i < kAdmitItems; i++) {
        run += dem[i];
        incl[i] = run;
        const uint32_t k = tid * kAdmitItems + i;
        if (k < Wn && run <= budget) fit++;
    }
    uint32_t cut;
    (void)block_excl_scan_u32<kAdmitThreads>(fit, sh_w32, &cut);
    const uint32_t par = a.parity;
#pragma unroll
    for (int i = 0; i < kAdmitItems; i++) {
        const uint32_t k = tid * kAdmitItems + i;
        if (k < cut) {
            const uint32_t s = slot[i];
            const uint32_t w = P.sfc[s];
            b.adm_slot[par][k] = s;
            b.adm_id[par][k] = a.id_base + idoff[i];
            b.adm_strat[par][k] = (uint8_t)sfc_strat(w);
            P.stamp[s] = a.step;
            P.sfc[s] = w & 0xffffu;  // StarvationCnt <- 0
            if (k == cut - 1) ctl->budget_used = incl[i];
        }
    }
    if (tid == 0 && cut == 0) ctl->budget_used = 0;
    __syncthreads();

    // preempted: admitted last step, still READY, not admitted now
    const uint32_t n_prev = ctl->n_prev;
    const uint32_t prev = par ^ 1u;
    uint32_t flag[kAdmitItems];
    uint32_t nf = 0;
#pragma unroll
    for (int i = 0; i < kAdmitItems; i++) {
        const uint32_t k = tid * kAdmitItems + i;
        flag[i] = 0;
        if (k < n_prev) {
            const uint32_t s = b.adm_slot[prev][k];
            flag[i] = (sfc_state(P.sfc[s]) == ST_READY && P.stamp[s] != a.step) ? 1u : 0u;
        }
        nf += flag[i];
    }
    uint32_t npre;
    uint32_t pos = block_excl_scan_u32<kAdmitThreads>(nf, sh_w32, &npre);
#pragma unroll
    for (int i = 0; i < kAdmitItems; i++) {
        const uint32_t k = tid * kAdmitItems + i;
        if (flag[i]) b.pre_id[pos++] = b.adm_id[prev][k];
    }
    if (tid == 0) {
        ctl->n_admitted = cut;
        ctl->n_preempted = npre;
        ctl->blocked_head = (n_elig > 0 && cut == 0) ? 1u : 0u;
        ctl->budget = budget;
        ctl->n_elig_out = n_elig;
        ctl->pinned_out = pinned;
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
    P.sfc[s] = sfc_pack(ST_READY, r.has, sfc_starv(w), sfc_strat(w), sfc_cnt(w));
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
    k_events<<<1, 1024, 0, s>>>(b, c, a);
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
