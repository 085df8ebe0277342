// kernels_small.cu -- the one-CTA small-pool step kernel (its own translation unit: the grid
// kernel's code layout stays as it is).
#include "fused_dev.cuh"

namespace lamps {

namespace {

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
    uint32_t kdem[kSmallPer], kw[kSmallPer];  // the admission's demand blk(ctx + 1) and state word
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
        const uint32_t dm = (uint32_t)blk((uint64_t)ctx + 1u, c);
#pragma unroll
        for (int q = 0; q < kSmallPer; q++)  // packed to the front (no dynamic register index)
            if (q == (int)nk) { key[q] = k; kdem[q] = dm; kw[q] = w; }
        nk++;
        kmin = min(kmin, (unsigned long long)k);
        kmax = max(kmax, (unsigned long long)k);
    }
    // ---- compaction into keys[0] (block scan), the pinned total, this step's key bounds
    uint32_t n;
    const uint32_t pos = block_excl_scan_u32<kFT>(nk, sm.l.w32, &n);
    // keys (and, up to kHeadPre keys, their demand / state words) stay in shared memory for
    // range_sort_tma (no copy to stage: the sort reads them where the compaction put them);
    // the few-hundred-key all-pairs sort and the forced fallback read them from keys[0]
    const bool onchip = n > kSmallSort && n <= kTmaMax && !(a.flags & kStepForceFallback) && !(a.tune & 4u);
    const bool pay = onchip && n <= kHeadPre;
    uint32_t* const Hd = tma_head_dem(sm.l);
    uint32_t* const Hw = tma_head_st(sm.l);
#pragma unroll
    for (int q = 0; q < kSmallPer; q++)
        if ((uint32_t)q < nk) {
            if (onchip) {
                sm.l.b[pos + q] = key[q];
                if (pay) { Hd[pos + q] = kdem[q]; Hw[pos + q] = kw[q]; }
            } else {
                b.keys[0][pos + q] = key[q];
            }
        }
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
        __syncwarp();  // every lane's reads above before lane 0 overwrites entries 0 / 1
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
    } else if (onchip) {
        written = range_sort_tma(sm.l, n, b.keys[1], 0u, vb, nullptr, pay, false, false);
    } else if (n > 1u && !(a.flags & kStepForceFallback)) {
        written = LAMPS_RANGE_SORT(sm.l, b.keys[0], n, b.keys[1], vb, nullptr, &b.pool, a.id_base_mod, &c, dsm, wsm);
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
    const uint64_t* srt = written && !kSortedInA ? reinterpret_cast<const uint64_t*>(sm.l.b) : sm.l.a;
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
    uint32_t* htab = written && !kSortedInA ? reinterpret_cast<uint32_t*>(sm.l.a) : reinterpret_cast<uint32_t*>(sm.l.b);
    const bool dw = written && stage && !onchip;
    const bool dq = written && pay;  // range_sort_tma: the payload by sorted position beside the keys
    const uint32_t* b32 = reinterpret_cast<const uint32_t*>(sm.l.b);  // small_sort's staged arrays
    static_assert(kHeadTC <= kHeadD, "small_sort's staged arrays lie past the hash table");
    admit_cta(b, c, a, srt, n, pinned_all, sm.l.adm, use_h ? htab : nullptr, use_h ? hs : 0u, nullptr,
              dq ? Hd : (dw ? dsm : (tiny ? b32 + kHeadD : nullptr)), dq ? Hw : (dw ? wsm : (tiny ? b32 + kHeadW : nullptr)));
    if (b.trace && tid == 0) b.trace[3] = clock64();
}

}  // namespace

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

}  // namespace lamps
