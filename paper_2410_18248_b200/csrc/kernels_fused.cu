// kernels_fused.cu -- the whole scheduling step (A0 default update .. A5) as ONE cooperative
// kernel, one 1024-thread CTA per SM (see fused_dev.cuh for the phases and the on-chip sorts).
#include "fused_dev.cuh"

namespace lamps {

namespace {

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

    if (bid == 0 && tid == 32u) {  // CTA 0: the admission's first loads (the previous admitted list) -> L2
        const uint32_t prv = a.parity ^ 1u;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(ctl));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b.adm_slot[prv]), "r"(((a.max_batch + 3u) & ~3u) * 4u)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b.adm_id[prv]), "r"(((a.max_batch + 1u) & ~1u) * 8u)
                     : "memory");
    }
    const bool hr0 = (a.flags & kStepHeadOnly) && G > 1u && !a.cold;  // head-only R (hr below)
    if (tid == 0 && !a.cold && !hr0 && bins_fit(G) && s_hi > s_lo)  // the slots' range hints -> shared memory
        range_hint_issue(sm.s.hbar, reinterpret_cast<uint8_t*>(sm.s.cnt), b.rhint, s_lo, s_hi);
    TRACE(0);
    if (b.trace && tid == 0) {  // diagnostics: the kernel's start on the global clock (slot 29)
        unsigned long long g0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        b.trace[(size_t)bid * kTraceSlots + 29] = g0;
    }
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
    if (tid == 0) { sm.s.novf = 0u; sm.s.nmiss = 0u; }
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
            // A1 + A2 (score_lean), A3: starvation, counter, key.  (A second instance with the
            // shifts as immediates was measured: the score phase gains 0.2 us, the step loses
            // 2 us -- the step's code is fetched cold every step and grew)
            uint64_t sc, wp, wd, ws;
            const uint32_t strat = score_lean(ctx, pre, api, rp, pp, pend, has, c, sc, wp, wd, ws);
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
    // binned R (warm steps with the full R): layout over sm.s.cnt / start (free in warm steps)
    const bool binm = !a.cold && !hr0 && bins_fit(G);
    uint8_t* const rbase = reinterpret_cast<uint8_t*>(sm.s.cnt);
    uint8_t* const rvb = rbase;                                                 // range hints by position
    uint64_t* const bins = reinterpret_cast<uint64_t*>(rbase + kRbBins);        // [G][kBinCap]
    uint32_t* const ovl = reinterpret_cast<uint32_t*>(rbase + kRbOvl);          // position | index << 14
    uint16_t* const mq = reinterpret_cast<uint16_t*>(rbase + kRbMiss);          // queued hint misses
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
    // (after the barrier above: the table was copied by other threads' cp.async)
    const uint32_t NB = sm.btab[kTabNB];  // buckets of this step's table
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
    // warm head-only steps (F3): only the head matters -- range 0 = keys below the first
    // splitter, every other key "range 1" (kept on chip for the fallback, never stored)
    const bool hr = head_mode && !a.cold && G > 1u;
    if (binm) {
        // binned R (warm steps): one pass over the keys -- each key's range from its slot's hint
        // (the range it had in the last ranking step, copied to shared memory at kernel start:
        // the splitters move little from step to step) verified by two compares, then its place
        // in the range's bin (kBinCap keys; the rest by position in the overflow list, with its
        // index in the range's run).  Keys whose hint misses are queued and searched after the
        // pass (a miss inside the pass would make its whole warp search); their hints are updated.
        const unsigned long long* spl = sm.s.spl;
        uint8_t* const rvp = rvb + (s_lo & 15u);
        auto bin_add = [&](uint32_t i, uint64_t k, uint32_t rg) {
            const uint32_t j = atomicAdd(&sm.s.lcnt[rg], 1u);
            if (j < kBinCap) bins[rg * kBinCap + j] = k;
            else ovl[atomicAdd(&sm.s.novf, 1u)] = i | (j << 14);
        };
        auto search_add = [&](uint32_t i, uint64_t k) {
            uint32_t r = 0;
#pragma unroll
            for (uint32_t st = kMaxCtas / 2u; st; st >>= 1) r = k >= spl[spl_pos(r + st)] ? r + st : r;
            const uint32_t rg = min(r, G - 1u);
            rvp[i] = (uint8_t)rg;
            b.rhint[s_lo + i] = (uint8_t)rg;
            bin_add(i, k, rg);
        };
        if (s_hi > s_lo) range_hint_wait(sm.s.hbar);  // (issued at kernel start)
        for (uint32_t i = tid; i < npos; i += kFT) {
            const uint32_t q = i >> 1;
            if (!((sm.s.vmask[2u * (q >> 5) + (i & 1u)] >> (q & 31u)) & 1u)) continue;
            const uint64_t k = sm.s.kbuf[i];
            const uint32_t h = rvp[i];
            // the hint's range or a neighbour (the order drifts by the keys that changed since:
            // e.g. newly starving keys move every other key back by their number)
            const uint32_t hm = h ? h - 1u : 0u;
            const unsigned long long sm1 = spl[spl_pos(hm)], s0 = spl[spl_pos(h)], s1 = spl[spl_pos(h + 1u)],
                                     s2 = spl[spl_pos(h + 2u)];
            const uint32_t rg = k < s0 ? (k >= sm1 || hm == 0u ? hm : 255u) : (k < s1 ? h : (k < s2 ? h + 1u : 255u));
            if (h < G && rg < G) {
                if (rg != h) {
                    rvp[i] = (uint8_t)rg;
                    b.rhint[s_lo + i] = (uint8_t)rg;
                }
                bin_add(i, k, rg);
            } else {
                const uint32_t m = atomicAdd(&sm.s.nmiss, 1u);
                if (m < kMissCap) mq[m] = (uint16_t)i;
                else search_add(i, k);
            }
        }
        __syncthreads();
        const uint32_t nm = min(sm.s.nmiss, kMissCap);
        for (uint32_t m = tid; m < nm; m += kFT) {
            const uint32_t i = mq[m];
            search_add(i, sm.s.kbuf[i]);
        }
        if (b.trace && tid == 0) {  // diagnostics: hint misses, overflow keys
            b.trace[(size_t)bid * kTraceSlots + 16] = sm.s.nmiss;
            b.trace[(size_t)bid * kTraceSlots + 17] = sm.s.novf;
        }
    } else if (hr) {
        const unsigned long long s1 = sm.s.spl[spl_pos(1)];
        for (uint32_t i = tid; i < npos; i += kFT) {
            const uint32_t q = i >> 1;
            if (!((sm.s.vmask[2u * (q >> 5) + (i & 1u)] >> (q & 31u)) & 1u)) continue;
            const uint32_t rg = sm.s.kbuf[i] >= s1 ? 1u : 0u;
            rv[i] = (uint8_t)rg;
            atomicAdd(&sm.s.lcnt[rg], 1u);
        }
    } else if (!binm) {  // cold steps: a binary search over the splitters (seeds the range hints)
        const unsigned long long* spl = sm.s.spl;
        uint8_t* const hint = b.rhint + s_lo;
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
                const uint32_t rg = min(r[u], G - 1u), i = i0 + (uint32_t)u * kFT;
                rv[i] = (uint8_t)rg;
                hint[i] = (uint8_t)rg;
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
    if (!binm) {
        if (tid < (uint32_t)kMaxCtas) sm.s.lst[tid] = sm.s.lcnt[tid];
        __syncthreads();
        (void)smem_excl_scan<kFT, 1>(sm.s.lst, kMaxCtas, sm.s.w32);
        if (tid < (uint32_t)kMaxCtas) sm.s.lcnt[tid] = sm.s.lst[tid];  // run cursors
    }
    __syncthreads();
    TRACE(5);
    if (!binm) {
        for (uint32_t i = tid; i < npos; i += kFT) {
            const uint32_t q = i >> 1;
            if (!((sm.s.vmask[2u * (q >> 5) + (i & 1u)] >> (q & 31u)) & 1u)) continue;
            if (hr && rv[i]) continue;  // head-only: only the head is placed and stored
            const uint32_t r = rv[i], lp = atomicAdd(&sm.s.lcnt[r], 1u);  // order within a run is free
            kb2[lp] = sm.s.kbuf[i];
            rr[lp] = (uint8_t)r;
        }
        __syncthreads();
    }
    TRACE(12);
    // warm steps: range 0's keys (the admission head; run 0 = kb2[0, lst[1])) get their payload
    // -- demand blk(ctx + 1) and state word, this CTA's own slots (L2) -- stored beside them, so
    // CTA 0 sorts the head with it instead of gathering it after its sort
    const bool hpay = !a.cold && G > 1u && !(a.flags & kStepMerge);
    auto store_key = [&](uint32_t r, uint32_t pos, uint64_t k) {
        if (pos < (uint32_t)kKcap) {  // else: overflow -> fallback
            b.keys[0][(size_t)r * kKcap + pos] = k;
            if (hpay && r == 0u) {
                const uint32_t slot = (a.id_base_mod + (uint32_t)(k & c.cap_mask)) & c.cap_mask;
                b.hd[pos] = (uint32_t)blk((uint64_t)b.pool.ctx[slot] + 1u, c);
                b.hw[pos] = b.pool.sfc[slot];
            }
        }
    };
    if (binm) {  // the bins (a warp per range, coalesced) and the overflow list
        // warp 0 takes the head's bin alone (its payload loads are the phase's latency chain);
        // the other warps share the other ranges, the highest threads the overflow list
        for (uint32_t r = warp == 0u ? 0u : warp - 1u + (G > 1u ? 1u : G); r < G; r += warp == 0u ? G : (uint32_t)kFW - 1u) {
            const uint32_t m = min(sm.s.lcnt[r], kBinCap), gb = sm.s.gbase[r];
            for (uint32_t l = lane; l < m; l += 32u) store_key(r, gb + l, bins[r * kBinCap + l]);
        }
        const uint8_t* const rvp = rvb + (s_lo & 15u);
        for (uint32_t o = kFT - 1u - tid; o < sm.s.novf; o += kFT) {
            const uint32_t e = ovl[o], i = e & 0x3fffu, r = rvp[i];
            store_key(r, sm.s.gbase[r] + (e >> 14), sm.s.kbuf[i]);
        }
    }
    const uint32_t n0 = sm.s.lst[1];
    for (uint32_t i = tid; i < (binm ? 0u : (hr ? sm.s.lcnt[0] : nk_cta)); i += kFT) {  // (head-only: run 0 = [0, lcnt[0]))
        const uint32_t r = rr[i], pos = sm.s.gbase[r] + (i - sm.s.lst[r]);
        if (pos < (uint32_t)kKcap) {  // else: overflow -> fallback
            const uint64_t k = kb2[i];
            b.keys[0][(size_t)r * kKcap + pos] = k;
            if (hpay && i < n0) {
                const uint32_t slot = (a.id_base_mod + (uint32_t)(k & c.cap_mask)) & c.cap_mask;
                b.hd[pos] = (uint32_t)blk((uint64_t)b.pool.ctx[slot] + 1u, c);
                b.hw[pos] = b.pool.sfc[slot];
            }
        }
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
        for (int j = 0; j < kMaxCtas / 32; j++) {  // (head-only: "range 1" is every other key, not sorted)
            tot += v[j];
            big |= (v[j] > (uint32_t)kKcap && !(hr && lane * (kMaxCtas / 32) + (uint32_t)j > 0u)) ? 1u : 0u;
        }
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
        __syncwarp();
        if (lane == 0) {
            sm.l.w32[0] = nq;
            sm.l.w32[1] = big;
            // this range's keys (CTA 0: and the head's payload) -> shared memory by bulk copies
            // (range_sort_tma), when this CTA will sort its range by it (the same conditions as below)
            const uint32_t rn0 = sm.l.rsz[bid], re0 = sm.l.rsz[0];
            const bool fb0 = fallback || big;
            const bool ho0 = head_mode && !fb0 && re0 >= min(nq, a.max_batch + 32u);
            const bool sorts = !fb0 && !(hr && !ho0) && (!ho0 || bid == 0);
            const bool keep = bid == 0 && rn0 <= kHeadPre && !(a.flags & kStepMerge);
            const bool pay = keep && !a.cold && G > 1u;  // R stored the head's payload (hpay)
            uint32_t tm = 0;
            if (sorts && (rn0 > kSmallSort || (a.tune & 4u)) && rn0 <= kTmaMax && rn0) {
                tm = 1u | (keep ? 2u : 0u) | (pay ? 4u : 0u);
                range_stage_issue(sm.l, b.keys[0] + (size_t)bid * kKcap, rn0, pay ? b.hd : nullptr, pay ? b.hw : nullptr);
            }
            sm.l.w32[2] = tm;
        }
    }
    if (bid == 0 && warp == 2) {  // A5's budget: the pinned total (beside the range sizes' round trip)
        unsigned long long pa = 0;
        for (uint32_t r = lane; r < G; r += 32) pa += __ldcg(&b.pin_part[r]);
#pragma unroll
        for (int o = 16; o; o >>= 1) pa += __shfl_xor_sync(0xffffffffu, pa, o);
        if (lane == 0) sm.pin_all = pa;
    }
    __syncthreads();
    n = sm.l.w32[0];
    fallback = fallback || sm.l.w32[1] != 0u;
    const uint32_t tmode = sm.l.w32[2];  // (read before the range sort's scan reuses w32)
    const bool tma = (tmode & 1u) != 0u;
    rsz = sm.l.rsz[bid];
    rpre = sm.l.rpre[bid];
    const uint32_t r_end0 = sm.l.rsz[0];
    // head-only mode (F3): CTA 0 ranks the head; the others stop here, unless the head range
    // does not hold the keys the admission needs (then every range is sorted)
    const bool head_only = head_mode && !fallback && r_end0 >= min(n, a.max_batch + 32u);
    if (hr && !head_only) fallback = true;  // head-only R placed only the head: the global LSD ranks the rest
    // positions of the next step's splitters in this step's order: the head (range 0) ends
    // at max_batch + kHeadMargin keys, the other ranges share the rest evenly
    const uint32_t q1 = G > 1u ? min(n, a.max_batch + kHeadMargin) : n;
    // position of grid entry f (0 .. 16 G) in this step's order: range 0's 16 segments over
    // [0, q1), the other ranges' over [q1, n) evenly (past the last key: the last key)
    auto qf = [&](uint32_t f) -> uint32_t { return grid_q(f, q1, n, G); };
    unsigned long long* spl_next = b.spl + (size_t)(a.parity ^ 1u) * kSplG;
    // head-only: the grid is kept (the other ranges were not sorted), except range 0's entries,
    // which CTA 0 refreshes from its sorted head when it holds more than q1 keys
    const bool hrefresh = head_only && r_end0 > q1;
    if (head_only && bid == G - 1u)
        for (uint32_t f = tid + (hrefresh ? kSeg + 1u : 0u); f <= kSeg * G; f += kFT)
            spl_next[f] = __ldcg(&b.spl[(size_t)a.parity * kSplG + f]);
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
    bool head_tq = false;    // CTA 0: head keys in sm.l.b, demands / states (if staged) beside (range_sort_tma)
    bool kept = false;       // the sorted range is in shared memory at sm.l.b + (rpre & 1) (range_sort_tma)
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
        if (tma) {  // staged by the bulk copy issued after the barrier; written to keys1 directly
            TRACE(13);
            // (CTA 0's head: plain stores, so no bulk copy is outstanding behind its admission)
            written = range_sort_tma(sm.l, rn, b.keys[1] + rpre, rpre & 1u, vb, tr ? tr + 32 : nullptr, (tmode & 4u) != 0u,
                                     true, bid != 0u);
            head_tq = (tmode & 2u) && written;
            kept = written;
            if (!written) {  // a counter held too many keys: sort the placed range (sm.a) by LSD
                unsigned long long o, an;
                block_or_and(sm.l, sm.l.a, rn, o, an);
                const uint64_t* r = local_lsd(sm.l, sm.l.a, sm.l.b, rn, o ^ an);
                if (r != sm.l.a)
                    for (uint32_t i = tid; i < rn; i += kFT) sm.l.a[i] = r[i];
                __syncthreads();
            }
        } else if (rn <= kSmallSort && !(a.tune & 4u)) {
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
            const bool hpay0 = stage && !a.cold && G > 1u;  // (merge steps never stage)
            written = LAMPS_RANGE_SORT(sm.l, src, rn, b.keys[1] + rpre, vb, tr ? tr + 32 : nullptr, &b.pool,
                                      a.id_base_mod, &c, stage ? sm.l.pos + kHeadPre : nullptr,
                                      stage ? sm.l.pos + 2u * kHeadPre : nullptr, hpay0 ? b.hd : nullptr,
                                      hpay0 ? b.hw : nullptr);
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
        if (tid == kFT - 1u) {  // the next step's grid entries that fall in this range: [gf[0], gf[1])
            sm.l.gf[0] = grid_f(rpre, q1, n, G);
            sm.l.gf[1] = grid_f(rpre + rn, q1, n, G);
        }
        __syncthreads();  // the range's keys are in place (visible to this CTA's threads)
        if (!a.cold) TRACE(10);  // (slots 10 / 11: cold steps' bucket phases; diagnostics here)
        const uint32_t gf0 = sm.l.gf[0], gf1 = sm.l.gf[1];
        // the next step's grid entries that fall in this range
        if (!head_only && rn) {  // (grid entries [gf0, gf1): grid_f in the range sizes' pass)
            const uint64_t* K = sm.l.b + (rpre & 1u);
            for (uint32_t f = gf0 + tid; f < gf1; f += kFT) {
                const uint32_t q = qf(f);
                spl_next[f] = kept ? K[q - rpre] : __ldcg(&b.keys[1][q]);
            }
        }
        if (hrefresh && bid == 0 && tid <= (uint32_t)kSeg) spl_next[tid] = __ldcg(&b.keys[1][qf(tid)]);
        if (!a.cold) TRACE(11);
        final_buf = 1;
        passes = 1;
    } else if (fallback) {
        if (tma) range_stage_wait(sm.l);  // the bulk copy lands before shared memory is reused
        {   // the keys compacted into keys0 (this CTA's at the prefix of the CTAs' key counts)
            uint32_t off = 0;
            {
                const uint32_t q = tid < bid ? __ldcg(&b.nk_part[tid]) : 0u;
                uint32_t tot;
                (void)block_excl_scan_u32<kFT>(q, sm.l.w32, &tot);
                off = tot;
            }
            // kb2 (this CTA's keys, compacted by R) is intact: since the barrier only PhaseL's
            // small arrays past sm.l.b (w32, rsz, rpre) were written.  Head-only R placed only
            // the head in kb2: then the keys come from kbuf / vmask (intact likewise; any order)
            if (hr) {
                uint32_t* ctr = &sm.l.w32[kFW];
                if (tid == 0) *ctr = 0u;
                __syncthreads();
                for (uint32_t i = tid; i < npos; i += kFT) {
                    const uint32_t q = i >> 1;
                    if ((sm.s.vmask[2u * (q >> 5) + (i & 1u)] >> (q & 31u)) & 1u)
                        b.keys[0][off + atomicAdd(ctr, 1u)] = sm.s.kbuf[i];
                }
            } else if (binm) {  // binned R: the bins and the overflow list (intact likewise)
                uint32_t* ctr = &sm.l.w32[kFW];
                if (tid == 0) *ctr = 0u;
                __syncthreads();
                for (uint32_t r = warp; r < G; r += (uint32_t)kFW) {
                    const uint32_t m = min(sm.s.lcnt[r], kBinCap);
                    const uint32_t o0 = lane == 0 && m ? atomicAdd(ctr, m) : 0u, ob = __shfl_sync(0xffffffffu, o0, 0);
                    for (uint32_t l = lane; l < m; l += 32u) b.keys[0][off + ob + l] = bins[r * kBinCap + l];
                }
                __syncthreads();
                const uint32_t nb = *ctr;
                for (uint32_t o = tid; o < sm.s.novf; o += kFT) b.keys[0][off + nb + o] = sm.s.kbuf[ovl[o] & 0x3fffu];
            } else {
                for (uint32_t i = tid; i < nk_cta; i += kFT) b.keys[0][off + i] = kb2[i];
            }
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
        if (tma) range_stage_wait(sm.l);  // (cold head-only steps) no copy outlives the CTA
        final_buf = 1;  // head-only: CTA 0 ranked the head; this CTA is done
        passes = 1;
    }
    // the next step's splitters past the last key, and (after the LSD) all of them
    if (bid == 0 && !head_only && n == 0)  // no keys: an empty grid
        for (uint32_t f = tid; f <= kSeg * G; f += kFT) spl_next[f] = 0ull;
    unsigned long long pinned_all = 0;  // (CTA 0: sm.pin_all, summed right after the grid barrier)

    TRACE(8);
    // ---------------- A: admission by CTA 0
    // CTA 0 may start as soon as the head it needs is sorted: without the fallback
    // the keys [0, rsz[0]) are sorted by CTA 0 itself.
    const uint32_t need = min(n, a.max_batch);  // the admission (or the merge records) reads keys [0, need)
    const bool wait = fallback || r_end0 < need;
    if (b.trace && bid == 0 && tid == 0) {  // diagnostics: the head's size, whether CTA 0 waits
        b.trace[56] = r_end0;
        b.trace[57] = wait ? 1u : 0u;
    }
    if (wait && tma && tid == 0) bulk_store_done();  // CTA 0 reads the ranges from keys1
    if (wait) grid_barrier(b.flags, G, ++bar);
    if (fallback && bid == 0 && n)
        for (uint32_t f = tid; f <= kSeg * G; f += kFT) spl_next[f] = __ldcg(&b.keys[final_buf][qf(f)]);
    if (bid != 0) {
        if (tma && tid == 0) bulk_store_read_wait();  // the range's bulk store has left shared memory
        return;
    }
    if (tma && tid == 0 && (a.flags & kStepMerge)) bulk_store_done();  // the records / merge read keys1
    pinned_all = sm.pin_all;
    if (tid == 0) {
        ctl->n_passes = passes;
        ctl->final_buf = final_buf;
        if (fallback) atomicAdd(&ctl->fallbacks, 1u);  // a reduction, no load on the path
        ctl->n_ranked = head_only ? r_end0 : n;  // head-only: keys [0, hb_r) are ranked
    }
    TRACE(15);
    // CTA 0 holds [0, need) in shared memory unless it waited (or its range sort wrote them out)
    const bool hl = head_loop && !wait;  // head keys in sm.l.b, demands / states in sm.l.pos
    const bool hq = head_tq && !wait;    // head keys in sm.l.b, demands / states (if staged) beside
    const uint64_t* head = wait ? b.keys[final_buf]
                                : ((hl || hq) ? (hq || !kSortedInA ? reinterpret_cast<const uint64_t*>(sm.l.b) : sm.l.a)
                                              : (written ? b.keys[final_buf] : sm.l.a));
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
        if (b.trace && tid == 0) b.trace[58] = clock64();
        for (uint32_t i = tid; i < ((nv + 32u) & ~31u); i += kFT) {  // whole warps (the shuffles below)
            // the 32-B record as two 16-B vectors built in registers: a warp stores 1 KB of
            // whole sectors per destination (a struct copied field by field through local
            // memory made 4 partial-sector stores per record: 17 us for 8 x 1025 records)
            ulonglong2 v0 = make_ulonglong2(0ull, 0ull), v1 = v0;
            if (i > nv) {
            } else if (i == 0) {  // MergeHdr {pinned, kv_total, n_valid | n_local << 32, pad}
                v0 = make_ulonglong2(pinned_all, a.kv_total);
                v1 = make_ulonglong2((unsigned long long)nv | ((unsigned long long)n << 32), 0ull);
            } else {       // MergeRec {sk, gid, demand | slot << 32, pad}
                const uint64_t k = head[i - 1];
                const uint64_t lid = a.id_base + (k & idmask);
                const uint32_t slot = (uint32_t)(lid & c.cap_mask);
                const uint32_t dem = dw ? reinterpret_cast<const uint32_t*>(sm.l.b)[kHeadD + i - 1]
                                        : (uint32_t)blk((uint64_t)b.pool.ctx[slot] + 1u, c);
                v0 = make_ulonglong2(k >> c.IB, lid * a.world + a.rank);
                v1 = make_ulonglong2((unsigned long long)dem | ((unsigned long long)slot << 32), 0ull);
            }
            if (p2p) {
                // the warp's 32 records are 64 consecutive 16-B chunks of each destination:
                // two stores of 32 consecutive chunks (whole sectors) per destination, lane l
                // of store h holding chunk 32 h + l = half (l & 1) of record 16 h + l / 2
                const uint32_t i0 = i - lane;
                ulonglong2 w[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint32_t sl = 16u * h + (lane >> 1);
                    const unsigned long long a0 = __shfl_sync(0xffffffffu, v0.x, sl), a1 = __shfl_sync(0xffffffffu, v0.y, sl);
                    const unsigned long long b0 = __shfl_sync(0xffffffffu, v1.x, sl), b1 = __shfl_sync(0xffffffffu, v1.y, sl);
                    w[h] = (lane & 1u) ? make_ulonglong2(b0, b1) : make_ulonglong2(a0, a1);
                }
                for (uint32_t p = 0; p < W; p++) {
                    ulonglong2* d = reinterpret_cast<ulonglong2*>(tail.xp[p] + slot0 + i0);
#pragma unroll
                    for (int h = 0; h < 2; h++)
                        if (i0 + 16u * h + (lane >> 1) <= nv) d[32u * h + lane] = w[h];  // records <= nv only
                }
            } else if (i <= nv) {
                ulonglong2* d = reinterpret_cast<ulonglong2*>(b.xsend + i);
                d[0] = v0;
                d[1] = v1;
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
    uint32_t* htab = (hl && !kSortedInA) || hq ? reinterpret_cast<uint32_t*>(sm.l.a) : reinterpret_cast<uint32_t*>(sm.l.b);
    const bool hqp = hq && (tmode & 4u);  // the TMA-staged head's payload
    admit_cta(b, c, a, head, n, pinned_all, sm.l.adm, use_h ? htab : nullptr, use_h ? hs : 0u,
              b.trace ? b.trace + 40 : nullptr,
              hl ? sm.l.pos + kHeadPre : (hqp ? tma_head_dem(sm.l) : (dw ? b32 + kHeadD : nullptr)),
              hl ? sm.l.pos + 2u * kHeadPre : (hqp ? tma_head_st(sm.l) : (dw ? b32 + kHeadW : nullptr)));
    if (tma && tid == 0) bulk_store_read_wait();
    TRACE(9);
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
