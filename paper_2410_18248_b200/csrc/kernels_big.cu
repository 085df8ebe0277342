// kernels_big.cu -- pools above the fused kernel's on-chip capacity (#SM x 10240 slots, up to
// 2^23): the warm-step design of k_fused (splitters = keys of the previous step's order, runs
// of keys into range regions, range sorts on chip) split at its grid barrier into two kernels,
// with several ranges per CTA:
//   k_big_score  (plain launch, one CTA per kBigSlots slots): the prologue's ingest, A0-A3 per
//                slot (the same device functions as k_fused), each key to its range (binary
//                search over the V splitters), the CTA's run of each range stored into the
//                range's region of keysR (one global atomic per nonempty range), and the
//                CTA's keys also stored compacted at its own stride (the fallback's input)
//   k_big_sort   (cooperative, one CTA per SM): ranges v = bid, bid + G, ... sorted on chip
//                (range_sort_loop) into their place in keys[1]; CTA 0 sorts range 0 (the
//                admission head) first and admits from it; the next step's grid entries.  A
//                range over its region's capacity sends every CTA to the global LSD over the
//                compacted keys, then CTA 0 admits.
// Cold steps (no grid yet) take the 3-kernel path and k_big_grid writes the grid from its
// sorted order.  Results identical to k_fused's (tests/test_parity_gpu.py, LAMPS_BIG_STEP).
#include "fused_dev.cuh"

namespace lamps {

namespace {

constexpr uint32_t kBigSlots = 8192;          // slots per k_big_score CTA
constexpr uint32_t kBigMaxRanges = 2048;
struct BigSmemA {
    uint64_t kbuf[kBigSlots];                 // 64 KB: keys by slot position
    uint64_t kb2[kBigSlots];                  // 64 KB: keys by range run
    uint16_t rv[kBigSlots];                   // 16 KB: range by position
    uint32_t vmask[kBigSlots / 32];           // which positions hold keys
    unsigned long long spl[kBigMaxRanges];    // 16 KB: splitters (range starts)
    uint32_t lcnt[kBigMaxRanges], lst[kBigMaxRanges], gbase[kBigMaxRanges];
    unsigned long long red[2][kFW];
    uint32_t w32[kFW + 1];
};
static_assert(sizeof(BigSmemA) <= 232448, "k_big_score shared memory exceeds 227 KB");

// position of grid entry f (0 .. 16 V) in an order of n keys: range 0's 16 segments over
// [0, q1), the other ranges' over [q1, n) evenly (as k_fused)
__device__ __forceinline__ uint32_t big_qf(uint32_t f, uint32_t n, uint32_t q1, uint32_t V) {
    const uint64_t p = f <= (uint32_t)kSeg ? (uint64_t)q1 * f / kSeg
                                           : q1 + (uint64_t)(f - kSeg) * (uint64_t)(n - q1) / ((uint64_t)kSeg * (V - 1u));
    return n ? (uint32_t)min(p, (uint64_t)(n - 1u)) : 0u;
}

template <bool DBG>
__global__ void __launch_bounds__(kFT, 1) k_big_score(const __grid_constant__ Bufs b, const __grid_constant__ Cost c,
                                                      StepArgs a, const __grid_constant__ InlineStage inl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BigSmemA& sm = *reinterpret_cast<BigSmemA*>(smem_raw);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, bid = blockIdx.x;
    const uint32_t V = b.big_ranges;
    const uint32_t s_lo = bid * b.big_cta_slots, s_hi = min(c.cap, s_lo + b.big_cta_slots);  // <= kBigSlots
    const uint32_t npos = s_hi > s_lo ? s_hi - s_lo : 0u;
    if (warp == 0) {  // the CTA's seven SoA ranges into L2 (bulk prefetches)
        for (uint32_t q = lane; q < 7u * ((npos + 1023u) / 1024u); q += 32u) {
            const uint32_t ai = q % 7u, base = s_lo + (q / 7u) * 1024u;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b.pool.sfc + (size_t)ai * b.pool.stride + base),
                         "r"(min(1024u, s_hi - base) * 4u) : "memory");
        }
    }
    for (uint32_t r = tid; r < V; r += kFT) {
        sm.spl[r] = __ldg(&b.big_spl[(size_t)a.parity * (kSeg * kBigMaxRanges + kSeg) + kSeg * r]);
        sm.lcnt[r] = 0u;
    }
    if (a.n_ev | a.n_ret | a.n_sub) {  // ingest on this CTA's slots (as k_fused's prologue)
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
    }
    __syncthreads();
    // ---- S: one slot per thread per round
    const Pool& P = b.pool;
    uint32_t pinned = 0;
    for (uint32_t i0 = 0; i0 < npos; i0 += kFT) {
        const uint32_t i = i0 + tid, slot = s_lo + i;
        bool has_key = false;
        uint64_t key = 0;
        if (i < npos) {
            uint32_t w = __ldcg(&P.sfc[slot]), ctx = __ldcg(&P.ctx[slot]), pre = __ldcg(&P.pre[slot]),
                     pend = __ldcg(&P.pend[slot]);
            const uint32_t api = __ldcg(&P.api[slot]), resp = __ldcg(&P.resp[slot]), post = __ldcg(&P.post[slot]);
            if (w & SFC_RAN) {  // A0: the previous batch generated one token
                ctx += 1u;
                pre = pre ? pre - 1u : 0u;
                pend = 0u;
                P.ctx[slot] = ctx;
                P.pre[slot] = pre;
                P.pend[slot] = 0u;
            }
            const uint32_t st = sfc_state(w);
            pinned += st == ST_PP ? (ctx + c.B - 1u) >> c.lgB : 0u;
            if (st == ST_READY) {
                const uint32_t has = sfc_has(w), rp = has ? resp : 0u, pp = has ? post : 0u;
                if (c.lean && (ctx | pre | rp | pp) < (1u << 18)) {
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
                    const ColdOut o = score_slot_cold<DBG>(P, c, a.id_base_mod, b.dbg, slot, w, ctx, pre, api, resp,
                                                           post, pend);
                    key = o.key;
                    w = o.w;
                }
                P.sfc[slot] = w;
                has_key = true;
            }
            sm.kbuf[i] = key;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, has_key);
        if (lane == 0 && i0 + warp * 32u < npos) sm.vmask[(i0 >> 5) + warp] = m;
    }
    // ---- the CTA's pinned blocks and key count
    unsigned long long pin64 = pinned;
#pragma unroll
    for (int o = 16; o; o >>= 1) pin64 += __shfl_xor_sync(0xffffffffu, pin64, o);
    if (lane == 0) sm.red[0][warp] = pin64;
    __syncthreads();
    // ---- R: each key to its range (the largest r with spl[r] <= key; spl[0] = 0)
    for (uint32_t i = tid; i < npos; i += kFT) {
        if (!((sm.vmask[i >> 5] >> (i & 31u)) & 1u)) continue;
        const uint64_t k = sm.kbuf[i];
        uint32_t lo = 0, hi = V;  // [lo, hi): the answer is in it
        while (hi - lo > 1u) {
            const uint32_t mid = (lo + hi) >> 1;
            if (k >= sm.spl[mid]) lo = mid; else hi = mid;
        }
        sm.rv[i] = (uint16_t)lo;
        atomicAdd(&sm.lcnt[lo], 1u);
    }
    __syncthreads();
    uint32_t* rcur = b.big_rcur + (size_t)a.parity * kBigMaxRanges;
    for (uint32_t r = tid; r < V; r += kFT) {
        const uint32_t m = sm.lcnt[r];
        sm.gbase[r] = m ? atomicAdd(&rcur[r], m) : 0u;
        sm.lst[r] = m;
    }
    __syncthreads();
    const uint32_t nk = smem_excl_scan<kFT, kBigMaxRanges / kFT + 1>(sm.lst, V, sm.w32);
    for (uint32_t r = tid; r < V; r += kFT) sm.lcnt[r] = sm.lst[r];  // run cursors
    if (tid == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kFW; w++) t += sm.red[0][w];
        b.pin_part[bid] = t;
        b.nk_part[bid] = nk;
    }
    __syncthreads();
    for (uint32_t i = tid; i < npos; i += kFT) {
        if (!((sm.vmask[i >> 5] >> (i & 31u)) & 1u)) continue;
        sm.kb2[atomicAdd(&sm.lcnt[sm.rv[i]], 1u)] = sm.kbuf[i];
    }
    __syncthreads();
    uint64_t* keysC = b.big_keysc + (size_t)bid * kBigSlots;
    bool over = false;
    for (uint32_t j = tid; j < nk; j += kFT) {
        uint32_t lo = 0, hi = V;  // the run holding kb2[j]: the last range with lst <= j
        while (hi - lo > 1u) {
            const uint32_t mid = (lo + hi) >> 1;
            if (sm.lst[mid] <= j) lo = mid; else hi = mid;
        }
        while (lo + 1u < V && sm.lst[lo + 1u] <= j) lo++;  // (empty runs share a start)
        const uint64_t k = sm.kb2[j];
        const uint32_t pos = sm.gbase[lo] + (j - sm.lst[lo]);
        if (pos < (uint32_t)kKcap) b.big_keysr[(size_t)lo * kKcap + pos] = k;
        else over = true;
        keysC[j] = k;  // the fallback's input (this CTA's keys at its own stride)
    }
    if (__syncthreads_or(over) && tid == 0) b.big_over[a.parity] = 1u;
}

template <bool DBG>
__global__ void __launch_bounds__(kFT, 1) k_big_sort(const __grid_constant__ Bufs b, const __grid_constant__ Cost c,
                                                     StepArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FusedSmem& sm = *reinterpret_cast<FusedSmem*>(smem_raw);
    Ctl* ctl = b.ctl;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t G = gridDim.x, bid = blockIdx.x;
    const uint32_t V = b.big_ranges, GA = b.big_grid;
    const uint32_t vb = c.SB + c.IB;
    const size_t spg = kSeg * kBigMaxRanges + kSeg;
    const unsigned long long* spl_cur = b.big_spl + (size_t)a.parity * spg;
    unsigned long long* spl_next = b.big_spl + (size_t)(a.parity ^ 1u) * spg;
    uint32_t* rcur = b.big_rcur + (size_t)a.parity * kBigMaxRanges;
    if (bid == 0) {  // the next step's accumulators
        for (uint32_t r = tid; r < V; r += kFT) b.big_rcur[(size_t)(a.parity ^ 1u) * kBigMaxRanges + r] = 0u;
        if (tid == 0) b.big_over[a.parity ^ 1u] = 0u;
    }
    // ---- sizes, positions, key count, pinned total (every CTA; one round trip); the range
    // sizes and positions live past FusedSmem (the range sorts use all of PhaseL)
    uint32_t* rsz = reinterpret_cast<uint32_t*>(smem_raw + sizeof(FusedSmem));  // [V]
    uint32_t* rpre = rsz + kBigMaxRanges;                                        // [V]
    for (uint32_t r = tid; r < V; r += kFT) rsz[r] = rpre[r] = __ldcg(&rcur[r]);
    unsigned long long pin = 0;
    uint32_t nq = 0;
    for (uint32_t q = tid; q < GA; q += kFT) {
        pin += __ldcg(&b.pin_part[q]);
        nq += __ldcg(&b.nk_part[q]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        pin += __shfl_xor_sync(0xffffffffu, pin, o);
        nq += __shfl_xor_sync(0xffffffffu, nq, o);
    }
    if (lane == 0) { sm.l.red[0][warp] = pin; sm.l.red[1][warp] = nq; }
    __syncthreads();
    (void)smem_excl_scan<kFT, kBigMaxRanges / kFT + 1>(rpre, V, sm.l.w32);
    bool big = false;
    for (uint32_t r = tid; r < V; r += kFT) big |= rsz[r] > (uint32_t)kKcap;
    big = __syncthreads_or(big || __ldcg(&b.big_over[a.parity]) != 0u || (a.flags & kStepForceFallback));
    unsigned long long pinned_all = 0;
    uint32_t n = 0;
    for (int w = 0; w < kFW; w++) { pinned_all += sm.l.red[0][w]; n += (uint32_t)sm.l.red[1][w]; }
    const uint32_t q1 = V > 1u ? min(n, a.max_batch + kHeadMargin) : n;
    const uint32_t need = min(n, a.max_batch);
    uint32_t bar = a.step * kBarPerStep;
    uint32_t final_buf = 1, passes = 1;
    bool admitted = false;
    // admission by CTA 0 (A5) from `head` (with the staged demand / state words when given);
    // the preempted check's hash table in whichever key buffer does not hold the head
    auto admit = [&](const uint64_t* head, bool on_chip, const uint32_t* dsm, const uint32_t* wsm) {
        if (tid == 0) sm.l.adm.w64[0] = pinned_all;
        __syncthreads();
        if (tid == 0) {
            ctl->n_passes = passes;
            ctl->final_buf = final_buf;
            if (big) atomicAdd(&ctl->fallbacks, 1u);
            ctl->n_ranked = n;
        }
        uint32_t hs = 1024;
        while (hs < 2u * a.max_batch) hs <<= 1;
        const bool use_h = hs <= kHeadTC;
        uint32_t* htab = on_chip && head == sm.l.a ? reinterpret_cast<uint32_t*>(sm.l.b) : reinterpret_cast<uint32_t*>(sm.l.a);
        admit_cta(b, c, a, head, n, pinned_all, sm.l.adm, use_h ? htab : nullptr, use_h ? hs : 0u, nullptr, dsm, wsm);
    };
    if (!big) {
        // ---- L: this CTA's ranges; CTA 0 starts with range 0 (the head) and admits from it
        for (uint32_t v = bid; v < V; v += G) {
            const uint32_t rn = rsz[v], rp = rpre[v];
            if (warp == 1 && lane <= (uint32_t)kSeg) {
                const unsigned long long fk = __ldcg(&spl_cur[kSeg * v + lane]);
                sm.l.fine[lane] = fk;
                sm.l.fcode[lane] = key_code(fk, vb);
            }
            __syncthreads();
            const uint64_t* src = b.big_keysr + (size_t)v * kKcap;
            const bool stage = v == 0 && rn <= kHeadPre;
            // ranges other than the staged head: the keys into shared memory by one bulk copy
            // and the shared-memory range sort (plain stores out: nothing asynchronous is left
            // behind when the next range reuses shared memory)
            const bool tma = !stage && rn > kSmallSort && rn <= kTmaMax && !(a.tune & 4u);
            if (tma && tid == 0) range_stage_issue(sm.l, src, rn);
            bool written = false;
            if (rn && tma) {
                written = range_sort_tma(sm.l, rn, b.keys[1] + rp, rp & 1u, vb, nullptr, false, true, false);
                if (!written) {  // a counter held too many keys: the placed range by LSD
                    unsigned long long o, an;
                    block_or_and(sm.l, sm.l.a, rn, o, an);
                    const uint64_t* r = local_lsd(sm.l, sm.l.a, sm.l.b, rn, o ^ an);
                    if (r != sm.l.a)
                        for (uint32_t i = tid; i < rn; i += kFT) sm.l.a[i] = r[i];
                    __syncthreads();
                    for (uint32_t i = tid; i < rn; i += kFT) b.keys[1][rp + i] = sm.l.a[i];
                }
            } else if (rn) {
                written = range_sort_loop(sm.l, src, rn, b.keys[1] + rp, vb, nullptr, &b.pool, a.id_base_mod, &c,
                                          stage ? sm.l.pos + kHeadPre : nullptr, stage ? sm.l.pos + 2u * kHeadPre : nullptr);
                if (!written) {  // a counter held too many keys: the placed range by LSD
                    unsigned long long o, an;
                    block_or_and(sm.l, sm.l.a, rn, o, an);
                    const uint64_t* r = local_lsd(sm.l, sm.l.a, sm.l.b, rn, o ^ an);
                    if (r != sm.l.a)
                        for (uint32_t i = tid; i < rn; i += kFT) sm.l.a[i] = r[i];
                    __syncthreads();
                    for (uint32_t i = tid; i < rn; i += kFT) b.keys[1][rp + i] = sm.l.a[i];
                }
            }
            __syncthreads();
            // the next step's grid entries that fall in this range: a window of f around the
            // exact inverse of big_qf, each candidate checked
            if (rn) {
                const uint32_t fmax = kSeg * V + 1u;
                uint32_t fa = fmax, fb = 0;
                if (rp < q1 || V == 1u) { fa = 0; fb = kSeg + 1u; }
                if (V > 1u && rp + rn > q1) {
                    const uint64_t D = n - q1, E = (uint64_t)kSeg * (V - 1u);
                    const uint32_t lo_q = max(rp, q1), hi_q = rp + rn;
                    const uint64_t flo = D ? kSeg + (uint64_t)(lo_q - q1) * E / D : (uint64_t)kSeg;
                    const uint64_t fhi = (hi_q >= n || !D) ? (uint64_t)fmax : kSeg + ((uint64_t)(hi_q - q1) * E + D - 1) / D + 2u;
                    fa = min(fa, (uint32_t)(flo > 1u ? flo - 1u : 0u));
                    fb = max(fb, (uint32_t)min(fhi, (uint64_t)fmax));
                }
                if (rp + rn >= n) fb = fmax;  // the last key's range: every f clamped to n - 1
                for (uint32_t f = fa + tid; f < fb; f += kFT) {
                    const uint32_t q = big_qf(f, n, q1, V);
                    if (q >= rp && q < rp + rn) spl_next[f] = __ldcg(&b.keys[1][q]);
                }
            }
            if (v == 0 && rn >= need) {  // CTA 0: the head it holds covers the admission
                const uint64_t* head = written ? reinterpret_cast<const uint64_t*>(sm.l.b) : sm.l.a;
                const bool dw = written && stage;
                admit(head, true, dw ? sm.l.pos + kHeadPre : nullptr, dw ? sm.l.pos + 2u * kHeadPre : nullptr);
                admitted = true;
                __syncthreads();
            }
        }
        if (bid == 0 && n == 0)
            for (uint32_t f = tid; f <= kSeg * V; f += kFT) spl_next[f] = 0ull;
        (void)admitted;
        if (rsz[0] < need) {  // grid-uniform: the head does not cover the admission
            grid_barrier(b.flags, G, ++bar);
            if (bid == 0) admit(b.keys[1], false, nullptr, nullptr);
        }
        return;
    }
    // ---- fallback: the keys compacted into keys[0] (prefix of the score CTAs' counts), the
    // grid-synchronous LSD, the admission, the grid from the sorted order
    for (uint32_t q = bid; q < GA; q += G) {
        uint32_t off = 0;
        for (uint32_t p = tid; p < q; p += kFT) off += __ldcg(&b.nk_part[p]);
#pragma unroll
        for (int o = 16; o; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
        if (lane == 0) sm.l.w32[warp] = off;
        __syncthreads();
        off = 0;
        for (int w = 0; w < kFW; w++) off += sm.l.w32[w];
        const uint32_t m = __ldcg(&b.nk_part[q]);
        for (uint32_t j = tid; j < m; j += kFT) b.keys[0][off + j] = __ldcg(&b.big_keysc[(size_t)q * kBigSlots + j]);
        __syncthreads();
    }
    grid_barrier(b.flags, G, ++bar);
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
    grid_barrier(b.flags, G, ++bar);
    if (bid == 0 && n)
        for (uint32_t f = tid; f <= kSeg * V; f += kFT) spl_next[f] = __ldcg(&b.keys[final_buf][big_qf(f, n, q1, V)]);
    if (bid == 0 && n == 0)
        for (uint32_t f = tid; f <= kSeg * V; f += kFT) spl_next[f] = 0ull;
    if (bid == 0) admit(b.keys[final_buf], false, nullptr, nullptr);
}

// cold steps: the grid from the 3-kernel path's sorted order (one thread per entry)
__global__ void k_big_grid(const __grid_constant__ Bufs b, StepArgs a) {
    const uint32_t V = b.big_ranges;
    const uint32_t n = (uint32_t)b.ctl->n_elig_out, fb = b.ctl->final_buf & 1u;
    const uint32_t q1 = V > 1u ? min(n, a.max_batch + kHeadMargin) : n;
    unsigned long long* spl_next = b.big_spl + (size_t)(a.parity ^ 1u) * (kSeg * kBigMaxRanges + kSeg);
    for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f <= kSeg * V; f += gridDim.x * blockDim.x)
        spl_next[f] = n ? __ldcg(&b.keys[fb][big_qf(f, n, q1, V)]) : 0ull;
    if (blockIdx.x == 0) {  // the accumulators of the first warm step (this parity's were never used)
        for (uint32_t r = threadIdx.x; r < V; r += blockDim.x) b.big_rcur[(size_t)(a.parity ^ 1u) * kBigMaxRanges + r] = 0u;
        if (threadIdx.x == 0) b.big_over[a.parity ^ 1u] = 0u;
    }
}

}  // namespace

uint32_t big_slots_per_cta() { return kBigSlots; }
uint32_t big_max_ranges() { return kBigMaxRanges; }

constexpr size_t kBigSortSmem = sizeof(FusedSmem) + 2u * kBigMaxRanges * 4u;
static_assert(kBigSortSmem <= 232448, "k_big_sort shared memory exceeds 227 KB");

cudaError_t launch_big(const Bufs& b, const Cost& c, const StepArgs& a, const InlineStage* inl, uint32_t sort_grid,
                       cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_big_score<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmemA));
        cudaFuncSetAttribute(k_big_score<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmemA));
        cudaFuncSetAttribute(k_big_sort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBigSortSmem);
        cudaFuncSetAttribute(k_big_sort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBigSortSmem);
        attr = true;
    }
    static const InlineStage kNone{};
    if (b.dbg)
        k_big_score<true><<<b.big_grid, kFT, sizeof(BigSmemA), s>>>(b, c, a, inl ? *inl : kNone);
    else
        k_big_score<false><<<b.big_grid, kFT, sizeof(BigSmemA), s>>>(b, c, a, inl ? *inl : kNone);
    if (cudaError_t e = cudaGetLastError()) return e;
    Bufs bb = b;
    Cost cc = c;
    StepArgs aa = a;
    void* args[] = {&bb, &cc, &aa};
    return cudaLaunchCooperativeKernel(b.dbg ? (const void*)k_big_sort<true> : (const void*)k_big_sort<false>,
                                       dim3(sort_grid), dim3(kFT), args, kBigSortSmem, s);
}

cudaError_t launch_big_grid(const Bufs& b, const StepArgs& a, cudaStream_t s) {
    k_big_grid<<<(kSeg * b.big_ranges + 1 + 255) / 256, 256, 0, s>>>(b, a);
    return cudaGetLastError();
}

}  // namespace lamps
