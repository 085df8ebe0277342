// merge_dev.cuh -- multi-GPU global admission as a device function.
// After the exchange every rank holds `world` runs of K records, each run sorted by
// (!starving, score, global id) -- the head of that rank's ranked order.  One CTA
// merges the runs (merge path, pairwise into an accumulator truncated to K), cuts the
// global order against the global budget and K, and admits this rank's share, which is
// a prefix of its own order.
#pragma once
#include "step_dev.cuh"

namespace lamps {

constexpr int kMT = 1024;

__device__ __forceinline__ bool rec_less(const unsigned long long* sk, const unsigned long long* gid,
                                         uint32_t x, uint32_t y) {
    return sk[x] < sk[y] || (sk[x] == sk[y] && gid[x] < gid[y]);
}

// out[0..lim) = first lim elements of merge(A[0..na), B[0..nb)) (indices into sk/gid), all threads
__device__ __forceinline__ void merge_path(const uint32_t* A, uint32_t na, const uint32_t* Bv, uint32_t nb,
                                           uint32_t* out, uint32_t lim, const unsigned long long* sk,
                                           const unsigned long long* gid) {
    const uint32_t tot = min(na + nb, lim);
    const uint32_t per = (tot + kMT - 1) / kMT;
    const uint32_t k0 = min(tot, threadIdx.x * per), k1 = min(tot, k0 + per);
    if (k0 < k1) {
        // co-rank: i elements from A, k0 - i from B, with A[i-1] < B[k0-i] and B[k0-i-1] < A[i]
        uint32_t lo = k0 > nb ? k0 - nb : 0u, hi = min(k0, na);
        while (lo < hi) {
            const uint32_t i = (lo + hi) >> 1;
            // too few from A if B[k0-i-1] > A[i]
            if (rec_less(sk, gid, A[i], Bv[k0 - i - 1])) lo = i + 1; else hi = i;
        }
        uint32_t i = lo, j = k0 - lo;
        for (uint32_t k = k0; k < k1; k++) {
            const bool takeA = j >= nb || (i < na && rec_less(sk, gid, A[i], Bv[j]));
            out[k] = takeA ? A[i++] : Bv[j++];
        }
    }
    __syncthreads();
}

// Merge of the W runs in xrecv ([W][K+1]: header + records), global cut, and admission
// of this rank's share, by one 1024-thread CTA.  smem_raw: merge_smem_bytes(W, K) bytes of
// scratch; adm / nv[32] / hsum[2] small shared structures.  Used by k_merge (after the
// NCCL all-gather or the loopback copies) and by the fused kernel's CTA 0 (after the
// in-kernel peer-memory exchange).
__device__ __forceinline__ void merge_admit_cta(const Bufs& b, const Cost& c, const StepArgs& a,
                                                const MergeRec* __restrict__ xrecv, unsigned char* smem_raw,
                                                AdmitSmem& adm, uint32_t* nv, unsigned long long* hsum,
                                                uint32_t* htab = nullptr, uint32_t hsize = 0,
                                                const uint32_t* dsm = nullptr, const uint32_t* wsm = nullptr,
                                                unsigned long long* tr = nullptr) {
#define MTRACE(k) do { if (tr && threadIdx.x == 0) tr[k] = clock64(); } while (0)
    const uint32_t W = a.world, K = a.max_batch, R = W * K;
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem_raw);
    unsigned long long* gid = sk + R;
    uint32_t* dem = reinterpret_cast<uint32_t*>(gid + R);
    uint32_t* acc = dem + R;
    uint32_t* tmp = acc + K;
    uint32_t* run = tmp + K;  // K indices of the run being merged
    const uint32_t tid = threadIdx.x;

    if (tid < 32) {  // the W headers in parallel (warp 0), sums by shuffles
        unsigned long long kv = 0, pin = 0;
        if (tid < W) {
            const MergeHdr h = *reinterpret_cast<const MergeHdr*>(xrecv + (size_t)tid * (K + 1));
            nv[tid] = h.n_valid;
            kv = h.kv_total;
            pin = h.pinned;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            kv += __shfl_xor_sync(0xffffffffu, kv, o);
            pin += __shfl_xor_sync(0xffffffffu, pin, o);
        }
        if (tid == 0) {
            hsum[0] = kv;
            hsum[1] = pin;
        }
    }
    __syncthreads();
    for (uint32_t f = tid; f < R; f += kMT) {
        const uint32_t r = f / K, i = f % K;
        if (i < nv[r]) {
            const MergeRec rec = xrecv[(size_t)r * (K + 1) + 1 + i];
            sk[f] = rec.sk;
            gid[f] = rec.gid;
            dem[f] = rec.demand;
        }
    }
    for (uint32_t i = tid; i < K; i += kMT) acc[i] = i;  // run 0
    __syncthreads();
    MTRACE(0);
    uint32_t na = nv[0];
    for (uint32_t r = 1; r < W; r++) {
        for (uint32_t i = tid; i < K; i += kMT) run[i] = r * K + i;
        __syncthreads();
        merge_path(acc, na, run, nv[r], tmp, K, sk, gid);
        na = min(na + nv[r], K);
        for (uint32_t i = tid; i < na; i += kMT) acc[i] = tmp[i];
        __syncthreads();
    }
    MTRACE(1);
    // global cut: longest prefix of the merged order within the budget (and K, every demand >= 1)
    const unsigned long long budget = hsum[0] > hsum[1] ? hsum[0] - hsum[1] : 0ull;
    const uint64_t Wn = (uint64_t)na < budget ? (uint64_t)na : budget;
    unsigned long long carry = 0, used = 0;
    uint32_t cut = 0, c_me = 0;
    unsigned long long d_me = 0;
    for (uint32_t base = 0; base < Wn; base += kMT) {
        const uint32_t k = base + tid;
        const uint32_t f = k < Wn ? acc[k] : 0u;
        const unsigned long long d = k < Wn ? dem[f] : 0ull;
        unsigned long long tot;
        const unsigned long long incl = carry + block_excl_scan_u64<kMT>(d, adm.w64, &tot) + d;
        const bool fit = k < Wn && incl <= budget;
        const uint32_t nfit = (uint32_t)__syncthreads_count(fit);
        const bool mine = fit && f / K == a.rank;
        c_me += (uint32_t)__syncthreads_count(mine);
        unsigned long long dm_tot;
        (void)block_excl_scan_u64<kMT>(mine ? d : 0ull, adm.w64, &dm_tot);
        d_me += dm_tot;
        if (fit && k == base + nfit - 1) hsum[0] = incl;  // global budget used (read after the loop)
        cut += nfit;
        carry += tot;
        if (nfit < min((uint64_t)kMT, Wn - base)) break;
    }
    __syncthreads();
    used = cut ? hsum[0] : 0ull;
    MTRACE(2);
    const MergeHdr* mh = reinterpret_cast<const MergeHdr*>(xrecv + (size_t)a.rank * (K + 1));
    const uint32_t n_local = mh->n_local;
    const unsigned long long pin_local = mh->pinned;
    unsigned long long total_valid = 0;
    for (uint32_t r = 0; r < W; r++) total_valid += nv[r];
    __syncthreads();
    // admit this rank's share: the first c_me keys of its own order (exactly within d_me)
    StepArgs la = a;
    la.kv_total = d_me;
    la.max_batch = c_me;
    admit_cta(b, c, la, b.keys[b.ctl->final_buf & 1u], n_local, 0ull, adm, htab, hsize, nullptr, dsm, wsm);
    MTRACE(3);
#undef MTRACE
    __syncthreads();
    if (tid == 0) {
        Ctl* ctl = b.ctl;
        ctl->budget = budget;
        ctl->budget_used = used;
        ctl->blocked_head = (total_valid > 0 && cut == 0) ? 1u : 0u;
        ctl->pinned_out = pin_local;
        publish_host_result(b);
    }
}

}  // namespace lamps
