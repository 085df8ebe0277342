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

// The W headers (warp 0): valid counts nv[r], sums of kv_total / pinned into hsum.
__device__ __forceinline__ void merge_headers(const MergeRec* __restrict__ xrecv, uint32_t W, uint32_t K, uint32_t* nv,
                                              unsigned long long* hsum) {
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
}

// Global cut over the merged order (its first na entries; entry k's demand and source rank
// from `at(k)`) against the global budget and K (every demand >= 1), then the admission of
// this rank's share -- the first c_me keys of its own order, exactly within d_me -- and the
// step summary.  One 1024-thread CTA.
template <class At>
__device__ __forceinline__ void merge_cut_admit(const Bufs& b, const Cost& c, const StepArgs& a,
                                                const MergeRec* __restrict__ xrecv, uint32_t na, At at,
                                                AdmitSmem& adm, const uint32_t* nv, unsigned long long* hsum,
                                                uint32_t* htab, uint32_t hsize, const uint32_t* dsm,
                                                const uint32_t* wsm, unsigned long long* tr) {
    const uint32_t W = a.world, K = a.max_batch;
    const uint32_t tid = threadIdx.x;
    const unsigned long long budget = hsum[0] > hsum[1] ? hsum[0] - hsum[1] : 0ull;
    const uint64_t Wn = (uint64_t)na < budget ? (uint64_t)na : budget;
    unsigned long long carry = 0, used = 0;
    uint32_t cut = 0, c_me = 0;
    unsigned long long d_me = 0;
    for (uint32_t base = 0; base < Wn; base += kMT) {
        const uint32_t k = base + tid;
        uint32_t src = 0;
        unsigned long long d = 0;
        if (k < Wn) at(k, d, src);
        unsigned long long tot;
        const unsigned long long incl = carry + block_excl_scan_u64<kMT>(d, adm.w64, &tot) + d;
        const bool fit = k < Wn && incl <= budget;
        const uint32_t nfit = (uint32_t)__syncthreads_count(fit);
        const bool mine = fit && src == a.rank;
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
    if (tr && tid == 0) tr[2] = clock64();
    const MergeHdr* mh = reinterpret_cast<const MergeHdr*>(xrecv + (size_t)a.rank * (K + 1));
    const uint32_t n_local = mh->n_local;
    const unsigned long long pin_local = mh->pinned;
    unsigned long long total_valid = 0;
    for (uint32_t r = 0; r < W; r++) total_valid += nv[r];
    __syncthreads();
    StepArgs la = a;
    la.kv_total = d_me;
    la.max_batch = c_me;
    admit_cta(b, c, la, b.keys[b.ctl->final_buf & 1u], n_local, 0ull, adm, htab, hsize, nullptr, dsm, wsm);
    if (tr && tid == 0) tr[3] = clock64();
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
    const uint32_t W = a.world, K = a.max_batch, R = W * K;
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem_raw);
    unsigned long long* gid = sk + R;
    uint32_t* dem = reinterpret_cast<uint32_t*>(gid + R);
    uint32_t* acc = dem + R;
    uint32_t* tmp = acc + K;
    uint32_t* run = tmp + K;  // K indices of the run being merged
    const uint32_t tid = threadIdx.x;
    merge_headers(xrecv, W, K, nv, hsum);
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
    if (tr && tid == 0) tr[0] = clock64();
    uint32_t na = nv[0];
    for (uint32_t r = 1; r < W; r++) {
        for (uint32_t i = tid; i < K; i += kMT) run[i] = r * K + i;
        __syncthreads();
        merge_path(acc, na, run, nv[r], tmp, K, sk, gid);
        na = min(na + nv[r], K);
        for (uint32_t i = tid; i < na; i += kMT) acc[i] = tmp[i];
        __syncthreads();
    }
    if (tr && tid == 0) tr[1] = clock64();
    merge_cut_admit(b, c, a, xrecv, na, [&](uint32_t k, unsigned long long& d, uint32_t& src) {
        const uint32_t f = acc[k];
        d = dem[f];
        src = f / K;
    }, adm, nv, hsum, htab, hsize, dsm, wsm, tr);
}

// ---------------------------------------------------------------------------
// Large exchanges (world * K records beyond one CTA's shared memory; the NCCL / loopback
// transports): the merged order by RANK, grid-wide.  Records are unique, so record x of
// run r (its index i_x there) is at position  i_x + sum_{r' != r} |{y in run r' : y < x}|
// of the merged order; each count is a binary search in the other (sorted) run.
//   merge_count:  cnt[r'][r * K + i] for every valid record (r, i) and run r' (one thread each)
//   merge_place:  order[pos] = xrecv index of the record, for pos < K
//   then one CTA cuts and admits from order[] (merge_cut_admit).
__device__ __forceinline__ bool rec_less_g(const MergeRec& x, const MergeRec& y) {
    return x.sk < y.sk || (x.sk == y.sk && x.gid < y.gid);
}

__device__ __forceinline__ uint32_t run_valid(const MergeRec* __restrict__ xrecv, uint32_t K, uint32_t r) {
    return reinterpret_cast<const MergeHdr*>(xrecv + (size_t)r * (K + 1))->n_valid;
}

__device__ __forceinline__ void merge_count(const MergeRec* __restrict__ xrecv, uint32_t W, uint32_t K,
                                            uint32_t* __restrict__ cnt) {
    const uint64_t R = (uint64_t)W * K, total = R * W;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = (uint32_t)(p / R), f = (uint32_t)(p % R);  // other run o, record f = r * K + i
        const uint32_t r = f / K, i = f % K;
        if (i >= run_valid(xrecv, K, r)) continue;
        uint32_t c = i;
        if (o != r) {
            const MergeRec x = xrecv[(size_t)r * (K + 1) + 1 + i];
            const MergeRec* y = xrecv + (size_t)o * (K + 1) + 1;
            uint32_t lo = 0, hi = run_valid(xrecv, K, o);  // first y >= x (y != x: unique)
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (rec_less_g(y[mid], x)) lo = mid + 1; else hi = mid;
            }
            c = lo;
        }
        cnt[(size_t)o * R + f] = c;
    }
}

__device__ __forceinline__ void merge_place(const MergeRec* __restrict__ xrecv, uint32_t W, uint32_t K,
                                            const uint32_t* __restrict__ cnt, uint32_t* __restrict__ order) {
    const uint32_t R = W * K;
    for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < R; f += gridDim.x * blockDim.x) {
        const uint32_t r = f / K, i = f % K;
        if (i >= run_valid(xrecv, K, r)) continue;
        uint32_t pos = 0;
        for (uint32_t o = 0; o < W; o++) pos += cnt[(size_t)o * R + f];
        if (pos < K) order[pos] = r * (K + 1) + 1 + i;
    }
}

// One CTA after merge_place: the cut over order[0 .. min(K, sum nv)) and the admission.
__device__ __forceinline__ void merge_cut_from_order(const Bufs& b, const Cost& c, const StepArgs& a,
                                                     const MergeRec* __restrict__ xrecv,
                                                     const uint32_t* __restrict__ order, AdmitSmem& adm,
                                                     uint32_t* nv, unsigned long long* hsum) {
    const uint32_t W = a.world, K = a.max_batch;
    merge_headers(xrecv, W, K, nv, hsum);
    uint64_t tv = 0;
    for (uint32_t r = 0; r < W; r++) tv += nv[r];
    const uint32_t na = (uint32_t)min(tv, (uint64_t)K);
    merge_cut_admit(b, c, a, xrecv, na, [&](uint32_t k, unsigned long long& d, uint32_t& src) {
        const uint32_t f = order[k];
        d = xrecv[f].demand;
        src = f / (K + 1);
    }, adm, nv, hsum, nullptr, 0u, nullptr, nullptr, nullptr);
}

}  // namespace lamps
