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

// out[0..lim) = first lim elements of merge(A, B) where A(i) / B(j) give the record index of
// element i / j (na / nb elements), by the T threads lt = 0..T-1 of a group (merge path:
// each thread finds its co-rank by binary search, then merges its share sequentially).
template <class FA, class FB>
__device__ __forceinline__ void merge_path_grp(FA A, uint32_t na, FB B, uint32_t nb, uint32_t* out, uint32_t lim,
                                               uint32_t lt, uint32_t T, const unsigned long long* sk,
                                               const unsigned long long* gid) {
    const uint32_t tot = min(na + nb, lim);
    const uint32_t per = (tot + T - 1) / T;
    const uint32_t k0 = min(tot, lt * per), k1 = min(tot, k0 + per);
    if (k0 >= k1) return;
    uint32_t lo = k0 > nb ? k0 - nb : 0u, hi = min(k0, na);
    while (lo < hi) {
        const uint32_t i = (lo + hi) >> 1;
        if (rec_less(sk, gid, A(i), B(k0 - i - 1))) lo = i + 1; else hi = i;
    }
    uint32_t i = lo, j = k0 - lo;
    for (uint32_t k = k0; k < k1; k++) {
        const bool takeA = j >= nb || (i < na && rec_less(sk, gid, A(i), B(j)));
        out[k] = takeA ? A(i++) : B(j++);
    }
}

// Merge of the W runs in xrecv ([W][K+1]: header + records), global cut, and admission
// of this rank's share, by one 1024-thread CTA.  smem_raw: merge_smem_bytes(W, K) bytes of
// scratch; adm / nv[32] / hsum[2] small shared structures.  Used by k_merge (after the
// NCCL all-gather or the loopback copies) and by the fused kernel's CTA 0 (after the
// in-kernel peer-memory exchange).  The runs are merged as a tree -- pairs in parallel, each
// by its share of the CTA's threads, every output truncated to K -- ceil(log2 W) rounds.
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
    uint32_t* X = dem + R;                   // [ceil(W/2)][K] lists of odd rounds
    uint32_t* Y = X + ((W + 1) / 2) * K;     // [ceil(W/4) + 1][K] lists of even rounds
    uint32_t* nl = reinterpret_cast<uint32_t*>(&adm.w32[0]);  // list lengths (adm is free until the cut)
    const uint32_t tid = threadIdx.x;
    merge_headers(xrecv, W, K, nv, hsum);
    {   // the records into shared memory: consecutive threads load consecutive 16-B halves of a
        // run's records (whole sectors), four in flight per thread; half 0 = (sk, gid), half 1 =
        // (demand, slot)
        const ulonglong2* x2 = reinterpret_cast<const ulonglong2*>(xrecv);
        const uint32_t Q = 2u * R;
        for (uint32_t q0 = tid; q0 < Q; q0 += 4u * kMT) {
            ulonglong2 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t q = q0 + (uint32_t)u * kMT, r = q / (2u * K), cI = q % (2u * K), i = cI >> 1;
                if (q < Q && i < nv[r]) v[u] = __ldcg(x2 + ((size_t)r * (K + 1) + 1 + i) * 2 + (cI & 1u));
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t q = q0 + (uint32_t)u * kMT, r = q / (2u * K), cI = q % (2u * K), i = cI >> 1;
                if (q < Q && i < nv[r]) {
                    const uint32_t f = r * K + i;
                    if (cI & 1u) {
                        dem[f] = (uint32_t)v[u].x;
                    } else {
                        sk[f] = v[u].x;
                        gid[f] = v[u].y;
                    }
                }
            }
        }
    }
    if (tid < W) nl[tid] = nv[tid];
    __syncthreads();
    if (tr && tid == 0) tr[0] = clock64();
    // round 1 merges the runs (implicit lists r K + i) into X, later rounds X <-> Y
    uint32_t nlist = W;
    uint32_t* src = nullptr;  // nullptr: the runs themselves
    uint32_t* dst = X;
    while (nlist > 1) {
        const uint32_t M = nlist / 2, T = kMT / M;  // pairs this round (an odd last list is copied)
        const uint32_t g = tid / T, lt = tid % T;
        const uint32_t la = g < M ? nl[2 * g] : 0u, lb = g < M ? nl[2 * g + 1] : 0u;
        __syncthreads();  // every thread read nl before it is rewritten
        if (g < M) {
            uint32_t* o = dst + (size_t)g * K;
            if (src == nullptr) {
                const uint32_t ba = 2u * g * K, bb = (2u * g + 1u) * K;
                merge_path_grp([&](uint32_t i) { return ba + i; }, la, [&](uint32_t j) { return bb + j; }, lb, o, K,
                               lt, T, sk, gid);
            } else {
                const uint32_t* pa = src + (size_t)2 * g * K;
                const uint32_t* pb = src + (size_t)(2 * g + 1) * K;
                merge_path_grp([&](uint32_t i) { return pa[i]; }, la, [&](uint32_t j) { return pb[j]; }, lb, o, K,
                               lt, T, sk, gid);
            }
            if (lt == 0) nl[g] = min(la + lb, K);
        }
        if (nlist & 1u) {  // the unpaired last list moves to position M
            const uint32_t last = nlist - 1u, ln = nl[last];
            uint32_t* o = dst + (size_t)M * K;
            for (uint32_t i = tid; i < ln; i += kMT) o[i] = src ? src[(size_t)last * K + i] : last * K + i;
            __syncthreads();
            if (tid == 0) nl[M] = ln;
        }
        __syncthreads();
        nlist = M + (nlist & 1u);
        src = dst;
        dst = dst == X ? Y : X;
    }
    const uint32_t* acc = src;
    const uint32_t na = src ? nl[0] : nv[0];
    __syncthreads();
    if (tr && tid == 0) tr[1] = clock64();
    merge_cut_admit(b, c, a, xrecv, na, [&](uint32_t k, unsigned long long& d, uint32_t& srk) {
        const uint32_t f = acc ? acc[k] : k;
        d = dem[f];
        srk = f / K;
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
