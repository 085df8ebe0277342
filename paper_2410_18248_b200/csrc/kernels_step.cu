// kernels_step.cu -- A0 events (K0), A1-A3 strategy/score/key (K1),
// A5 admission (K3) and the ingest scatter kernels.  sm_100a, integer only.
#include "step_dev.cuh"

namespace lamps {

namespace {

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
    apply_event(b.pool, c, static_cast<const DevEvent*>(b.events)[e]);
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
    const uint32_t ngroups = (c.cap + 3u) >> 2;  // SoA arrays are padded to a multiple of 4
    unsigned long long pinned = 0, kor = 0, kand = ~0ull;

    for (uint32_t g0 = blockIdx.x * kScoreThreads; g0 < ngroups; g0 += gridDim.x * kScoreThreads) {
        const uint32_t g = g0 + tid;
        uint64_t key[4];
        uint32_t nk = 0;
        if (g < ngroups) nk = score_group<DBG>(b.pool, c, a.id_base_mod, b.dbg, g, key, pinned);
#pragma unroll
        for (int j = 0; j < 4; j++)
            if ((uint32_t)j < nk) { kor |= key[j]; kand &= key[j]; }

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
#pragma unroll
        for (int j = 0; j < 4; j++)
            if ((uint32_t)j < nk) dst[j] = key[j];
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
    __shared__ AdmitSmem sm;
    Ctl* ctl = b.ctl;
    const uint32_t n = ctl->n_elig;
    admit_cta(b, c, a, b.keys[ctl->final_buf & 1u], n, ctl->pinned, sm);
    if (threadIdx.x == 0) ctl->n_ranked = n;  // the 3-kernel path ranks everything
}

// ---------------------------------------------------------------------------
// ingest scatter kernels (Alg.1 intake P:965-969 and API return P:971-975)
// ---------------------------------------------------------------------------
__global__ void k_submit(Pool P, Cost c, const SubmitRec* rec, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    apply_submit(P, c, rec[i]);
}

__global__ void k_api_return(Pool P, Cost c, const ReturnRec* rec, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    apply_return(P, c, rec[i]);
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
