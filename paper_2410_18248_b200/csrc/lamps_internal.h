// lamps_internal.h -- shared declarations between the host runtime and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lamps_dev.cuh"

namespace lamps {

constexpr int kDigits = 8;          // 8-bit digits of a 64-bit key
constexpr int kBins = 256;
constexpr int kSortThreads = 256;   // onesweep pass CTA
constexpr int kSortItems = 8;       // keys per thread
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys per tile
constexpr int kScoreThreads = 256;  // K1 CTA
constexpr int kAdmitThreads = 1024; // K3 (single CTA)
constexpr int kMaxBatch = 16384;

// Device control block: per-step counters, the sort plan and the step summary.
struct Ctl {
    // ---- written by K0 (zeroed), K1
    uint32_t n_elig;                 // compacted eligible keys (K1 atomics)
    uint32_t k1_done;                // K1 finished-CTA counter (last-block plan)
    unsigned long long pinned;       // sum over PAUSED_P of blk(ctx)
    // ---- sort plan (K1 last block)
    uint32_t n_passes;               // radix passes that do work
    uint32_t shift[kDigits];         // bit offset of each active pass's digit
    uint32_t tile_ctr[kDigits];      // dynamic tile ids per pass
    // ---- summary (K3)
    uint32_t n_admitted, n_preempted, blocked_head, n_prev;
    unsigned long long budget, budget_used;
    unsigned long long n_elig_out, pinned_out;
};

struct StepArgs {
    uint64_t kv_total;
    uint64_t id_base;       // ids of this step's keys are id_base + offset
    uint32_t id_base_mod;   // id_base & cap_mask
    uint32_t step;          // step number (1-based), stamp for admitted slots
    uint32_t epoch;         // lookback epoch base (step * 8)
    uint32_t n_ev;
    uint32_t max_batch;
    uint32_t parity;        // admitted list buffer written this step
};

struct Bufs {
    Pool pool;
    Ctl* ctl;
    uint32_t* hist;          // [kDigits][kBins]  global digit histograms
    uint32_t* offs;          // [kDigits][kBins]  exclusive prefix per active pass
    unsigned long long* status;  // [max_tiles][kBins] decoupled look-back words
    uint64_t* keys[2];       // ping-pong key buffers, capacity + pad
    uint32_t* adm_slot[2];   // admitted slots, by parity
    uint64_t* adm_id[2];     // admitted ids
    uint8_t* adm_strat[2];
    uint64_t* pre_id;        // preempted ids
    const void* events;      // lamps_event[max_batch] (device)
    unsigned long long* dbg; // [cap][4] W_P, W_D, W_S, score (LAMPS_DEBUG_OUT) or null
    uint32_t max_tiles;
};

// launchers (kernels_step.cu / kernels_sort.cu)
cudaError_t launch_events(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s);
cudaError_t launch_score(const Bufs& b, const Cost& c, const StepArgs& a, int grid,
                         cudaStream_t s);
cudaError_t launch_sort(const Bufs& b, const Cost& c, const StepArgs& a, uint32_t cap,
                        cudaStream_t s, cudaEvent_t* mid_events);
cudaError_t launch_admit(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s);

// ingest records (host -> device staging)
struct SubmitRec {
    uint32_t slot, ctx, pre, api, resp, post, has, pad;
};
struct ReturnRec {
    uint32_t slot, actual, pre, api, resp, post, has, pad;
};
cudaError_t launch_submit(const Pool& p, const Cost& c, const SubmitRec* d_rec, uint32_t n,
                          cudaStream_t s);
cudaError_t launch_gather_u32(const uint32_t* src, const uint32_t* d_slots, uint32_t* d_out,
                              uint32_t n, cudaStream_t s);
cudaError_t launch_api_return(const Pool& p, const Cost& c, const ReturnRec* d_rec, uint32_t n,
                              cudaStream_t s);

}  // namespace lamps
