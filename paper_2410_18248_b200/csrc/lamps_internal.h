// lamps_internal.h -- shared declarations between the host runtime and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lamps_dev.cuh"

namespace lamps {

constexpr int kDigits = 8;          // 8-bit digits of a 64-bit key
constexpr int kBins = 256;
constexpr int kSortThreads = 1024;  // persistent sort CTA (one per SM)
constexpr int kSortItems = 8;       // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;  // 8192 keys per tile
constexpr int kSortMaxTilesPerCta = 8;               // capacity <= 2^23 over >= 128 CTAs
constexpr int kScoreThreads = 256;  // K1 CTA
constexpr int kAdmitThreads = 1024; // K3 (single CTA)
constexpr int kMaxBatch = 16384;
constexpr int kFusedKcap = 10240;    // keys per SM kept in shared memory by the fused step kernel
constexpr uint32_t kStepForceFallback = 1u;  // StepArgs.flags: fused kernel takes the global LSD
constexpr uint32_t kStepMerge = 2u;          // StepArgs.flags: emit top-K records, no local admission
constexpr uint32_t kStepHeadOnly = 4u;       // StepArgs.flags: rank only the admission head (F3)
constexpr uint32_t kStepP2P = 8u;            // StepArgs.flags: exchange by peer stores + merge in k_fused
constexpr uint32_t kStepP2PSys = 16u;        // StepArgs.flags: the peers are other GPUs (system scope)
constexpr uint32_t kMergeMaxRecords = 8192;  // world * max_batch of the in-kernel (P2P) merge's records
constexpr size_t kMergeSmemMax = 232448 - 4096;  // above: the grid-wide merge by rank (k_merge_count/place/cut)

// multi-GPU exchange: per rank one header followed by K records (32 B each)
struct MergeHdr {
    unsigned long long pinned, kv_total;
    uint32_t n_valid, n_local;
    unsigned long long pad;
};
struct MergeRec {
    unsigned long long sk;   // (!starving << SB) | score
    unsigned long long gid;  // global id = local id * world + rank
    uint32_t demand, slot;
    unsigned long long pad;
};
static_assert(sizeof(MergeHdr) == 32 && sizeof(MergeRec) == 32, "exchange records are 32 B");
// Peer-memory exchange buffer of one rank: records [2 parities][world][K + 1] (header +
// K records from each source rank), then flags [2][32] u32 (source rank's sequence number).
__host__ __device__ inline size_t p2p_rec_count(uint32_t world, uint32_t K) { return 2ull * world * (K + 1ull); }
__host__ __device__ inline size_t p2p_bytes(uint32_t world, uint32_t K) {
    return p2p_rec_count(world, K) * sizeof(MergeRec) + 2 * 32 * 4;
}
constexpr int kTraceSlots = 64;
constexpr uint32_t kBarPerStep = 64;  // grid-barrier values reserved per step

// Device control block: per-step counters, the sort plan and the step summary.
struct Ctl {
    // ---- accumulated by K1, reset by K3 for the next step
    uint32_t n_elig;                 // compacted eligible keys (K1 atomics)
    uint32_t pad0;
    unsigned long long pinned;       // sum over PAUSED_P of blk(ctx)
    // ---- sort (K2)
    uint32_t n_passes;               // radix passes that did work
    uint32_t final_buf;              // keys[final_buf] holds the ranked order
    uint32_t fallbacks;              // fused steps that needed the global LSD fallback
    uint32_t bar_count, bar_gen;     // grid barrier of the cooperative kernels
    // ---- summary (K3)
    uint32_t n_admitted, n_preempted, blocked_head, n_prev;
    unsigned long long budget, budget_used;
    unsigned long long n_elig_out, pinned_out;
    uint32_t n_ranked;               // keys of the ranked order available in keys[final_buf]
    uint32_t pad1;
};

// Step result delivered straight into mapped pinned host memory by the admission (one
// stream synchronisation per step, no device-to-host copies): summary, then the lists.
struct HostRes {
    unsigned long long n_elig, pinned, budget, budget_used;
    uint32_t n_admitted, n_preempted, blocked_head, final_buf;
    uint32_t xfail, pad;  // P2P: 1 = the peers' records did not arrive in time (no admission)
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
    uint32_t flags;         // kStepForceFallback, kStepMerge, kStepHeadOnly
    uint32_t world, rank;   // multi-GPU shards
    uint32_t xseq;          // peer-memory exchange: sequence number of this step's exchange
    uint32_t xtimeout_ms;   // peer-memory exchange: longest wait for the peers' flags
    uint32_t n_ret;         // fused path: API returns staged at Bufs::returns, applied in the prologue
    uint32_t n_sub;         // fused path: arrivals staged at Bufs::arrivals, applied in the prologue
    uint32_t inl;           // fused path: returns, arrivals, events read from the kernel's
                            // InlineStage parameter (records in that order) instead of Bufs
    uint32_t cold;          // fused: no splitters from a previous step (first step after init /
                            // import): ranges from a bucket histogram instead
    uint32_t tune;          // A/B knobs of the fused kernel (env LAMPS_TUNE at init; 0 = defaults):
                            // bit 0 uniform key ranges (no speed weights), bit 1 nearest-
                            // instead of first-boundary snapping of the range ends, bit 3
                            // one-sided speed weights (capped at 1 instead of 1.25), bit 2 the
                            // bucket range sort also for ranges of <= 384 keys, bit 4 no
                            // sparse-bucket sort for the head range
};

// A small iteration's staging (API returns, arrivals, events) carried in the fused kernel's
// parameter block: no copy operation before the launch.
constexpr uint32_t kInlineStage = 2048;
struct InlineStage {
    alignas(16) unsigned char bytes[kInlineStage];
};

struct Bufs {
    Pool pool;
    Ctl* ctl;
    unsigned long long* kmask;   // [2][max(score_grid, sort_grid)] per-block OR / AND of keys
    unsigned long long* pin_part;  // [sort_grid] per-CTA pinned sums (fused kernel)
    uint32_t* blocksum;      // LSD: [2][grid][kBins] digit counts
    uint32_t* btot;          // fused: [2][buckets] bucket totals by step parity; the other
                             // parity's array is zeroed during the step (zero at init)
    uint32_t* btab;          // fused: [2][136] bucket tables by step parity (kernels_fused.cu
                             // bucket_t); each cold step writes the next step's (bt_update)
    unsigned long long* spl; // fused: [2][256] range splitters by step parity; each step writes
                             // the next step's from its own sorted order
    uint32_t* rcur;          // fused: [2][256] keys written to each range, by step parity
    uint32_t* nk_part;       // fused: [grid] keys of each CTA
    uint32_t* hd;            // fused: [kFusedKcap] demand blk(ctx + 1) of range 0's keys (the admission
                             // head), beside range 0's region of keys[0] (warm steps)
    uint32_t* hw;            // fused: [kFusedKcap] their state words, likewise
    uint8_t* rhint;          // fused: [cap_pad] each slot's key range in the last step that ranked it
                             // (R's search starts there; any value is safe, it is verified)
    uint32_t score_grid, sort_grid;
    uint64_t* keys[2];       // ping-pong key buffers, capacity + pad
    uint32_t* adm_slot[2];   // admitted slots, by parity
    uint64_t* adm_id[2];     // admitted ids
    uint8_t* adm_strat[2];
    uint64_t* pre_id;        // preempted ids
    const void* events;      // lamps_event[max_batch] (device)
    const void* returns;     // ReturnRec[] staged by lamps_iterate (device, the ingest staging)
    const void* arrivals;    // SubmitRec[] staged by lamps_iterate (device, after the returns)
    unsigned long long* dbg; // [cap][4] W_P, W_D, W_S, score (LAMPS_DEBUG_OUT) or null
    unsigned long long* trace;  // [grid][16] clock64 at phase boundaries (LAMPS_TRACE) or null
    uint32_t* flags;         // grid barrier words (see sort_dev.cuh)
    float* cta_cost;         // fused: [grid] measured range-sort cycles per key of each CTA
                             // (EMA over steps; 0 = not measured): weights the key ranges
    HostRes* hres;           // mapped pinned host memory (device pointer): step summary
    unsigned long long* h_adm_id;  // mapped: admitted ids [max_batch]
    unsigned long long* h_pre_id;  // mapped: preempted ids [max_batch]
    uint8_t* h_adm_strat;          // mapped: admitted strategies [max_batch]
    MergeRec* const* xpeers; // peer-memory transport: [world] exchange buffers (device pointers,
                             // peers' mapped through CUDA IPC), layout p2p_* below
    MergeRec* xown;          // this rank's exchange buffer (the receive side)
    MergeRec* xsend;         // [1 + K] header + top-K records of this rank (world > 1)
    MergeRec* xrecv;         // [world][1 + K] all ranks' send buffers after the all-gather
    // pools above the fused kernel's capacity (kernels_big.cu): V ranges over the score CTAs
    uint32_t big_ranges;     // V (a multiple of the sort grid)
    uint32_t big_grid;       // k_big_score CTAs
    uint32_t big_cta_slots;  // slots per k_big_score CTA (<= kBigSlots; whole waves of #SM CTAs)
    unsigned long long* big_spl;  // [2][16 * kBigMaxRanges + 16] splitter grid by step parity
    uint32_t* big_rcur;      // [2][kBigMaxRanges] keys written to each range, by step parity
    uint32_t* big_over;      // [2] a range's region overflowed (this step: global-LSD fallback)
    uint64_t* big_keysr;     // [V][kFusedKcap] the range regions
    uint64_t* big_keysc;     // [big_grid][kBigSlots] each score CTA's keys (the fallback's input)
    uint32_t* xcnt;          // large merges: [world][world * K] counts of smaller records per other run
    uint32_t* xorder;        // large merges: [K] the merged order's first K records (xrecv indices)
};

// launchers (kernels_step.cu / kernels_sort.cu)
cudaError_t launch_events(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s);
cudaError_t launch_score(const Bufs& b, const Cost& c, const StepArgs& a, int grid,
                         cudaStream_t s);
cudaError_t launch_sort(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s);
int sort_blocks_per_sm();  // occupancy of the persistent sort kernel
size_t fused_smem_bytes();
int fused_blocks_per_sm();
uint32_t fused_max_buckets();
void fused_default_table(uint32_t vb, uint32_t* out136);  // the initial bucket table
cudaError_t launch_fused(const Bufs& b, const Cost& c, const StepArgs& a, const InlineStage* inl, uint32_t grid,
                         cudaStream_t s);
uint32_t small_max_cap();  // the one-CTA small-pool step kernel's capacity limit
cudaError_t launch_small(const Bufs& b, const Cost& c, const StepArgs& a, const InlineStage* inl, cudaStream_t s);
cudaError_t launch_merge(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s);
bool merge_is_large(uint32_t world, uint32_t K);  // world * K records beyond one CTA's shared memory
uint32_t big_slots_per_cta();
uint32_t big_max_ranges();
cudaError_t launch_big(const Bufs& b, const Cost& c, const StepArgs& a, const InlineStage* inl, uint32_t sort_grid,
                       cudaStream_t s);
cudaError_t launch_big_grid(const Bufs& b, const StepArgs& a, cudaStream_t s);
// merge scratch: sk, gid (8 B) and demand (4 B) per record of the W runs, 3 index arrays of K
__host__ __device__ inline size_t merge_smem_bytes(uint32_t world, uint32_t K) {
    const size_t R = (size_t)world * K;
    return R * 8 * 2 + R * 4 + ((size_t)(world + 1) / 2 + (world + 3) / 4 + 1) * K * 4;  // records; the tree's lists
}
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

// predictor ingest (kernels_ingest.cu, row F4): truth records in, predicted segments out
struct TruthRec {
    unsigned long long key;
    uint32_t pre, pre_bin, resp, post, api, has;
};
struct PredRec {
    uint32_t pre, resp, post, api;
};
static_assert(sizeof(TruthRec) == 32 && sizeof(PredRec) == 16, "ingest records");
cudaError_t launch_predict(const TruthRec* d_in, PredRec* d_out, uint32_t n, uint64_t seed, uint32_t len_ppm,
                           uint32_t api_ppm, cudaStream_t s);

}  // namespace lamps
