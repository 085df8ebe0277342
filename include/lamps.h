/*
 * lamps.h -- C ABI of the B200-native LAMPS scheduling pass (liblamps.so).
 *
 * LAMPS = "LLM API- and Memory-based Predictive Scheduling", arXiv 2410.18248
 * ("Fast Inference for Augmented Large Language Models").  Citations "P:<n>"
 * are lines of that paper's text; "R<n>" are the readings listed in
 * DESIGN.md where the paper is silent or ambiguous.
 *
 * One call of lamps_schedule_step is one iteration of Algorithm 1
 * over the whole request pool, run as one batched GPU pass on the handle's
 * CUDA stream:
 *   A0  apply the engine's events for the previously admitted batch
 *   A1  per READY request with an API: memory waste of Preserve / Discard /
 *       Swap (Eq. 1-3) and the argmin
 *   A2  memory-over-time score
 *   A3  starvation tag (Alg.1) and the 64-bit sort key
 *   A4  radix sort of the keys = ranked order (Alg.1)
 *   A5  admission: longest prefix of the ranked order whose KV-block demand
 *       fits the budget and max_batch (Alg.1), counters
 *
 * All device state is integer (tokens, KV blocks, ticks).  The only floating
 * point input, the predicted API duration in seconds, is quantised on the host
 * at ingest (R22).  No call falls back to the CPU: without a usable CUDA
 * device lamps_init fails with LAMPS_ECUDA.
 *
 * Threading: a handle is single-owner and not thread-safe; distinct handles
 * are independent.  Every call is synchronous with respect to the host unless
 * its name ends in _async.  On any error return the handle's state is
 * unchanged and lamps_last_error() describes the failure.
 */
#ifndef LAMPS_H
#define LAMPS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define LAMPS_OK 0
#define LAMPS_EINVAL (-1)  /* bad argument / infeasible request / bad event */
#define LAMPS_ENOSPC (-2)  /* pool full: the new id's slot is still occupied */
#define LAMPS_ENOENT (-3)  /* unknown id, or id in the wrong state for the call */
#define LAMPS_ENOTSUP (-4) /* feature not available in this build */
#define LAMPS_ECUDA (-5)   /* CUDA runtime error (no device, launch failure, ...) */
#define LAMPS_ENCCL (-6)   /* NCCL error (multi-GPU merge) */

/* ---- request states (Alg.1: WaitingQueue, PQueue, DQueue, SQueue) -------- */
#define LAMPS_FREE 0u
#define LAMPS_READY 1u
#define LAMPS_PAUSED_P 2u
#define LAMPS_PAUSED_D 3u
#define LAMPS_PAUSED_S 4u

/* ---- handling strategies ------------------------------------- */
#define LAMPS_PRESERVE 0u
#define LAMPS_DISCARD 1u
#define LAMPS_SWAP 2u
#define LAMPS_NONE 3u /* request has no further API call */

/* ---- engine events (Alg.1) --------------------------- */
#define LAMPS_EV_API_CALL 1u /* the token just generated triggered the API call */
#define LAMPS_EV_FINISHED 2u /* the request completed */

/* ---- config flags --------------------------------------------------------- */
#define LAMPS_DEBUG_OUT 1u /* keep per-slot W_P, W_D, W_S and score for export */
#define LAMPS_TIMING 2u    /* record CUDA events around each phase (lamps_timing_read) */
#define LAMPS_MULTI_KERNEL 4u   /* use the 3-kernel path even where the fused step kernel fits */
#define LAMPS_FORCE_FALLBACK 8u /* fused path: always take the global-LSD fallback (tests) */
#define LAMPS_TRACE 16u         /* fused path: record SM clock at phase boundaries (lamps_trace_read) */
#define LAMPS_MERGE 32u         /* world <= 1: still run the multi-shard exchange + merge over a 1-rank
                                   NCCL communicator (transport NCCL, nccl_id required); tests the
                                   NCCL path on one GPU */
#define LAMPS_HEAD_ONLY 64u     /* top-K fast path: rank only the head of the order the
                                   admission can reach (>= min(n_eligible, max_batch) keys, to the end
                                   of a bucket).  Admitted set, preempted list, counters and pool
                                   state are those of the full pass; lamps_ranked_keys returns the
                                   head only.  Fused path; the 3-kernel path ranks everything */

#define LAMPS_SHARE_DEVICE 128u /* P2P ranks co-resident on ONE device (lamps_p2p_connect_local, tests):
                                   the step kernel uses #SM / world CTAs so all ranks' kernels run
                                   at once; each rank needs its own stream */

#define LAMPS_GRID_STEP 256u    /* pools the one-CTA small-pool step kernel covers (capacity <= 4096,
                                   one shard) take the grid-wide fused step kernel instead (tests,
                                   measurements) */

#define LAMPS_BIG_STEP 512u     /* take the large-pool path (k_big_score + k_big_sort, several ranges per
                                   CTA; the default above #SM x 10240 slots) at any capacity (tests) */

#define LAMPS_INGEST_LIMIT (1u << 24) /* max tokens of one request (R21) */

typedef struct lamps_s lamps_t;

/*
 * Predictions for one segment of a request: its decode tokens up to its next
 * API call (or to completion), that API's duration and response length, and
 * the decode tokens after it (a multi-API request is a
 * chain of segments, each ending with one API call).
 */
typedef struct {
    uint32_t prompt_len;  /* lamps_submit only: initial context tokens */
    uint32_t pre_len;     /* predicted decode tokens before the API (or in total) */
    uint32_t resp_len;    /* predicted API response tokens           (has_api) */
    uint32_t post_len;    /* predicted decode tokens after the API    (has_api) */
    double api_seconds;   /* predicted API duration T_INT, seconds    (has_api);
                             quantised to ticks = llround(s * ticks_per_second) */
    uint32_t has_api;     /* 0 or 1; 0: resp_len, post_len, api_seconds ignored */
    uint32_t reserved;
} lamps_segment;

/* An engine report about a request admitted by the previous step. */
typedef struct {
    uint64_t id;
    uint32_t kind; /* LAMPS_EV_API_CALL or LAMPS_EV_FINISHED */
    uint32_t reserved;
} lamps_event;

typedef struct {
    uint32_t capacity;      /* pool slots: power of 2, <= 2^23; slot = id mod capacity */
    uint32_t block_tokens;  /* B, tokens per KV block: power of 2 (paged KV) */
    uint64_t tau;           /* ticks per decode iteration (R3); < 2^48 */
    uint64_t A1, A2;        /* T_fwd(c) = (A1*c + A2*c^2) >> SH ticks (R1); < 2^48 */
    uint64_t S0, S1;        /* T_swap(c) = c ? (S0 + S1*c) >> SH : 0 ticks (R2); < 2^48 */
    uint32_t SH;            /* fixed-point shift, <= 63 */
    uint64_t c_other;       /* C_other tokens (profiled, R4); < 2^32 */
    double ticks_per_second;          /* ingest quantisation scale, finite > 0 */
    uint32_t starvation_threshold;    /* StarvationT >= 1 (100 in P:1085) */
    uint32_t max_batch;               /* runningBatch size limit, 1..16384 */
    uint64_t kv_capacity_blocks;      /* static KV capacity: infeasibility check at
                                         ingest; every step's kv_total must be <= it */
    uint32_t score_bits, id_bits;     /* key layout: score_bits + id_bits + 1 <= 64,
                                         2^id_bits >= capacity */
    void* stream;                     /* cudaStream_t to run on (NULL = legacy default) */
    uint32_t flags;                   /* LAMPS_DEBUG_OUT, LAMPS_TIMING, ... */
    /* ---- multi-GPU: shard-parallel pools, global admission ------ */
    uint32_t world;                   /* number of shards (ranks); 0 or 1 = single shard */
    uint32_t rank;                    /* this shard, < world.  Shard r owns the global ids
                                         g with g mod world == r; its local id l is g / world */
    uint32_t transport;               /* LAMPS_XPORT_NCCL or LAMPS_XPORT_LOOPBACK */
    const void* nccl_id;              /* 128-byte ncclUniqueId (all ranks the same; from
                                         lamps_nccl_unique_id on one rank) */
    /* ---- rank policy ---------------------------------------- */
    uint32_t policy;                  /* LAMPS_POLICY_*: the score field of the key (R25) */
    uint32_t score_interval;          /* LAMPS only: selective score update (P:1080, P:1113,
                                         R26).  0 or 1 = every step; k <= 127 = a READY
                                         request keeps its strategy and score for k steps
                                         unless its segment changes (submit / API return) */
    /* ---- co-resident shards (appended) --------------------------------------- */
    uint32_t local_ranks;             /* LAMPS_SHARE_DEVICE: shards co-resident on this
                                         device (each step kernel takes #SM / local_ranks
                                         CTAs); 0 = world.  Fewer than world: the other
                                         shards are on other GPUs (system-scope exchange) */
} lamps_config;

/* rank policies (R25): lower key = earlier; starving requests first under all of them */
#define LAMPS_POLICY_LAMPS 0u     /* memory-over-time area */
#define LAMPS_POLICY_FCFS 1u      /* request id = arrival */
#define LAMPS_POLICY_SJF 2u       /* remaining iterations of the segment: decode tokens + owed
                                     prefill / swap-in ceil(pending / tau) */
#define LAMPS_POLICY_SJF_TOTAL 3u /* + API duration in decode iterations, ceil(ticks / tau) */

#define LAMPS_XPORT_NCCL 0u     /* one ncclAllGather per step over NVLink (libnccl.so.2) */
#define LAMPS_XPORT_LOOPBACK 1u /* all shards in this process on one device: lamps_group_step */
#define LAMPS_XPORT_P2P 2u      /* no library collective: inside the step kernel, CTA 0 stores its
                                   records straight into every rank's exchange buffer (CUDA IPC
                                   mappings over NVLink / NVSwitch), raises a flag on each, waits
                                   for all ranks' flags and merges + admits -- one kernel per step.
                                   Needs lamps_p2p_handle / lamps_p2p_connect after lamps_init
                                   (world 1: self-exchange, no connect needed) */

/*
 * Result of one step.  Host arrays are owned by the handle and stay valid until
 * the next call on it.  Device arrays likewise (they live in the workspace).
 */
typedef struct {
    uint64_t n_eligible;           /* |WaitingQueue| = READY requests this step */
    uint64_t pinned;               /* KV blocks held by Preserve-paused requests (R23) */
    uint64_t budget;               /* kv_total - pinned, clamped at 0 */
    uint64_t budget_used;          /* sum of demand blk(ctx+1) over the admitted (R19) */
    uint32_t n_admitted;           /* |runningBatch| */
    uint32_t n_preempted;          /* admitted last step, READY now, not admitted now */
    uint32_t blocked_head;         /* n_eligible > 0 and nothing admitted */
    uint32_t reserved;
    uint64_t id_base;              /* ids of this step's keys are id_base + (key & (2^id_bits-1)) */
    const uint64_t* admitted_ids;        /* host, ranked order, n_admitted */
    const uint8_t* admitted_strategy;    /* host, LAMPS_PRESERVE.. for each admitted */
    const uint64_t* preempted_ids;       /* host, n_preempted */
    const uint64_t* d_ranked_keys;       /* device, n_eligible ascending unique keys:
                                            key = (!starving << (SB+IB)) | (score << IB)
                                                  | (id - id_base) */
    const uint32_t* d_admitted_slots;    /* device, n_admitted */
} lamps_step_out;

/*
 * Snapshot view of the pool, one entry per slot (all arrays of length
 * capacity, caller-owned host memory).  Used by lamps_pool_import /
 * lamps_pool_export for tests, benches and checkpoints.
 * dbg_w (3 per slot: W_P, W_D, W_S) and dbg_score are export-only and need
 * LAMPS_DEBUG_OUT; they hold the values of the last step for READY slots (W
 * are 0 where a cached score was reused).  age / dirty / cached_score are the
 * selective-update state (R26); on import NULL means a fresh pool (every score
 * computed at the next step: age 0, dirty 1, cached_score 0).
 */
typedef struct {
    uint64_t* id;
    uint32_t *state, *has_api, *starving, *strategy, *cnt;
    uint32_t *ctx, *pre_rem, *api_ticks, *resp_len, *post_len, *pending;
    uint64_t* dbg_w;     /* may be NULL */
    uint64_t* dbg_score; /* may be NULL */
    uint32_t* age;       /* may be NULL; steps since the cached score was computed, <= 127 */
    uint32_t* dirty;     /* may be NULL; 1 = segment changed, recompute */
    uint64_t* cached_score; /* may be NULL */
} lamps_pool_io;

/*
 * lamps_init -- create a handle.  Two-phase: with d_workspace == NULL only
 * *ws_bytes is written (device bytes needed, 256-byte aligned).  Then call
 * again with a device buffer of at least that size (e.g. a torch uint8 CUDA
 * tensor) that the caller keeps alive until lamps_free.  All per-step device
 * state lives in that workspace.  The library itself allocates pinned host
 * staging / result buffers and, for the P2P transport only, the exchange
 * buffer (cudaMalloc, 2 x world x (max_batch + 1) x 32 B + flags): CUDA IPC
 * exports whole allocations, so it cannot be carved from the caller's buffer.
 * Both are released by lamps_free.
 * Errors: EINVAL (NULL pointer, invalid config field), ECUDA.
 */
int lamps_init(const lamps_config* cfg, void* d_workspace, size_t* ws_bytes, lamps_t** out);

/*
 * lamps_submit -- Alg.1 intake: n new requests arrive, in order.
 * Ids are assigned consecutively in arrival order and written to ids_out.
 * Each starts READY with ctx = prompt_len and owes its prefill,
 * pending = T_fwd(prompt_len).  Errors (nothing submitted):
 * EINVAL (NULL, has_api > 1, NaN/inf/negative/out-of-range duration,
 * prompt+pre+resp+post > LAMPS_INGEST_LIMIT, peak demand blk(...) >
 * kv_capacity_blocks), ENOSPC (the slot of a new id still holds a live request).
 */
int lamps_submit(lamps_t* h, const lamps_segment* segs, uint32_t n, uint64_t* ids_out);

/*
 * lamps_api_return -- Alg.1: the API of each PAUSED request ids[k]
 * returned actual_resp_len[k] tokens; next[k] holds the predictions of its
 * next segment (prompt_len ignored).  ctx grows by the response; the request
 * owes (R10) by its handling strategy D: T_fwd(ctx'), S: T_swap(C_i) +
 * T_fwd(ctx') - T_fwd(C_i), P: T_fwd(ctx') - T_fwd(C_i); it becomes READY.
 * Errors: ENOENT (unknown id or not PAUSED), EINVAL (duplicate id, bad
 * segment, infeasible) -- nothing applied.
 */
int lamps_api_return(lamps_t* h, const uint64_t* ids, const uint32_t* actual_resp_len,
                     const lamps_segment* next, uint32_t n);

/*
 * lamps_schedule_step -- one scheduling iteration (A0..A5 above).
 * ev[0..n_ev) (host memory) reports what happened to requests admitted by the
 * previous step; every other previously admitted request generated one token.
 * kv_total_blocks is the KV capacity available this step (<= kv_capacity_blocks).
 * Fills *out and returns after the GPU pass completed.
 * Errors: EINVAL (event for an id not admitted by the previous step,
 * duplicate event, unknown kind, kv_total_blocks too large), ECUDA.
 */
int lamps_schedule_step(lamps_t* h, const lamps_event* ev, uint32_t n_ev,
                        uint64_t kv_total_blocks, lamps_step_out* out);

/*
 * lamps_iterate -- one engine iteration in one call: the API returns, the new arrivals,
 * then one scheduling step with the engine's events, i.e. exactly
 *   lamps_api_return(returns); lamps_submit(arrivals); lamps_schedule_step(events)
 * but with one host synchronisation: every part is validated before any is applied (on
 * error nothing is applied), and on the fused path the returns, arrivals and events are
 * applied inside the step kernel's prologue (one staging copy, one kernel).  Arrivals are
 * ranked in this step; they cannot reuse the slots this iteration's FINISHED events free
 * (those are free from the next call on).  Arrival ids go to arrival_ids_out (may be NULL).
 * Errors: those of the three calls.
 */
typedef struct {
    const lamps_event* events;        /* reports on the previous step's batch */
    uint32_t n_events;
    uint32_t n_returns;
    const uint64_t* return_ids;       /* PAUSED requests whose API returned */
    const uint32_t* return_resp;      /* actual response tokens */
    const lamps_segment* return_next; /* predictions of their next segment */
    const lamps_segment* arrivals;    /* new requests, in arrival order */
    uint32_t n_arrivals;
    uint32_t reserved;
    uint64_t* arrival_ids_out;
    uint64_t kv_total_blocks;
} lamps_iteration;

int lamps_iterate(lamps_t* h, const lamps_iteration* it, lamps_step_out* out);

/* lamps_free -- release the handle (not the caller's workspace). */
int lamps_free(lamps_t* h);

/* ---- auxiliary entry points ---------------------------------------------- */

/* Last error message of the handle (static storage, never NULL). */
const char* lamps_last_error(const lamps_t* h);

/*
 * lamps_schedule_step_async -- the same step with no events, enqueued on the
 * handle's stream without waiting: nothing is copied to the host.  For
 * engines that capture the pass in their own stream/graph and for device-only
 * timing.  Fetch the result with lamps_step_result (which synchronises).
 */
int lamps_schedule_step_async(lamps_t* h, uint64_t kv_total_blocks);

/* Synchronise and fill *out with the last step's result. */
int lamps_step_result(lamps_t* h, lamps_step_out* out);

/*
 * lamps_pool_import -- replace the whole pool with a snapshot (io arrays of
 * length capacity).  Live slots (state != FREE) must hold ids with
 * id mod capacity == slot and id_base <= id < next_id, next_id - id_base <=
 * capacity.  The previous admitted list is cleared.  Errors: EINVAL.
 */
int lamps_pool_import(lamps_t* h, const lamps_pool_io* io, uint64_t id_base, uint64_t next_id);

/* lamps_pool_export -- copy the pool (and debug values if requested) to io. */
int lamps_pool_export(lamps_t* h, lamps_pool_io* io);

/* Copy the last step's ranked keys (n_eligible of them, or the head only under
 * LAMPS_HEAD_ONLY; *n_out receives the count) to host memory. */
int lamps_ranked_keys(lamps_t* h, uint64_t* host_out, uint64_t max_keys, uint64_t* n_out);

/*
 * Device-side launch statistics of the last step, for benches: the number of
 * kernels it launched and the number of radix passes that did work.
 */
int lamps_step_stats(lamps_t* h, uint32_t* kernels_launched, uint32_t* sort_passes);

/*
 * With LAMPS_TIMING: device time per phase summed over the steps recorded
 * since the last read (at most 4096 steps are kept), in milliseconds:
 * ms[0] = A0 events kernel, ms[1] = A1-A3 score/key kernel, ms[2] = A4 sort
 * (all radix passes), ms[3] = A5 admission kernel.  Synchronises the stream.
 */
int lamps_timing_read(lamps_t* h, double ms[4], uint32_t* n_steps);

/*
 * With LAMPS_TRACE on the fused path: the SM clock (clock64) of every CTA at
 * the phase boundaries of the last step, out[cta * 64 + k], k = 0 start,
 * 1 scored, 2 counts published, 3 after barrier 1, 4 count exchange done,
 * 5 after barrier 2, 6 scattered, 7 after barrier 3, 8 range sorted,
 * 9 admission done (CTA 0), 10..15 sub-phases, 16..31 range-sort sub-phases,
 * 30/31 range size / starving keys, 32..63 refinement levels of the
 * non-starving part (diagnostics; layout may change).
 * *n_cta receives the grid size.
 */
int lamps_trace_read(lamps_t* h, uint64_t* out, uint32_t max_words, uint32_t* n_cta);

/*
 * Multi-GPU.  With world > 1 a step ranks every shard's requests locally, takes
 * the head K (= max_batch, the GLOBAL batch limit) of the local order as
 * records, exchanges them with ONE all-gather, merges the world sorted runs
 * identically on every rank and cuts the global order against the global
 * budget (sum of kv_total - sum of pinned) and K; each rank admits its own
 * prefix.  The result equals one step over the union pool (global ids).
 * lamps_step_out then holds: n_eligible, pinned, n_admitted, n_preempted local;
 * budget, budget_used, blocked_head global.  Requires the fused path
 * (capacity <= #SM * 10240) and world * max_batch <= 8192.
 *
 * lamps_nccl_unique_id: fill out[128] with a new ncclUniqueId (LAMPS_ENCCL if
 * libnccl.so.2 cannot be loaded); broadcast it to every rank before lamps_init.
 */
int lamps_nccl_unique_id(void* out128);

/*
 * Loopback transport: one step of `world` shards that live in this process on
 * one device (handles created with transport LAMPS_XPORT_LOOPBACK, ranks
 * 0..world-1, same stream).  ev[r] / n_ev[r] / kv_total[r] / out[r] are the
 * per-shard arguments of lamps_schedule_step.  The all-gather is a device copy.
 */
int lamps_group_step(lamps_t* const* h, uint32_t world, const lamps_event* const* ev,
                     const uint32_t* n_ev, const uint64_t* kv_total, lamps_step_out* out);

/*
 * lamps_group_step_async -- the co-resident P2P shards of this process (n handles,
 * LAMPS_SHARE_DEVICE, one stream each, distinct ranks of one world; the other ranks may
 * live in other processes / on other GPUs and step in lockstep): enqueue one step on
 * every handle's stream without events and without waiting (results with
 * lamps_step_result per handle).  Every handle is validated before any is enqueued.
 * Errors: EINVAL (handles not such a group, kv_total > kv_capacity_blocks, pending
 * results unread on a handle is allowed), ECUDA.
 */
int lamps_group_step_async(lamps_t* const* h, uint32_t n, const uint64_t* kv_total);

/* ---- predictor ingest and error injection ---------------- */

#define LAMPS_NO_BIN 0xffffffffu
#define LAMPS_BIN_TOKENS 10u   /* predictor bins of 10 tokens */
#define LAMPS_MAX_BIN 49u      /* 50 bins */

/*
 * What is known about one segment before prediction: the measured values of
 * a trace (the INFERCEPT datasets carry them) or, for the length,
 * the length predictor's bin (the classifier itself -- OPT-125M +
 * a linear head -- needs trained weights and is out of scope).
 */
typedef struct {
    uint64_t key;        /* RNG stream of this record (e.g. the trace index); < 2^57 */
    uint32_t prompt_len; /* copied to the output */
    uint32_t pre_len;    /* measured decode tokens before the API (or in total) */
    uint32_t pre_bin;    /* LAMPS_NO_BIN, or the predictor's bin b <= LAMPS_MAX_BIN:
                            the length is the bin's midpoint 10 b + 5 */
    uint32_t resp_len;   /* API response tokens (has_api), copied */
    uint32_t post_len;   /* measured decode tokens after the API (has_api) */
    uint32_t api_ticks;  /* measured API duration in ticks, already quantised (R22) (has_api) */
    uint32_t has_api;    /* 0 or 1 */
    uint32_t reserved;   /* must be 0 */
} lamps_truth;

/*
 * Error injection of the paper's prediction study:
 * predicted = measured + error, error ~ N(0, p * measured), applied to the
 * output lengths (pre_len and post_len, p = len_error_ppm / 1e6) and to the API
 * duration (p = api_error_ppm / 1e6), clamped at 0 (reading R27).  The normal
 * draw is integer and counter-based, so it is reproducible bit for bit:
 *   w_k = splitmix64 output number n = (key*4 + field)*32 + k + 1 from `seed`
 *         (state seed + n * 0x9E3779B97F4A7C15, the standard finaliser),
 *         field 0 = pre_len, 1 = post_len, 2 = api_ticks, k = 0..16;
 *   X = sum_{k<16} popcount(w_k)  (Binomial(1024, 1/2): mean 512, sd 16);
 *   Z = (X - 512) * 2^16 + (w_16 >> 48) - 2^15   (z = Z / 2^20, sd ~ 1; the low
 *       term is a uniform dither across one binomial step);
 *   error = round-half-away(p_ppm * m * Z / (1e6 * 2^20)), exact 128-bit;
 *   predicted = min(max(m + error, 0), 2^24 (lengths) or 2^32 - 1 (ticks)).
 */
typedef struct {
    uint64_t seed;
    uint32_t len_error_ppm;  /* p for pre_len / post_len, parts per million, <= 10^7 */
    uint32_t api_error_ppm;  /* p for the API duration, parts per million, <= 10^7 */
} lamps_noise;

/*
 * lamps_predict -- turn n truths (host array) into predicted segments (host
 * array out[n], ready for lamps_submit / lamps_api_return).  Bin-to-length,
 * the normal draws and the rounding run on the GPU (k_predict) on the handle's
 * stream; out[k].api_seconds = api_ticks / ticks_per_second, which lamps_submit
 * quantises back to exactly api_ticks.  noise == NULL means no error (p = 0).
 * Synchronous.  Errors: EINVAL (NULL arrays with n > 0, has_api > 1, reserved
 * != 0, pre_bin out of range, key >= 2^57, ppm > 10^7), ECUDA.  The pool is
 * not touched.
 */
int lamps_predict(lamps_t* h, const lamps_truth* truth, uint32_t n, const lamps_noise* noise,
                  lamps_segment* out);

/*
 * Peer-memory transport (LAMPS_XPORT_P2P).  lamps_p2p_handle writes this rank's 64-byte
 * cudaIpcMemHandle of its exchange buffer (library-allocated, p2p layout) to out64;
 * the caller all-gathers the handles (e.g. torch.distributed) and passes them to
 * lamps_p2p_connect (world * 64 bytes, rank order), which maps every peer's buffer
 * (cudaIpcOpenMemHandle).  lamps_p2p_connect_local connects `world` handles of this
 * process that share one device (LAMPS_SHARE_DEVICE; the buffers are used directly).
 * Every rank must then call lamps_schedule_step the same number of times (the step
 * kernels wait for each other).  Errors: EINVAL (wrong transport / sizes), ECUDA.
 * A step whose peers' records do not all arrive within LAMPS_P2P_TIMEOUT_MS milliseconds
 * (environment variable read at lamps_init; default 10000) ends without admitting and
 * returns LAMPS_ENCCL ("peer exchange timed out"): the ranks are out of lockstep (a peer
 * died or stopped stepping) and the handles should be freed.
 */
int lamps_p2p_handle(lamps_t* h, void* out64);
int lamps_p2p_connect(lamps_t* h, const void* handles, size_t n_bytes);
int lamps_p2p_connect_local(lamps_t* const* hs, uint32_t world);

/* Library version (major << 16 | minor). */
uint32_t lamps_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LAMPS_H */
