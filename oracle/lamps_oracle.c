/*
 * lamps_oracle.c -- the CPU ORACLE for the LAMPS scheduling pass.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this file's
 * library.  The product path (include/lamps.h, paper_2410_18248_b200/) never
 * links, imports or calls it, and this file shares no code, header, table or
 * constant with that path.
 *
 * It is a plain, slow, obviously-correct transcription of the paper
 * (arXiv 2410.18248, "Fast Inference for Augmented Large Language Models",
 * /root/reference/PAPER.md, cited "P:<line>") in integer units, with the
 * readings of DESIGN.md section "Readings" (R1..R24) where the paper is silent.
 *
 *   - Eq. (1)-(3) memory waste of Preserve / Discard / Swap .... P:677-685
 *   - strategy = argmin waste, decided before scheduling ........ P:482
 *   - rank = area under predicted memory-over-time curve ........ P:1054-1057
 *   - only the next API counts (segments) ....................... P:1060-1063
 *   - Algorithm 1: sort, fill running batch, starvation counter . P:957-1028
 *   - starvation threshold, sticky tag, counter reset ........... P:1085
 *   - prefill cost shape k1*n^2*d ............................... P:1580
 *   - baseline rank keys FCFS / SJF / SJF by total length ....... P:818-822
 *   - selective score update (cached scores, refresh interval) .. P:1080
 *   - predictor bins (50 x 10 tokens) ........................... P:1115
 *   - error injection error ~ N(0, p*m) ......................... P:1450-1451
 *
 * Everything is computed with plain loops, exact 128-bit intermediates and
 * explicit clamps; sums are done by explicit summation (no closed forms), the
 * sort is qsort() with the three-level comparator, admission is a linear walk.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (see DESIGN.md "Oracle pins").  No function is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define O_OK 0
#define O_EINVAL (-1)
#define O_ENOSPC (-2)
#define O_ENOENT (-3)

/* request states (Alg.1: WaitingQueue, PQueue, DQueue, SQueue) */
#define O_FREE 0u
#define O_READY 1u
#define O_PAUSED_P 2u
#define O_PAUSED_D 3u
#define O_PAUSED_S 4u

/* handling strategies */
#define O_P 0u
#define O_D 1u
#define O_S 2u
#define O_NONE 3u

/* engine events (Alg.1 P:1004 "Remove finished", "encounterAPIcall") */
#define O_EV_API_CALL 1u
#define O_EV_FINISHED 2u

#define O_INGEST_LIMIT (1u << 24) /* reading R21: max tokens per request ingest */

/* rank policies (P:818-822 baselines, P:1078 LAMPS; reading R25) */
#define O_POL_LAMPS 0u
#define O_POL_FCFS 1u
#define O_POL_SJF 2u
#define O_POL_SJF_TOTAL 3u
#define O_MAX_INTERVAL 127u /* selective score update: refresh interval limit (R26) */

typedef struct {
    uint32_t capacity;      /* pool slots */
    uint32_t block_tokens;  /* B: tokens per KV block (paged KV) */
    uint64_t tau;           /* ticks per decode iteration (reading R3) */
    uint64_t A1, A2;        /* T_fwd(c) = (A1*c + A2*c^2) >> SH   (R1) */
    uint64_t S0, S1;        /* T_swap(c) = c ? (S0 + S1*c) >> SH : 0   (R2) */
    uint32_t SH;
    uint64_t c_other;       /* C_other, profiled (R4) */
    double ticks_per_second;
    uint32_t starvation_threshold; /* StarvationT, 100 in P:1085 */
    uint32_t max_batch;
    uint64_t kv_capacity_blocks;
    uint32_t score_bits;    /* scores clamp at 2^score_bits - 1 (R22) */
    uint32_t id_bits;
    uint32_t policy;        /* O_POL_* (R25) */
    uint32_t score_interval; /* LAMPS selective score update: refresh every k steps (R26); 0, 1 = always */
} ocfg;

typedef struct {
    uint64_t id;
    uint32_t state, has_api, starving, strategy, cnt;
    uint32_t ctx;       /* context tokens now */
    uint32_t pre_rem;   /* predicted decode tokens before next API / to completion */
    uint32_t api_ticks; /* predicted API duration T_INT, quantised */
    uint32_t resp_len;  /* predicted API response tokens */
    uint32_t post_len;  /* predicted decode tokens after the API */
    uint32_t pending;   /* ticks of prefill / swap-in owed */
    uint32_t age;       /* steps since the cached score was computed (R26) */
    uint32_t dirty;     /* segment changed since (submit / API return): recompute (R26) */
    uint64_t cached_score;
} oreq;

typedef struct {
    uint64_t id;
    uint32_t kind;
    uint32_t reserved;
} oevent;

typedef struct {
    uint32_t prompt_len, pre_len, resp_len, post_len;
    double api_seconds;
    uint32_t has_api;
    uint32_t pad;
} oseg;

typedef struct {
    uint64_t n_eligible;
    uint64_t pinned;
    uint64_t budget;
    uint64_t budget_used;
    uint32_t n_admitted;
    uint32_t n_preempted;
    uint32_t blocked_head;
    uint32_t pad;
} osummary;

/* ------------------------------------------------------------------ */
/* small arithmetic helpers                                           */
/* ------------------------------------------------------------------ */

static uint64_t clamp64(u128 x) { return x > (u128)UINT64_MAX ? UINT64_MAX : (uint64_t)x; }

/* blocks needed to hold n tokens: ceil(n / B), by integer division (paged KV) */
uint64_t o_blk(uint64_t n, uint32_t B) {
    uint64_t q = n / B;
    if (n % B != 0) q = q + 1;
    return q;
}

/* Ingest quantisation of a predicted API duration (reading R22):
 * ticks = llround(seconds * ticks_per_second), one IEEE multiply, round half
 * away from zero; rejected unless 0 <= result <= 2^32 - 1. */
int o_quantize(double seconds, double tps, uint32_t* ticks) {
    if (!isfinite(seconds) || seconds < 0.0) return O_EINVAL;
    if (!isfinite(tps) || !(tps > 0.0)) return O_EINVAL;
    volatile double x = seconds * tps; /* volatile: no contraction, no excess precision */
    if (!(x >= 0.0) || !(x < 4294967295.5)) return O_EINVAL;
    long long r = llround(x);
    if (r < 0 || r > 4294967295LL) return O_EINVAL;
    *ticks = (uint32_t)r;
    return O_OK;
}

int o_validate_cfg(const ocfg* c) {
    const uint64_t lim = (uint64_t)1 << 48;
    if (!c) return O_EINVAL;
    if (c->capacity == 0 || (c->capacity & (c->capacity - 1)) != 0) return O_EINVAL;
    if (c->capacity > (1u << 23)) return O_EINVAL;
    if (c->block_tokens == 0 || (c->block_tokens & (c->block_tokens - 1)) != 0) return O_EINVAL;
    if (c->A1 >= lim || c->A2 >= lim || c->S0 >= lim || c->S1 >= lim) return O_EINVAL;
    if (c->tau >= lim) return O_EINVAL;
    if (c->c_other > 0xffffffffull) return O_EINVAL;
    if (c->SH > 63) return O_EINVAL;
    if (!isfinite(c->ticks_per_second) || !(c->ticks_per_second > 0.0)) return O_EINVAL;
    if (c->starvation_threshold == 0) return O_EINVAL;
    if (c->max_batch == 0 || c->max_batch > 16384) return O_EINVAL;
    if (c->score_bits == 0 || c->id_bits == 0) return O_EINVAL;
    if (c->score_bits + c->id_bits + 1 > 64) return O_EINVAL;
    if (((uint64_t)1 << c->id_bits) < c->capacity) return O_EINVAL;
    if (c->policy > O_POL_SJF_TOTAL) return O_EINVAL;
    if ((c->policy == O_POL_SJF || c->policy == O_POL_SJF_TOTAL) && c->tau == 0) return O_EINVAL;
    if (c->score_interval > O_MAX_INTERVAL) return O_EINVAL;
    return O_OK;
}

/* T_fwd(C): model forwarding time for context C, with the Appendix
 * prefill shape k1*n^2*d plus a linear term (reading R1):
 *   T_fwd(c) = floor((A1*c + A2*c^2) / 2^SH), clamped to 2^64-1. */
uint64_t o_t_fwd(const ocfg* cfg, uint64_t c) {
    u128 lin = (u128)cfg->A1 * c;
    u128 quad = (u128)cfg->A2 * ((u128)c * c);
    u128 t = (lin + quad) >> cfg->SH;
    return clamp64(t);
}

/* T_swap(C): time to swap context C, reading R2:
 *   T_swap(0) = 0; else floor((S0 + S1*c) / 2^SH), clamped. */
uint64_t o_t_swap(const ocfg* cfg, uint64_t c) {
    if (c == 0) return 0;
    u128 t = ((u128)cfg->S0 + (u128)cfg->S1 * c) >> cfg->SH;
    return clamp64(t);
}

/* Eq. (1)-(3), with M dropped as a common factor (R5),
 * C_i = ctx + pre_rem (context at the API call),
 * C_other = c_other, C_batch = C_i + C_other (R4):
 *   W[0] = WastePreserve = T_INT * C_i
 *   W[1] = WasteDiscard  = T_fwd(C_i)*C_i + T_fwd(C_i)*C_other
 *   W[2] = WasteSwap     = 2 * T_swap(C_i) * C_batch
 * each clamped to 2^64-1. */
void o_wastes(const ocfg* cfg, uint64_t ctx, uint64_t pre_rem, uint64_t api_ticks,
              uint64_t W[3]) {
    uint64_t c_i = ctx + pre_rem;
    uint64_t c_batch = c_i + cfg->c_other;
    u128 wp = (u128)api_ticks * c_i;
    uint64_t tf = o_t_fwd(cfg, c_i);
    u128 wd = (u128)tf * c_i + (u128)tf * cfg->c_other;
    uint64_t ts = o_t_swap(cfg, c_i);
    u128 ws = (u128)2 * ts * c_batch;
    W[0] = clamp64(wp);
    W[1] = clamp64(wd);
    W[2] = clamp64(ws);
}

/* "INFERCEPT dynamically selects a strategy that minimizes memory waste"
 * (P:685); LAMPS makes the same choice before scheduling.  Ties go to
 * the first in the order Preserve, Discard, Swap (reading R6). */
uint32_t o_argmin3(const uint64_t W[3]) {
    uint32_t best = 0;
    for (uint32_t k = 1; k < 3; k++)
        if (W[k] < W[best]) best = k;
    return best;
}

/* HandlingRanking(r) (Alg.1 line P:979): the integral of the predicted
 * memory-over-time curve (curve shapes P:1054, Fig. P:909-933)
 * in KV blocks x ticks, over the remaining life of the request up to and
 * including its NEXT API call, reading R7-R10:
 *   pending rectangle  : blk(ctx) for `pending` ticks (owed prefill / swap-in)
 *   pre-API decode ramp: for j = 1..pre_rem, blk(ctx+j) for tau ticks each
 *   API phase          : P: blk(C_i) held for T_INT ticks
 *                        D: blk(C_i+resp) for T_fwd(C_i+resp) ticks (recompute)
 *                        S: blk(C_i) for T_swap(C_i) ticks, twice (out and in)
 *   post-API ramp      : for j = 1..post_len, blk(C_i+resp+j) for tau ticks
 * The sum is clamped to 2^score_bits - 1 (R22); the running sum is capped at
 * 2^score_bits, which cannot change the clamped result because every term is
 * non-negative. */
uint64_t o_score(const ocfg* cfg, const oreq* r, uint32_t strategy) {
    const uint32_t B = cfg->block_tokens;
    const u128 cap = (u128)1 << cfg->score_bits;
    u128 area = 0;
#define O_ADD(term)                       \
    do {                                  \
        area = area + (u128)(term);       \
        if (area > cap) area = cap;       \
    } while (0)

    O_ADD((u128)o_blk(r->ctx, B) * r->pending);
    for (uint64_t j = 1; j <= r->pre_rem; j++) O_ADD((u128)cfg->tau * o_blk((uint64_t)r->ctx + j, B));

    uint64_t c_i = (uint64_t)r->ctx + r->pre_rem;
    if (r->has_api) {
        if (strategy == O_P) {
            O_ADD((u128)o_blk(c_i, B) * r->api_ticks);
        } else if (strategy == O_D) {
            uint64_t c_re = c_i + r->resp_len;
            O_ADD((u128)o_blk(c_re, B) * o_t_fwd(cfg, c_re));
        } else if (strategy == O_S) {
            O_ADD((u128)o_blk(c_i, B) * o_t_swap(cfg, c_i)); /* swap-out */
            O_ADD((u128)o_blk(c_i, B) * o_t_swap(cfg, c_i)); /* swap-in  */
        }
        uint64_t c_post = c_i + r->resp_len;
        for (uint64_t j = 1; j <= r->post_len; j++) O_ADD((u128)cfg->tau * o_blk(c_post + j, B));
    }
#undef O_ADD
    u128 maxs = cap - 1;
    return (uint64_t)(area < maxs ? area : maxs);
}

/* Baseline rank keys (reading R25), lower = earlier, clamped to 2^score_bits - 1:
 *   FCFS      : 0 for every request, so the order is the request id, i.e. arrival
 *               ("determines their order based on request ID")
 *   SJF       : remaining length of the current segment in decode iterations:
 *               pre_rem + post_len + the owed prefill / swap-in, ceil(pending / tau)
 *               ("based only on length"; "a post-API part of length 2
 *               (including recomputation)")
 *   SJF_TOTAL : SJF + the API duration in decode iterations, ceil(api_ticks / tau)
 *               ("output length plus API duration")
 * LAMPS is o_score. */
static uint64_t ceil_div(uint64_t a, uint64_t b) {
    uint64_t q = a / b;
    if (a % b != 0) q = q + 1;
    return q;
}

uint64_t o_policy_score(const ocfg* cfg, const oreq* r) {
    uint64_t v = 0;
    if (cfg->policy == O_POL_SJF || cfg->policy == O_POL_SJF_TOTAL) {
        v = r->pre_rem;
        if (r->has_api) v = v + r->post_len;
        v = v + ceil_div(r->pending, cfg->tau);
    }
    if (cfg->policy == O_POL_SJF_TOTAL && r->has_api) v = v + ceil_div(r->api_ticks, cfg->tau);
    uint64_t maxs = (cfg->score_bits >= 64) ? UINT64_MAX : (((uint64_t)1 << cfg->score_bits) - 1);
    return v < maxs ? v : maxs;
}

/* ------------------------------------------------------------------ */
/* ingest: submit (Alg.1) and API return (Alg.1)  */
/* ------------------------------------------------------------------ */

static int seg_check(const ocfg* cfg, uint64_t ctx0, const oseg* s, uint32_t* ticks) {
    if (s->has_api > 1) return O_EINVAL;
    uint64_t total = ctx0 + s->pre_len;
    *ticks = 0;
    if (s->has_api) {
        total += (uint64_t)s->resp_len + s->post_len;
        if (o_quantize(s->api_seconds, cfg->ticks_per_second, ticks) != O_OK) return O_EINVAL;
    }
    if (total > O_INGEST_LIMIT) return O_EINVAL;
    /* a request that can never fit is reported infeasible */
    if (o_blk(total, cfg->block_tokens) > cfg->kv_capacity_blocks) return O_EINVAL;
    return O_OK;
}

/* Submit n requests: ids are assigned in arrival order starting at *next_id;
 * slot = id mod capacity must be free (else ENOSPC).  ctx = prompt_len,
 * pending = T_fwd(prompt_len) (the prefill owed), state READY.
 * All-or-nothing: on any error the pool is unchanged. */
int o_submit(const ocfg* cfg, oreq* pool, uint64_t* next_id, const oseg* segs, uint32_t n,
             uint64_t* ids_out) {
    uint32_t* ticks = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    if (!ticks) return O_EINVAL;
    for (uint32_t k = 0; k < n; k++) {
        if (seg_check(cfg, segs[k].prompt_len, &segs[k], &ticks[k]) != O_OK) {
            free(ticks);
            return O_EINVAL;
        }
        uint64_t id = *next_id + k;
        if (n > cfg->capacity || pool[id % cfg->capacity].state != O_FREE) {
            free(ticks);
            return O_ENOSPC;
        }
    }
    for (uint32_t k = 0; k < n; k++) {
        uint64_t id = *next_id + k;
        oreq* r = &pool[id % cfg->capacity];
        memset(r, 0, sizeof(*r));
        r->id = id;
        r->state = O_READY;
        r->has_api = segs[k].has_api;
        r->starving = 0;
        r->strategy = O_NONE;
        r->cnt = 0;
        r->ctx = segs[k].prompt_len;
        r->pre_rem = segs[k].pre_len;
        r->api_ticks = segs[k].has_api ? ticks[k] : 0;
        r->resp_len = segs[k].has_api ? segs[k].resp_len : 0;
        r->post_len = segs[k].has_api ? segs[k].post_len : 0;
        uint64_t pf = o_t_fwd(cfg, r->ctx);
        r->pending = pf > 0xffffffffull ? 0xffffffffu : (uint32_t)pf;
        r->dirty = 1; /* a new segment: its score is computed at the next step (R26) */
        if (ids_out) ids_out[k] = id;
    }
    *next_id += n;
    free(ticks);
    return O_OK;
}

static oreq* find_live(const ocfg* cfg, oreq* pool, uint64_t id) {
    oreq* r = &pool[id % cfg->capacity];
    if (r->state == O_FREE || r->id != id) return NULL;
    return r;
}

/* API return (Alg.1; multi-API re-entry as a new segment,
 * P:1060-1063).  ctx grows by the actual response tokens; the request owes
 * (reading R10) the work its frozen strategy left undone:
 *   D: T_fwd(ctx')                       (full recompute)
 *   S: T_swap(C_i) + T_fwd(ctx') - T_fwd(C_i)   (swap-in + prefill of the response)
 *   P: T_fwd(ctx') - T_fwd(C_i)          (prefill of the response)
 * with C_i = ctx before the response. */
int o_api_return(const ocfg* cfg, oreq* pool, const uint64_t* ids, const uint32_t* actual_resp,
                 const oseg* next, uint32_t n) {
    uint32_t* ticks = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    if (!ticks) return O_EINVAL;
    for (uint32_t k = 0; k < n; k++) {
        oreq* r = find_live(cfg, pool, ids[k]);
        if (!r || r->state < O_PAUSED_P) {
            free(ticks);
            return O_ENOENT;
        }
        for (uint32_t q = 0; q < k; q++)
            if (ids[q] == ids[k]) {
                free(ticks);
                return O_EINVAL;
            }
        uint64_t ctx1 = (uint64_t)r->ctx + actual_resp[k];
        if (seg_check(cfg, ctx1, &next[k], &ticks[k]) != O_OK) {
            free(ticks);
            return O_EINVAL;
        }
    }
    for (uint32_t k = 0; k < n; k++) {
        oreq* r = find_live(cfg, pool, ids[k]);
        uint64_t c_i = r->ctx;
        uint64_t ctx1 = c_i + actual_resp[k];
        uint64_t owed;
        uint64_t f1 = o_t_fwd(cfg, ctx1), f0 = o_t_fwd(cfg, c_i);
        uint64_t inc = f1 >= f0 ? f1 - f0 : 0;
        if (r->state == O_PAUSED_D) {
            owed = f1;
        } else if (r->state == O_PAUSED_S) {
            u128 s = (u128)o_t_swap(cfg, c_i) + inc;
            owed = clamp64(s);
        } else {
            owed = inc;
        }
        r->pending = owed > 0xffffffffull ? 0xffffffffu : (uint32_t)owed;
        r->ctx = (uint32_t)ctx1;
        r->pre_rem = next[k].pre_len;
        r->has_api = next[k].has_api;
        r->api_ticks = next[k].has_api ? ticks[k] : 0;
        r->resp_len = next[k].has_api ? next[k].resp_len : 0;
        r->post_len = next[k].has_api ? next[k].post_len : 0;
        r->state = O_READY;
        r->dirty = 1; /* a new segment: recompute its score (R26) */
    }
    free(ticks);
    return O_OK;
}

/* ------------------------------------------------------------------ */
/* one scheduling iteration: Algorithm 1 body            */
/* ------------------------------------------------------------------ */

typedef struct {
    uint64_t id;
    uint64_t score;
    uint32_t starving;
    uint32_t slot;
} oent;

/* Sort(WaitingQueue) by r.score; starving requests at the head with
 * their relative rank kept (Alg.1); equal scores by request
 * id, i.e. arrival order ("index of the requests"). */
static int ent_cmp(const void* a, const void* b) {
    const oent* x = (const oent*)a;
    const oent* y = (const oent*)b;
    if (x->starving != y->starving) return x->starving ? -1 : 1;
    if (x->score != y->score) return x->score < y->score ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return 0;
}

/*
 * One step.  Inputs: the pool (one oreq per slot, mutated), the ids admitted
 * by the previous step, the engine events observed while executing them, and
 * the KV blocks available this step.  Outputs: summary, ranked order, the
 * admitted prefix, the preempted list, and per-slot debug values.
 *
 *  A0  events.  Every previously admitted request executed one iteration
 *      (iteration-level scheduling): ctx += 1, pre_rem -= 1 (not
 *      below 0), pending = 0.  Then, in array order: API_CALL routes the
 *      request to P/D/S (Alg.1) by argmin waste at C_i = ctx and
 *      resets its counter unless it is starving; FINISHED frees it
 *      (P:1004).
 *  A1  strategy = argmin(Eq.1-3) for READY requests with an API.
 *  A2  score = memory-over-time area.
 *  A3  starving |= cnt >= StarvationT (Alg.1; sticky).
 *  A4  sort.
 *  A5  fill runningBatch while it is not full: budget =
 *      kv_total - sum over Preserve-paused of blk(ctx) (R23); walk the ranked
 *      queue accumulating blk(ctx+1) (R19); stop at the first request that
 *      does not fit or at max_batch (R15).  Admitted -> cnt = 0, others
 *      cnt += 1 (Alg.1; saturating at 65535).
 *
 * Output arrays must hold: ranked_* >= capacity, adm_* >= max_batch,
 * pre_id >= n_prev, dbg >= 4*capacity (W_P, W_D, W_S, score per slot),
 * dbg_strategy >= capacity.  dbg / dbg_strategy may be NULL.
 * Returns O_EINVAL (pool unchanged) on invalid events or kv_total.
 */
int o_step(const ocfg* cfg, oreq* pool, const uint64_t* prev_adm, uint32_t n_prev,
           const oevent* ev, uint32_t n_ev, uint64_t kv_total, osummary* out,
           uint64_t* ranked_id, uint64_t* ranked_score, uint8_t* ranked_starving,
           uint64_t* adm_id, uint8_t* adm_strategy, uint64_t* pre_id, uint64_t* dbg,
           uint8_t* dbg_strategy) {
    const uint32_t cap = cfg->capacity;
    const uint32_t B = cfg->block_tokens;

    /* ---- validation (state unchanged on error) ---- */
    if (kv_total > cfg->kv_capacity_blocks) return O_EINVAL;
    for (uint32_t e = 0; e < n_ev; e++) {
        int found = 0;
        if (ev[e].kind != O_EV_API_CALL && ev[e].kind != O_EV_FINISHED) return O_EINVAL;
        for (uint32_t k = 0; k < n_prev; k++)
            if (prev_adm[k] == ev[e].id) found = 1;
        if (!found) return O_EINVAL;
        for (uint32_t q = 0; q < e; q++)
            if (ev[q].id == ev[e].id) return O_EINVAL;
    }

    /* ---- A0: the previous batch executed one iteration ---- */
    for (uint32_t k = 0; k < n_prev; k++) {
        oreq* r = find_live(cfg, pool, prev_adm[k]);
        if (!r || r->state != O_READY) continue;
        r->ctx = r->ctx + 1;
        r->pre_rem = r->pre_rem > 0 ? r->pre_rem - 1 : 0;
        r->pending = 0;
    }
    for (uint32_t e = 0; e < n_ev; e++) {
        oreq* r = find_live(cfg, pool, ev[e].id);
        if (!r) continue;
        if (ev[e].kind == O_EV_FINISHED) {
            r->state = O_FREE;
        } else {
            /* Alg.1: the request is routed by r.handling, the label of the ranking
             * pass that admitted it (reading R11); a request without one (never ranked
             * with an API ahead) takes the argmin of Eq. (1)-(3) at C_i = ctx */
            r->pre_rem = 0;
            if (r->strategy == O_NONE) {
                uint64_t W[3];
                o_wastes(cfg, r->ctx, 0, r->api_ticks, W);
                r->strategy = o_argmin3(W);
            }
            r->state = O_PAUSED_P + r->strategy;
            if (!r->starving) r->cnt = 0;
        }
    }

    /* ---- pinned Preserve blocks (R23) and the waiting queue E ---- */
    uint64_t pinned = 0;
    uint32_t n_e = 0;
    oent* E = (oent*)malloc(sizeof(oent) * (cap ? cap : 1));
    if (!E) return O_EINVAL;
    for (uint32_t s = 0; s < cap; s++) {
        oreq* r = &pool[s];
        if (dbg) {
            dbg[4 * s + 0] = dbg[4 * s + 1] = dbg[4 * s + 2] = dbg[4 * s + 3] = 0;
        }
        if (dbg_strategy) dbg_strategy[s] = O_NONE;
        if (r->state == O_PAUSED_P) pinned += o_blk(r->ctx, B);
        if (r->state != O_READY) continue;

        /* A1 + A2.  LAMPS with selective score update (reading R26):
         * a READY request keeps the strategy and score of its last computation
         * unless its segment changed or that computation is score_interval steps
         * old.  Baseline policies (R25) rank by their own key, always fresh; their
         * strategy is still the argmin of Eq. (1)-(3). */
        uint64_t W[3] = {0, 0, 0};
        uint32_t strat = O_NONE;
        uint64_t sc;
        int fresh = cfg->policy != O_POL_LAMPS || cfg->score_interval <= 1 || r->dirty ||
                    r->age + 1 >= cfg->score_interval;
        if (fresh) {
            if (r->has_api) {
                o_wastes(cfg, r->ctx, r->pre_rem, r->api_ticks, W);
                strat = o_argmin3(W);
            }
            r->strategy = strat;
            sc = cfg->policy == O_POL_LAMPS ? o_score(cfg, r, strat) : o_policy_score(cfg, r);
            if (cfg->policy == O_POL_LAMPS && cfg->score_interval > 1) r->cached_score = sc; /* the cache exists only then */
            r->age = 0;
            r->dirty = 0;
        } else {
            strat = r->strategy;
            sc = r->cached_score;
            r->age = r->age + 1;
        }
        /* A3 */
        if (r->cnt >= cfg->starvation_threshold) r->starving = 1;

        E[n_e].id = r->id;
        E[n_e].score = sc;
        E[n_e].starving = r->starving;
        E[n_e].slot = s;
        n_e++;
        if (dbg) {
            dbg[4 * s + 0] = W[0];
            dbg[4 * s + 1] = W[1];
            dbg[4 * s + 2] = W[2];
            dbg[4 * s + 3] = sc;
        }
        if (dbg_strategy) dbg_strategy[s] = (uint8_t)strat;
    }

    /* ---- A4 ---- */
    qsort(E, n_e, sizeof(oent), ent_cmp);

    /* ---- A5 ---- */
    uint64_t budget = kv_total > pinned ? kv_total - pinned : 0;
    uint64_t used = 0;
    uint32_t n_adm = 0;
    for (uint32_t k = 0; k < n_e; k++) {
        if (n_adm == cfg->max_batch) break;
        oreq* r = &pool[E[k].slot];
        uint64_t d = o_blk((uint64_t)r->ctx + 1, B);
        if (used + d > budget) break;
        used += d;
        adm_id[n_adm] = r->id;
        adm_strategy[n_adm] = (uint8_t)r->strategy;
        n_adm++;
    }
    for (uint32_t k = 0; k < n_e; k++) {
        oreq* r = &pool[E[k].slot];
        if (k < n_adm)
            r->cnt = 0;
        else
            r->cnt = r->cnt < 65535 ? r->cnt + 1 : 65535;
        ranked_id[k] = E[k].id;
        ranked_score[k] = E[k].score;
        ranked_starving[k] = (uint8_t)E[k].starving;
    }

    /* preempted: previously admitted, still READY, not admitted now */
    uint32_t n_pre = 0;
    for (uint32_t k = 0; k < n_prev; k++) {
        oreq* r = find_live(cfg, pool, prev_adm[k]);
        if (!r || r->state != O_READY) continue;
        int again = 0;
        for (uint32_t q = 0; q < n_adm; q++)
            if (adm_id[q] == prev_adm[k]) again = 1;
        if (!again) pre_id[n_pre++] = prev_adm[k];
    }

    out->n_eligible = n_e;
    out->pinned = pinned;
    out->budget = budget;
    out->budget_used = used;
    out->n_admitted = n_adm;
    out->n_preempted = n_pre;
    out->blocked_head = (n_e > 0 && n_adm == 0) ? 1u : 0u;
    free(E);
    return O_OK;
}

/* ------------------------------------------------------------------ */
/* Predictor ingest and error injection (row F4, reading R27)         */
/* ------------------------------------------------------------------ */

typedef struct {
    uint64_t key;
    uint32_t prompt_len, pre_len, pre_bin, resp_len, post_len, api_ticks, has_api, reserved;
} otruth;

typedef struct {
    uint32_t pre_len, resp_len, post_len, api_ticks;
} opred;

#define O_NO_BIN 0xffffffffu

/* splitmix64 (Steele, Lea, Flood 2014; Vigna's reference C): the generator's
 * state advances by the golden gamma before every output, so output number n
 * (1-based) of the generator seeded with `seed` is next() called on the state
 * seed + (n - 1) * gamma. */
static uint64_t o_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t o_splitmix_output(uint64_t seed, uint64_t n) {
    uint64_t state = seed + (n - 1) * 0x9E3779B97F4A7C15ull;
    return o_splitmix_next(&state);
}

/* number of one bits, bit by bit */
static uint32_t o_popcount(uint64_t w) {
    uint32_t c = 0;
    for (int b = 0; b < 64; b++)
        if ((w >> b) & 1ull) c = c + 1;
    return c;
}

/* The normal draw of reading R27 for (key, field), in units of 2^-20:
 * X = number of one bits in the 16 words n0 .. n0+15, Binomial(1024, 1/2)
 * (mean 512, standard deviation sqrt(1024/4) = 16), standardised and scaled:
 * (X - 512) / 16 * 2^20 = (X - 512) * 2^16; plus the top 16 bits of word
 * n0+16 centred, a uniform dither across one binomial step (1/16). */
int64_t o_normal_q20(uint64_t seed, uint64_t key, uint32_t field) {
    const uint64_t n0 = (key * 4 + field) * 32 + 1;
    uint32_t X = 0;
    for (uint32_t k = 0; k < 16; k++) X += o_popcount(o_splitmix_output(seed, n0 + k));
    const int64_t U = (int64_t)(o_splitmix_output(seed, n0 + 16) >> 48);
    return ((int64_t)X - 512) * 65536 + (U - 32768);
}

/* predicted = measured + error, error = p * m * z with
 * p = ppm / 10^6 and z = Z / 2^20, rounded half away from zero, then clamped
 * at 0 and at `hi` (reading R27). */
uint32_t o_perturb(uint32_t m, uint32_t ppm, int64_t Z, uint64_t hi) {
    const u128 num_mag = (u128)ppm * m * (u128)(Z < 0 ? -Z : Z);
    const u128 den = (u128)1000000 * 1048576;
    u128 q = num_mag / den;
    const u128 r = num_mag % den;
    if (2 * r >= den) q = q + 1; /* half away from zero (on the magnitude) */
    int64_t v = (int64_t)m;
    if (Z < 0) v = v - (int64_t)q;
    else v = v + (int64_t)q;
    if (v < 0) v = 0;
    if ((uint64_t)v > hi) v = (int64_t)hi;
    return (uint32_t)v;
}

/* Truths -> predicted segment fields.  pre_len comes from the bin midpoint
 * 10 b + 5 when a bin is given (50 bins of 10 tokens); the output
 * lengths (pre, post) get p = len_ppm, the API duration p = api_ppm; the
 * response length is passed through. */
int o_predict(const otruth* t, uint32_t n, uint64_t seed, uint32_t len_ppm, uint32_t api_ppm, opred* out) {
    if (len_ppm > 10000000u || api_ppm > 10000000u) return O_EINVAL;
    for (uint32_t k = 0; k < n; k++) {
        if (t[k].has_api > 1 || t[k].reserved != 0) return O_EINVAL;
        if (t[k].pre_bin != O_NO_BIN && t[k].pre_bin > 49) return O_EINVAL;
        if ((t[k].key >> 57) != 0) return O_EINVAL;
    }
    for (uint32_t k = 0; k < n; k++) {
        uint32_t pre = t[k].pre_len;
        if (t[k].pre_bin != O_NO_BIN) pre = 10 * t[k].pre_bin + 5;
        opred r = {0, 0, 0, 0};
        r.pre_len = pre;
        if (len_ppm != 0) r.pre_len = o_perturb(pre, len_ppm, o_normal_q20(seed, t[k].key, 0), O_INGEST_LIMIT);
        if (t[k].has_api) {
            r.resp_len = t[k].resp_len;
            r.post_len = t[k].post_len;
            r.api_ticks = t[k].api_ticks;
            if (len_ppm != 0)
                r.post_len = o_perturb(t[k].post_len, len_ppm, o_normal_q20(seed, t[k].key, 1), O_INGEST_LIMIT);
            if (api_ppm != 0)
                r.api_ticks = o_perturb(t[k].api_ticks, api_ppm, o_normal_q20(seed, t[k].key, 2), 4294967295ull);
        }
        out[k] = r;
    }
    return O_OK;
}

/* size helpers so the Python wrapper can check its struct layouts */
uint32_t o_sizeof_req(void) { return (uint32_t)sizeof(oreq); }
uint32_t o_sizeof_cfg(void) { return (uint32_t)sizeof(ocfg); }
uint32_t o_sizeof_seg(void) { return (uint32_t)sizeof(oseg); }
uint32_t o_sizeof_summary(void) { return (uint32_t)sizeof(osummary); }
uint32_t o_sizeof_event(void) { return (uint32_t)sizeof(oevent); }
