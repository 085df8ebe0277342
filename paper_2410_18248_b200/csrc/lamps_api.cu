// lamps_api.cu -- host runtime behind include/lamps.h.
//
// Validation, ingest quantisation, the host shadow of request liveness (id
// window, paused/ready), workspace carving, pinned staging and the launch
// sequence of one step: K0 events -> K1 score/key -> K2 radix passes -> K3
// admission.  Every step of the method runs in the kernels; the host only
// moves inputs and outputs.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "lamps.h"
#include "lamps_internal.h"

using namespace lamps;

namespace {

constexpr uint32_t kIngestChunk = 65536;
constexpr uint32_t kTimingRing = 4096;
constexpr size_t kAlign = 256;
enum : uint8_t { H_FREE = 0, H_READY = 1, H_PAUSED = 2 };

size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// Ingest quantisation (reading R22): ticks = round-half-away(seconds * tps),
// one IEEE double multiply; accepted iff the result is in [0, 2^32 - 1].
bool quantize(double seconds, double tps, uint32_t* out) {
    if (!std::isfinite(seconds) || seconds < 0.0) return false;
    volatile double x = seconds * tps;
    const double xv = x;
    if (!(xv >= 0.0) || !(xv < 4294967295.5)) return false;
    const double r = std::round(xv);
    if (r > 4294967295.0) return false;
    *out = (uint32_t)r;
    return true;
}

// ---- NCCL, loaded at run time (only multi-GPU handles need it) ----------------
typedef void* nccl_comm_t;
struct NcclApi {
    void* so = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    int (*commInitRank)(nccl_comm_t*, int, const void* /* by value 128 B, see call */, int) = nullptr;
    int (*allGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*commDestroy)(nccl_comm_t) = nullptr;
    const char* (*getErrorString)(int) = nullptr;
    bool load() {
        if (so) return true;
        so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!so) return false;
        getUniqueId = (int (*)(void*))dlsym(so, "ncclGetUniqueId");
        allGather = (int (*)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t))dlsym(so, "ncclAllGather");
        commDestroy = (int (*)(nccl_comm_t))dlsym(so, "ncclCommDestroy");
        getErrorString = (const char* (*)(int))dlsym(so, "ncclGetErrorString");
        return getUniqueId && allGather && commDestroy && dlsym(so, "ncclCommInitRank");
    }
};
NcclApi g_nccl;
struct NcclId { char internal[128]; };  // ncclUniqueId is passed by value
typedef int (*CommInitRankFn)(nccl_comm_t*, int, NcclId, int);
constexpr int kNcclUint8 = 1;  // ncclUint8 in ncclDataType_t

// Exchange buffers exported by this process: a handle of one of them is mapped to its own
// pointer by lamps_p2p_connect (CUDA IPC cannot open a handle in the exporting process), so
// co-resident shards of this process and shards in other processes connect the same way.
std::mutex g_exp_mu;
std::vector<std::pair<cudaIpcMemHandle_t, MergeRec*>> g_exported;

struct Layout {
    size_t off = 0;
    size_t take(size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes);
        return o;
    }
};

}  // namespace

struct lamps_s {
    lamps_config cfg{};
    cudaStream_t stream = nullptr;
    Cost cost{};
    Bufs b{};
    uint32_t cap = 0, cap_pad = 0, score_grid = 0, sort_grid = 0, fused_grid = 0;
    uint32_t big_ranges = 0, big_grid = 0, big_cta_slots = 0;
    bool fused = false;
    bool small = false;   // fused family: the one-CTA small-pool step kernel (k_small)
    bool big = false;     // pools above the fused kernel's capacity: k_big_score + k_big_sort
    bool cold = true;     // fused: no splitters yet (StepArgs.cold); a fused step writes the next's
    uint32_t world = 1, rank = 0;
    bool merge = false;  // merge_mode(cfg)
    // peer-memory transport
    MergeRec* xbuf = nullptr;            // own exchange buffer (cudaMalloc, IPC-exportable)
    MergeRec** d_peers = nullptr;        // device table of the world ranks' buffers
    std::vector<void*> peer_open;        // IPC mappings to close
    bool p2p_ready = false;
    uint32_t xseq = 0;
    uint32_t xtimeout_ms = 10000;  // P2P: longest wait for the peers (env LAMPS_P2P_TIMEOUT_MS)
    uint32_t tune = 0;  // StepArgs.tune, from env LAMPS_TUNE (A/B measurements)
    uint32_t ret_pending = 0;  // API returns staged for the next fused step's prologue
    uint32_t sub_pending = 0;  // arrivals staged for the next fused step's prologue
    bool inl_pending = false;  // ... staged in `inl` (the kernel's parameter block)
    InlineStage inl{};
    nccl_comm_t comm = nullptr;
    uint8_t* ws = nullptr;
    // device ingest staging (inside the workspace)
    void* d_ingest = nullptr;
    const void* d_events = nullptr;
    uint32_t* d_gather = nullptr;
    // host shadow
    std::vector<uint8_t> hstate;
    std::vector<uint32_t> hctx;  // host shadow of each slot's context length (ingest checks
                                 // without a device round trip): submit, +1 per admission
                                 // (applied by the next step's A0), + response at API return
    bool shadow_ok = true;       // false once a step's admitted list went unread (async use)
    std::vector<uint32_t> adm_mark;  // per slot: step that last admitted it (event validation)
    std::vector<uint32_t> ev_mark;   // per slot: tag of the last event batch naming it
    uint32_t ev_tag = 0;
    uint32_t fetched_step = 0;   // last step whose admitted list entered the shadow
    uint64_t next_id = 0, id_base = 0;
    uint32_t step = 0;
    std::vector<uint64_t> prev_adm;
    bool prev_known = true;
    uint64_t last_id_base = 0;
    uint32_t last_kernels = 0;
    // pinned host buffers
    void* h_ingest = nullptr;
    lamps_event* h_ev = nullptr;
    Ctl* h_ctl = nullptr;
    uint64_t* h_adm_ids = nullptr;
    uint8_t* h_adm_strat = nullptr;
    uint64_t* h_pre_ids = nullptr;
    bool have_result = false;
    // mapped pinned result block (written by the admission kernel)
    void* h_res = nullptr;
    HostRes* hres = nullptr;
    // staging reuse: the last host-to-device copy out of h_ingest
    cudaEvent_t ing_ev = nullptr;
    bool ing_pending = false;
    // timing ring
    std::vector<cudaEvent_t> tev;
    uint32_t t_count = 0, t_head = 0;
    std::string err;
};

namespace {

int fail(lamps_t* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    return code;
}

int cuda_fail(lamps_t* h, cudaError_t e, const char* where) {
    return fail(h, LAMPS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(h, call)                                        \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
    } while (0)

bool pow2(uint64_t x) { return x && !(x & (x - 1)); }

const char* validate_cfg(const lamps_config* c) {
    const uint64_t lim = 1ull << 48;
    if (!pow2(c->capacity) || c->capacity > (1u << 23)) return "capacity must be a power of 2 <= 2^23";
    if (!pow2(c->block_tokens)) return "block_tokens must be a power of 2";
    if (c->tau >= lim || c->A1 >= lim || c->A2 >= lim || c->S0 >= lim || c->S1 >= lim)
        return "tau, A1, A2, S0, S1 must be < 2^48";
    if (c->SH > 63) return "SH must be <= 63";
    if (c->c_other > 0xffffffffull) return "c_other must be < 2^32";
    if (!std::isfinite(c->ticks_per_second) || !(c->ticks_per_second > 0.0))
        return "ticks_per_second must be finite and > 0";
    if (c->starvation_threshold == 0) return "starvation_threshold must be >= 1";
    if (c->max_batch == 0 || c->max_batch > (uint32_t)kMaxBatch) return "max_batch must be 1..16384";
    if (c->score_bits == 0 || c->id_bits == 0 || c->score_bits + c->id_bits + 1 > 64)
        return "need score_bits, id_bits >= 1 and score_bits + id_bits + 1 <= 64";
    if (c->id_bits < 64 && (1ull << c->id_bits) < c->capacity) return "2^id_bits must be >= capacity";
    if (c->policy > LAMPS_POLICY_SJF_TOTAL) return "unknown policy";
    if ((c->policy == LAMPS_POLICY_SJF || c->policy == LAMPS_POLICY_SJF_TOTAL) && c->tau == 0)
        return "SJF and SJF_TOTAL need tau >= 1";
    if (c->score_interval > 127) return "score_interval must be <= 127";
    if (c->world > 1 || (c->flags & LAMPS_MERGE)) {
        if (c->world > 32 || c->rank >= (c->world > 1 ? c->world : 1u)) return "need rank < world <= 32";
        if (c->transport == LAMPS_XPORT_P2P && (uint64_t)c->world * c->max_batch > kMergeMaxRecords)
            return "P2P transport: world * max_batch must be <= 8192 (the in-kernel merge); NCCL / loopback merge any";
        if (c->transport > LAMPS_XPORT_P2P) return "unknown transport";
        if (c->local_ranks > (c->world > 1 ? c->world : 1u)) return "local_ranks must be <= world";
        if (c->transport == LAMPS_XPORT_NCCL && !c->nccl_id) return "NCCL transport needs nccl_id";
        if (c->world <= 1 && c->transport == LAMPS_XPORT_LOOPBACK)
            return "LAMPS_MERGE at world 1 needs the NCCL or P2P transport";
        if (c->transport == LAMPS_XPORT_P2P &&
            merge_smem_bytes(c->world > 1 ? c->world : 1u, c->max_batch) + 1024 > fused_smem_bytes())
            return "P2P transport: world * max_batch too large for the in-kernel merge";
    }
    return nullptr;
}

// the multi-shard path (records, all-gather, merge kernel): world > 1, or a
// 1-rank NCCL communicator when LAMPS_MERGE is set (exercises the exchange on one GPU)
bool merge_mode(const lamps_config& c) { return c.world > 1 || (c.flags & LAMPS_MERGE); }

size_t carve(lamps_t* h, uint8_t* base) {
    // base == nullptr: size only
    const uint32_t cap_pad = h->cap_pad;
    const uint32_t mb = h->cfg.max_batch;
    Layout L;
    size_t o_soa[10];  // sfc, ctx, pre, api, resp, post, pend, stamp, score cache lo / hi
    for (int i = 0; i < 10; i++) o_soa[i] = L.take((size_t)cap_pad * 4);
    // keys0: in the fused kernel, range r's keys are written to [r * kFusedKcap, ...)
    size_t o_keys0 = L.take(std::max((size_t)cap_pad + kSortTile, h->fused ? (size_t)h->fused_grid * kFusedKcap : 0) * 8);
    size_t o_keys1 = L.take(((size_t)cap_pad + kSortTile) * 8);
    const uint32_t gmax = std::max(std::max(h->score_grid, h->big_grid), std::max(h->sort_grid, h->fused_grid));
    size_t o_kmask = L.take((size_t)2 * gmax * 8);
    size_t o_pin = L.take((size_t)gmax * 8);
    size_t o_flags = L.take((size_t)32 * 4 * (2 + 16));  // grid barrier: release word, 16 group counters, root
    const size_t bsum_lsd = (size_t)2 * gmax * kBins * 4;
    size_t o_bsum = L.take(bsum_lsd);
    size_t o_btot = h->fused ? L.take((size_t)2 * fused_max_buckets() * 4) : 0;
    size_t o_btab = h->fused ? L.take((size_t)2 * 136 * 4) : 0;
    size_t o_spl = h->fused ? L.take((size_t)2 * (16 * 256 + 16) * 8) : 0;  // kernels_fused.cu kSplG
    size_t o_rcur = h->fused ? L.take((size_t)2 * 256 * 4) : 0;
    size_t o_nkp = L.take((size_t)gmax * 4);
    size_t o_hd = h->fused ? L.take((size_t)kFusedKcap * 4) : 0, o_hw = h->fused ? L.take((size_t)kFusedKcap * 4) : 0;
    size_t o_rh = h->fused ? L.take((size_t)cap_pad + 16) : 0;
    const size_t bigr = big_max_ranges();
    size_t o_bspl = h->big ? L.take((size_t)2 * (16 * bigr + 16) * 8) : 0;
    size_t o_brc = h->big ? L.take((size_t)2 * bigr * 4) : 0;
    size_t o_bov = h->big ? L.take(64) : 0;
    size_t o_bkr = h->big ? L.take((size_t)h->big_ranges * kFusedKcap * 8) : 0;
    size_t o_bkc = h->big ? L.take((size_t)h->big_grid * big_slots_per_cta() * 8) : 0;
    size_t o_ctl = L.take(sizeof(Ctl));
    size_t o_ctasm = L.take((size_t)gmax * 4);
    size_t o_as0 = L.take((size_t)mb * 4), o_as1 = L.take((size_t)mb * 4);
    size_t o_ai0 = L.take((size_t)mb * 8), o_ai1 = L.take((size_t)mb * 8);
    size_t o_at0 = L.take(mb), o_at1 = L.take(mb);
    size_t o_pre = L.take((size_t)mb * 8);
    size_t o_ev = L.take((size_t)mb * sizeof(lamps_event));
    size_t o_ing = L.take((size_t)kIngestChunk * sizeof(SubmitRec));
    size_t o_gat = L.take((size_t)kIngestChunk * 4);
    size_t o_dbg = (h->cfg.flags & LAMPS_DEBUG_OUT) ? L.take((size_t)cap_pad * 32) : 0;
    size_t o_trace = (h->cfg.flags & LAMPS_TRACE) ? L.take((size_t)gmax * kTraceSlots * 8) : 0;
    const uint32_t world = h->cfg.world > 1 ? h->cfg.world : 1;
    const bool merge = merge_mode(h->cfg);
    size_t o_xs = merge ? L.take(((size_t)mb + 1) * sizeof(MergeRec)) : 0;
    size_t o_xr = merge ? L.take((size_t)world * ((size_t)mb + 1) * sizeof(MergeRec)) : 0;
    const bool large = merge && merge_is_large(world, mb);
    size_t o_xc = large ? L.take((size_t)world * world * mb * 4) : 0;
    size_t o_xo = large ? L.take((size_t)mb * 4) : 0;
    if (!base) return L.off;
    h->b.xsend = merge ? reinterpret_cast<MergeRec*>(base + o_xs) : nullptr;
    h->b.xrecv = merge ? reinterpret_cast<MergeRec*>(base + o_xr) : nullptr;
    h->b.xcnt = large ? reinterpret_cast<uint32_t*>(base + o_xc) : nullptr;
    h->b.xorder = large ? reinterpret_cast<uint32_t*>(base + o_xo) : nullptr;
    uint32_t* soa[10];
    for (int i = 0; i < 10; i++) soa[i] = reinterpret_cast<uint32_t*>(base + o_soa[i]);
    h->b.pool = Pool{soa[0], soa[1], soa[2], soa[3], soa[4], soa[5], soa[6], soa[7], soa[8], soa[9], cap_pad};
    for (int i = 1; i < 8; i++)
        if (soa[i] != soa[0] + (size_t)i * cap_pad) return 0;  // layout invariant used by the kernels
    h->b.keys[0] = reinterpret_cast<uint64_t*>(base + o_keys0);
    h->b.keys[1] = reinterpret_cast<uint64_t*>(base + o_keys1);
    h->b.kmask = reinterpret_cast<unsigned long long*>(base + o_kmask);
    h->b.pin_part = reinterpret_cast<unsigned long long*>(base + o_pin);
    h->b.flags = reinterpret_cast<uint32_t*>(base + o_flags);
    h->b.blocksum = reinterpret_cast<uint32_t*>(base + o_bsum);
    h->b.btot = h->fused ? reinterpret_cast<uint32_t*>(base + o_btot) : nullptr;
    h->b.btab = h->fused ? reinterpret_cast<uint32_t*>(base + o_btab) : nullptr;
    h->b.spl = h->fused ? reinterpret_cast<unsigned long long*>(base + o_spl) : nullptr;
    h->b.rcur = h->fused ? reinterpret_cast<uint32_t*>(base + o_rcur) : nullptr;
    h->b.nk_part = reinterpret_cast<uint32_t*>(base + o_nkp);
    h->b.hd = h->fused ? reinterpret_cast<uint32_t*>(base + o_hd) : nullptr;
    h->b.hw = h->fused ? reinterpret_cast<uint32_t*>(base + o_hw) : nullptr;
    h->b.rhint = h->fused ? base + o_rh : nullptr;
    h->b.big_ranges = h->big_ranges;
    h->b.big_grid = h->big_grid;
    h->b.big_cta_slots = h->big_cta_slots;
    h->b.big_spl = h->big ? reinterpret_cast<unsigned long long*>(base + o_bspl) : nullptr;
    h->b.big_rcur = h->big ? reinterpret_cast<uint32_t*>(base + o_brc) : nullptr;
    h->b.big_over = h->big ? reinterpret_cast<uint32_t*>(base + o_bov) : nullptr;
    h->b.big_keysr = h->big ? reinterpret_cast<uint64_t*>(base + o_bkr) : nullptr;
    h->b.big_keysc = h->big ? reinterpret_cast<uint64_t*>(base + o_bkc) : nullptr;
    h->b.score_grid = h->score_grid;
    h->b.sort_grid = h->sort_grid;
    h->b.ctl = reinterpret_cast<Ctl*>(base + o_ctl);
    h->b.cta_cost = reinterpret_cast<float*>(base + o_ctasm);
    h->b.adm_slot[0] = reinterpret_cast<uint32_t*>(base + o_as0);
    h->b.adm_slot[1] = reinterpret_cast<uint32_t*>(base + o_as1);
    h->b.adm_id[0] = reinterpret_cast<uint64_t*>(base + o_ai0);
    h->b.adm_id[1] = reinterpret_cast<uint64_t*>(base + o_ai1);
    h->b.adm_strat[0] = base + o_at0;
    h->b.adm_strat[1] = base + o_at1;
    h->b.pre_id = reinterpret_cast<uint64_t*>(base + o_pre);
    h->b.events = base + o_ev;
    h->d_events = h->b.events;
    h->d_ingest = base + o_ing;
    h->b.returns = h->d_ingest;
    h->d_gather = reinterpret_cast<uint32_t*>(base + o_gat);
    h->b.dbg = (h->cfg.flags & LAMPS_DEBUG_OUT) ? reinterpret_cast<unsigned long long*>(base + o_dbg)
                                                  : nullptr;
    h->b.trace = (h->cfg.flags & LAMPS_TRACE) ? reinterpret_cast<unsigned long long*>(base + o_trace) : nullptr;
    return L.off;
}

// Grid sizes.  Device attributes are needed only when a device exists; the
// size query (phase 1 of lamps_init) assumes the largest B200 grids so the
// reported size is an upper bound.
void grids(lamps_t* h, bool query_device) {
    int sms = 148, sort_occ = 1, fused_occ = 1;
    if (query_device) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sort_occ = sort_blocks_per_sm();
        fused_occ = fused_blocks_per_sm();
    }
    h->fused_grid = (uint32_t)std::max(1, sms * std::max(fused_occ, 1));
    if ((h->cfg.flags & LAMPS_SHARE_DEVICE) && h->cfg.world > 1) {  // co-resident ranks split the SMs
        const uint32_t lr = h->cfg.local_ranks ? std::min(h->cfg.local_ranks, h->cfg.world) : h->cfg.world;
        h->fused_grid = std::max<uint32_t>(1u, h->fused_grid / lr);
    }
    if (const char* gv = std::getenv("LAMPS_FUSED_GRID"))  // measurements: a smaller step grid
        h->fused_grid = std::max<uint32_t>(1u, std::min<uint32_t>(h->fused_grid, (uint32_t)std::strtoul(gv, nullptr, 0)));
    {
        const uint32_t groups = (h->cap + 3) / 4;
        const uint32_t gpc = (groups + h->fused_grid - 1) / h->fused_grid;
        h->fused = !(h->cfg.flags & LAMPS_MULTI_KERNEL) && gpc * 4u <= (uint32_t)kFusedKcap && fused_occ >= 1 &&
                   h->fused_grid <= 255u;  // range weights (kMaxCtas) cover up to 255 CTAs
    }
    // small pools: the whole step in one CTA (k_small), no grid barriers
    h->small = h->fused && h->cap <= small_max_cap() && !merge_mode(h->cfg) && !(h->cfg.flags & LAMPS_GRID_STEP) &&
               !((h->cfg.flags & LAMPS_SHARE_DEVICE) && h->cfg.world > 1);
    if (!query_device) {  // size query: assume the fused path may be chosen
        h->fused = !(h->cfg.flags & LAMPS_MULTI_KERNEL) && h->cap <= 148u * (uint32_t)kFusedKcap;
        h->fused_grid = std::max<uint32_t>(h->fused_grid, 296u);
    }
    // pools above the fused kernel's capacity (or LAMPS_BIG_STEP): several ranges per CTA
    h->big = !(h->cfg.flags & LAMPS_MULTI_KERNEL) && !merge_mode(h->cfg) &&
             ((h->cfg.flags & LAMPS_BIG_STEP) || !h->fused) && fused_occ >= 1;
    if (h->big) {
        h->fused = false;
        h->small = false;
        const uint32_t G = std::max<uint32_t>(h->fused_grid, 1u);
        const uint64_t per = (uint64_t)G * 7168u;  // ~6300 eligible keys per range at 88 % READY
        h->big_ranges = (uint32_t)std::min<uint64_t>((uint64_t)G * ((h->cap + per - 1) / per), big_max_ranges());
        // whole waves of one CTA per SM: the fewest waves whose CTAs hold <= 8192 slots each
        const uint64_t sms_u = (uint64_t)std::max(sms, 1), mx = big_slots_per_cta();
        const uint64_t waves = (h->cap + sms_u * mx - 1) / (sms_u * mx);
        uint64_t spc = (h->cap + sms_u * waves - 1) / (sms_u * waves);
        spc = std::min<uint64_t>((spc + 31) & ~31ull, mx);
        h->big_cta_slots = (uint32_t)spc;
        h->big_grid = (uint32_t)((h->cap + spc - 1) / spc);
    }
    const uint32_t groups = (h->cap + 3) / 4;
    const uint32_t want = (groups + kScoreThreads - 1) / kScoreThreads;
    h->score_grid = std::max<uint32_t>(1, std::min<uint32_t>(want, (uint32_t)sms * 7));
    h->sort_grid = (uint32_t)std::max(1, sms * std::max(sort_occ, 1));
    if (!query_device) h->sort_grid = std::max<uint32_t>(h->sort_grid, 148u * 2u);
}

// Cost::fast: prove, with exact 128-bit arithmetic, that the unchecked 64-bit
// fast path (lamps_dev.cuh strategy_score_fast) cannot overflow for any slot
// whose context values stay below L = kFastCtxLimit: every intermediate and the
// final sum must stay < 2^63.
bool fast_bounds_ok(const lamps_config& c) {
    typedef unsigned __int128 U;
    const U L = (U)kFastCtxLimit, lim = (U)1 << 63;
    const uint64_t m32 = 1ull << 32;
    if (c.A1 >= m32 || c.A2 >= m32 || c.S0 >= m32 || c.S1 >= m32 || c.tau >= m32 || c.c_other >= (1ull << 26))
        return false;
    if ((L - 1) * (L - 1) >= ((U)1 << 40)) return false;  // mul32x40 operand bound (x^2, ramps)
    const U api_max = 0xffffffffull, pend_max = 0xffffffffull;
    const U tf_in = (U)c.A1 * L + (U)c.A2 * L * L;         // T_fwd before the shift
    const U ts_in = (U)c.S0 + (U)c.S1 * L;
    if (tf_in >= lim || ts_in >= lim) return false;
    const U tf = tf_in >> c.SH, ts = ts_in >> c.SH;
    const U cb = L + c.c_other;
    const U blkL = (L + c.block_tokens - 1) / c.block_tokens;
    const U ramp = L * blkL;                                // >= F(n) for n <= L
    const U wd = tf * cb, ws = 2 * ts * cb, wp = api_max * L;
    if (wd >= lim || ws >= lim || wp >= lim) return false;
    const U t_pend = blkL * pend_max, t_ramp = (U)c.tau * ramp;
    U t_api = blkL * api_max;
    if (blkL * tf > t_api) t_api = blkL * tf;
    if (2 * blkL * ts > t_api) t_api = 2 * blkL * ts;
    if (L * c.block_tokens >= lim) return false;
    return t_pend + 2 * t_ramp + t_api < lim;
}

// segment validation shared by submit and api_return; ctx0 = context before the segment
const char* check_segment(const lamps_t* h, uint64_t ctx0, const lamps_segment& s, uint32_t* ticks) {
    if (s.has_api > 1) return "has_api must be 0 or 1";
    uint64_t total = ctx0 + s.pre_len;
    *ticks = 0;
    if (s.has_api) {
        total += (uint64_t)s.resp_len + s.post_len;
        if (!quantize(s.api_seconds, h->cfg.ticks_per_second, ticks))
            return "api_seconds is NaN, infinite, negative or out of range after quantisation";
    }
    if (total > LAMPS_INGEST_LIMIT) return "request longer than LAMPS_INGEST_LIMIT tokens";
    const uint64_t B = h->cfg.block_tokens;
    if ((total + B - 1) / B > h->cfg.kv_capacity_blocks)
        return "request can never fit: peak KV demand exceeds kv_capacity_blocks";
    return nullptr;
}

bool id_live(const lamps_t* h, uint64_t id) {
    if (id < h->id_base || id >= h->next_id) return false;
    return h->hstate[id & h->cost.cap_mask] != H_FREE;
}

void advance_id_base(lamps_t* h) {
    while (h->id_base < h->next_id && h->hstate[h->id_base & h->cost.cap_mask] == H_FREE) h->id_base++;
}

void record_timing(lamps_t* h, int k) {
    if (!(h->cfg.flags & LAMPS_TIMING)) return;
    cudaEventRecord(h->tev[(size_t)h->t_head * 5 + k], h->stream);
}

// Enqueue K0..K3 for one step on the handle's stream.
StepArgs make_args(lamps_t* h, uint64_t kv_total, uint32_t n_ev) {
    StepArgs a{};
    a.kv_total = kv_total;
    a.id_base = h->id_base;
    a.id_base_mod = (uint32_t)(h->id_base & h->cost.cap_mask);
    a.step = h->step;
    a.epoch = h->step * 8u;
    a.n_ev = n_ev;
    a.max_batch = h->cfg.max_batch;
    a.parity = h->step & 1u;
    a.flags = (h->cfg.flags & LAMPS_FORCE_FALLBACK) ? kStepForceFallback : 0u;
    a.world = h->world;
    a.rank = h->rank;
    a.tune = h->tune;
    a.n_ret = h->fused ? h->ret_pending : 0u;
    a.n_sub = h->fused ? h->sub_pending : 0u;
    a.inl = h->fused && h->inl_pending ? 1u : 0u;
    a.cold = h->cold ? 1u : 0u;
    if (h->merge) a.flags |= kStepMerge;
    if (h->merge && h->cfg.transport == LAMPS_XPORT_P2P) {
        a.flags |= kStepP2P;
        // peers on other GPUs: system scope (co-resident shards only: device scope)
        const bool all_local = (h->cfg.flags & LAMPS_SHARE_DEVICE) &&
                               (h->cfg.local_ranks == 0 || h->cfg.local_ranks >= h->world);
        if (h->world > 1 && !all_local) a.flags |= kStepP2PSys;
        a.xseq = h->xseq;
        a.xtimeout_ms = h->xtimeout_ms;
    }
    if (h->cfg.flags & LAMPS_HEAD_ONLY) a.flags |= kStepHeadOnly;
    return a;
}

// phase 1: events, scoring, ranking (and, single shard, admission)
int enqueue_phase1(lamps_t* h, uint64_t kv_total, uint32_t n_ev) {
    const bool timing = (h->cfg.flags & LAMPS_TIMING) != 0;
    if (h->merge && h->cfg.transport == LAMPS_XPORT_P2P && !h->p2p_ready)
        return fail(h, LAMPS_EINVAL, "P2P transport: call lamps_p2p_connect first");
    if (timing && h->t_count == kTimingRing) return fail(h, LAMPS_EINVAL, "timing ring full: call lamps_timing_read");
    // after every check: every rank steps in lockstep, so the sequence numbers agree
    if (h->merge && h->cfg.transport == LAMPS_XPORT_P2P) h->xseq++;
    if (h->have_result && h->fetched_step != h->step) h->shadow_ok = false;  // an unread admitted list
    h->step++;
    const StepArgs a = make_args(h, kv_total, n_ev);
    h->last_id_base = h->id_base;
    record_timing(h, 0);
    if (!h->fused) CU(h, launch_events(h->b, h->cost, a, h->stream));  // fused: in the kernel's prologue
    record_timing(h, 1);
    if (h->fused) {
        if (h->small)
            CU(h, launch_small(h->b, h->cost, a, a.inl ? &h->inl : nullptr, h->stream));
        else
            CU(h, launch_fused(h->b, h->cost, a, a.inl ? &h->inl : nullptr, h->fused_grid, h->stream));
        h->cold = false;  // the kernel wrote the next step's splitters
        record_timing(h, 2);
        record_timing(h, 3);
    } else if (h->big && !h->cold) {  // warm large-pool step (events applied by k_events above)
        StepArgs ab = a;
        ab.n_ev = 0;
        CU(h, launch_big(h->b, h->cost, ab, nullptr, h->fused_grid, h->stream));
        record_timing(h, 2);
        record_timing(h, 3);
    } else {
        CU(h, launch_score(h->b, h->cost, a, (int)h->score_grid, h->stream));
        record_timing(h, 2);
        CU(h, launch_sort(h->b, h->cost, a, h->stream));
        record_timing(h, 3);
        CU(h, launch_admit(h->b, h->cost, a, h->stream));
        if (h->big) {  // cold large-pool step: the next step's grid from this order
            CU(h, launch_big_grid(h->b, a, h->stream));
            h->cold = false;
        }
    }
    h->last_kernels = (h->fused ? 1 : (h->big && a.cold == 0 ? 2 : 3 + (h->big ? 1 : 0))) + (!h->fused && n_ev ? 1 : 0);
    h->ret_pending = 0;
    h->sub_pending = 0;
    h->inl_pending = false;
    return LAMPS_OK;
}

// phase 2 (world > 1): exchange the top-K records, merge, admit this rank's share
int enqueue_phase2(lamps_t* h, uint64_t kv_total, uint32_t n_ev, bool exchange) {
    if (h->merge && h->cfg.transport != LAMPS_XPORT_P2P) {  // P2P: exchanged and merged in k_fused
        const StepArgs a = make_args(h, kv_total, n_ev);
        if (exchange) {
            const size_t bytes = ((size_t)h->cfg.max_batch + 1) * sizeof(MergeRec);
            const int r = g_nccl.allGather(h->b.xsend, h->b.xrecv, bytes, kNcclUint8, h->comm, h->stream);
            if (r != 0)
                return fail(h, LAMPS_ENCCL, std::string("ncclAllGather: ") +
                                                (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error"));
        }
        CU(h, launch_merge(h->b, h->cost, a, h->stream));
        h->last_kernels += merge_is_large(h->world, h->cfg.max_batch) ? 3 : 1;
    }
    record_timing(h, 4);
    if (h->cfg.flags & LAMPS_TIMING) {
        h->t_head = (h->t_head + 1) % kTimingRing;
        h->t_count++;
    }
    h->have_result = true;
    return LAMPS_OK;
}

int enqueue_step(lamps_t* h, uint64_t kv_total, uint32_t n_ev) {
    if (h->world > 1 && h->cfg.transport == LAMPS_XPORT_LOOPBACK)
        return fail(h, LAMPS_EINVAL, "loopback shards step together: use lamps_group_step");
    if (h->world > 1 && (h->cfg.flags & LAMPS_SHARE_DEVICE))
        return fail(h, LAMPS_EINVAL, "ranks sharing one device step together: use lamps_group_step");
    int rc = enqueue_phase1(h, kv_total, n_ev);
    if (rc) return rc;
    return enqueue_phase2(h, kv_total, n_ev, true);
}

int fetch_result(lamps_t* h, lamps_step_out* out) {
    // the admission kernel wrote the summary and the lists into mapped host memory
    CU(h, cudaStreamSynchronize(h->stream));
    const HostRes& R = *h->hres;
    if (h->merge && h->cfg.transport == LAMPS_XPORT_P2P && R.xfail)
        return fail(h, LAMPS_ENCCL, "peer exchange timed out: a rank did not step (ranks out of lockstep)");
    const uint32_t par = h->step & 1u;
    const uint64_t* adm = h->h_adm_ids;
    h->prev_adm.assign(adm, adm + R.n_admitted);
    if (h->fetched_step != h->step) {
        for (uint32_t k = 0; k < R.n_admitted; k++) {
            const uint32_t sl = (uint32_t)(adm[k] & h->cost.cap_mask);
            h->hctx[sl] += 1u;  // the next step's A0
            h->adm_mark[sl] = h->step;
        }
        h->fetched_step = h->step;
    }
    h->prev_known = true;
    if (out) {
        std::memset(out, 0, sizeof(*out));
        out->n_eligible = R.n_elig;
        out->pinned = R.pinned;
        out->budget = R.budget;
        out->budget_used = R.budget_used;
        out->n_admitted = R.n_admitted;
        out->n_preempted = R.n_preempted;
        out->blocked_head = R.blocked_head;
        out->id_base = h->last_id_base;
        out->admitted_ids = h->h_adm_ids;
        out->admitted_strategy = h->h_adm_strat;
        out->preempted_ids = h->h_pre_ids;
        out->d_ranked_keys = h->b.keys[R.final_buf & 1u];
        out->d_admitted_slots = h->b.adm_slot[par];
    }
    return LAMPS_OK;
}

// Rebuild the context shadow from the device (after async steps whose admitted lists the
// host never read): the device ctx plus the pending A0 of the last step's admitted slots.
int resync_shadow(lamps_t* h) {
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaMemcpy(h->hctx.data(), h->b.pool.ctx, (size_t)h->cap * 4, cudaMemcpyDeviceToHost));
    if (h->have_result) {
        CU(h, cudaMemcpy(h->h_ctl, h->b.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
        const uint32_t n = h->h_ctl->n_admitted;
        std::vector<uint32_t> slots(n);
        if (n) CU(h, cudaMemcpy(slots.data(), h->b.adm_slot[h->step & 1u], (size_t)n * 4, cudaMemcpyDeviceToHost));
        for (uint32_t k = 0; k < n; k++) h->hctx[slots[k]] += 1u;
    }
    h->fetched_step = h->step;
    h->shadow_ok = true;
    return LAMPS_OK;
}

// the pinned ingest staging may be rewritten once its last host-to-device copy is done
int staging_wait(lamps_t* h) {
    if (h->ing_pending) {
        CU(h, cudaEventSynchronize(h->ing_ev));
        h->ing_pending = false;
    }
    return LAMPS_OK;
}

int staging_copied(lamps_t* h) {
    CU(h, cudaEventRecord(h->ing_ev, h->stream));
    h->ing_pending = true;
    return LAMPS_OK;
}

// ---- validation and staging shared by the single calls and lamps_iterate ----------

// submit: the segments (pure checks; ticks out)
int check_submit(lamps_t* h, const lamps_segment* segs, uint32_t n, std::vector<uint32_t>& ticks) {
    if (n && !segs) return fail(h, LAMPS_EINVAL, "segs is NULL");
    ticks.assign(n, 0u);
    for (uint32_t k = 0; k < n; k++) {
        if (const char* m = check_segment(h, segs[k].prompt_len, segs[k], &ticks[k]))
            return fail(h, LAMPS_EINVAL, std::string("submit[") + std::to_string(k) + "]: " + m);
    }
    return LAMPS_OK;
}

// submit: the id window and free slots, counting the slots in freed[0..nf) (sorted) as free
int window_submit(lamps_t* h, uint32_t n, const uint32_t* freed, uint32_t nf) {
    auto is_free = [&](uint32_t sl) {
        return h->hstate[sl] == H_FREE || (nf && std::binary_search(freed, freed + nf, sl));
    };
    uint64_t base = h->id_base;
    while (nf && base < h->next_id && is_free((uint32_t)(base & h->cost.cap_mask))) base++;
    if (h->next_id + n - base > h->cap) return fail(h, LAMPS_ENOSPC, "pool full (id window)");
    for (uint32_t k = 0; k < n; k++)
        if (!is_free((uint32_t)((h->next_id + k) & h->cost.cap_mask)))
            return fail(h, LAMPS_ENOSPC, "pool full (slot occupied)");
    return LAMPS_OK;
}

int do_submit(lamps_t* h, const lamps_segment* segs, uint32_t n, const std::vector<uint32_t>& ticks,
              uint64_t* ids_out) {
    SubmitRec* rec = static_cast<SubmitRec*>(h->h_ingest);
    for (uint32_t k0 = 0; k0 < n; k0 += kIngestChunk) {
        const uint32_t m = std::min(kIngestChunk, n - k0);
        if (int rc = staging_wait(h)) return rc;
        for (uint32_t i = 0; i < m; i++) {
            const lamps_segment& s = segs[k0 + i];
            SubmitRec& r = rec[i];
            r.slot = (uint32_t)((h->next_id + k0 + i) & h->cost.cap_mask);
            r.ctx = s.prompt_len;
            r.pre = s.pre_len;
            r.has = s.has_api;
            r.api = s.has_api ? ticks[k0 + i] : 0u;
            r.resp = s.has_api ? s.resp_len : 0u;
            r.post = s.has_api ? s.post_len : 0u;
            r.pad = 0;
        }
        CU(h, cudaMemcpyAsync(h->d_ingest, rec, (size_t)m * sizeof(SubmitRec), cudaMemcpyHostToDevice, h->stream));
        if (int rc = staging_copied(h)) return rc;
        CU(h, launch_submit(h->b.pool, h->cost, static_cast<const SubmitRec*>(h->d_ingest), m, h->stream));
    }
    for (uint32_t k = 0; k < n; k++) {
        h->hstate[(h->next_id + k) & h->cost.cap_mask] = H_READY;
        h->hctx[(h->next_id + k) & h->cost.cap_mask] = segs[k].prompt_len;
        if (ids_out) ids_out[k] = h->next_id + k;
    }
    h->next_id += n;
    return LAMPS_OK;
}

// API returns: ids PAUSED, distinct, segments valid against the context shadow
int check_returns(lamps_t* h, const uint64_t* ids, const uint32_t* actual, const lamps_segment* next, uint32_t n,
                  std::vector<uint32_t>& ticks, std::vector<uint32_t>& ctx) {
    if (n && (!ids || !actual || !next)) return fail(h, LAMPS_EINVAL, "NULL argument");
    for (uint32_t k = 0; k < n; k++) {
        if (!id_live(h, ids[k]) || h->hstate[ids[k] & h->cost.cap_mask] != H_PAUSED)
            return fail(h, LAMPS_ENOENT, "api_return: id unknown or not paused");
    }
    {
        std::vector<uint64_t> s(ids, ids + n);
        std::sort(s.begin(), s.end());
        if (std::adjacent_find(s.begin(), s.end()) != s.end())
            return fail(h, LAMPS_EINVAL, "api_return: duplicate id");
    }
    ticks.assign(n, 0u);
    ctx.assign(n, 0u);
    if (!h->shadow_ok) {
        const int rc = resync_shadow(h);
        if (rc) return rc;
    }
    for (uint32_t k = 0; k < n; k++) ctx[k] = h->hctx[ids[k] & h->cost.cap_mask];
    for (uint32_t k = 0; k < n; k++) {
        if (const char* m = check_segment(h, (uint64_t)ctx[k] + actual[k], next[k], &ticks[k]))
            return fail(h, LAMPS_EINVAL, std::string("api_return[") + std::to_string(k) + "]: " + m);
    }
    return LAMPS_OK;
}

// API returns: staged to the device; applied by k_api_return now, or (prologue, one
// chunk) by the next fused step kernel before it scores
int do_returns(lamps_t* h, const uint64_t* ids, const uint32_t* actual, const lamps_segment* next, uint32_t n,
               const std::vector<uint32_t>& ticks, const std::vector<uint32_t>& ctx, bool prologue) {
    ReturnRec* rec = static_cast<ReturnRec*>(h->h_ingest);
    for (uint32_t k0 = 0; k0 < n; k0 += kIngestChunk) {
        const uint32_t m = std::min(kIngestChunk, n - k0);
        if (int rc = staging_wait(h)) return rc;
        for (uint32_t i = 0; i < m; i++) {
            const lamps_segment& s = next[k0 + i];
            ReturnRec& r = rec[i];
            r.slot = (uint32_t)(ids[k0 + i] & h->cost.cap_mask);
            r.actual = actual[k0 + i];
            r.pre = s.pre_len;
            r.has = s.has_api;
            r.api = s.has_api ? ticks[k0 + i] : 0u;
            r.resp = s.has_api ? s.resp_len : 0u;
            r.post = s.has_api ? s.post_len : 0u;
            r.pad = 0;
        }
        CU(h, cudaMemcpyAsync(h->d_ingest, rec, (size_t)m * sizeof(ReturnRec), cudaMemcpyHostToDevice, h->stream));
        if (int rc = staging_copied(h)) return rc;
        if (prologue)
            h->ret_pending = m;  // the caller guarantees n <= kIngestChunk
        else
            CU(h, launch_api_return(h->b.pool, h->cost, static_cast<const ReturnRec*>(h->d_ingest), m, h->stream));
    }
    for (uint32_t k = 0; k < n; k++) {
        h->hstate[ids[k] & h->cost.cap_mask] = H_READY;
        h->hctx[ids[k] & h->cost.cap_mask] = ctx[k] + actual[k];
    }
    return LAMPS_OK;
}

// events: valid against the previous admitted list (pure checks)
int check_events(lamps_t* h, const lamps_event* ev, uint32_t n_ev, uint64_t kv_total_blocks) {
    if (n_ev && !ev) return fail(h, LAMPS_EINVAL, "events is NULL");
    if (kv_total_blocks > h->cfg.kv_capacity_blocks)
        return fail(h, LAMPS_EINVAL, "kv_total_blocks exceeds kv_capacity_blocks");
    if (n_ev) {
        if (!h->prev_known) {  // previous step ran async: fetch its admitted list
            int rc = fetch_result(h, nullptr);
            if (rc) return rc;
        }
        if (n_ev > h->prev_adm.size()) return fail(h, LAMPS_EINVAL, "more events than admitted requests");
        // O(n_ev): a valid event names a live id whose slot the previous step admitted,
        // at most once (per-slot marks; the live id of a slot is unique)
        const uint32_t tag = ++h->ev_tag;
        for (uint32_t e = 0; e < n_ev; e++) {
            if (ev[e].kind != LAMPS_EV_API_CALL && ev[e].kind != LAMPS_EV_FINISHED)
                return fail(h, LAMPS_EINVAL, "unknown event kind");
            const uint32_t sl = (uint32_t)(ev[e].id & h->cost.cap_mask);
            if (!id_live(h, ev[e].id) || h->adm_mark[sl] != h->step || h->fetched_step != h->step)
                return fail(h, LAMPS_EINVAL, "event for a request not admitted by the previous step");
            if (h->ev_mark[sl] == tag) return fail(h, LAMPS_EINVAL, "duplicate event id");
            h->ev_mark[sl] = tag;
        }
    }
    return LAMPS_OK;
}

// events: liveness shadow updated (the events already staged)
void events_staged(lamps_t* h, const lamps_event* ev, uint32_t n_ev) {
    if (!n_ev) return;
    for (uint32_t e = 0; e < n_ev; e++)
        h->hstate[ev[e].id & h->cost.cap_mask] = ev[e].kind == LAMPS_EV_FINISHED ? H_FREE : H_PAUSED;
    advance_id_base(h);
}

// events: staged to the device, liveness shadow updated
int stage_events(lamps_t* h, const lamps_event* ev, uint32_t n_ev) {
    h->b.events = h->d_events;
    if (!h->ret_pending && !h->sub_pending) h->inl_pending = false;  // no stale inline staging
    if (!n_ev) return LAMPS_OK;
    if (h->fused && !h->ret_pending && !h->sub_pending && (size_t)n_ev * sizeof(lamps_event) <= kInlineStage) {
        std::memcpy(h->inl.bytes, ev, (size_t)n_ev * sizeof(lamps_event));  // the kernel's parameters
        h->inl_pending = true;
        events_staged(h, ev, n_ev);
        return LAMPS_OK;
    }
    std::memcpy(h->h_ev, ev, (size_t)n_ev * sizeof(lamps_event));
    CU(h, cudaMemcpyAsync(const_cast<void*>(h->d_events), h->h_ev, (size_t)n_ev * sizeof(lamps_event),
                          cudaMemcpyHostToDevice, h->stream));
    events_staged(h, ev, n_ev);
    return LAMPS_OK;
}

// the step's own preconditions, checked before anything is staged (so that a rejected
// step leaves the handle unchanged; after staging only a CUDA error can fail it)
int step_precheck(lamps_t* h, bool group = false) {
    if (!group && h->world > 1 && h->cfg.transport == LAMPS_XPORT_LOOPBACK)
        return fail(h, LAMPS_EINVAL, "loopback shards step together: use lamps_group_step");
    if (!group && h->world > 1 && (h->cfg.flags & LAMPS_SHARE_DEVICE))
        return fail(h, LAMPS_EINVAL, "ranks sharing one device step together: use lamps_group_step");
    if (h->merge && h->cfg.transport == LAMPS_XPORT_P2P && !h->p2p_ready)
        return fail(h, LAMPS_EINVAL, "P2P transport: call lamps_p2p_connect first");
    if ((h->cfg.flags & LAMPS_TIMING) && h->t_count == kTimingRing)
        return fail(h, LAMPS_EINVAL, "timing ring full: call lamps_timing_read");
    return LAMPS_OK;
}

// host-side part of a step: validate the events against the previous admitted
// list, stage them to the device, update the liveness shadow (state unchanged on error)
int prepare_step(lamps_t* h, const lamps_event* ev, uint32_t n_ev, uint64_t kv_total_blocks) {
    if (int rc = check_events(h, ev, n_ev, kv_total_blocks)) return rc;
    if (int rc = step_precheck(h)) return rc;
    return stage_events(h, ev, n_ev);
}

}  // namespace

extern "C" {

uint32_t lamps_version(void) { return (1u << 16) | 0u; }

const char* lamps_last_error(const lamps_t* h) {
    if (!h) return "null handle";
    return h->err.c_str();
}

int lamps_init(const lamps_config* cfg, void* d_workspace, size_t* ws_bytes, lamps_t** out) {
    if (!cfg || !ws_bytes) return LAMPS_EINVAL;
    if (validate_cfg(cfg)) return LAMPS_EINVAL;
    lamps_t tmp;
    tmp.cfg = *cfg;
    tmp.cap = cfg->capacity;
    tmp.cap_pad = std::max<uint32_t>(cfg->capacity, 1024u);
    grids(&tmp, false);
    const size_t need = carve(&tmp, nullptr);
    if (!d_workspace) {
        *ws_bytes = need;
        return LAMPS_OK;
    }
    if (!out) return LAMPS_EINVAL;
    if (*ws_bytes < need || (reinterpret_cast<uintptr_t>(d_workspace) & (kAlign - 1))) return LAMPS_EINVAL;
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return LAMPS_ECUDA;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, d_workspace) != cudaSuccess || attr.type != cudaMemoryTypeDevice)
        return LAMPS_EINVAL;

    lamps_t* h = new lamps_t();
    h->cfg = *cfg;
    h->stream = static_cast<cudaStream_t>(cfg->stream);
    h->cap = cfg->capacity;
    h->cap_pad = tmp.cap_pad;
    h->ws = static_cast<uint8_t*>(d_workspace);
    grids(h, true);
    if (h->sort_grid > tmp.sort_grid || h->score_grid > tmp.score_grid ||
        (h->fused && (!tmp.fused || h->fused_grid > tmp.fused_grid))) {
        delete h;
        return LAMPS_ENOTSUP;  // device larger than the sizing assumption
    }
    if ((uint64_t)h->sort_grid * kSortMaxTilesPerCta * kSortTile < h->cap) {
        delete h;
        return LAMPS_ENOTSUP;
    }
    if (const char* tv = std::getenv("LAMPS_TUNE")) h->tune = (uint32_t)std::strtoul(tv, nullptr, 0);
    if (const char* xv = std::getenv("LAMPS_P2P_TIMEOUT_MS"))
        h->xtimeout_ms = std::max<uint32_t>(1u, (uint32_t)std::strtoul(xv, nullptr, 0));
    h->world = cfg->world > 1 ? cfg->world : 1;
    h->rank = cfg->world > 1 ? cfg->rank : 0;
    h->merge = merge_mode(*cfg);
    if (h->merge && !h->fused) {
        delete h;
        return LAMPS_ENOTSUP;  // multi-GPU merge is implemented on the fused path
    }
    carve(h, h->ws);
    Cost& c = h->cost;
    c.tau = cfg->tau; c.A1 = cfg->A1; c.A2 = cfg->A2; c.S0 = cfg->S0; c.S1 = cfg->S1;
    c.c_other = cfg->c_other; c.SH = cfg->SH;
    c.B = cfg->block_tokens;
    c.lgB = 0;
    while ((1u << c.lgB) < c.B) c.lgB++;
    c.T = cfg->starvation_threshold;
    c.SB = cfg->score_bits; c.IB = cfg->id_bits;
    c.score_max = (cfg->score_bits >= 64) ? ~0ull : ((1ull << cfg->score_bits) - 1ull);
    c.nsbit = 1ull << (cfg->score_bits + cfg->id_bits);  // <= 2^63 (SB + IB + 1 <= 64)
    c.cap = cfg->capacity; c.cap_mask = cfg->capacity - 1u;
    c.fast = fast_bounds_ok(*cfg) ? 1u : 0u;
    c.policy = cfg->policy;
    c.interval = cfg->score_interval;
    c.cache = (cfg->policy == LAMPS_POLICY_LAMPS && cfg->score_interval > 1) ? 1u : 0u;
    c.lean = (c.fast && c.lgB >= 1 && cfg->policy == LAMPS_POLICY_LAMPS && !c.cache) ? 1u : 0u;
    h->hstate.assign(h->cap, H_FREE);
    auto cleanup = [&](int code, const char*) { lamps_free(h); return code; };
    if (cudaMemsetAsync(h->ws, 0, need, h->stream) != cudaSuccess) return cleanup(LAMPS_ECUDA, "memset");
    if (cudaHostAlloc(&h->h_ingest, (size_t)kIngestChunk * sizeof(SubmitRec), cudaHostAllocDefault) ||
        cudaHostAlloc((void**)&h->h_ev, (size_t)cfg->max_batch * sizeof(lamps_event), cudaHostAllocDefault) ||
        cudaHostAlloc((void**)&h->h_ctl, sizeof(Ctl), cudaHostAllocDefault) ||
        cudaHostAlloc(&h->h_res, sizeof(HostRes) + (size_t)cfg->max_batch * 17, cudaHostAllocMapped) ||
        cudaEventCreateWithFlags(&h->ing_ev, cudaEventDisableTiming))
        return cleanup(LAMPS_ECUDA, "cudaHostAlloc");
    {   // result block: summary | admitted ids | preempted ids | admitted strategies
        uint8_t* hb = static_cast<uint8_t*>(h->h_res);
        uint8_t* db = nullptr;
        if (cudaHostGetDevicePointer((void**)&db, h->h_res, 0) != cudaSuccess)
            return cleanup(LAMPS_ECUDA, "cudaHostGetDevicePointer");
        const size_t o_adm = sizeof(HostRes), o_pre = o_adm + (size_t)cfg->max_batch * 8,
                     o_str = o_pre + (size_t)cfg->max_batch * 8;
        h->hres = reinterpret_cast<HostRes*>(hb);
        h->h_adm_ids = reinterpret_cast<uint64_t*>(hb + o_adm);
        h->h_pre_ids = reinterpret_cast<uint64_t*>(hb + o_pre);
        h->h_adm_strat = hb + o_str;
        std::memset(hb, 0, o_str + cfg->max_batch);
        h->b.hres = reinterpret_cast<HostRes*>(db);
        h->b.h_adm_id = reinterpret_cast<unsigned long long*>(db + o_adm);
        h->b.h_pre_id = reinterpret_cast<unsigned long long*>(db + o_pre);
        h->b.h_adm_strat = db + o_str;
    }
    h->hctx.assign(h->cap, 0u);
    h->adm_mark.assign(h->cap, 0u);
    h->ev_mark.assign(h->cap, 0u);

    if (cfg->flags & LAMPS_TIMING) {
        h->tev.resize((size_t)kTimingRing * 5);
        for (auto& e : h->tev)
            if (cudaEventCreate(&e) != cudaSuccess) return cleanup(LAMPS_ECUDA, "event");
    }
    if (h->fused) {  // both parities' bucket tables start as the default (kernels_fused.cu)
        uint32_t* tab = static_cast<uint32_t*>(h->h_ingest);
        fused_default_table(cfg->score_bits + cfg->id_bits, tab);
        std::memcpy(tab + 136, tab, 136 * 4);
        if (cudaMemcpyAsync(h->b.btab, tab, 2 * 136 * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
            return cleanup(LAMPS_ECUDA, "bucket table");
    }
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) return cleanup(LAMPS_ECUDA, "sync");
    if (h->merge && cfg->transport == LAMPS_XPORT_P2P) {
        const size_t xb = p2p_bytes(h->world, cfg->max_batch);
        if (cudaMalloc((void**)&h->xbuf, xb) != cudaSuccess ||
            cudaMalloc((void**)&h->d_peers, (size_t)h->world * sizeof(MergeRec*)) != cudaSuccess ||
            cudaMemset(h->xbuf, 0, xb) != cudaSuccess)
            return cleanup(LAMPS_ECUDA, "P2P exchange buffer");
        h->b.xown = h->xbuf;
        h->b.xpeers = h->d_peers;
        if (h->world == 1) {  // self-exchange: the same kernel path with one rank
            if (cudaMemcpy(h->d_peers, &h->xbuf, sizeof(MergeRec*), cudaMemcpyHostToDevice) != cudaSuccess)
                return cleanup(LAMPS_ECUDA, "P2P table");
            h->p2p_ready = true;
        }
    }
    if (h->merge && cfg->transport == LAMPS_XPORT_NCCL) {
        if (!g_nccl.load()) return cleanup(LAMPS_ENCCL, "libnccl.so.2 not loadable");
        NcclId id;
        std::memcpy(id.internal, cfg->nccl_id, sizeof(id.internal));
        CommInitRankFn init = (CommInitRankFn)dlsym(g_nccl.so, "ncclCommInitRank");
        if (init(&h->comm, (int)h->world, id, (int)h->rank) != 0) return cleanup(LAMPS_ENCCL, "ncclCommInitRank");
    }
    *out = h;
    return LAMPS_OK;
}

int lamps_free(lamps_t* h) {
    if (!h) return LAMPS_EINVAL;
    cudaStreamSynchronize(h->stream);
    for (void* p : h->peer_open) cudaIpcCloseMemHandle(p);
    if (h->d_peers) cudaFree(h->d_peers);
    if (h->xbuf) {
        std::lock_guard<std::mutex> lk(g_exp_mu);
        for (size_t i = 0; i < g_exported.size(); i++)
            if (g_exported[i].second == h->xbuf) {
                g_exported.erase(g_exported.begin() + (long)i);
                break;
            }
    }
    if (h->xbuf) cudaFree(h->xbuf);
    if (h->comm && g_nccl.commDestroy) g_nccl.commDestroy(h->comm);
    for (auto& e : h->tev)
        if (e) cudaEventDestroy(e);
    if (h->h_ingest) cudaFreeHost(h->h_ingest);
    if (h->h_ev) cudaFreeHost(h->h_ev);
    if (h->h_ctl) cudaFreeHost(h->h_ctl);
    if (h->h_res) cudaFreeHost(h->h_res);
    if (h->ing_ev) cudaEventDestroy(h->ing_ev);
    delete h;
    return LAMPS_OK;
}

int lamps_submit(lamps_t* h, const lamps_segment* segs, uint32_t n, uint64_t* ids_out) {
    if (!h) return LAMPS_EINVAL;
    std::vector<uint32_t> ticks;
    if (int rc = check_submit(h, segs, n, ticks)) return rc;
    if (int rc = window_submit(h, n, nullptr, 0)) return rc;
    return do_submit(h, segs, n, ticks, ids_out);
}

int lamps_predict(lamps_t* h, const lamps_truth* truth, uint32_t n, const lamps_noise* noise,
                  lamps_segment* out) {
    if (!h) return LAMPS_EINVAL;
    if (n && (!truth || !out)) return fail(h, LAMPS_EINVAL, "NULL argument");
    const uint64_t seed = noise ? noise->seed : 0ull;
    const uint32_t lp = noise ? noise->len_error_ppm : 0u, ap = noise ? noise->api_error_ppm : 0u;
    if (lp > 10000000u || ap > 10000000u) return fail(h, LAMPS_EINVAL, "error ppm above 10^7");
    for (uint32_t k = 0; k < n; k++) {
        const lamps_truth& t = truth[k];
        if (t.has_api > 1 || t.reserved)
            return fail(h, LAMPS_EINVAL, "predict[" + std::to_string(k) + "]: has_api > 1 or reserved != 0");
        if (t.pre_bin != LAMPS_NO_BIN && t.pre_bin > LAMPS_MAX_BIN)
            return fail(h, LAMPS_EINVAL, "predict[" + std::to_string(k) + "]: pre_bin out of range");
        if (t.key >> 57) return fail(h, LAMPS_EINVAL, "predict[" + std::to_string(k) + "]: key >= 2^57");
    }
    constexpr uint32_t kChunk = kIngestChunk / 2;  // truths + predictions fit the staging buffer
    static_assert((size_t)kChunk * (sizeof(TruthRec) + sizeof(PredRec)) <= (size_t)kIngestChunk * sizeof(SubmitRec),
                  "predict staging");
    TruthRec* tin = static_cast<TruthRec*>(h->h_ingest);
    PredRec* pout = reinterpret_cast<PredRec*>(tin + kChunk);
    TruthRec* d_in = static_cast<TruthRec*>(h->d_ingest);
    PredRec* d_out = reinterpret_cast<PredRec*>(d_in + kChunk);
    for (uint32_t k0 = 0; k0 < n; k0 += kChunk) {
        const uint32_t m = std::min(kChunk, n - k0);
        if (int rc = staging_wait(h)) return rc;
        for (uint32_t i = 0; i < m; i++) {
            const lamps_truth& t = truth[k0 + i];
            tin[i] = TruthRec{t.key, t.pre_len, t.pre_bin, t.resp_len, t.post_len, t.api_ticks, t.has_api};
        }
        CU(h, cudaMemcpyAsync(d_in, tin, (size_t)m * sizeof(TruthRec), cudaMemcpyHostToDevice, h->stream));
        CU(h, launch_predict(d_in, d_out, m, seed, lp, ap, h->stream));
        CU(h, cudaMemcpyAsync(pout, d_out, (size_t)m * sizeof(PredRec), cudaMemcpyDeviceToHost, h->stream));
        CU(h, cudaStreamSynchronize(h->stream));
        for (uint32_t i = 0; i < m; i++) {
            lamps_segment& s = out[k0 + i];
            const PredRec& r = pout[i];
            s.prompt_len = truth[k0 + i].prompt_len;
            s.pre_len = r.pre;
            s.resp_len = r.resp;
            s.post_len = r.post;
            s.has_api = truth[k0 + i].has_api;
            // |ticks/tps * tps - ticks| <= 2^-52 * 2^32 << 1/2: quantises back to r.api exactly
            s.api_seconds = (double)r.api / h->cfg.ticks_per_second;
            s.reserved = 0;
        }
    }
    return LAMPS_OK;
}

int lamps_api_return(lamps_t* h, const uint64_t* ids, const uint32_t* actual_resp_len,
                     const lamps_segment* next, uint32_t n) {
    if (!h) return LAMPS_EINVAL;
    std::vector<uint32_t> ticks, ctx;
    if (int rc = check_returns(h, ids, actual_resp_len, next, n, ticks, ctx)) return rc;
    return do_returns(h, ids, actual_resp_len, next, n, ticks, ctx, false);
}

int lamps_schedule_step(lamps_t* h, const lamps_event* ev, uint32_t n_ev, uint64_t kv_total_blocks,
                        lamps_step_out* out) {
    if (!h) return LAMPS_EINVAL;
    int rc = prepare_step(h, ev, n_ev, kv_total_blocks);
    if (rc) return rc;
    rc = enqueue_step(h, kv_total_blocks, n_ev);
    if (rc) return rc;
    return fetch_result(h, out);
}

int lamps_iterate(lamps_t* h, const lamps_iteration* it, lamps_step_out* out) {
    if (!h || !it) return LAMPS_EINVAL;
    if (int rc = step_precheck(h)) return rc;  // world > 1 refusals etc. before any host work
    const uint32_t nr = it->n_returns, ne = it->n_events, na = it->n_arrivals;
    // 1. everything is validated before anything is applied
    std::vector<uint32_t> rticks, rctx, aticks;
    if (int rc = check_returns(h, it->return_ids, it->return_resp, it->return_next, nr, rticks, rctx)) return rc;
    if (int rc = check_submit(h, it->arrivals, na, aticks)) return rc;
    if (int rc = window_submit(h, na, nullptr, 0)) return rc;
    if (int rc = check_events(h, it->events, ne, it->kv_total_blocks)) return rc;
    // 2. API returns, arrivals and the events: on the fused path staged together and applied
    //    in the step kernel's prologue -- up to kInlineStage bytes inside the kernel's parameter
    //    block (no copy), else with one copy; otherwise returns and arrivals by their own
    //    kernels before the step
    const size_t rbytes = (size_t)(nr + na) * sizeof(ReturnRec), ebytes = (size_t)ne * sizeof(lamps_event);
    bool ev_staged = false;
    h->inl_pending = false;
    if (h->fused && rbytes + ebytes <= (size_t)kIngestChunk * sizeof(SubmitRec)) {
        const bool inl = rbytes + ebytes <= kInlineStage;
        if (!inl) {
            if (int rc = staging_wait(h)) return rc;
        }
        ReturnRec* rr = inl ? reinterpret_cast<ReturnRec*>(h->inl.bytes) : static_cast<ReturnRec*>(h->h_ingest);
        SubmitRec* sr = reinterpret_cast<SubmitRec*>(rr + nr);
        static_assert(sizeof(ReturnRec) == sizeof(SubmitRec), "one staging layout");
        for (uint32_t i = 0; i < nr; i++) {
            const lamps_segment& sg = it->return_next[i];
            ReturnRec& r = rr[i];
            r.slot = (uint32_t)(it->return_ids[i] & h->cost.cap_mask);
            r.actual = it->return_resp[i];
            r.pre = sg.pre_len;
            r.has = sg.has_api;
            r.api = sg.has_api ? rticks[i] : 0u;
            r.resp = sg.has_api ? sg.resp_len : 0u;
            r.post = sg.has_api ? sg.post_len : 0u;
            r.pad = 0;
        }
        for (uint32_t i = 0; i < na; i++) {
            const lamps_segment& sg = it->arrivals[i];
            SubmitRec& r = sr[i];
            r.slot = (uint32_t)((h->next_id + i) & h->cost.cap_mask);
            r.ctx = sg.prompt_len;
            r.pre = sg.pre_len;
            r.has = sg.has_api;
            r.api = sg.has_api ? aticks[i] : 0u;
            r.resp = sg.has_api ? sg.resp_len : 0u;
            r.post = sg.has_api ? sg.post_len : 0u;
            r.pad = 0;
        }
        if (ne) std::memcpy(reinterpret_cast<uint8_t*>(rr) + rbytes, it->events, ebytes);  // 16 B aligned
        h->inl_pending = inl;
        if (!inl && rbytes + ebytes) {
            CU(h, cudaMemcpyAsync(h->d_ingest, rr, rbytes + ebytes, cudaMemcpyHostToDevice, h->stream));
            if (int rc = staging_copied(h)) return rc;
        }
        h->b.events = static_cast<const uint8_t*>(h->d_ingest) + rbytes;
        ev_staged = true;
        h->ret_pending = nr;
        h->sub_pending = na;
        h->b.arrivals = static_cast<const ReturnRec*>(h->d_ingest) + nr;
        for (uint32_t k = 0; k < nr; k++) {
            h->hstate[it->return_ids[k] & h->cost.cap_mask] = H_READY;
            h->hctx[it->return_ids[k] & h->cost.cap_mask] = rctx[k] + it->return_resp[k];
        }
        for (uint32_t k = 0; k < na; k++) {
            h->hstate[(h->next_id + k) & h->cost.cap_mask] = H_READY;
            h->hctx[(h->next_id + k) & h->cost.cap_mask] = it->arrivals[k].prompt_len;
            if (it->arrival_ids_out) it->arrival_ids_out[k] = h->next_id + k;
        }
        h->next_id += na;
    } else {
        if (int rc = do_returns(h, it->return_ids, it->return_resp, it->return_next, nr, rticks, rctx, false))
            return rc;
        if (int rc = do_submit(h, it->arrivals, na, aticks, it->arrival_ids_out)) return rc;
    }
    // 3. the step with the events, its result (the one host synchronisation)
    if (ev_staged)
        events_staged(h, it->events, ne);
    else if (int rc = stage_events(h, it->events, ne))
        return rc;
    if (int rc = enqueue_step(h, it->kv_total_blocks, ne)) return rc;
    return fetch_result(h, out);
}

// A step group: loopback handles are ranks 0..n-1 of a world of n; P2P handles are distinct
// ranks of one world (n <= world: the other ranks step in other processes).
int check_group(lamps_t* const* hs, uint32_t n, bool p2p) {
    uint64_t seen = 0;
    for (uint32_t r = 0; r < n; r++) {
        if (!hs[r] || hs[r]->cfg.max_batch != hs[0]->cfg.max_batch || hs[r]->world != hs[0]->world)
            return fail(hs[0], LAMPS_EINVAL, "group: handles of one world");
        if (!p2p && (hs[r]->world != n || hs[r]->rank != r))
            return fail(hs[0], LAMPS_EINVAL, "group: loopback handles must be ranks 0..world-1");
        if (p2p && (hs[r]->rank >= hs[r]->world || (seen >> hs[r]->rank) & 1ull))
            return fail(hs[0], LAMPS_EINVAL, "group: P2P handles must be distinct ranks");
        seen |= 1ull << hs[r]->rank;
    }
    return LAMPS_OK;
}

int lamps_group_step(lamps_t* const* hs, uint32_t world, const lamps_event* const* ev, const uint32_t* n_ev,
                     const uint64_t* kv_total, lamps_step_out* out) {
    if (!hs || !n_ev || !kv_total || world < 2 || world > 32) return LAMPS_EINVAL;
    const bool p2p = hs[0] && hs[0]->cfg.transport == LAMPS_XPORT_P2P;
    if (int rc = check_group(hs, world, p2p)) return rc;
    for (uint32_t r = 0; r < world; r++) {
        if (!p2p && (hs[r]->cfg.transport != LAMPS_XPORT_LOOPBACK || hs[r]->stream != hs[0]->stream))
            return fail(hs[0], LAMPS_EINVAL, "group: loopback handles on one stream");
        if (p2p && (hs[r]->cfg.transport != LAMPS_XPORT_P2P || !(hs[r]->cfg.flags & LAMPS_SHARE_DEVICE) ||
                    (r && hs[r]->stream == hs[0]->stream)))
            return fail(hs[0], LAMPS_EINVAL, "group: P2P handles need LAMPS_SHARE_DEVICE and one stream each");
    }
    // two passes: every shard is validated before any shard is staged, so a refused shard
    // leaves every handle unchanged (staging itself can fail only on a CUDA error)
    for (uint32_t r = 0; r < world; r++) {
        if (int rc = check_events(hs[r], ev ? ev[r] : nullptr, n_ev[r], kv_total[r])) return rc;
        if (int rc = step_precheck(hs[r], true)) return rc;
    }
    for (uint32_t r = 0; r < world; r++) {
        int rc = stage_events(hs[r], ev ? ev[r] : nullptr, n_ev[r]);
        if (rc) return rc;
    }
    for (uint32_t r = 0; r < world; r++) {
        int rc = enqueue_phase1(hs[r], kv_total[r], n_ev[r]);
        if (rc) return rc;
    }
    const size_t bytes = ((size_t)hs[0]->cfg.max_batch + 1) * sizeof(MergeRec);
    for (uint32_t d = 0; d < world && !p2p; d++)
        for (uint32_t r = 0; r < world; r++)
            CU(hs[d], cudaMemcpyAsync(reinterpret_cast<uint8_t*>(hs[d]->b.xrecv) + r * bytes, hs[r]->b.xsend, bytes,
                                      cudaMemcpyDeviceToDevice, hs[d]->stream));
    for (uint32_t r = 0; r < world; r++) {
        int rc = enqueue_phase2(hs[r], kv_total[r], n_ev[r], false);
        if (rc) return rc;
    }
    for (uint32_t r = 0; r < world; r++) {
        int rc = fetch_result(hs[r], out ? &out[r] : nullptr);
        if (rc) return rc;
    }
    return LAMPS_OK;
}

int lamps_group_step_async(lamps_t* const* hs, uint32_t n, const uint64_t* kv_total) {
    if (!hs || !kv_total || n < 1 || n > 32 || !hs[0]) return LAMPS_EINVAL;
    if (int rc = check_group(hs, n, true)) return rc;
    for (uint32_t r = 0; r < n; r++) {
        if (hs[r]->cfg.transport != LAMPS_XPORT_P2P || !(hs[r]->cfg.flags & LAMPS_SHARE_DEVICE) || hs[r]->world < 2 ||
            (r && hs[r]->stream == hs[0]->stream))
            return fail(hs[0], LAMPS_EINVAL, "group async: P2P handles with LAMPS_SHARE_DEVICE and one stream each");
        if (int rc = check_events(hs[r], nullptr, 0, kv_total[r])) return rc;
        if (int rc = step_precheck(hs[r], true)) return rc;
    }
    for (uint32_t r = 0; r < n; r++)
        if (int rc = stage_events(hs[r], nullptr, 0)) return rc;
    for (uint32_t r = 0; r < n; r++) {
        if (int rc = enqueue_phase1(hs[r], kv_total[r], 0)) return rc;
        if (int rc = enqueue_phase2(hs[r], kv_total[r], 0, false)) return rc;
    }
    return LAMPS_OK;
}

int lamps_p2p_handle(lamps_t* h, void* out64) {
    if (!h || !out64) return LAMPS_EINVAL;
    if (!h->xbuf) return fail(h, LAMPS_EINVAL, "not a P2P-transport handle");
    cudaIpcMemHandle_t hd;
    CU(h, cudaIpcGetMemHandle(&hd, h->xbuf));
    std::memcpy(out64, &hd, sizeof(hd));
    std::lock_guard<std::mutex> lk(g_exp_mu);
    for (auto& e : g_exported)
        if (e.second == h->xbuf) return LAMPS_OK;
    g_exported.emplace_back(hd, h->xbuf);
    return LAMPS_OK;
}

int lamps_p2p_connect(lamps_t* h, const void* handles, size_t n_bytes) {
    if (!h || !handles) return LAMPS_EINVAL;
    if (!h->xbuf) return fail(h, LAMPS_EINVAL, "not a P2P-transport handle");
    if (n_bytes != (size_t)h->world * sizeof(cudaIpcMemHandle_t)) return fail(h, LAMPS_EINVAL, "need world handles");
    std::vector<MergeRec*> tab(h->world);
    for (uint32_t r = 0; r < h->world; r++) {
        if (r == h->rank) { tab[r] = h->xbuf; continue; }
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(hd), sizeof(hd));
        MergeRec* own = nullptr;
        {
            std::lock_guard<std::mutex> lk(g_exp_mu);
            for (auto& e : g_exported)
                if (!std::memcmp(&e.first, &hd, sizeof(hd))) own = e.second;
        }
        if (own) {  // exported by this process (a co-resident shard)
            tab[r] = own;
            continue;
        }
        void* p = nullptr;
        CU(h, cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
        h->peer_open.push_back(p);
        tab[r] = static_cast<MergeRec*>(p);
    }
    CU(h, cudaMemcpy(h->d_peers, tab.data(), tab.size() * sizeof(MergeRec*), cudaMemcpyHostToDevice));
    h->p2p_ready = true;
    return LAMPS_OK;
}

int lamps_p2p_connect_local(lamps_t* const* hs, uint32_t world) {
    if (!hs || world < 1 || world > 32) return LAMPS_EINVAL;
    std::vector<MergeRec*> tab(world);
    for (uint32_t r = 0; r < world; r++) {
        if (!hs[r] || !hs[r]->xbuf || hs[r]->world != world || hs[r]->rank != r) return LAMPS_EINVAL;
        tab[r] = hs[r]->xbuf;
    }
    for (uint32_t r = 0; r < world; r++) {
        CU(hs[r], cudaMemcpy(hs[r]->d_peers, tab.data(), tab.size() * sizeof(MergeRec*), cudaMemcpyHostToDevice));
        hs[r]->p2p_ready = true;
    }
    return LAMPS_OK;
}

int lamps_nccl_unique_id(void* out128) {
    if (!out128) return LAMPS_EINVAL;
    if (!g_nccl.load()) return LAMPS_ENCCL;
    return g_nccl.getUniqueId(out128) == 0 ? LAMPS_OK : LAMPS_ENCCL;
}

int lamps_schedule_step_async(lamps_t* h, uint64_t kv_total_blocks) {
    if (!h) return LAMPS_EINVAL;
    if (kv_total_blocks > h->cfg.kv_capacity_blocks)
        return fail(h, LAMPS_EINVAL, "kv_total_blocks exceeds kv_capacity_blocks");
    if (int rc0 = step_precheck(h)) return rc0;  // before enqueue_phase1 bumps the exchange sequence
    int rc = enqueue_step(h, kv_total_blocks, 0);
    if (rc) return rc;
    h->prev_known = false;
    return LAMPS_OK;
}

int lamps_step_result(lamps_t* h, lamps_step_out* out) {
    if (!h || !out) return LAMPS_EINVAL;
    if (!h->have_result) return fail(h, LAMPS_EINVAL, "no step has run");
    return fetch_result(h, out);
}

int lamps_pool_import(lamps_t* h, const lamps_pool_io* io, uint64_t id_base, uint64_t next_id) {
    if (!h || !io) return LAMPS_EINVAL;
    if (!io->id || !io->state || !io->has_api || !io->starving || !io->strategy || !io->cnt || !io->ctx ||
        !io->pre_rem || !io->api_ticks || !io->resp_len || !io->post_len || !io->pending)
        return fail(h, LAMPS_EINVAL, "import: NULL array");
    if (next_id < id_base || next_id - id_base > h->cap) return fail(h, LAMPS_EINVAL, "import: bad id window");
    const uint32_t cap = h->cap, cp = h->cap_pad;
    std::vector<uint32_t> sfc(cp, 0u);
    std::vector<uint8_t> hs(cap, H_FREE);
    for (uint32_t s = 0; s < cap; s++) {
        const uint32_t st = io->state[s];
        if (st > LAMPS_PAUSED_S) return fail(h, LAMPS_EINVAL, "import: bad state");
        if (st == LAMPS_FREE) continue;
        const uint64_t id = io->id[s];
        if (id < id_base || id >= next_id || (id & h->cost.cap_mask) != s)
            return fail(h, LAMPS_EINVAL, "import: id outside the window or in the wrong slot");
        if (io->has_api[s] > 1 || io->starving[s] > 1 || io->strategy[s] > 3 || io->cnt[s] > 65535 ||
            (io->age && io->age[s] > 127) || (io->dirty && io->dirty[s] > 1))
            return fail(h, LAMPS_EINVAL, "import: field out of range");
        sfc[s] = sfc_pack(st, io->has_api[s], io->starving[s], io->strategy[s], io->cnt[s]) |
                 ((io->age ? io->age[s] : 0u) << SFC_AGE_SHIFT) | ((io->dirty ? io->dirty[s] : 1u) ? SFC_DIRTY : 0u);
        hs[s] = st == LAMPS_READY ? H_READY : H_PAUSED;
    }
    // ingest staged by a failed lamps_iterate must not reach the imported pool
    if (int rc = staging_wait(h)) return rc;
    h->ret_pending = 0;
    h->sub_pending = 0;
    h->inl_pending = false;
    h->cold = true;  // the imported pool's distribution is unknown: bucket-histogram ranges first
    const Pool& P = h->b.pool;
    const uint32_t* src[6] = {io->ctx, io->pre_rem, io->api_ticks, io->resp_len, io->post_len, io->pending};
    uint32_t* dst[6] = {P.ctx, P.pre, P.api, P.resp, P.post, P.pend};
    std::vector<uint32_t> tmp(cp, 0u);
    CU(h, cudaMemcpyAsync(P.sfc, sfc.data(), (size_t)cp * 4, cudaMemcpyHostToDevice, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    for (int f = 0; f < 6; f++) {
        for (uint32_t s = 0; s < cap; s++) tmp[s] = io->state[s] == LAMPS_FREE ? 0u : src[f][s];
        CU(h, cudaMemcpyAsync(dst[f], tmp.data(), (size_t)cp * 4, cudaMemcpyHostToDevice, h->stream));
        CU(h, cudaStreamSynchronize(h->stream));
    }
    for (int half = 0; half < 2; half++) {  // cached scores (R26)
        for (uint32_t s = 0; s < cap; s++) {
            const uint64_t v = (io->cached_score && io->state[s] != LAMPS_FREE) ? io->cached_score[s] : 0ull;
            tmp[s] = half ? (uint32_t)(v >> 32) : (uint32_t)v;
        }
        CU(h, cudaMemcpyAsync(half ? P.schi : P.sclo, tmp.data(), (size_t)cp * 4, cudaMemcpyHostToDevice, h->stream));
        CU(h, cudaStreamSynchronize(h->stream));
    }
    CU(h, cudaMemsetAsync(P.stamp, 0, (size_t)cp * 4, h->stream));
    CU(h, cudaMemsetAsync(h->b.ctl, 0, sizeof(Ctl), h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    h->hstate.swap(hs);
    for (uint32_t s2 = 0; s2 < cap; s2++) h->hctx[s2] = io->state[s2] == LAMPS_FREE ? 0u : io->ctx[s2];
    h->shadow_ok = true;
    h->fetched_step = h->step;
    std::fill(h->adm_mark.begin(), h->adm_mark.end(), 0u);  // previous admitted list cleared
    h->id_base = id_base;
    h->next_id = next_id;
    advance_id_base(h);
    h->prev_adm.clear();
    h->prev_known = true;
    h->have_result = false;
    return LAMPS_OK;
}

int lamps_pool_export(lamps_t* h, lamps_pool_io* io) {
    if (!h || !io) return LAMPS_EINVAL;
    if ((io->dbg_w || io->dbg_score) && !h->b.dbg)
        return fail(h, LAMPS_EINVAL, "export: debug values need LAMPS_DEBUG_OUT");
    const uint32_t cap = h->cap;
    const Pool& P = h->b.pool;
    std::vector<uint32_t> sfc(cap);
    CU(h, cudaStreamSynchronize(h->stream));
    CU(h, cudaMemcpy(sfc.data(), P.sfc, (size_t)cap * 4, cudaMemcpyDeviceToHost));
    const uint32_t* src[6] = {P.ctx, P.pre, P.api, P.resp, P.post, P.pend};
    uint32_t* dst[6] = {io->ctx, io->pre_rem, io->api_ticks, io->resp_len, io->post_len, io->pending};
    for (int f = 0; f < 6; f++)
        if (dst[f]) CU(h, cudaMemcpy(dst[f], src[f], (size_t)cap * 4, cudaMemcpyDeviceToHost));
    for (uint32_t s = 0; s < cap; s++) {
        const uint32_t w = sfc[s];
        if (io->state) io->state[s] = sfc_state(w);
        if (io->has_api) io->has_api[s] = sfc_has(w);
        if (io->starving) io->starving[s] = sfc_starv(w);
        if (io->strategy) io->strategy[s] = sfc_strat(w);
        if (io->cnt) io->cnt[s] = sfc_cnt(w);
        if (io->age) io->age[s] = sfc_age(w);
        if (io->dirty) io->dirty[s] = (w & SFC_DIRTY) ? 1u : 0u;
        if (io->id)
            io->id[s] = sfc_state(w) == LAMPS_FREE ? 0ull
                                                    : h->id_base + ((s - h->id_base) & h->cost.cap_mask);
    }
    if (io->cached_score) {
        std::vector<uint32_t> lo(cap), hi(cap);
        CU(h, cudaMemcpy(lo.data(), P.sclo, (size_t)cap * 4, cudaMemcpyDeviceToHost));
        CU(h, cudaMemcpy(hi.data(), P.schi, (size_t)cap * 4, cudaMemcpyDeviceToHost));
        for (uint32_t s = 0; s < cap; s++) io->cached_score[s] = ((uint64_t)hi[s] << 32) | lo[s];
    }
    if (io->dbg_w || io->dbg_score) {
        std::vector<unsigned long long> d((size_t)cap * 4);
        CU(h, cudaMemcpy(d.data(), h->b.dbg, (size_t)cap * 32, cudaMemcpyDeviceToHost));
        for (uint32_t s = 0; s < cap; s++) {
            if (io->dbg_w)
                for (int k = 0; k < 3; k++) io->dbg_w[3 * (size_t)s + k] = d[4 * (size_t)s + k];
            if (io->dbg_score) io->dbg_score[s] = d[4 * (size_t)s + 3];
        }
    }
    return LAMPS_OK;
}

int lamps_ranked_keys(lamps_t* h, uint64_t* host_out, uint64_t max_keys, uint64_t* n_out) {
    if (!h || !n_out) return LAMPS_EINVAL;
    CU(h, cudaMemcpyAsync(h->h_ctl, h->b.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    const uint64_t n = h->h_ctl->n_ranked;  // n_eligible, or the head only (LAMPS_HEAD_ONLY)
    *n_out = n;
    if (host_out && max_keys) {
        const uint64_t m = std::min(n, max_keys);
        if (m) CU(h, cudaMemcpy(host_out, h->b.keys[h->h_ctl->final_buf & 1u], m * 8, cudaMemcpyDeviceToHost));
    }
    return LAMPS_OK;
}

int lamps_step_stats(lamps_t* h, uint32_t* kernels_launched, uint32_t* sort_passes) {
    if (!h) return LAMPS_EINVAL;
    CU(h, cudaMemcpyAsync(h->h_ctl, h->b.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    if (kernels_launched) *kernels_launched = h->last_kernels;
    if (sort_passes) *sort_passes = h->h_ctl->n_passes;
    return LAMPS_OK;
}

int lamps_trace_read(lamps_t* h, uint64_t* out, uint32_t max_words, uint32_t* n_cta) {
    if (!h || !out || !n_cta) return LAMPS_EINVAL;
    if (!h->b.trace) return fail(h, LAMPS_EINVAL, "tracing needs LAMPS_TRACE");
    if (!h->fused) return fail(h, LAMPS_ENOTSUP, "tracing is implemented for the fused path");
    CU(h, cudaStreamSynchronize(h->stream));
    const size_t words = std::min<size_t>(max_words, (size_t)h->fused_grid * kTraceSlots);
    CU(h, cudaMemcpy(out, h->b.trace, words * 8, cudaMemcpyDeviceToHost));
    *n_cta = h->fused_grid;
    return LAMPS_OK;
}

int lamps_timing_read(lamps_t* h, double ms[4], uint32_t* n_steps) {
    if (!h || !ms) return LAMPS_EINVAL;
    if (!(h->cfg.flags & LAMPS_TIMING)) return fail(h, LAMPS_EINVAL, "timing needs LAMPS_TIMING");
    CU(h, cudaStreamSynchronize(h->stream));
    for (int k = 0; k < 4; k++) ms[k] = 0.0;
    const uint32_t n = h->t_count;
    const uint32_t first = (h->t_head + kTimingRing - n) % kTimingRing;
    for (uint32_t i = 0; i < n; i++) {
        const size_t r = (size_t)((first + i) % kTimingRing) * 5;
        for (int k = 0; k < 4; k++) {
            float t = 0.f;
            CU(h, cudaEventElapsedTime(&t, h->tev[r + k], h->tev[r + k + 1]));
            ms[k] += t;
        }
    }
    if (n_steps) *n_steps = n;
    h->t_count = 0;
    return LAMPS_OK;
}

}  // extern "C"
