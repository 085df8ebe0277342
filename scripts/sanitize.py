"""Driver for compute-sanitizer runs (scripts/sanitize.sh): a short closed loop through
every step path -- the fused kernel (iterate: returns, arrivals and events in the
prologue), the 3-kernel path, the forced global-sort fallback, the head-only ranking, the
score cache, the baseline policies, the world-1 P2P exchange + in-kernel merge -- plus the
predictor ingest.  No parity checks here (the tests do those); the sanitizer checks memory
accesses, shared-memory races, barrier use and uninitialised reads.

usage: python scripts/sanitize.py [mode ...]   (default: all modes)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2410_18248_b200 import Scheduler  # noqa: E402
from paper_2410_18248_b200 import lamps as L  # noqa: E402

STEPS = int(os.environ.get("STEPS", "12"))


def segs(rows):
    a = np.zeros(len(rows), L.SEGMENT_DTYPE)
    for k, r in enumerate(rows):
        for f in ("prompt_len", "pre_len", "resp_len", "post_len", "api_seconds", "has_api"):
            a[k][f] = r.get(f, 0)
    return a


def closed_loop(name, cname="C3", n_req=1500, flags=0, transport=None, **over):
    cfg = gen.lib_config(cname, **over)
    kv = gen.CONFIGS[cname]["kv_total"]
    kw = {} if transport is None else dict(transport=transport)
    s = Scheduler(cfg, flags=flags, **kw)
    reqs = gen.requests(cname, n_req, seed=3)
    drv = gen.ClosedLoop(reqs, gen.PROFILES[gen.CONFIGS[cname]["profile"]]["tau"], 600, 6.0, 3)
    prev, n_adm = [], 0
    for t in range(STEPS):
        rids, resp, rrows = drv.api_returns(t)
        idx, arows = drv.arrivals(t)
        ev = drv.events(t, prev)
        g, gids = s.iterate(events=ev, ret_ids=rids, ret_resp=resp, ret_next=segs(rrows), arrivals=segs(arows),
                            kv_total=kv)
        if len(arows):
            drv.on_submitted(idx, gids)
        prev = g["admitted_id"]
        n_adm += len(prev)
    s.close()
    print(f"{name}: {STEPS} steps, {n_adm} admissions", flush=True)


def predict():
    cfg = gen.lib_config("C3")
    s = Scheduler(cfg)
    t = gen.truths("C3", 500, seed=1)
    truth = np.zeros(len(t["key"]), L.TRUTH_DTYPE)
    for f in truth.dtype.names:
        if f in t:
            truth[f] = t[f]
    truth["pre_bin"] = L.LAMPS_NO_BIN
    out = s.predict(truth, seed=5, len_error_ppm=200_000, api_error_ppm=100_000)
    print(f"predict: {len(out)} segments", flush=True)
    s.close()


def c5(flags=0):
    """The bench pool (2^20 slots): the planned head, full-size ranges, the weights."""
    cfg = gen.lib_config("C5")
    snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99, n=cfg["capacity"] - 8192)
    s = Scheduler(cfg, flags=flags)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    for _ in range(STEPS):
        g = s.step(kv_total=gen.CONFIGS["C5"]["kv_total"])
    print(f"c5 flags={flags}: {STEPS} steps, {g['n_eligible']} eligible, {g['n_admitted']} admitted", flush=True)
    s.close()


def large_merge(world=4, K=4096):
    """Loopback shards whose world * K records exceed one CTA's shared memory: the grid-wide
    merge by rank (k_merge_count / k_merge_place / k_merge_cut)."""
    cfg = gen.lib_config("C4", max_batch=K)
    cfg["capacity"] = 32768
    stream = torch.cuda.current_stream()
    S = [Scheduler(cfg, world=world, rank=r, transport=L.LAMPS_XPORT_LOOPBACK, stream=stream) for r in range(world)]
    for r, sh in enumerate(S):
        snap = gen.snapshot("C4", seed=r, n=25000, capacity=32768, id_base=1000)
        sh.import_pool(snap, snap["id_base"], snap["next_id"])
    for _ in range(max(2, STEPS // 3)):
        outs = Scheduler.group_step(S, None, [250_000] * world)
    print(f"large_merge W={world} K={K}: {sum(o['n_admitted'] for o in outs)} admitted", flush=True)
    for sh in S:
        sh.close()


def c4_head_only():
    """The fused kernel's head-only ranking (warm steps place only the head) on C4."""
    cfg = gen.lib_config("C4")
    snap = gen.snapshot("C4", seed=0, id_base=77)
    s = Scheduler(cfg, flags=L.LAMPS_HEAD_ONLY)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    for _ in range(STEPS):
        g = s.step(kv_total=gen.CONFIGS["C4"]["kv_total"])
    print(f"c4_head_only: {g['n_eligible']} eligible, {g['n_admitted']} admitted", flush=True)
    s.close()


MODES = {
    "fused": lambda: closed_loop("fused"),  # C3: the one-CTA small-pool kernel
    "grid": lambda: closed_loop("grid", flags=L.LAMPS_GRID_STEP),  # C3 on the grid-wide fused kernel
    "small_fallback": lambda: closed_loop("small_fallback", flags=L.LAMPS_FORCE_FALLBACK),
    "grid_fallback": lambda: closed_loop("grid_fallback", flags=L.LAMPS_GRID_STEP | L.LAMPS_FORCE_FALLBACK),
    "multi": lambda: closed_loop("multi", flags=L.LAMPS_MULTI_KERNEL),
    "head_only": lambda: closed_loop("head_only", flags=L.LAMPS_HEAD_ONLY),
    "interval10": lambda: closed_loop("interval10", score_interval=10),
    "sjf": lambda: closed_loop("sjf", policy=L.LAMPS_POLICY_SJF),
    "fcfs": lambda: closed_loop("fcfs", policy=L.LAMPS_POLICY_FCFS),
    "starve": lambda: closed_loop("starve", cname="C1", n_req=16, starvation_threshold=3),
    "p2p_merge": lambda: closed_loop("p2p_merge", flags=L.LAMPS_MERGE, transport=L.LAMPS_XPORT_P2P),
    "predict": predict,
    "c5": c5,
    "c5_head_only": lambda: c5(L.LAMPS_HEAD_ONLY),
    "c4_head_only": c4_head_only,
    "large_merge": large_merge,
    "big": lambda: closed_loop("big", flags=L.LAMPS_BIG_STEP),  # the large-pool path on C3
    "big_fallback": lambda: closed_loop("big_fallback", flags=L.LAMPS_BIG_STEP | L.LAMPS_FORCE_FALLBACK),
}

if __name__ == "__main__":
    torch.cuda.init()
    for m in sys.argv[1:] or list(MODES):
        MODES[m]()
