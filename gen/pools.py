"""Seeded synthetic request pools and request specs.

This module draws INPUTS only; it holds none of the method's arithmetic (no
waste, no strategy argmin, no score, no sort, no admission, no T_fwd/T_swap).
It feeds both the CUDA path and the oracle, which each compute everything
else independently.

Distributions (Table 2):
  prompt   lognormal(median, sigma) clipped to [lo, hi]  (256/0.8/[16,2048];
           ToolBench 1024/0.8/[128,4096])
  pre_len  10*b + 5, b ~ U{0..49}  (50 bins of 10 tokens)
  post_len U[1, 200]
  API      class uniform over the config's classes; duration truncated-normal
           (mean, std) of Table 2, in integer ticks (1 us); calls per request
           truncated-normal of Table 2 "Num", rounded, >= 1 (multi-API only)
  resp_len per-class constant (Math 8, QA 64, VE 32, Chatbot 128, Image 16,
           TTS 16, ToolBench 96)
Snapshot state mix: 75% READY / 25% PAUSED (Preserve-paused capped at 40% of
the KV budget, the excess stays READY); READY progress ~ U[0, pre_len];
20% of READY slots are fresh arrivals owing a prefill of ~100 ticks/token;
cnt ~ U{0..T-1} (1% at T..T+19); 5% already starving.  PAUSED slots get a handling label by
a generator heuristic (short API classes -> P, long -> D below 440 tokens of
context else S); it only needs to look plausible, not to be the argmin.
"""
from __future__ import annotations

import numpy as np

from .configs import API_CLASSES, CONFIGS, PROFILES

FREE, READY, PAUSED_P, PAUSED_D, PAUSED_S = 0, 1, 2, 3, 4
P, D, S, NONE = 0, 1, 2, 3

SEED_BASE = 0x2410182480


def rng_for(cname: str, seed: int = 0) -> np.random.Generator:
    k = int(cname[1:]) if cname[1:].isdigit() else 0
    return np.random.Generator(np.random.PCG64(SEED_BASE + 1000 * k + seed))


def _lognormal_clip(rng, n, median, sigma, lo, hi):
    x = np.exp(np.log(median) + sigma * rng.standard_normal(n))
    return np.clip(np.rint(x), lo, hi).astype(np.int64)


def _truncnorm(rng, n, mean, std, lo=0.0):
    x = mean + std * rng.standard_normal(n)
    bad = x < lo
    while bad.any():
        x[bad] = mean + std * rng.standard_normal(int(bad.sum()))
        bad = x < lo
    return x


def _class_arrays(rng, n, classes):
    ci = rng.integers(0, len(classes), n)
    dur_s = np.zeros(n)
    resp = np.zeros(n, np.int64)
    num = np.zeros(n, np.int64)
    for k, c in enumerate(classes):
        m = ci == k
        cnt = int(m.sum())
        if cnt == 0:
            continue
        st = API_CLASSES[c]
        dur_s[m] = _truncnorm(rng, cnt, *st["dur"])
        resp[m] = st["resp"]
        num[m] = np.maximum(1, np.rint(_truncnorm(rng, cnt, *st["num"], lo=-1e9))).astype(np.int64)
    return ci, dur_s, resp, num


def snapshot(cname: str, seed: int = 0, id_base: int = 0, n: int | None = None,
             capacity: int | None = None, **over) -> dict:
    """A per-slot pool snapshot: dict of arrays of length `capacity` plus 'id'.

    Slots hold ids id_base .. id_base+n-1 (slot = id mod capacity, so a
    non-zero id_base exercises ring wrap-around); the remaining slots are FREE.
    """
    c = dict(CONFIGS[cname]); c.update(over)
    n = c["n"] if n is None else n
    cap = c["capacity"] if capacity is None else capacity
    assert n <= cap
    rng = rng_for(cname, seed)
    med, sig, lo, hi = c["prompt"]
    prompt = _lognormal_clip(rng, n, med, sig, lo, hi)
    pre_len = 10 * rng.integers(0, 50, n) + 5
    post_len = rng.integers(1, 201, n)
    ci, dur_s, resp, num = _class_arrays(rng, n, c["classes"])
    ticks = np.rint(dur_s * 1e6).astype(np.int64)  # integer input ticks (us)

    # earlier segments already done (multi-API): extra context from finished segments
    if c["multi_api"]:
        done_calls = np.minimum((rng.random(n) * num).astype(np.int64), 6)
        extra = done_calls * (resp + rng.integers(1, 201, n))
        has_api = (rng.random(n) >= 0.1).astype(np.int64)  # 10% in their final segment
    else:
        extra = np.zeros(n, np.int64)
        has_api = (rng.random(n) >= 0.1).astype(np.int64)  # 10% already past their API

    u = rng.random(n)
    state = np.where(u < 0.75, READY, 0)
    paused = u >= 0.75
    long_api = dur_s > 2.0
    ctx_at_api = prompt + extra + pre_len
    lab = np.where(~long_api, PAUSED_P, np.where(ctx_at_api < 440, PAUSED_D, PAUSED_S))
    # Preserve-paused requests hold their KV on the GPU, so only as many as fit in
    # ~40% of the KV budget can be paused that way at once; the rest are READY.
    pblk = -(-(ctx_at_api) // PROFILES[c["profile"]]["block_tokens"])
    isP = paused & (lab == PAUSED_P)
    keep = np.cumsum(np.where(isP, pblk, 0)) <= int(0.4 * c["kv_total"])
    drop = isP & ~keep
    paused = paused & ~drop
    state = np.where(drop, READY, state)
    state = np.where(paused, lab, state)
    has_api = np.where(paused, 1, has_api)

    progress = (rng.random(n) * (pre_len + 1)).astype(np.int64)
    progress = np.minimum(progress, pre_len)
    ctx = np.where(paused, prompt + extra + pre_len, prompt + extra + progress)
    pre_rem = np.where(paused, 0, pre_len - progress)
    fresh = (~paused) & (rng.random(n) < 0.2)
    ctx = np.where(fresh, prompt + extra, ctx)
    pre_rem = np.where(fresh, pre_len, pre_rem)
    pending = np.where(fresh, prompt * 100 + rng.integers(0, 1000, n), 0)
    T = c["starvation_threshold"]
    cnt = rng.integers(0, T, n)
    cnt = np.where(rng.random(n) < 0.01, T + rng.integers(0, 20, n), cnt)  # 1% hit T now
    starving = (rng.random(n) < 0.05).astype(np.int64)
    strategy = np.where(paused, lab - PAUSED_P, NONE)
    cnt = np.where(paused & (starving == 0), 0, cnt)

    api_ticks = np.where(has_api == 1, ticks, 0)
    resp_len = np.where(has_api == 1, resp, 0)
    post = np.where(has_api == 1, post_len, 0)

    ids = id_base + np.arange(n, dtype=np.int64)
    slots = ids % cap
    out = {f: np.zeros(cap, np.int64) for f in
           ("id", "state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem",
            "api_ticks", "resp_len", "post_len", "pending")}
    out["strategy"][:] = NONE
    for f, v in (("id", ids), ("state", state), ("has_api", has_api), ("starving", starving),
                 ("strategy", strategy), ("cnt", cnt), ("ctx", ctx), ("pre_rem", pre_rem),
                 ("api_ticks", api_ticks), ("resp_len", resp_len), ("post_len", post),
                 ("pending", pending)):
        out[f][slots] = v
    # FREE slots: id is the would-be id of the window (unused by either side)
    free = np.ones(cap, bool); free[slots] = False
    out["id"][free] = 0
    out["next_id"] = int(id_base + n)
    out["id_base"] = int(id_base)
    out["capacity"] = cap
    return out


def requests(cname: str, n: int, seed: int = 0, **over) -> list:
    """Ground-truth request specs for closed-loop traces.

    Each request: dict(prompt, segs=[(decode_tokens, api_seconds, resp_len), ...],
    final=decode tokens after the last API).  Predictions are exact (no error injection).
    """
    c = dict(CONFIGS[cname]); c.update(over)
    rng = rng_for(cname, 7919 + seed)
    med, sig, lo, hi = c["prompt"]
    prompt = _lognormal_clip(rng, n, med, sig, lo, hi)
    ci, dur_s, resp, num = _class_arrays(rng, n, c["classes"])
    out = []
    for k in range(n):
        calls = int(min(num[k], 4)) if c["multi_api"] else 1
        if not c["multi_api"] and rng.random() < 0.1:
            calls = 0
        segs = []
        for j in range(calls):
            st = API_CLASSES[c["classes"][ci[k]]]
            d = float(_truncnorm(rng, 1, *st["dur"])[0]) if j else float(dur_s[k])
            segs.append((int(10 * rng.integers(0, 50) + 5), d, int(resp[k])))
        out.append(dict(prompt=int(prompt[k]), segs=segs, final=int(rng.integers(1, 201))))
    return out


def truths(cname: str, n: int, seed: int = 0, bins: bool = False, key0: int = 0, **over) -> dict:
    """Measured values of n first segments for the predictor ingest (row F4), as plain
    arrays (the caller packs them into its own record type): prompt, pre_len (or the
    predictor's bin b with pre_len = 0 when bins=True), resp_len, post_len, api_ticks
    (quantised measured duration, 1 us ticks), has_api, key = key0 + index."""
    c = dict(CONFIGS[cname]); c.update(over)
    rng = rng_for(cname, 104729 + seed)
    med, sig, lo, hi = c["prompt"]
    prompt = _lognormal_clip(rng, n, med, sig, lo, hi)
    b = rng.integers(0, 50, n)
    ci, dur_s, resp, num = _class_arrays(rng, n, c["classes"])
    has = (rng.random(n) >= 0.1).astype(np.int64)
    post = rng.integers(1, 201, n)
    return {
        "key": key0 + np.arange(n, dtype=np.int64),
        "prompt_len": prompt,
        "pre_len": np.zeros(n, np.int64) if bins else 10 * b + 5 + rng.integers(-4, 5, n),
        "pre_bin": b if bins else np.full(n, 0xFFFFFFFF, np.int64),
        "resp_len": np.where(has == 1, resp, 0),
        "post_len": np.where(has == 1, post, 0),
        "api_ticks": np.where(has == 1, np.rint(dur_s * 1e6).astype(np.int64), 0),
        "has_api": has,
    }
