"""Iteration-level serving engine at workload scale, driving the scheduling pass through
its public API (part 2).

Every step is one decode iteration of tau ticks.  The engine holds the TRUE request
(gen.requests: segments of decode tokens, API duration, response length, and the
final decode run); the scheduler is told PREDICTED segments, produced by the
backend's predictor ingest (lamps_predict: error ~ N(0, p*m), row F4).
Per step:

  1. arrivals (Poisson, ``rate`` requests per second) are submitted;
  2. API calls that finished return with their true response, and the next
     segment's prediction;
  3. the previously admitted batch generated one token each: a request that
     reached its TRUE pre-API length reports API_CALL, one that reached its true
     final length reports FINISHED (misprediction: the pass clamps pre_rem at 0
     and waits for the event, R24);
  4. one lamps_schedule_step over the whole pool ranks and admits (A0-A5).

The engine's physics are the pass's own iteration semantics (a prefill or
recomputation runs in the iteration that admits it, as in vLLM's chunk-free
prefill); an API call returns after ceil(true duration / tau) steps.  Metrics:
per-request completion time (finish step + 1 - arrival step) x tau, and
throughput.  No method arithmetic lives here.
"""
from __future__ import annotations

import math

import numpy as np

import gen

EV_API_CALL, EV_FINISHED = 1, 2
EVENT_DTYPE = np.dtype([("id", np.uint64), ("kind", np.uint32), ("reserved", np.uint32)], align=True)
TRUTH_DTYPE = np.dtype([("key", np.uint64), ("prompt_len", np.uint32), ("pre_len", np.uint32),
                        ("pre_bin", np.uint32), ("resp_len", np.uint32), ("post_len", np.uint32),
                        ("api_ticks", np.uint32), ("has_api", np.uint32), ("reserved", np.uint32)], align=True)
NO_BIN = 0xFFFFFFFF
KEY_STRIDE = 64  # RNG stream key = request index * 64 + segment


class SchedulerBackend:
    """The CUDA pass (paper_2410_18248_b200.Scheduler) as the engine's scheduler."""

    def __init__(self, cfg: dict, flags: int = 0):
        from paper_2410_18248_b200 import Scheduler
        self.s = Scheduler(cfg, flags=flags)

    def predict(self, truth, seed, len_ppm, api_ppm):
        return self.s.predict(truth, seed=seed, len_error_ppm=len_ppm, api_error_ppm=api_ppm)

    def submit(self, segs):
        return self.s.submit(segs)

    def api_return(self, ids, resp, segs):
        self.s.api_return(ids, resp, segs)

    def step(self, ev, kv_total):
        return self.s.step(ev, kv_total)

    def close(self):
        self.s.close()


def _truth_rows(reqs, items, tps):
    """items: (request index, segment k, prompt_len) -> TRUTH_DTYPE records of the true segment k."""
    t = np.zeros(len(items), TRUTH_DTYPE)
    for j, (i, k, prompt) in enumerate(items):
        r = reqs[i]
        segs = r["segs"]
        t[j]["key"] = i * KEY_STRIDE + k
        t[j]["prompt_len"] = prompt
        t[j]["pre_bin"] = NO_BIN
        if k < len(segs):
            t[j]["pre_len"] = segs[k][0]
            t[j]["has_api"] = 1
            t[j]["api_ticks"] = int(round(segs[k][1] * tps))
            t[j]["resp_len"] = segs[k][2]
            t[j]["post_len"] = segs[k + 1][0] if k + 1 < len(segs) else r["final"]
        else:
            t[j]["pre_len"] = r["final"]
    return t


def run(cname: str, n_req: int, rate: float, backend, *, seed: int = 0, kv_total: int | None = None,
        len_error_ppm: int = 0, api_error_ppm: int = 0, noise_seed: int = 1, max_steps: int = 200_000,
        profile: str | None = None, reqs=None, api_scale: float = 1.0) -> dict:
    """Run the closed loop until every request finished (or max_steps).  Returns metrics.
    api_scale multiplies every true API duration (regimes where queueing, not the API wait,
    dominates the completion time)."""
    c = gen.CONFIGS[cname]
    prof = gen.PROFILES[profile or c["profile"]]
    tau, tps = prof["tau"], prof["ticks_per_second"]
    kv = c["kv_total"] if kv_total is None else kv_total
    reqs = gen.requests(cname, n_req, seed=seed) if reqs is None else reqs
    if api_scale != 1.0:
        reqs = [dict(r, segs=[(p, d * api_scale, resp) for (p, d, resp) in r["segs"]]) for r in reqs]
    rng = np.random.Generator(np.random.PCG64(0xF2 + seed))
    per_step = rate * tau / tps
    arrive = []
    t = 0.0
    for _ in range(n_req):  # Poisson arrivals: exponential gaps, in steps
        t += rng.exponential(1.0 / per_step) if per_step > 0 else 0.0
        arrive.append(int(t))
    by_step = {}
    for i, a in enumerate(arrive):
        by_step.setdefault(a, []).append(i)

    rid_req, seg, tok = {}, {}, {}
    returns = {}
    done_at = np.full(n_req, -1, np.int64)
    prev = np.zeros(0, np.uint64)
    admitted_total = preempted_total = 0
    n_done = 0
    step = 0
    for step in range(max_steps):
        idx = by_step.get(step, [])
        if idx:
            truth = _truth_rows(reqs, [(i, 0, reqs[i]["prompt"]) for i in idx], tps)
            segs = backend.predict(truth, noise_seed, len_error_ppm, api_error_ppm)
            ids = backend.submit(segs)
            for i, rid in zip(idx, ids):
                rid_req[int(rid)], seg[int(rid)], tok[int(rid)] = i, 0, 0
        back = returns.pop(step, [])
        if back:
            items, resp = [], []
            for rid in back:
                i = rid_req[rid]
                k = seg[rid]
                resp.append(reqs[i]["segs"][k][2])
                seg[rid], tok[rid] = k + 1, 0
                items.append((i, k + 1, 0))
            segs = backend.predict(_truth_rows(reqs, items, tps), noise_seed, len_error_ppm, api_error_ppm)
            backend.api_return(np.array(back, np.uint64), np.array(resp, np.uint32), segs)
        ev = []
        for rid in prev:
            rid = int(rid)
            i, k = rid_req[rid], seg[rid]
            tok[rid] += 1
            r = reqs[i]
            need = r["segs"][k][0] if k < len(r["segs"]) else r["final"]
            if tok[rid] >= need:
                if k < len(r["segs"]):
                    ev.append((rid, EV_API_CALL))
                    wait = max(1, math.ceil(round(r["segs"][k][1] * tps) / tau))
                    returns.setdefault(step + wait, []).append(rid)
                else:
                    ev.append((rid, EV_FINISHED))
                    done_at[i] = step
                    n_done += 1
        e = np.zeros(len(ev), EVENT_DTYPE)
        for j, (rid, kind) in enumerate(ev):
            e[j]["id"], e[j]["kind"] = rid, kind
        if n_done == n_req:
            break
        g = backend.step(e, kv)
        prev = g["admitted_id"]
        admitted_total += g["n_admitted"]
        preempted_total += g["n_preempted"]
    fin = done_at >= 0
    arr = np.array(arrive)
    jct = (done_at[fin] + 1 - arr[fin]) * tau / tps
    span = (done_at[fin].max() + 1) * tau / tps if fin.any() else float("nan")
    return {
        "config": cname, "n_req": n_req, "rate": rate, "steps": step + 1, "finished": int(fin.sum()),
        "jct_mean_s": float(jct.mean()) if fin.any() else float("nan"),
        "jct_median_s": float(np.median(jct)) if fin.any() else float("nan"),
        "jct_p99_s": float(np.percentile(jct, 99)) if fin.any() else float("nan"),
        "throughput_rps": float(fin.sum() / span) if fin.any() else 0.0,
        "admitted_per_step": admitted_total / max(1, step + 1),
        "preempted_total": int(preempted_total),
        "len_error_ppm": len_error_ppm, "api_error_ppm": api_error_ppm,
        "done_step": done_at.tolist(),
    }
