"""The worked example's unit model (Table 1).

Time advances in units of one decode iteration; memory is counted in tokens (one
unit per context token, prompt 0, B = 1); the budget is 6 units; at most
``max_running`` requests run per unit (one in the example, "only one request can run
at a time").  Engine rules (the paper's stylised vLLM engine):

  * iteration-level preemptive priority: every unit the ranker orders the READY
    requests; a preempted request keeps its KV resident;
  * admission: walk the ranked order and run the first request(s) whose peak
    footprint up to the end of its current segment fits next to everything resident
    (``resident of the others + ctx + remaining recompute/decode <= budget``):
    "R3's pre-API part cannot run during R1's API call because it will not release
    memory before the API response completes", "leaving only 1 unit
    available, which is insufficient to start the post-API part of R2";
  * at its API call a request takes the handling label the ranker gave it (the
    pass's argmin, Eq. 1-3): Preserve keeps its KV resident for the call, Discard
    frees it and recomputes its context at one iteration per token on return
    ("a post-API part of length 2 (including recomputation)"), Swap moves it
    to host memory and back at no time cost;
  * API durations are whole units; completion time = the end of the last unit.

The engine passes the ranker the state a scheduler sees: ctx, remaining decode
tokens, API duration, post-API tokens, and the owed recomputation as ``pending``
ticks (recompute tokens x tau).  No method arithmetic lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

FREE, READY, PAUSED_P, PAUSED_D, PAUSED_S = 0, 1, 2, 3, 4
P, D, S, NONE = 0, 1, 2, 3


@dataclass
class UnitRequest:
    pre: int        # decode tokens before the API call
    api_iters: int  # API duration, iterations
    post: int       # decode tokens after the API
    arrival: int = 0
    # engine state
    ctx: int = 0
    resident: int = 0
    recompute: int = 0
    pre_rem: int = 0
    seg: int = 0
    state: int = FREE
    label: int = NONE
    api_label: int = NONE  # handling strategy taken at the API call
    ret_at: int = -1
    done_at: int = -1
    ran: list = field(default_factory=list)


def _fields(reqs, ids, cap, tau):
    f = {k: [0] * cap for k in ("id", "state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem",
                                "api_ticks", "resp_len", "post_len", "pending")}
    f["strategy"] = [NONE] * cap
    for r, i in zip(reqs, ids):
        if r.state == FREE:
            continue
        s = i % cap
        f["id"][s] = i
        f["state"][s] = r.state
        has = 1 if r.seg == 0 else 0
        f["has_api"][s] = has
        f["ctx"][s] = r.ctx
        f["pre_rem"][s] = r.pre_rem
        f["api_ticks"][s] = r.api_iters * tau if has else 0
        f["post_len"][s] = r.post if has else 0
        f["pending"][s] = r.recompute * tau
        if r.state in (PAUSED_P, PAUSED_D, PAUSED_S):
            f["strategy"][s] = r.label
    return f


def simulate_unit(specs, ranker, budget=6, max_running=1, tau=1, cap=16, id_base=0, horizon=1000):
    """Run the unit model to completion.  specs: list of (pre, api_iters, post) or
    UnitRequest; ids are id_base + arrival index.  Returns (requests, timeline) where
    timeline[t] = ids that ran in unit [t, t+1)."""
    reqs = [s if isinstance(s, UnitRequest) else UnitRequest(*s) for s in specs]
    ids = [id_base + k for k in range(len(reqs))]
    by_id = dict(zip(ids, reqs))
    timeline = []
    for t in range(horizon):
        for r in reqs:  # arrivals and API returns at time t
            if r.state == FREE and r.arrival == t and r.done_at < 0:
                r.state, r.seg, r.pre_rem = READY, 0, r.pre
            if r.state in (PAUSED_P, PAUSED_D, PAUSED_S) and r.ret_at == t:
                if r.state == PAUSED_D:
                    r.resident, r.recompute = 0, r.ctx
                elif r.state == PAUSED_S:
                    r.resident = r.ctx  # swapped back in, no time cost
                r.state, r.seg, r.pre_rem = READY, 1, r.post
        if all(r.done_at >= 0 for r in reqs):
            break
        ready = [i for i, r in by_id.items() if r.state == READY]
        ran = []
        if ready:
            order, labels = ranker.rank(_fields(reqs, ids, cap, tau), id_base, id_base + len(reqs))
            for i, lab in labels.items():
                if by_id[i].state == READY:
                    by_id[i].label = lab
            resident = sum(r.resident for r in reqs)
            for i in order:
                if len(ran) == max_running:
                    break
                r = by_id[i]
                peak = r.ctx + r.pre_rem  # context at the end of the current segment
                if resident - r.resident + peak <= budget:
                    ran.append(i)
                    resident += peak - r.resident
        for i in ran:
            r = by_id[i]
            r.ran.append(t)
            if r.recompute:
                r.recompute -= 1
                r.resident += 1
            else:
                r.ctx += 1
                r.resident += 1
                r.pre_rem -= 1
            if r.recompute == 0 and r.pre_rem == 0:
                if r.seg == 0:
                    r.api_label = r.label
                    r.state = {P: PAUSED_P, D: PAUSED_D, S: PAUSED_S}[r.label]
                    r.ret_at = t + 1 + r.api_iters
                    if r.state != PAUSED_P:
                        r.resident = 0
                else:
                    r.state, r.done_at, r.resident = FREE, t + 1, 0
        timeline.append(ran)
        assert sum(r.resident for r in reqs) <= budget, "engine invariant: resident KV within the budget"
    return reqs, timeline


def average_jct(reqs) -> Fraction:
    return Fraction(sum(r.done_at - r.arrival for r in reqs), len(reqs))
