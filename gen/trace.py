"""Closed-loop trace driver: the "engine" side of a scheduling loop.

It turns each step's admitted list into the next step's inputs -- engine events
(API_CALL when a request has generated the last token before its API, FINISHED
at the end), API returns (after ceil(duration / tau) steps of pause) and new
arrivals.  It is shared host code that plays the engine for BOTH
implementations under test; it contains none of the method's arithmetic
(strategies, scores, order and admission all come from the implementations).
Predictions are exact: the segment the scheduler is told about is the one the
engine then runs.
"""
from __future__ import annotations

import math

import numpy as np

EV_API_CALL, EV_FINISHED = 1, 2


def seg_row(req: dict, k: int, ctx_prompt: int | None = None) -> dict:
    """Prediction record for segment k of a request (lamps_segment fields)."""
    segs = req["segs"]
    dec = segs[k][0] if k < len(segs) else req["final"]
    row = dict(prompt_len=req["prompt"] if ctx_prompt is None else ctx_prompt, pre_len=dec,
               resp_len=0, post_len=0, api_seconds=0.0, has_api=0)
    if k < len(segs):
        row.update(has_api=1, api_seconds=segs[k][1], resp_len=segs[k][2],
                   post_len=segs[k + 1][0] if k + 1 < len(segs) else req["final"])
    return row


class ClosedLoop:
    def __init__(self, reqs: list, tau_ticks: int, initial: int, per_step: float, seed: int = 0):
        self.reqs = reqs
        self.tau = tau_ticks
        rng = np.random.Generator(np.random.PCG64(0xC105ED + seed))
        self.arrive_at = {}
        t = 0
        for i in range(len(reqs)):
            if i >= initial:
                t += int(rng.poisson(1.0 / per_step)) if per_step > 0 else 1
            self.arrive_at.setdefault(t if i >= initial else 0, []).append(i)
        self.id_req = {}      # id -> request index
        self.seg = {}         # id -> current segment index
        self.tok = {}         # id -> tokens generated in the current segment
        self.returns = {}     # step -> list of ids
        self.finished = 0

    def arrivals(self, t: int):
        idx = self.arrive_at.get(t, [])
        return idx, [seg_row(self.reqs[i], 0) for i in idx]

    def on_submitted(self, idx, ids):
        for i, rid in zip(idx, ids):
            rid = int(rid)
            self.id_req[rid] = i
            self.seg[rid] = 0
            self.tok[rid] = 0

    def events(self, t: int, prev_admitted) -> np.ndarray:
        """Engine report for the iteration that ran the previous admitted batch."""
        ev = []
        for rid in prev_admitted:
            rid = int(rid)
            req = self.reqs[self.id_req[rid]]
            k = self.seg[rid]
            self.tok[rid] += 1
            need = req["segs"][k][0] if k < len(req["segs"]) else req["final"]
            if self.tok[rid] >= need:
                if k < len(req["segs"]):
                    ev.append((rid, EV_API_CALL))
                    steps = max(1, math.ceil(req["segs"][k][1] * 1e6 / self.tau))
                    self.returns.setdefault(t + steps, []).append(rid)
                else:
                    ev.append((rid, EV_FINISHED))
                    self.finished += 1
        a = np.zeros(len(ev), np.dtype([("id", np.uint64), ("kind", np.uint32),
                                        ("reserved", np.uint32)], align=True))
        for j, (rid, kind) in enumerate(ev):
            a[j]["id"], a[j]["kind"] = rid, kind
        return a

    def api_returns(self, t: int):
        ids = self.returns.pop(t, [])
        resp, rows = [], []
        for rid in ids:
            req = self.reqs[self.id_req[rid]]
            k = self.seg[rid]
            resp.append(req["segs"][k][2])
            self.seg[rid] = k + 1
            self.tok[rid] = 0
            rows.append(seg_row(req, k + 1, ctx_prompt=0))
        return ids, resp, rows
