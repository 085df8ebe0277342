"""CPU oracle for the LAMPS scheduling pass -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``include/lamps.h`` and ``paper_2410_18248_b200``) never imports it, and it
shares no code with that path.

The arithmetic lives in ``lamps_oracle.c`` (plain C, plain loops, exact
128-bit intermediates; every function cites PAPER.md).  This module is only
ctypes marshalling around it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lamps_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ENOSPC, ENOENT = 0, -1, -2, -3
FREE, READY, PAUSED_P, PAUSED_D, PAUSED_S = 0, 1, 2, 3, 4
P, D, S, NONE = 0, 1, 2, 3
POL_LAMPS, POL_FCFS, POL_SJF, POL_SJF_TOTAL = 0, 1, 2, 3
EV_API_CALL, EV_FINISHED = 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction, so the quantiser is one IEEE multiply)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
             "-fno-fast-math", "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class OCfg(ctypes.Structure):
    _fields_ = [
        ("capacity", ctypes.c_uint32), ("block_tokens", ctypes.c_uint32),
        ("tau", ctypes.c_uint64), ("A1", ctypes.c_uint64), ("A2", ctypes.c_uint64),
        ("S0", ctypes.c_uint64), ("S1", ctypes.c_uint64), ("SH", ctypes.c_uint32),
        ("c_other", ctypes.c_uint64), ("ticks_per_second", ctypes.c_double),
        ("starvation_threshold", ctypes.c_uint32), ("max_batch", ctypes.c_uint32),
        ("kv_capacity_blocks", ctypes.c_uint64), ("score_bits", ctypes.c_uint32),
        ("id_bits", ctypes.c_uint32), ("policy", ctypes.c_uint32), ("score_interval", ctypes.c_uint32),
    ]


class OSummary(ctypes.Structure):
    _fields_ = [
        ("n_eligible", ctypes.c_uint64), ("pinned", ctypes.c_uint64),
        ("budget", ctypes.c_uint64), ("budget_used", ctypes.c_uint64),
        ("n_admitted", ctypes.c_uint32), ("n_preempted", ctypes.c_uint32),
        ("blocked_head", ctypes.c_uint32), ("pad", ctypes.c_uint32),
    ]


REQ_DTYPE = np.dtype([
    ("id", np.uint64), ("state", np.uint32), ("has_api", np.uint32),
    ("starving", np.uint32), ("strategy", np.uint32), ("cnt", np.uint32),
    ("ctx", np.uint32), ("pre_rem", np.uint32), ("api_ticks", np.uint32),
    ("resp_len", np.uint32), ("post_len", np.uint32), ("pending", np.uint32),
    ("age", np.uint32), ("dirty", np.uint32), ("cached_score", np.uint64),
], align=True)
# snapshot fields that may be absent (defaults: a fresh pool, every score to be computed)
REQ_DEFAULTS = {"age": 0, "dirty": 1, "cached_score": 0}

EVENT_DTYPE = np.dtype([("id", np.uint64), ("kind", np.uint32), ("reserved", np.uint32)], align=True)

SEG_DTYPE = np.dtype([
    ("prompt_len", np.uint32), ("pre_len", np.uint32), ("resp_len", np.uint32),
    ("post_len", np.uint32), ("api_seconds", np.float64), ("has_api", np.uint32),
    ("pad", np.uint32),
], align=True)

_lib_handle = None


def lib():
    global _lib_handle
    if _lib_handle is None:
        L = ctypes.CDLL(build())
        u64, u32, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double
        vp = ctypes.c_void_p
        L.o_blk.restype = u64; L.o_blk.argtypes = [u64, u32]
        L.o_quantize.restype = ctypes.c_int
        L.o_quantize.argtypes = [dbl, dbl, ctypes.POINTER(u32)]
        L.o_validate_cfg.restype = ctypes.c_int; L.o_validate_cfg.argtypes = [vp]
        L.o_t_fwd.restype = u64; L.o_t_fwd.argtypes = [vp, u64]
        L.o_t_swap.restype = u64; L.o_t_swap.argtypes = [vp, u64]
        L.o_wastes.restype = None; L.o_wastes.argtypes = [vp, u64, u64, u64, vp]
        L.o_argmin3.restype = u32; L.o_argmin3.argtypes = [vp]
        L.o_score.restype = u64; L.o_score.argtypes = [vp, vp, u32]
        L.o_policy_score.restype = u64; L.o_policy_score.argtypes = [vp, vp]
        L.o_submit.restype = ctypes.c_int
        L.o_submit.argtypes = [vp, vp, ctypes.POINTER(u64), vp, u32, vp]
        L.o_api_return.restype = ctypes.c_int
        L.o_api_return.argtypes = [vp, vp, vp, vp, vp, u32]
        L.o_step.restype = ctypes.c_int
        L.o_step.argtypes = [vp, vp, vp, u32, vp, u32, u64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.o_splitmix_output.restype = u64; L.o_splitmix_output.argtypes = [u64, u64]
        L.o_normal_q20.restype = ctypes.c_int64; L.o_normal_q20.argtypes = [u64, u64, u32]
        L.o_perturb.restype = u32; L.o_perturb.argtypes = [u32, u32, ctypes.c_int64, u64]
        L.o_predict.restype = ctypes.c_int; L.o_predict.argtypes = [vp, u32, u64, u32, u32, vp]
        for n in ("o_sizeof_req", "o_sizeof_cfg", "o_sizeof_seg", "o_sizeof_summary"):
            getattr(L, n).restype = u32
        assert L.o_sizeof_req() == REQ_DTYPE.itemsize
        assert L.o_sizeof_cfg() == ctypes.sizeof(OCfg)
        assert L.o_sizeof_seg() == SEG_DTYPE.itemsize
        assert L.o_sizeof_summary() == ctypes.sizeof(OSummary)
        _lib_handle = L
    return _lib_handle


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def make_cfg(d: dict) -> OCfg:
    """Build the oracle's config struct from a plain dict of integers."""
    c = OCfg()
    for name, _ in OCfg._fields_:
        setattr(c, name, d.get(name, 0) if name in ("policy", "score_interval") else d[name])
    return c


# ---------------------------------------------------------------- scalars
def blk(n: int, B: int) -> int:
    return int(lib().o_blk(n, B))


def quantize(seconds: float, tps: float):
    t = ctypes.c_uint32(0)
    rc = lib().o_quantize(float(seconds), float(tps), ctypes.byref(t))
    return rc, int(t.value)


def validate_cfg(cfg: OCfg) -> int:
    return int(lib().o_validate_cfg(ctypes.byref(cfg)))


def t_fwd(cfg: OCfg, c: int) -> int:
    return int(lib().o_t_fwd(ctypes.byref(cfg), c))


def t_swap(cfg: OCfg, c: int) -> int:
    return int(lib().o_t_swap(ctypes.byref(cfg), c))


def wastes(cfg: OCfg, ctx: int, pre_rem: int, api_ticks: int):
    W = np.zeros(3, np.uint64)
    lib().o_wastes(ctypes.byref(cfg), ctx, pre_rem, api_ticks, _ptr(W))
    return [int(x) for x in W]


def argmin3(W) -> int:
    a = np.asarray(W, dtype=np.uint64)
    return int(lib().o_argmin3(_ptr(a)))


def score(cfg: OCfg, *, ctx, pre_rem, api_ticks=0, resp_len=0, post_len=0, pending=0,
          has_api=1, strategy=P) -> int:
    r = np.zeros(1, REQ_DTYPE)
    r["ctx"], r["pre_rem"], r["api_ticks"] = ctx, pre_rem, api_ticks
    r["resp_len"], r["post_len"], r["pending"], r["has_api"] = resp_len, post_len, pending, has_api
    r["state"] = READY
    return int(lib().o_score(ctypes.byref(cfg), _ptr(r), strategy))


def policy_score(cfg: OCfg, *, pre_rem, post_len=0, api_ticks=0, has_api=1, pending=0) -> int:
    r = np.zeros(1, REQ_DTYPE)
    r["pre_rem"], r["post_len"], r["api_ticks"], r["has_api"] = pre_rem, post_len, api_ticks, has_api
    r["pending"] = pending
    r["state"] = READY
    return int(lib().o_policy_score(ctypes.byref(cfg), _ptr(r)))


def segments(rows) -> np.ndarray:
    """rows: iterable of dicts/tuples (prompt_len, pre_len, resp_len, post_len, api_seconds, has_api)."""
    rows = list(rows)
    a = np.zeros(len(rows), SEG_DTYPE)
    for k, r in enumerate(rows):
        if isinstance(r, dict):
            for f in ("prompt_len", "pre_len", "resp_len", "post_len", "api_seconds", "has_api"):
                a[k][f] = r.get(f, 0)
        else:
            (a[k]["prompt_len"], a[k]["pre_len"], a[k]["resp_len"], a[k]["post_len"],
             a[k]["api_seconds"], a[k]["has_api"]) = r
    return a


# ---------------------------------------------------------------- F4 ingest
TRUTH_DTYPE = np.dtype([("key", np.uint64), ("prompt_len", np.uint32), ("pre_len", np.uint32),
                        ("pre_bin", np.uint32), ("resp_len", np.uint32), ("post_len", np.uint32),
                        ("api_ticks", np.uint32), ("has_api", np.uint32), ("reserved", np.uint32)], align=True)
PRED_DTYPE = np.dtype([("pre_len", np.uint32), ("resp_len", np.uint32), ("post_len", np.uint32),
                       ("api_ticks", np.uint32)])
NO_BIN = 0xFFFFFFFF


def splitmix_output(seed: int, n: int) -> int:
    return int(lib().o_splitmix_output(seed, n))


def normal_q20(seed: int, key: int, field: int) -> int:
    return int(lib().o_normal_q20(seed, key, field))


def perturb(m: int, ppm: int, Z: int, hi: int) -> int:
    return int(lib().o_perturb(m, ppm, Z, hi))


def predict(truth: np.ndarray, seed: int = 0, len_error_ppm: int = 0, api_error_ppm: int = 0):
    """Truths (TRUTH_DTYPE) -> (rc, predictions PRED_DTYPE)."""
    truth = np.ascontiguousarray(truth, TRUTH_DTYPE)
    out = np.zeros(max(len(truth), 1), PRED_DTYPE)
    rc = int(lib().o_predict(_ptr(truth), len(truth), seed, len_error_ppm, api_error_ppm, _ptr(out)))
    return rc, out[:len(truth)]


# ---------------------------------------------------------------- pool
class OraclePool:
    """The oracle's request pool: one record per slot (slot = id mod capacity)."""

    def __init__(self, cfg: dict):
        self.cfg_dict = dict(cfg)
        self.cfg = make_cfg(cfg)
        rc = validate_cfg(self.cfg)
        if rc != OK:
            raise ValueError(f"oracle: invalid config ({rc})")
        self.cap = int(cfg["capacity"])
        self.pool = np.zeros(self.cap, REQ_DTYPE)
        self.next_id = 0
        self.prev_adm = np.zeros(0, np.uint64)

    def load(self, fields: dict, next_id: int, prev_admitted=None):
        """Load a per-slot snapshot (dict of arrays, length capacity, incl. 'id')."""
        for f in REQ_DTYPE.names:
            v = fields[f] if f in fields else REQ_DEFAULTS[f]
            self.pool[f] = np.asarray(v).astype(REQ_DTYPE[f])
        self.next_id = int(next_id)
        self.prev_adm = np.asarray(prev_admitted if prev_admitted is not None else [], np.uint64)

    def submit(self, segs: np.ndarray):
        ids = np.zeros(max(len(segs), 1), np.uint64)
        nid = ctypes.c_uint64(self.next_id)
        rc = lib().o_submit(ctypes.byref(self.cfg), _ptr(self.pool), ctypes.byref(nid),
                            _ptr(segs), len(segs), _ptr(ids))
        if rc == OK:
            self.next_id = int(nid.value)
        return rc, ids[:len(segs)]

    def api_return(self, ids, actual_resp, next_segs: np.ndarray) -> int:
        ids = np.ascontiguousarray(ids, np.uint64)
        ar = np.ascontiguousarray(actual_resp, np.uint32)
        return int(lib().o_api_return(ctypes.byref(self.cfg), _ptr(self.pool), _ptr(ids),
                                      _ptr(ar), _ptr(next_segs), len(ids)))

    def step(self, events=None, kv_total: int = 0, debug: bool = False):
        ev = np.zeros(0, EVENT_DTYPE) if events is None else np.ascontiguousarray(events, EVENT_DTYPE)
        cap, mb = self.cap, int(self.cfg.max_batch)
        summ = OSummary()
        r_id = np.zeros(cap, np.uint64); r_sc = np.zeros(cap, np.uint64); r_st = np.zeros(cap, np.uint8)
        a_id = np.zeros(mb, np.uint64); a_st = np.zeros(mb, np.uint8)
        p_id = np.zeros(max(len(self.prev_adm), 1), np.uint64)
        dbg = np.zeros(4 * cap, np.uint64) if debug else None
        dbs = np.zeros(cap, np.uint8) if debug else None
        prev = np.ascontiguousarray(self.prev_adm, np.uint64)
        rc = lib().o_step(ctypes.byref(self.cfg), _ptr(self.pool), _ptr(prev), len(prev),
                          _ptr(ev), len(ev), int(kv_total), ctypes.byref(summ),
                          _ptr(r_id), _ptr(r_sc), _ptr(r_st), _ptr(a_id), _ptr(a_st), _ptr(p_id),
                          _ptr(dbg), _ptr(dbs))
        if rc != OK:
            return {"rc": rc}
        n_e, n_a, n_p = int(summ.n_eligible), int(summ.n_admitted), int(summ.n_preempted)
        self.prev_adm = a_id[:n_a].copy()
        out = {
            "rc": rc, "n_eligible": n_e, "pinned": int(summ.pinned), "budget": int(summ.budget),
            "budget_used": int(summ.budget_used), "n_admitted": n_a, "n_preempted": n_p,
            "blocked_head": int(summ.blocked_head),
            "ranked_id": r_id[:n_e], "ranked_score": r_sc[:n_e], "ranked_starving": r_st[:n_e],
            "admitted_id": a_id[:n_a], "admitted_strategy": a_st[:n_a], "preempted_id": p_id[:n_p],
        }
        if debug:
            d4 = dbg.reshape(cap, 4)
            out.update({"W_P": d4[:, 0].copy(), "W_D": d4[:, 1].copy(), "W_S": d4[:, 2].copy(),
                        "score": d4[:, 3].copy(), "strategy": dbs})
        return out
