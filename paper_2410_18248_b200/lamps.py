"""ctypes binding of liblamps.so (include/lamps.h).

Argument marshalling only: every step of the scheduling pass runs in the CUDA
kernels behind the C ABI.  PyTorch provides the device workspace (a uint8 CUDA
tensor the handle keeps alive) and the stream.  If the library or a CUDA device
is missing, calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

LAMPS_OK, LAMPS_EINVAL, LAMPS_ENOSPC, LAMPS_ENOENT, LAMPS_ENOTSUP, LAMPS_ECUDA, LAMPS_ENCCL = 0, -1, -2, -3, -4, -5, -6
LAMPS_FREE, LAMPS_READY, LAMPS_PAUSED_P, LAMPS_PAUSED_D, LAMPS_PAUSED_S = 0, 1, 2, 3, 4
LAMPS_PRESERVE, LAMPS_DISCARD, LAMPS_SWAP, LAMPS_NONE = 0, 1, 2, 3
LAMPS_EV_API_CALL, LAMPS_EV_FINISHED = 1, 2
LAMPS_DEBUG_OUT, LAMPS_TIMING, LAMPS_MULTI_KERNEL, LAMPS_FORCE_FALLBACK, LAMPS_TRACE, LAMPS_MERGE = 1, 2, 4, 8, 16, 32
LAMPS_HEAD_ONLY = 64
LAMPS_POLICY_LAMPS, LAMPS_POLICY_FCFS, LAMPS_POLICY_SJF, LAMPS_POLICY_SJF_TOTAL = 0, 1, 2, 3
LAMPS_XPORT_NCCL, LAMPS_XPORT_LOOPBACK, LAMPS_XPORT_P2P = 0, 1, 2
LAMPS_SHARE_DEVICE = 128
LAMPS_GRID_STEP = 256  # small pools: the grid-wide fused kernel instead of the one-CTA kernel
LAMPS_BIG_STEP = 512  # the large-pool path (several ranges per CTA) at any capacity

u32, u64, dbl, vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class lamps_segment(ctypes.Structure):
    _fields_ = [("prompt_len", u32), ("pre_len", u32), ("resp_len", u32), ("post_len", u32),
                ("api_seconds", dbl), ("has_api", u32), ("reserved", u32)]


class lamps_event(ctypes.Structure):
    _fields_ = [("id", u64), ("kind", u32), ("reserved", u32)]


class lamps_config(ctypes.Structure):
    _fields_ = [("capacity", u32), ("block_tokens", u32), ("tau", u64), ("A1", u64), ("A2", u64),
                ("S0", u64), ("S1", u64), ("SH", u32), ("c_other", u64),
                ("ticks_per_second", dbl), ("starvation_threshold", u32), ("max_batch", u32),
                ("kv_capacity_blocks", u64), ("score_bits", u32), ("id_bits", u32),
                ("stream", vp), ("flags", u32), ("world", u32), ("rank", u32), ("transport", u32),
                ("nccl_id", vp), ("policy", u32), ("score_interval", u32), ("local_ranks", u32)]


class lamps_step_out(ctypes.Structure):
    _fields_ = [("n_eligible", u64), ("pinned", u64), ("budget", u64), ("budget_used", u64),
                ("n_admitted", u32), ("n_preempted", u32), ("blocked_head", u32), ("reserved", u32),
                ("id_base", u64), ("admitted_ids", ctypes.POINTER(u64)),
                ("admitted_strategy", ctypes.POINTER(ctypes.c_uint8)),
                ("preempted_ids", ctypes.POINTER(u64)), ("d_ranked_keys", vp),
                ("d_admitted_slots", vp)]


class lamps_pool_io(ctypes.Structure):
    _fields_ = [("id", vp), ("state", vp), ("has_api", vp), ("starving", vp), ("strategy", vp),
                ("cnt", vp), ("ctx", vp), ("pre_rem", vp), ("api_ticks", vp), ("resp_len", vp),
                ("post_len", vp), ("pending", vp), ("dbg_w", vp), ("dbg_score", vp),
                ("age", vp), ("dirty", vp), ("cached_score", vp)]


SEGMENT_DTYPE = np.dtype([("prompt_len", np.uint32), ("pre_len", np.uint32), ("resp_len", np.uint32),
                          ("post_len", np.uint32), ("api_seconds", np.float64), ("has_api", np.uint32),
                          ("reserved", np.uint32)], align=True)
TRUTH_DTYPE = np.dtype([("key", np.uint64), ("prompt_len", np.uint32), ("pre_len", np.uint32),
                        ("pre_bin", np.uint32), ("resp_len", np.uint32), ("post_len", np.uint32),
                        ("api_ticks", np.uint32), ("has_api", np.uint32), ("reserved", np.uint32)], align=True)
LAMPS_NO_BIN = 0xFFFFFFFF


class lamps_iteration(ctypes.Structure):
    _fields_ = [("events", vp), ("n_events", u32), ("n_returns", u32), ("return_ids", vp),
                ("return_resp", vp), ("return_next", vp), ("arrivals", vp), ("n_arrivals", u32),
                ("reserved", u32), ("arrival_ids_out", vp), ("kv_total_blocks", u64)]


_NO_IDS = np.zeros(0, np.uint64)
_NO_IDS.flags.writeable = False


class lamps_noise(ctypes.Structure):
    _fields_ = [("seed", u64), ("len_error_ppm", u32), ("api_error_ppm", u32)]


EVENT_DTYPE = np.dtype([("id", np.uint64), ("kind", np.uint32), ("reserved", np.uint32)], align=True)
POOL_U32_FIELDS = ("state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem", "api_ticks",
                   "resp_len", "post_len", "pending")

_L = None


def lib() -> ctypes.CDLL:
    """Load liblamps.so (building it first if it is missing or stale)."""
    global _L
    if _L is None:
        path = os.environ.get("LAMPS_LIB") or _build.LIB  # LAMPS_LIB: another build (A/B runs)
        if path == _build.LIB and (not os.path.exists(path) or _build.stale()):
            _build.build()
        L = ctypes.CDLL(path)
        c_int, P = ctypes.c_int, ctypes.POINTER
        sig = {
            "lamps_init": (c_int, [P(lamps_config), vp, P(ctypes.c_size_t), P(vp)]),
            "lamps_submit": (c_int, [vp, vp, u32, vp]),
            "lamps_api_return": (c_int, [vp, vp, vp, vp, u32]),
            "lamps_schedule_step": (c_int, [vp, vp, u32, u64, P(lamps_step_out)]),
            "lamps_free": (c_int, [vp]),
            "lamps_last_error": (ctypes.c_char_p, [vp]),
            "lamps_schedule_step_async": (c_int, [vp, u64]),
            "lamps_step_result": (c_int, [vp, P(lamps_step_out)]),
            "lamps_pool_import": (c_int, [vp, P(lamps_pool_io), u64, u64]),
            "lamps_pool_export": (c_int, [vp, P(lamps_pool_io)]),
            "lamps_ranked_keys": (c_int, [vp, vp, u64, P(u64)]),
            "lamps_step_stats": (c_int, [vp, P(u32), P(u32)]),
            "lamps_timing_read": (c_int, [vp, P(dbl), P(u32)]),
            "lamps_trace_read": (c_int, [vp, vp, u32, P(u32)]),
            "lamps_nccl_unique_id": (c_int, [vp]),
            "lamps_group_step": (c_int, [vp, u32, vp, vp, vp, vp]),
            "lamps_group_step_async": (c_int, [vp, u32, vp]),
            "lamps_version": (u32, []),
            "lamps_predict": (c_int, [vp, vp, u32, P(lamps_noise), vp]),
            "lamps_p2p_handle": (c_int, [vp, vp]),
            "lamps_iterate": (c_int, [vp, P(lamps_iteration), P(lamps_step_out)]),
            "lamps_p2p_connect": (c_int, [vp, vp, ctypes.c_size_t]),
            "lamps_p2p_connect_local": (c_int, [vp, u32]),
        }
        for name, (res, args) in sig.items():
            if path != _build.LIB and not hasattr(L, name):
                continue  # an older build loaded for an A/B run
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _L = L
    return _L


class LampsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"lamps error {code}: {msg}")
        self.code = code


def _p(a):
    # the raw address (the caller keeps the array alive across the call)
    return None if a is None else a.ctypes.data


# ---- thin wrappers with the C names (return codes, no exceptions) ----------
def lamps_init(cfg: lamps_config, d_workspace, ws_bytes: int):
    h = vp()
    n = ctypes.c_size_t(ws_bytes)
    rc = lib().lamps_init(ctypes.byref(cfg), d_workspace, ctypes.byref(n), ctypes.byref(h))
    return rc, h, n.value


def lamps_workspace_bytes(cfg: lamps_config) -> int:
    n = ctypes.c_size_t(0)
    rc = lib().lamps_init(ctypes.byref(cfg), None, ctypes.byref(n), None)
    if rc != LAMPS_OK:
        raise LampsError(rc, "invalid config")
    return n.value


def lamps_submit(h, segs: np.ndarray, ids_out: np.ndarray) -> int:
    return lib().lamps_submit(h, _p(segs), len(segs), _p(ids_out))


def lamps_api_return(h, ids: np.ndarray, actual: np.ndarray, nxt: np.ndarray) -> int:
    return lib().lamps_api_return(h, _p(ids), _p(actual), _p(nxt), len(ids))


def lamps_schedule_step(h, ev: np.ndarray, kv_total: int, out: lamps_step_out) -> int:
    return lib().lamps_schedule_step(h, _p(ev) if len(ev) else None, len(ev), kv_total, ctypes.byref(out))


def lamps_free(h) -> int:
    return lib().lamps_free(h)


def lamps_last_error(h) -> str:
    return lib().lamps_last_error(h).decode()


# ---- Scheduler: the user-facing object --------------------------------------
class Scheduler:
    """One LAMPS scheduling pass handle on the current CUDA device.

    cfg: dict with the lamps_config integer fields (see gen.lib_config for an
    example).  flags: LAMPS_DEBUG_OUT | LAMPS_TIMING.
    """

    def __init__(self, cfg: dict, flags: int = 0, stream=None, device=None, world: int = 1, rank: int = 0,
                 transport: int = LAMPS_XPORT_NCCL, nccl_id: bytes = None, local_ranks: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise LampsError(LAMPS_ECUDA, "no CUDA device: the LAMPS pass has no CPU fallback")
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        c = lamps_config()
        for name, _ in lamps_config._fields_:
            if name in cfg:
                setattr(c, name, cfg[name])
        c.flags = flags
        c.stream = ctypes.c_void_p(self.stream.cuda_stream)
        c.world, c.rank, c.transport, c.local_ranks = world, rank, transport, local_ranks
        self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        c.nccl_id = ctypes.cast(self._nccl_id, vp) if self._nccl_id is not None else None
        self.world, self.rank = world, rank
        self.cfg = c
        self.capacity = int(cfg["capacity"])
        self.max_batch = int(cfg["max_batch"])
        self.id_bits, self.score_bits = int(cfg["id_bits"]), int(cfg["score_bits"])
        n = lamps_workspace_bytes(c)
        self.workspace = torch.empty(n, dtype=torch.uint8, device=self.device)
        rc, h, _ = lamps_init(c, ctypes.c_void_p(self.workspace.data_ptr()), n)
        if rc != LAMPS_OK:
            raise LampsError(rc, "lamps_init failed")
        self.h = h
        self._out = lamps_step_out()
        self._it = lamps_iteration()

    def _check(self, rc):
        if rc != LAMPS_OK:
            raise LampsError(rc, lamps_last_error(self.h))

    def close(self):
        if getattr(self, "h", None):
            lamps_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- ingest
    @staticmethod
    def segments(rows) -> np.ndarray:
        rows = list(rows)
        a = np.zeros(len(rows), SEGMENT_DTYPE)
        for k, r in enumerate(rows):
            for f in ("prompt_len", "pre_len", "resp_len", "post_len", "api_seconds", "has_api"):
                a[k][f] = r.get(f, 0)
        return a

    def submit(self, segs: np.ndarray) -> np.ndarray:
        segs = np.ascontiguousarray(segs, SEGMENT_DTYPE)
        ids = np.zeros(max(len(segs), 1), np.uint64)
        self._check(lamps_submit(self.h, segs, ids))
        return ids[:len(segs)]

    def submit_rc(self, segs: np.ndarray):
        segs = np.ascontiguousarray(segs, SEGMENT_DTYPE)
        ids = np.zeros(max(len(segs), 1), np.uint64)
        return lamps_submit(self.h, segs, ids), ids[:len(segs)]

    def predict_rc(self, truth: np.ndarray, seed: int = 0, len_error_ppm: int = 0, api_error_ppm: int = 0,
                   noise: bool = True):
        """lamps_predict: truths (TRUTH_DTYPE) -> predicted segments (SEGMENT_DTYPE), row F4."""
        truth = np.ascontiguousarray(truth, TRUTH_DTYPE)
        out = np.zeros(max(len(truth), 1), SEGMENT_DTYPE)
        nz = lamps_noise(seed, len_error_ppm, api_error_ppm)
        rc = lib().lamps_predict(self.h, _p(truth), len(truth), ctypes.byref(nz) if noise else None, _p(out))
        return rc, out[:len(truth)]

    def predict(self, truth: np.ndarray, seed: int = 0, len_error_ppm: int = 0, api_error_ppm: int = 0):
        rc, out = self.predict_rc(truth, seed, len_error_ppm, api_error_ppm)
        self._check(rc)
        return out

    def api_return_rc(self, ids, actual, nxt) -> int:
        return lamps_api_return(self.h, np.ascontiguousarray(ids, np.uint64),
                                np.ascontiguousarray(actual, np.uint32),
                                np.ascontiguousarray(nxt, SEGMENT_DTYPE))

    def api_return(self, ids, actual, nxt):
        self._check(self.api_return_rc(ids, actual, nxt))

    # ---- step
    def _views(self, out: lamps_step_out):
        """numpy views of the handle's result lists (fixed host buffers), made once."""
        key = (ctypes.addressof(out.admitted_ids.contents) if out.admitted_ids else 0,
               ctypes.addressof(out.preempted_ids.contents) if out.preempted_ids else 0)
        if getattr(self, "_vkey", None) != key:
            mb = int(self.cfg.max_batch)
            self._vkey = key
            self._vadm = np.ctypeslib.as_array(out.admitted_ids, (mb,)) if key[0] else None
            self._vstr = np.ctypeslib.as_array(out.admitted_strategy, (mb,)) if key[0] else None
            self._vpre = np.ctypeslib.as_array(out.preempted_ids, (mb,)) if key[1] else None
        return self._vadm, self._vstr, self._vpre

    def _result(self, out: lamps_step_out) -> dict:
        na, npr = out.n_admitted, out.n_preempted
        va, vs, vp_ = self._views(out)
        return {
            "rc": 0, "n_eligible": int(out.n_eligible), "pinned": int(out.pinned),
            "budget": int(out.budget), "budget_used": int(out.budget_used), "n_admitted": int(na),
            "n_preempted": int(npr), "blocked_head": int(out.blocked_head), "id_base": int(out.id_base),
            "admitted_id": va[:na].copy() if na else np.zeros(0, np.uint64),
            "admitted_strategy": vs[:na].copy() if na else np.zeros(0, np.uint8),
            "preempted_id": vp_[:npr].copy() if npr else np.zeros(0, np.uint64),
        }

    def step_rc(self, events=None, kv_total: int = 0):
        ev = np.zeros(0, EVENT_DTYPE) if events is None else np.ascontiguousarray(events, EVENT_DTYPE)
        rc = lamps_schedule_step(self.h, ev, int(kv_total), self._out)
        return rc

    def step(self, events=None, kv_total: int = 0) -> dict:
        self._check(self.step_rc(events, kv_total))
        return self._result(self._out)

    def iterate_rc(self, events=None, ret_ids=None, ret_resp=None, ret_next=None, arrivals=None,
                   kv_total: int = 0):
        """lamps_iterate: API returns, one step with the events, arrivals -- one sync.
        Returns (rc, result dict or None, arrival ids)."""
        it = self._it  # one struct per handle, every field set on each call
        keep = []
        if events is not None and len(events):
            ev = np.ascontiguousarray(events, EVENT_DTYPE); keep.append(ev)
            it.events, it.n_events = _p(ev), len(ev)
        else:
            it.events, it.n_events = None, 0
        if ret_ids is not None and len(ret_ids):
            ri = np.ascontiguousarray(ret_ids, np.uint64)
            rr = np.ascontiguousarray(ret_resp, np.uint32)
            rn = np.ascontiguousarray(ret_next, SEGMENT_DTYPE)
            keep += [ri, rr, rn]
            it.return_ids, it.return_resp, it.return_next, it.n_returns = _p(ri), _p(rr), _p(rn), len(ri)
        else:
            it.return_ids = it.return_resp = it.return_next = None
            it.n_returns = 0
        ids = _NO_IDS
        if arrivals is not None and len(arrivals):
            ar = np.ascontiguousarray(arrivals, SEGMENT_DTYPE)
            ids = np.zeros(len(ar), np.uint64)
            keep += [ar, ids]
            it.arrivals, it.n_arrivals, it.arrival_ids_out = _p(ar), len(ar), _p(ids)
        else:
            it.arrivals, it.n_arrivals, it.arrival_ids_out = None, 0, None
        it.kv_total_blocks = int(kv_total)
        rc = lib().lamps_iterate(self.h, ctypes.byref(it), ctypes.byref(self._out))
        return rc, (self._result(self._out) if rc == LAMPS_OK else None), ids

    def iterate(self, events=None, ret_ids=None, ret_resp=None, ret_next=None, arrivals=None, kv_total: int = 0):
        rc, out, ids = self.iterate_rc(events, ret_ids, ret_resp, ret_next, arrivals, kv_total)
        self._check(rc)
        return out, ids

    def step_async(self, kv_total: int):
        self._check(lib().lamps_schedule_step_async(self.h, int(kv_total)))

    def result(self) -> dict:
        self._check(lib().lamps_step_result(self.h, ctypes.byref(self._out)))
        return self._result(self._out)

    def ranked_keys(self) -> np.ndarray:
        n = u64(0)
        self._check(lib().lamps_ranked_keys(self.h, None, 0, ctypes.byref(n)))
        a = np.zeros(max(int(n.value), 1), np.uint64)
        self._check(lib().lamps_ranked_keys(self.h, _p(a), int(n.value), ctypes.byref(n)))
        return a[:int(n.value)]

    def decode_keys(self, keys: np.ndarray, id_base: int):
        IB, SB = self.id_bits, self.score_bits
        keys = keys.astype(np.uint64)
        idoff = keys & np.uint64((1 << IB) - 1)
        score = (keys >> np.uint64(IB)) & np.uint64((1 << SB) - 1)
        starving = 1 - ((keys >> np.uint64(IB + SB)) & np.uint64(1))
        return idoff + np.uint64(id_base), score, starving.astype(np.uint8)

    def stats(self):
        k, p = u32(0), u32(0)
        self._check(lib().lamps_step_stats(self.h, ctypes.byref(k), ctypes.byref(p)))
        return int(k.value), int(p.value)

    def trace(self):
        """Per-CTA SM clocks at the fused kernel's phase boundaries (LAMPS_TRACE)."""
        out = np.zeros(512 * 64, np.uint64)
        n = u32(0)
        self._check(lib().lamps_trace_read(self.h, _p(out), len(out), ctypes.byref(n)))
        return out[:n.value * 64].reshape(n.value, 64)

    def timing(self):
        ms = (dbl * 4)()
        n = u32(0)
        self._check(lib().lamps_timing_read(self.h, ms, ctypes.byref(n)))
        return list(ms), int(n.value)

    # ---- multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        rc = lib().lamps_nccl_unique_id(buf)
        if rc != LAMPS_OK:
            raise LampsError(rc, "ncclGetUniqueId failed (libnccl.so.2)")
        return buf.raw

    @staticmethod
    def group_step(shards, events=None, kv_totals=None) -> list:
        """One step of loopback shards (same device and stream), see lamps_group_step."""
        W = len(shards)
        evs = [np.zeros(0, EVENT_DTYPE) if events is None or events[r] is None
               else np.ascontiguousarray(events[r], EVENT_DTYPE) for r in range(W)]
        ev_ptrs = (vp * W)(*[e.ctypes.data if len(e) else None for e in evs])
        n_ev = (u32 * W)(*[len(e) for e in evs])
        kv = (u64 * W)(*[int(x) for x in kv_totals])
        outs = (lamps_step_out * W)()
        hs = (vp * W)(*[s.h for s in shards])
        rc = lib().lamps_group_step(hs, W, ev_ptrs, n_ev, kv, outs)
        if rc != LAMPS_OK:
            raise LampsError(rc, lamps_last_error(shards[0].h))
        return [shards[r]._result(outs[r]) for r in range(W)]

    # ---- peer-memory transport (LAMPS_XPORT_P2P)
    @staticmethod
    def group_step_async(shards, kv_totals):
        """Enqueue one step on every co-resident P2P shard of this process (each on its own
        stream; the other ranks of the world step in lockstep elsewhere), lamps_group_step_async.
        Results: shard.result()."""
        W = len(shards)
        kv = (u64 * W)(*[int(x) for x in kv_totals])
        hs = (vp * W)(*[s.h for s in shards])
        rc = lib().lamps_group_step_async(hs, W, kv)
        if rc != LAMPS_OK:
            raise LampsError(rc, lamps_last_error(shards[0].h))

    def p2p_handle(self) -> bytes:
        """This rank's 64-byte CUDA IPC handle of its exchange buffer."""
        buf = ctypes.create_string_buffer(64)
        self._check(lib().lamps_p2p_handle(self.h, buf))
        return buf.raw

    def p2p_connect(self, handles: list):
        """Map every rank's exchange buffer (handles in rank order, from p2p_handle)."""
        blob = b"".join(handles)
        self._check(lib().lamps_p2p_connect(self.h, blob, len(blob)))

    @staticmethod
    def p2p_connect_local(shards):
        """Connect P2P ranks that live in this process on one device (LAMPS_SHARE_DEVICE)."""
        hs = (vp * len(shards))(*[s.h for s in shards])
        rc = lib().lamps_p2p_connect_local(hs, len(shards))
        if rc != LAMPS_OK:
            raise LampsError(rc, lamps_last_error(shards[0].h))

    # ---- snapshots
    def import_pool(self, fields: dict, id_base: int, next_id: int):
        cap = self.capacity
        keep = {"id": np.ascontiguousarray(np.asarray(fields["id"])[:cap], np.uint64)}
        for f in POOL_U32_FIELDS:
            keep[f] = np.ascontiguousarray(np.asarray(fields[f])[:cap], np.uint32)
        for f in ("age", "dirty"):  # selective-update state (optional: a fresh pool)
            if f in fields:
                keep[f] = np.ascontiguousarray(np.asarray(fields[f])[:cap], np.uint32)
        if "cached_score" in fields:
            keep["cached_score"] = np.ascontiguousarray(np.asarray(fields["cached_score"])[:cap], np.uint64)
        io = lamps_pool_io(**{k: _p(v) for k, v in keep.items()})
        self._check(lib().lamps_pool_import(self.h, ctypes.byref(io), int(id_base), int(next_id)))

    def export_pool(self, debug: bool = False) -> dict:
        cap = self.capacity
        out = {"id": np.zeros(cap, np.uint64)}
        for f in POOL_U32_FIELDS + ("age", "dirty"):
            out[f] = np.zeros(cap, np.uint32)
        out["cached_score"] = np.zeros(cap, np.uint64)
        io = lamps_pool_io(**{k: _p(v) for k, v in out.items()})
        if debug:
            out["dbg_w"] = np.zeros(3 * cap, np.uint64)
            out["dbg_score"] = np.zeros(cap, np.uint64)
            io.dbg_w, io.dbg_score = _p(out["dbg_w"]), _p(out["dbg_score"])
        self._check(lib().lamps_pool_export(self.h, ctypes.byref(io)))
        if debug:
            w = out.pop("dbg_w").reshape(cap, 3)
            out["W_P"], out["W_D"], out["W_S"] = w[:, 0].copy(), w[:, 1].copy(), w[:, 2].copy()
            out["score"] = out.pop("dbg_score")
        return out
