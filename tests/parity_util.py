"""Helpers for GPU <-> oracle parity tests (bit-exact comparison)."""
import numpy as np

import gen
import oracle as O

FIELDS = ("state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem", "api_ticks",
          "resp_len", "post_len", "pending", "age", "dirty")


# fused step kernel (one-CTA k_small for capacity <= 4096); LAMPS_MULTI_KERNEL; LAMPS_FORCE_FALLBACK;
# LAMPS_HEAD_ONLY (F3 top-K fast path); LAMPS_GRID_STEP (small pools on the grid-wide fused kernel);
# LAMPS_BIG_STEP (the large-pool path -- several ranges per CTA -- at any capacity)
PATH_FLAGS = {"fused": 0, "multi": 4, "fallback": 8, "head": 64, "grid": 256, "grid_fallback": 256 | 8,
              "big": 512, "big_fallback": 512 | 8}


def make_pair(cfg: dict, debug=True, path="fused"):
    from paper_2410_18248_b200 import Scheduler, LAMPS_DEBUG_OUT
    s = Scheduler(cfg, flags=(LAMPS_DEBUG_OUT if debug else 0) | PATH_FLAGS[path])
    o = O.OraclePool(cfg)
    return s, o


def load_both(s, o, snap):
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    o.load(snap, snap["next_id"])


def seg_rows_to_arrays(rows):
    from paper_2410_18248_b200.lamps import SEGMENT_DTYPE
    a = np.zeros(len(rows), SEGMENT_DTYPE)
    b = np.zeros(len(rows), O.SEG_DTYPE)
    for k, r in enumerate(rows):
        for f in ("prompt_len", "pre_len", "resp_len", "post_len", "api_seconds", "has_api"):
            a[k][f] = r.get(f, 0)
            b[k][f] = r.get(f, 0)
    return a, b


def compare_outputs(s, g, r, where=""):
    assert r["rc"] == 0, where
    for k in ("n_eligible", "pinned", "budget", "budget_used", "n_admitted", "n_preempted", "blocked_head"):
        assert g[k] == r[k], (where, k, g[k], r[k])
    assert np.array_equal(g["admitted_id"], r["admitted_id"]), where
    assert np.array_equal(g["admitted_strategy"], r["admitted_strategy"]), where
    assert np.array_equal(g["preempted_id"], r["preempted_id"]), where
    keys = s.ranked_keys()
    m = len(keys)
    if s.cfg.flags & 64:  # LAMPS_HEAD_ONLY (F3): a prefix, at least as long as the admission can reach
        assert min(r["n_eligible"], s.cfg.max_batch) <= m <= r["n_eligible"], (where, m)
    else:
        assert m == r["n_eligible"], where
    ids, score, starving = s.decode_keys(keys, g["id_base"])
    assert np.array_equal(ids, r["ranked_id"][:m]), (where, "ranked ids")
    assert np.array_equal(score, r["ranked_score"][:m]), (where, "ranked scores")
    assert np.array_equal(starving, r["ranked_starving"][:m]), (where, "ranked starving")


def compare_state(s, o, r=None, where=""):
    e = s.export_pool(debug=r is not None and "W_P" in r)
    P = o.pool
    live = P["state"] != O.FREE
    assert np.array_equal(e["state"], P["state"].astype(np.uint32)), where
    for f in FIELDS:
        a, b = e[f][live], P[f][live].astype(np.uint32)
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0][:5]
            raise AssertionError(f"{where}: field {f} differs at live slots {np.nonzero(live)[0][bad]}: "
                                 f"gpu {a[bad]} oracle {b[bad]}")
    assert np.array_equal(e["id"][live], P["id"][live]), where
    if o.cfg.policy == O.POL_LAMPS and o.cfg.score_interval > 1:  # the score cache (R26)
        assert np.array_equal(e["cached_score"][live], P["cached_score"][live]), (where, "cached_score")
    if r is not None and "W_P" in r:
        ready = P["state"] == O.READY
        for f in ("W_P", "W_D", "W_S", "score"):
            a, b = e[f][ready], r[f][ready]
            if not np.array_equal(a, b):
                bad = np.nonzero(a != b)[0][:5]
                raise AssertionError(f"{where}: debug {f} differs: gpu {a[bad]} oracle {b[bad]}")
        assert np.array_equal(e["strategy"][ready], r["strategy"][ready].astype(np.uint32)), where


def snapshot_step_parity(cname, seed=0, id_base=0, steps=3, debug=True, path="fused", **over):
    cfg = gen.lib_config(cname, **{k: v for k, v in over.items()
                                   if k in ("max_batch", "starvation_threshold", "score_bits", "id_bits", "policy",
                                            "score_interval")})
    snap = gen.snapshot(cname, seed=seed, id_base=id_base,
                        **{k: v for k, v in over.items() if k in ("n", "capacity")})
    if "capacity" in over:
        cfg["capacity"] = over["capacity"]
    s, o = make_pair(cfg, debug=debug, path=path)
    load_both(s, o, snap)
    kv = over.get("kv_total", gen.CONFIGS[cname]["kv_total"])
    outs = []
    for t in range(steps):
        g = s.step(kv_total=kv)
        r = o.step(kv_total=kv, debug=debug)
        compare_outputs(s, g, r, where=f"{cname} seed {seed} step {t}")
        compare_state(s, o, r if debug else None, where=f"{cname} seed {seed} step {t}")
        outs.append(g)
    s.close()
    return outs
