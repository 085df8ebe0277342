"""GPU <-> oracle parity: bit-exact strategy, wastes, score, ranked order,
admitted set, counters, preempted list and the whole pool state, through the
C ABI (liblamps.so), on seeded synthetic pools of the paper's workloads and on
closed-loop traces.  Needs a B200."""
import math
import random

import numpy as np
import pytest

import gen
import oracle as O
from parity_util import (compare_outputs, compare_state, load_both, make_pair, seg_rows_to_arrays,
                         snapshot_step_parity)

pytestmark = pytest.mark.gpu


PATHS = ["fused", "multi", "fallback", "head", "grid", "grid_fallback", "big", "big_fallback"]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cname,seed,id_base", [
    ("C1", 0, 0), ("C1", 1, 5), ("C2", 0, 0), ("C2", 1, 12345), ("C3", 0, 0), ("C3", 2, 777),
    ("C4", 0, 0), ("C4", 1, 3 * 131072 + 17),
])
def test_snapshot_parity(cname, seed, id_base, path):
    snapshot_step_parity(cname, seed=seed, id_base=id_base, steps=3, path=path)


@pytest.mark.slow
@pytest.mark.parametrize("path", ["fused", "multi", "head", "fallback"])
def test_c5_full_size_parity(path):
    # BASELINE.json's 1M-request pool in the launch configuration bench.py times
    snapshot_step_parity("C5", seed=0, id_base=(1 << 20) * 7 + 99, steps=2, path=path)


@pytest.mark.slow
def test_pool_above_fused_capacity_parity():
    # 2^21 slots: above the fused kernel's 148 x 10240, the large-pool path (k_big_score +
    # k_big_sort, two ranges per CTA); the first step is the cold 3-kernel one
    snapshot_step_parity("C5", seed=1, n=1 << 21, capacity=1 << 21, id_base=(1 << 21) * 3 + 5, steps=3, id_bits=21,
                         path="fused")


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n", [1, 2, 5, 1023, 1024, 1025, 8191, 8192, 8193, 12287, 12288, 12289, 30000])
def test_tile_boundaries(n, path):
    # ragged tails around the 8192-key sort tile, the 12288-key shared-memory range and
    # the 1024-thread score rounds
    snapshot_step_parity("C2", seed=n, n=n, capacity=32768, steps=2, path=path)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cap", [1, 2, 4, 8])
def test_tiny_capacity(cap, path):
    snapshot_step_parity("C1", seed=cap, n=cap, capacity=cap, steps=3, path=path)


@pytest.mark.parametrize("path", ["fused", "multi", "head"])
def test_equal_scores_large_bucket(path):
    # 40000 identical requests: one bucket far larger than a shared-memory range,
    # so the fused kernel must take its in-kernel global LSD fallback; order = ids
    n = 40000
    snap = gen.snapshot("C4", seed=9, n=n, capacity=65536, id_base=65536 * 3 + 5)
    for f, v in (("state", 1), ("has_api", 1), ("ctx", 700), ("pre_rem", 40), ("api_ticks", 500000),
                 ("resp_len", 96), ("post_len", 30), ("pending", 0), ("starving", 0), ("cnt", 3)):
        live = snap["state"] != 0
        snap[f][live] = v
    cfg = gen.lib_config("C4")
    cfg["capacity"] = 65536
    from parity_util import compare_outputs, compare_state, load_both, make_pair
    s, o = make_pair(cfg, debug=False, path=path)
    load_both(s, o, snap)
    for t in range(2):
        g, r = s.step(kv_total=10000), o.step(kv_total=10000)
        compare_outputs(s, g, r, where=f"equal t={t}")
    compare_state(s, o)


@pytest.mark.parametrize("path", PATHS)
def test_many_equal_scores_in_one_range(path):
    # 3000 identical requests among 6000: one sub-bucket far above the rank-by-comparison
    # limit inside a shared-memory range, so the fused kernel's local LSD fallback runs
    snap = gen.snapshot("C2", seed=4, n=6000, capacity=8192, id_base=8192 * 2 + 1)
    idx = np.nonzero(snap["state"] != 0)[0][::2]
    for f, v in (("state", 1), ("has_api", 1), ("ctx", 400), ("pre_rem", 25), ("api_ticks", 700000),
                 ("resp_len", 64), ("post_len", 60), ("pending", 0), ("starving", 0), ("cnt", 1)):
        snap[f][idx] = v
    cfg = gen.lib_config("C2")
    cfg["capacity"] = 8192
    s, o = make_pair(cfg, debug=True, path=path)
    load_both(s, o, snap)
    for t in range(2):
        g, r = s.step(kv_total=3000), o.step(kv_total=3000, debug=True)
        compare_outputs(s, g, r, where=f"equal-range t={t}")
        compare_state(s, o, r, where=f"equal-range t={t}")


def _custom(cfg_over, recs, kv, steps=2, id_base=0, path="fused"):
    cfg = gen.lib_config("C1")
    cfg.update(cfg_over)
    cap = cfg["capacity"]
    snap = {f: np.zeros(cap, np.int64) for f in O.REQ_DTYPE.names}
    snap["strategy"][:] = O.NONE
    for i, r in enumerate(recs):
        sl = (id_base + i) % cap
        snap["id"][sl] = id_base + i
        for k, v in r.items():
            snap[k][sl] = v
        snap["state"][sl] = r.get("state", O.READY)
    snap["id_base"], snap["next_id"] = id_base, id_base + len(recs)
    s, o = make_pair(cfg, path=path)
    load_both(s, o, snap)
    for t in range(steps):
        g, r = s.step(kv_total=kv), o.step(kv_total=kv, debug=True)
        compare_outputs(s, g, r, where=f"step {t}")
        compare_state(s, o, r, where=f"step {t}")
    return g


@pytest.mark.parametrize("path", PATHS)
def test_empty_pool_and_zero_budget(path):
    g = _custom(dict(capacity=16), [], kv=10, path=path)
    assert g["n_eligible"] == 0 and g["blocked_head"] == 0
    recs = [dict(ctx=10, pre_rem=5) for _ in range(5)]
    g = _custom(dict(capacity=16), recs, kv=0, path=path)
    assert g["n_admitted"] == 0 and g["blocked_head"] == 1


@pytest.mark.parametrize("path", PATHS)
def test_all_equal_scores_break_ties_by_id(path):
    recs = [dict(ctx=100, pre_rem=50, has_api=1, api_ticks=10 ** 6, resp_len=8, post_len=9) for _ in range(16)]
    g = _custom(dict(capacity=16, max_batch=7), recs, kv=10 ** 6, id_base=(1 << 30) + 3, path=path)
    assert list(g["admitted_id"]) == list(range((1 << 30) + 3, (1 << 30) + 10))


@pytest.mark.parametrize("path", PATHS)
def test_all_starving_and_threshold_boundary(path):
    recs = [dict(ctx=50 + i, pre_rem=10 * i, starving=1) for i in range(8)]
    recs += [dict(ctx=5, pre_rem=1, cnt=99), dict(ctx=5, pre_rem=1, cnt=100)]
    _custom(dict(capacity=16, max_batch=3, starvation_threshold=100), recs, kv=10 ** 4, steps=4, path=path)


@pytest.mark.parametrize("path", PATHS)
def test_max_batch_one_and_misprediction(path):
    recs = [dict(ctx=10 * i, pre_rem=0, has_api=1, api_ticks=5, resp_len=3, post_len=2) for i in range(6)]
    _custom(dict(capacity=8, max_batch=1), recs, kv=10 ** 4, steps=6, path=path)


@pytest.mark.parametrize("path", PATHS)
def test_score_saturation_and_narrow_id_window(path):
    recs = [dict(ctx=1000 + i, pre_rem=400, has_api=1, api_ticks=10 ** 9, resp_len=8, post_len=100)
            for i in range(16)]
    _custom(dict(capacity=16, score_bits=12, id_bits=4), recs, kv=10 ** 4, id_base=2 ** 40 + 11, path=path)


@pytest.mark.parametrize("path", PATHS)
def test_extreme_cost_constants_saturate_like_the_oracle(path):
    big = (1 << 48) - 1
    recs = [dict(ctx=(1 << 24) - 5 * i, pre_rem=3000 * i, has_api=1, api_ticks=(1 << 32) - 1 - i,
                 resp_len=7 * i, post_len=1000, pending=(1 << 32) - 1) for i in range(8)]
    _custom(dict(capacity=8, A1=big, A2=big, S0=big, S1=big, tau=big, c_other=(1 << 32) - 1, SH=3,
                 score_bits=50, id_bits=13, kv_capacity_blocks=1 << 62), recs, kv=1 << 40, path=path)


def test_quantiser_parity_through_submit():
    cfg = gen.lib_config("C2")
    cfg["capacity"] = 1 << 16
    s, o = make_pair(cfg, debug=False)
    rng = random.Random(5)
    rows = []
    for k in range(60000):
        x = rng.choice([rng.uniform(0, 100), (rng.randrange(10 ** 7) + 0.5) / 1e6, 9e-5, 28.6, 0.69, 1.72])
        if k % 3 == 0:
            x = math.nextafter(x, 0 if k % 2 else 1e9)
        rows.append(dict(prompt_len=10, pre_len=5, resp_len=1, post_len=1, api_seconds=x, has_api=1))
    a, b = seg_rows_to_arrays(rows)
    ids = s.submit(a)
    rc, ido = o.submit(b)
    assert rc == 0 and np.array_equal(ids, ido)
    e = s.export_pool()
    live = o.pool["state"] != 0
    assert np.array_equal(e["api_ticks"][live], o.pool["api_ticks"][live])
    assert np.array_equal(e["pending"][live], o.pool["pending"][live])


def test_ingest_errors_match_oracle():
    cfg = gen.lib_config("C1")
    cfg.update(capacity=4, kv_capacity_blocks=100)
    s, o = make_pair(cfg, debug=False)
    ok = [dict(prompt_len=10, pre_len=5, has_api=1, api_seconds=0.5, resp_len=3, post_len=4)] * 3
    cases = [ok, ok[:2], [dict(prompt_len=1600, pre_len=5)], [dict(prompt_len=1, api_seconds=float("nan"), has_api=1)],
             [dict(prompt_len=1, api_seconds=-1.0, has_api=1)], [dict(prompt_len=1 << 24, pre_len=1)],
             [dict(prompt_len=1, has_api=2)], [dict(prompt_len=1, api_seconds=5000.0, has_api=1)]]
    for rows in cases:
        a, b = seg_rows_to_arrays(rows)
        rg, _ = s.submit_rc(a)
        ro, _ = o.submit(b)
        assert rg == ro, rows
    compare_state(s, o)
    a, b = seg_rows_to_arrays([dict(pre_len=1)])
    assert s.api_return_rc([0], [1], a) == o.api_return([0], [1], b) == O.ENOENT
    assert s.api_return_rc([99], [1], a) == o.api_return([99], [1], b) == O.ENOENT
    # events for requests not admitted / kv_total above capacity
    ev = np.zeros(1, O.EVENT_DTYPE); ev[0]["id"], ev[0]["kind"] = 1, 2
    assert s.step_rc(ev, 10) == O.EINVAL and o.step(ev, 10)["rc"] == O.EINVAL
    assert s.step_rc(None, 101) == O.EINVAL and o.step(None, 101)["rc"] == O.EINVAL


def closed_loop(cname, n_req, steps, initial, per_step, kv=None, seed=0, state_every=10, path="fused", **over):
    cfg = gen.lib_config(cname, **over)
    kv = gen.CONFIGS[cname]["kv_total"] if kv is None else kv
    s, o = make_pair(cfg, debug=False, path=path)
    reqs = gen.requests(cname, n_req, seed=seed)
    drv = gen.ClosedLoop(reqs, gen.PROFILES[gen.CONFIGS[cname]["profile"]]["tau"], initial, per_step, seed)
    prev = []
    stats = dict(api=0, fin=0, adm=0, pre=0, starving=0)
    for t in range(steps):
        idx, rows = drv.arrivals(t)
        if rows:
            a, b = seg_rows_to_arrays(rows)
            ids = s.submit(a)
            rc, ido = o.submit(b)
            assert rc == 0 and np.array_equal(ids, ido)
            drv.on_submitted(idx, ids)
        ids, resp, rows = drv.api_returns(t)
        if ids:
            a, b = seg_rows_to_arrays(rows)
            s.api_return(ids, resp, a)
            assert o.api_return(ids, resp, b) == 0
        ev = drv.events(t, prev)
        stats["api"] += int((ev["kind"] == 1).sum()); stats["fin"] += int((ev["kind"] == 2).sum())
        g = s.step(ev, kv)
        r = o.step(ev, kv)
        compare_outputs(s, g, r, where=f"{cname} t={t}")
        if t % state_every == 0 or t == steps - 1:
            compare_state(s, o, where=f"{cname} t={t}")
        prev = g["admitted_id"]
        stats["adm"] += g["n_admitted"]; stats["pre"] += g["n_preempted"]
        stats["starving"] = max(stats["starving"], int(o.pool["starving"].sum()))
    return stats


def test_closed_loop_c1_300_steps():
    st = closed_loop("C1", 16, 300, 16, 0)
    assert st["api"] > 0 and st["fin"] > 0


def test_closed_loop_c1_starvation_fires():
    # tight KV budget and threshold 20 so deferred requests get tagged
    st = closed_loop("C1", 16, 300, 16, 0, kv=60, starvation_threshold=20)
    assert st["starving"] > 0 and st["pre"] > 0


@pytest.mark.parametrize("path", PATHS)
def test_closed_loop_c2(path):
    st = closed_loop("C2", 1500, 150, 600, 6.0, path=path)
    assert st["api"] > 0 and st["fin"] > 0


@pytest.mark.parametrize("path", PATHS)
def test_closed_loop_c3_multi_api(path):
    st = closed_loop("C3", 1500, 150, 600, 6.0, path=path)
    assert st["api"] > 0


@pytest.mark.slow
def test_closed_loop_c4_toolbench():
    closed_loop("C4", 60000, 40, 50000, 200.0, state_every=20)
