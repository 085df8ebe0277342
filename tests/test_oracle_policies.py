"""Oracle pins for SURVEY row F1: the baseline rank keys (FCFS, SJF, SJF by total
length; reading R25) and LAMPS's selective score update (reading R26).  Every
check is against the paper's worked example, a closed form, or an invariant of
the definition -- not a retyped formula."""
import numpy as np
import pytest

import gen
import oracle as O

POL = {"LAMPS": O.POL_LAMPS, "FCFS": O.POL_FCFS, "SJF": O.POL_SJF, "SJF_TOTAL": O.POL_SJF_TOTAL}


def unit_cfg(policy, tau=1, **over):
    d = dict(capacity=16, block_tokens=1, tau=tau, A1=0, A2=1, S0=0, S1=1, SH=0, c_other=0,
             ticks_per_second=1.0, starvation_threshold=100, max_batch=16, kv_capacity_blocks=1 << 20,
             score_bits=40, id_bits=23, policy=policy, score_interval=0)
    d.update(over)
    return d


def table1_pool(cfg, g):
    o = O.OraclePool(cfg)
    rows = []
    for name in ("R1", "R2", "R3"):
        r = g["requests"][name]
        rows.append(dict(prompt_len=0, pre_len=r["pre"], resp_len=0, post_len=r["post"],
                         api_seconds=float(r["api_iters"] * g["tau"]), has_api=1))
    rc, ids = o.submit(O.segments(rows))
    assert rc == O.OK
    return o, ids


@pytest.mark.parametrize("pol", ["FCFS", "SJF", "SJF_TOTAL"])
def test_worked_example_orders(golden, pol):
    """the three baseline orders of the Table 1 requests."""
    g = golden["policies"]
    o, ids = table1_pool(unit_cfg(POL[pol], tau=g["tau"]), g)
    r = o.step(kv_total=1000)
    names = {int(i): n for i, n in zip(ids, ("R1", "R2", "R3"))}
    assert [names[int(i)] for i in r["ranked_id"]] == g["expect"][pol]["order"]
    keys = {names[int(i)]: int(s) for i, s in zip(r["ranked_id"], r["ranked_score"])}
    assert keys == g["expect"][pol]["keys"]


def test_policy_score_closed_forms():
    cfg = O.make_cfg(unit_cfg(O.POL_SJF_TOTAL, tau=10))
    # ceil(api_ticks / tau): 0 -> 0, 1..10 -> 1, 11 -> 2
    for api, it in ((0, 0), (1, 1), (10, 1), (11, 2), (25, 3)):
        assert O.policy_score(cfg, pre_rem=4, post_len=3, api_ticks=api) == 4 + 3 + it
    assert O.policy_score(cfg, pre_rem=4, post_len=3, api_ticks=25, has_api=0) == 4  # no API: no post, no API
    sjf = O.make_cfg(unit_cfg(O.POL_SJF))
    assert O.policy_score(sjf, pre_rem=7, post_len=5, api_ticks=99) == 12
    fcfs = O.make_cfg(unit_cfg(O.POL_FCFS))
    assert O.policy_score(fcfs, pre_rem=7, post_len=5, api_ticks=99) == 0
    # owed prefill / swap-in counts in iterations ("a post-API part of length 2
    # (including recomputation)"): ceil(pending / tau)
    sjf10 = O.make_cfg(unit_cfg(O.POL_SJF, tau=10))
    for pend, it in ((0, 0), (1, 1), (10, 1), (11, 2)):
        assert O.policy_score(sjf10, pre_rem=1, post_len=0, has_api=0, pending=pend) == 1 + it
        assert O.policy_score(cfg, pre_rem=4, post_len=3, api_ticks=25, pending=pend) == 4 + 3 + 3 + it
    small = O.make_cfg(unit_cfg(O.POL_SJF, score_bits=3))
    assert O.policy_score(small, pre_rem=100, post_len=0) == 7  # clamp 2^SB - 1


def test_policy_validation():
    assert O.validate_cfg(O.make_cfg(unit_cfg(4))) == O.EINVAL
    assert O.validate_cfg(O.make_cfg(unit_cfg(O.POL_SJF_TOTAL, tau=0))) == O.EINVAL
    assert O.validate_cfg(O.make_cfg(unit_cfg(O.POL_SJF, tau=0))) == O.EINVAL  # ceil(pending / tau)
    assert O.validate_cfg(O.make_cfg(unit_cfg(O.POL_FCFS, tau=0))) == O.OK
    assert O.validate_cfg(O.make_cfg(unit_cfg(O.POL_LAMPS, score_interval=127))) == O.OK
    assert O.validate_cfg(O.make_cfg(unit_cfg(O.POL_LAMPS, score_interval=128))) == O.EINVAL


def _ranked_keys(r):
    return [(1 - int(s), int(sc), int(i)) for s, sc, i in zip(r["ranked_starving"], r["ranked_score"], r["ranked_id"])]


@pytest.mark.parametrize("seed", range(6))
def test_fcfs_is_id_order_within_starvation_class(seed):
    """FCFS ranks by request id; starving requests first."""
    cfg = gen.lib_config("C2", policy=O.POL_FCFS)
    snap = gen.snapshot("C2", seed=seed, id_base=123)
    o = O.OraclePool(cfg)
    o.load(snap, snap["next_id"])
    r = o.step(kv_total=3000)
    assert np.all(r["ranked_score"] == 0)
    st = r["ranked_starving"].astype(int)
    assert np.all(np.diff(st) <= 0)  # starving block first
    for part in (st == 1, st == 0):
        assert np.all(np.diff(r["ranked_id"][part].astype(np.int64)) > 0)


@pytest.mark.parametrize("seed", range(6))
def test_sjf_sorted_by_remaining_tokens(seed):
    cfg = gen.lib_config("C3", policy=O.POL_SJF)
    snap = gen.snapshot("C3", seed=seed, id_base=7)
    o = O.OraclePool(cfg)
    o.load(snap, snap["next_id"])
    r = o.step(kv_total=640)
    P = o.pool
    slot = {int(i): k for k, i in enumerate(P["id"])}
    tau = cfg["tau"]
    rem = [int(P["pre_rem"][slot[int(i)]]) + (int(P["post_len"][slot[int(i)]]) if P["has_api"][slot[int(i)]] else 0)
           + -(-int(P["pending"][slot[int(i)]]) // tau) for i in r["ranked_id"]]
    assert [int(x) for x in r["ranked_score"]] == rem
    keys = _ranked_keys(r)
    assert keys == sorted(keys)


def test_lamps_equals_sjf_without_apis():
    """with no API calls (and nothing owed, ctx 0, B = 1) the LAMPS area
    tau * L (L + 1) / 2 is increasing in L, so LAMPS ranks exactly as SJF."""
    rng = np.random.default_rng(5)
    rows = [dict(prompt_len=0, pre_len=int(x), has_api=0) for x in rng.integers(1, 300, 14)]
    orders = {}
    for pol in (O.POL_LAMPS, O.POL_SJF):
        o = O.OraclePool(unit_cfg(pol, tau=3))
        o.submit(O.segments(rows))
        orders[pol] = list(o.step(kv_total=10)["ranked_id"])
    assert orders[O.POL_LAMPS] == orders[O.POL_SJF]


def _run_single(interval, steps, api_at=None):
    """One request, always admitted (ample budget): the uncached score changes every
    step (ctx grows, pre_rem shrinks); returns the reported scores."""
    o = O.OraclePool(unit_cfg(O.POL_LAMPS, tau=5, block_tokens=1, score_interval=interval))
    rc, ids = o.submit(O.segments([dict(prompt_len=3, pre_len=40, resp_len=2, post_len=6,
                                        api_seconds=9.0, has_api=1)]))
    out = []
    for t in range(1, steps + 1):
        ev = None
        if api_at is not None and t == api_at:
            ev = np.zeros(1, O.EVENT_DTYPE)
            ev["id"], ev["kind"] = ids[0], O.EV_API_CALL
        r = o.step(ev, kv_total=10_000)
        assert r["rc"] == 0
        if api_at is not None and t == api_at:
            segs = O.segments([dict(prompt_len=0, pre_len=11, resp_len=0, post_len=0, api_seconds=0.0, has_api=0)])
            assert o.api_return(ids, [2], segs) == O.OK
            out.append(None)
            continue
        out.append(int(r["ranked_score"][0]))
    return out


@pytest.mark.parametrize("k", [2, 3, 10])
def test_selective_update_refresh_schedule(k):
    """P:1080, P:1113 (R26): with interval k the reported score is the fresh score of
    the last refresh step; refreshes at steps 1, 1+k, 1+2k, ..."""
    fresh = _run_single(0, 25)
    cached = _run_single(k, 25)
    assert len(set(fresh)) == 25  # the fresh score changes every step
    for t in range(1, 26):
        t0 = 1 + ((t - 1) // k) * k
        assert cached[t - 1] == fresh[t0 - 1], (t, t0)


def test_selective_update_interval_one_is_fresh():
    assert _run_single(1, 20) == _run_single(0, 20)


def test_selective_update_new_segment_is_fresh():
    """An API return starts a new segment: scored afresh at the next
    step whatever the age of the cached score."""
    a = _run_single(10, 12, api_at=4)
    b = _run_single(0, 12, api_at=4)
    assert a[4] == b[4]  # step 5: first step of the new segment
    assert a[5:] == [a[4]] * 7  # then cached again (steps 6..12 < 5 + 10)
    assert a[:3] == [b[0]] * 3


@pytest.mark.parametrize("pol", [O.POL_FCFS, O.POL_SJF, O.POL_SJF_TOTAL])
def test_baselines_ignore_interval(pol):
    """baseline keys are always fresh."""
    res = []
    for interval in (0, 10):
        cfg = gen.lib_config("C2", policy=pol, score_interval=interval)
        snap = gen.snapshot("C2", seed=2, id_base=50)
        o = O.OraclePool(cfg)
        o.load(snap, snap["next_id"])
        outs = []
        for _ in range(4):
            r = o.step(kv_total=3000)
            outs.append((list(r["ranked_id"]), list(r["ranked_score"]), list(r["admitted_id"])))
        res.append(outs)
    assert res[0] == res[1]
