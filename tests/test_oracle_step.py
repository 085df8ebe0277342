"""Pins for the oracle's whole step (A0 events .. A5 admission, counters) and
its ingest calls, against hand traces, Algorithm 1's text, invariants and
brute force (permutation and subset enumeration on pools of <= 8 requests).
"""
import itertools
import random

import numpy as np
import pytest

import gen
import oracle as O


def cfgd(**over):
    d = dict(capacity=16, block_tokens=16, tau=1, A1=0, A2=0, S0=0, S1=0, SH=0, c_other=0,
             ticks_per_second=1e6, starvation_threshold=100, max_batch=16,
             kv_capacity_blocks=1 << 40, score_bits=40, id_bits=23)
    d.update(over)
    return d


def pool_of(cfg, recs, next_id=None, prev=()):
    p = O.OraclePool(cfg)
    cap = cfg["capacity"]
    f = {k: np.zeros(cap, np.int64) for k in O.REQ_DTYPE.names}
    f["strategy"][:] = O.NONE
    for r in recs:
        s = r["id"] % cap
        for k in O.REQ_DTYPE.names:
            if k in r:
                f[k][s] = r[k]
        f["state"][s] = r.get("state", O.READY)
        f["strategy"][s] = r.get("strategy", O.NONE)
    p.load(f, next_id if next_id is not None else max([r["id"] for r in recs] + [-1]) + 1, prev)
    return p


def ev(*pairs):
    a = np.zeros(len(pairs), O.EVENT_DTYPE)
    for k, (i, kind) in enumerate(pairs):
        a[k]["id"], a[k]["kind"] = i, kind
    return a


# ------------------------------------------------------------------ A5 admission
def test_form_batch_spec_example(golden):
    row = golden["spec_examples"]["form_batch"][0]
    # two READY requests, no API; demands blk(ctx+1) with B=1 -> ctx = demand-1
    c = cfgd(block_tokens=1)
    p = pool_of(c, [dict(id=0, ctx=row["demands"][0] - 1, pre_rem=1),
                    dict(id=1, ctx=row["demands"][1] - 1, pre_rem=50)])
    out = p.step(kv_total=row["budget"])
    assert list(out["ranked_id"]) == [0, 1]
    assert out["n_admitted"] == row["expect_admitted"] and out["budget_used"] == 5
    assert p.pool["cnt"][0] == 0 and p.pool["cnt"][1] == 1  # Alg.1


def test_prefix_rule_no_skip_fit():
    # R15: stop at the first request that does not fit (Alg.1 in-order fill)
    c = cfgd(block_tokens=1)
    p = pool_of(c, [dict(id=0, ctx=0, pre_rem=1), dict(id=1, ctx=9, pre_rem=2),
                    dict(id=2, ctx=0, pre_rem=400)])
    out = p.step(kv_total=5)
    assert list(out["ranked_id"]) == [0, 1, 2]
    assert list(out["admitted_id"]) == [0] and out["budget_used"] == 1


def test_max_batch_limit_and_blocked_head():
    c = cfgd(block_tokens=1, max_batch=2)
    p = pool_of(c, [dict(id=i, ctx=0, pre_rem=i + 1) for i in range(5)])
    assert p.step(kv_total=100)["n_admitted"] == 2
    p = pool_of(c, [dict(id=0, ctx=10, pre_rem=1)])
    out = p.step(kv_total=5)
    assert out["n_admitted"] == 0 and out["blocked_head"] == 1
    p = pool_of(c, [])
    out = p.step(kv_total=5)
    assert out["n_eligible"] == 0 and out["blocked_head"] == 0


def test_pinned_preserve_blocks_reduce_budget():
    # R23: Preserve-paused requests keep their KV (Fig. P:909-933 (a))
    c = cfgd(block_tokens=16)
    recs = [dict(id=0, state=O.PAUSED_P, ctx=33, strategy=O.P),     # 3 blocks pinned
            dict(id=1, state=O.PAUSED_D, ctx=1000, strategy=O.D),   # holds nothing
            dict(id=2, state=O.PAUSED_S, ctx=1000, strategy=O.S),   # holds nothing
            dict(id=3, ctx=15, pre_rem=1)]                            # demand blk(16) = 1
    p = pool_of(c, recs)
    out = p.step(kv_total=4)
    assert out["pinned"] == 3 and out["budget"] == 1 and out["n_admitted"] == 1
    p = pool_of(c, recs)
    out = p.step(kv_total=3)
    assert out["budget"] == 0 and out["n_admitted"] == 0 and out["blocked_head"] == 1
    p = pool_of(c, recs)
    assert p.step(kv_total=2)["budget"] == 0  # clamped at 0


# ------------------------------------------------------------------ A3 starvation
def test_starvation_threshold_boundary(golden):
    for row in golden["spec_examples"]["starvation"]:
        c = cfgd(block_tokens=1, starvation_threshold=row["T"])
        # the starving candidate has the worse score; budget for one request
        p = pool_of(c, [dict(id=0, ctx=0, pre_rem=1), dict(id=1, ctx=0, pre_rem=9, cnt=row["cnt"])])
        out = p.step(kv_total=1)
        head = int(out["ranked_id"][0])
        assert (head == 1) == bool(row["expect"])
        assert int(p.pool["starving"][1]) == row["expect"]


def test_two_starving_keep_rank_order():
    # S:255 / P:1085: "relative order of prioritized ... requests is maintained"
    c = cfgd(block_tokens=1, starvation_threshold=5)
    p = pool_of(c, [dict(id=0, ctx=0, pre_rem=1), dict(id=1, ctx=0, pre_rem=30, cnt=5),
                    dict(id=2, ctx=0, pre_rem=20, cnt=7), dict(id=3, ctx=0, pre_rem=2)])
    out = p.step(kv_total=100)
    assert list(out["ranked_id"]) == [2, 1, 0, 3]
    assert list(out["ranked_starving"]) == [1, 1, 0, 0]


def test_deferred_T_steps_is_head_at_step_T_plus_1():
    # Alg.1: a request deferred T consecutive iterations is tagged and
    # placed at the head; the tag is sticky.
    T = 4
    c = cfgd(block_tokens=1, starvation_threshold=T, max_batch=1)
    p = pool_of(c, [dict(id=0, ctx=0, pre_rem=1000), dict(id=1, ctx=0, pre_rem=10 ** 6)])
    # id 0 always wins on score while not starving; id 1 is deferred every step
    for step in range(T):
        out = p.step(kv_total=10 ** 6)
        assert list(out["admitted_id"]) == [0]
    out = p.step(kv_total=10 ** 6)
    assert list(out["admitted_id"]) == [1] and list(out["ranked_starving"][:1]) == [1]
    assert list(out["preempted_id"]) == [0]
    for _ in range(3):
        out = p.step(kv_total=10 ** 6)
        assert list(out["admitted_id"]) == [1]


def test_starving_tag_survives_api_call():
    c = cfgd(block_tokens=1, starvation_threshold=2, A1=1, tau=1)
    p = pool_of(c, [dict(id=0, ctx=5, pre_rem=1, has_api=1, api_ticks=10, starving=1, cnt=9)])
    out = p.step(kv_total=100)
    assert list(out["admitted_id"]) == [0]
    p.step(ev((0, O.EV_API_CALL)), kv_total=100)
    assert p.pool["state"][0] >= O.PAUSED_P and p.pool["starving"][0] == 1
    # not starving: counter resets on API entry
    p = pool_of(c, [dict(id=0, ctx=5, pre_rem=1, has_api=1, api_ticks=10, cnt=1)])
    p.step(kv_total=100)
    p.pool["cnt"][0] = 1  # pretend it had waited once before (cnt is 0 after admission)
    p.step(ev((0, O.EV_API_CALL)), kv_total=100)
    assert p.pool["cnt"][0] == 0 and p.pool["starving"][0] == 0


# ------------------------------------------------------------------ A0 events
def test_events_iteration_semantics():
    c = cfgd(block_tokens=16, A1=1 << 4, SH=4, S1=1 << 4, S0=0, c_other=0, tau=3)
    recs = [dict(id=0, ctx=10, pre_rem=5, pending=77),
            dict(id=1, ctx=20, pre_rem=1, has_api=1, api_ticks=1),      # short API -> P
            dict(id=2, ctx=30, pre_rem=1, has_api=1, api_ticks=10 ** 6),  # long, D vs S
            dict(id=3, ctx=40, pre_rem=0)]
    p = pool_of(c, recs, prev=[0, 1, 2, 3])
    out = p.step(ev((1, O.EV_API_CALL), (2, O.EV_API_CALL), (3, O.EV_FINISHED)), kv_total=1000)
    P = p.pool
    assert (P["ctx"][0], P["pre_rem"][0], P["pending"][0]) == (11, 4, 0)
    # request 1: ctx 21, W_P = 1*21 = 21 < W_D = 21*21 -> Preserve
    assert P["state"][1] == O.PAUSED_P and P["ctx"][1] == 21 and P["pre_rem"][1] == 0
    # request 2: ctx 31, W_D = 31*31 = 961, W_S = 2*31*31 = 1922 -> Discard
    assert P["state"][2] == O.PAUSED_D
    assert P["state"][3] == O.FREE
    assert out["n_eligible"] == 1 and out["pinned"] == 2  # blk(21) = 2
    assert list(out["preempted_id"]) == []


def test_event_validation_leaves_state_unchanged():
    c = cfgd()
    p = pool_of(c, [dict(id=0, ctx=1, pre_rem=1), dict(id=1, ctx=1, pre_rem=1)], prev=[0])
    snap = p.pool.copy()
    assert p.step(ev((1, O.EV_FINISHED)), kv_total=10)["rc"] == O.EINVAL   # not admitted last step
    assert p.step(ev((0, 7)), kv_total=10)["rc"] == O.EINVAL               # bad kind
    assert p.step(ev((0, 1), (0, 2)), kv_total=10)["rc"] == O.EINVAL       # duplicate
    assert p.step(kv_total=(1 << 40) + 1)["rc"] == O.EINVAL                 # above capacity
    assert (p.pool == snap).all()


# ------------------------------------------------------------------ ingest
def test_submit_and_api_return_pending_by_strategy():
    # T_fwd(c) = c (A1 = 2^SH), T_swap(c) = 100 + c
    c = cfgd(block_tokens=16, A1=1 << 8, SH=8, S0=100 << 8, S1=1 << 8, capacity=8)
    p = O.OraclePool(c)
    segs = O.segments([(50, 3, 7, 4, 1e-3, 1), (60, 3, 7, 4, 30.0, 1), (70, 3, 7, 4, 30.0, 1)])
    rc, ids = p.submit(segs)
    assert rc == O.OK and list(ids) == [0, 1, 2]
    assert list(p.pool["pending"][:3]) == [50, 60, 70]          # T_fwd(prompt)
    assert list(p.pool["api_ticks"][:3]) == [1000, 30_000_000, 30_000_000]
    # paused by hand in each strategy at C_i = ctx
    p.pool["state"][:3] = [O.PAUSED_P, O.PAUSED_D, O.PAUSED_S]
    nxt = O.segments([(0, 5, 0, 0, 0.0, 0)] * 3)
    assert p.api_return([0, 1, 2], [7, 7, 7], nxt) == O.OK
    P = p.pool
    assert list(P["ctx"][:3]) == [57, 67, 77]
    assert P["pending"][0] == 7                 # P: T_fwd(57) - T_fwd(50)
    assert P["pending"][1] == 67                # D: T_fwd(67)
    assert P["pending"][2] == (100 + 70) + 7    # S: T_swap(70) + T_fwd(77) - T_fwd(70)
    assert list(P["state"][:3]) == [O.READY] * 3 and list(P["has_api"][:3]) == [0] * 3
    assert list(P["api_ticks"][:3]) == [0] * 3 and list(P["pre_rem"][:3]) == [5] * 3


def test_submit_errors_are_atomic():
    c = cfgd(capacity=4, kv_capacity_blocks=10, block_tokens=16)
    p = O.OraclePool(c)
    ok = O.segments([(10, 5, 0, 0, 0.0, 0)] * 3)
    assert p.submit(ok)[0] == O.OK
    snap = p.pool.copy()
    assert p.submit(O.segments([(10, 5, 0, 0, 0.0, 0)] * 2))[0] == O.ENOSPC
    assert p.submit(O.segments([(150, 20, 0, 0, 0.0, 0)]))[0] == O.EINVAL      # 170 tok > 10 blocks
    assert p.submit(O.segments([(1, 1, 1, 1, float("nan"), 1)]))[0] == O.EINVAL
    assert p.submit(O.segments([(1, 1, 1, 1, -1.0, 1)]))[0] == O.EINVAL
    assert p.submit(O.segments([(1 << 24, 1, 0, 0, 0.0, 0)]))[0] == O.EINVAL
    assert p.submit(O.segments([(1, 1, 0, 0, 0.0, 2)]))[0] == O.EINVAL
    assert (p.pool == snap).all() and p.next_id == 3
    assert p.api_return([0], [1], O.segments([(0, 1, 0, 0, 0.0, 0)])) == O.ENOENT  # READY
    assert p.api_return([9], [1], O.segments([(0, 1, 0, 0, 0.0, 0)])) == O.ENOENT  # unknown


# ------------------------------------------------------------------ brute force
def _brute_step(cfg, recs, kv_total):
    """Whole pipeline by enumeration, composing the separately pinned scalar
    functions: strategy by enumerating the three wastes, order by enumerating
    all permutations, admission by enumerating all subsets."""
    c = O.make_cfg(cfg)
    B = cfg["block_tokens"]
    E = []
    pinned = 0
    for r in recs:
        if r.get("state", O.READY) == O.PAUSED_P:
            pinned += O.blk(r["ctx"], B)
        if r.get("state", O.READY) != O.READY:
            continue
        if r.get("has_api", 0):
            W = O.wastes(c, r["ctx"], r["pre_rem"], r.get("api_ticks", 0))
            strat = min((0, 1, 2), key=lambda k: (W[k], k))
        else:
            strat = O.NONE
        sc = O.score(c, ctx=r["ctx"], pre_rem=r["pre_rem"], api_ticks=r.get("api_ticks", 0),
                     resp_len=r.get("resp_len", 0), post_len=r.get("post_len", 0),
                     pending=r.get("pending", 0), has_api=r.get("has_api", 0), strategy=strat)
        starving = int(r.get("starving", 0) or r.get("cnt", 0) >= cfg["starvation_threshold"])
        E.append((r["id"], sc, starving, O.blk(r["ctx"] + 1, B), strat))

    def before(a, b):  # a ranks ahead of b
        if a[2] != b[2]:
            return a[2] > b[2]
        if a[1] != b[1]:
            return a[1] < b[1]
        return a[0] < b[0]

    order = None
    for perm in itertools.permutations(E):
        if all(before(perm[i], perm[i + 1]) for i in range(len(perm) - 1)):
            assert order is None  # unique
            order = list(perm)
    order = order or []
    budget = max(kv_total - pinned, 0)
    best = ()
    for m in range(1 << len(order)):
        sub = [i for i in range(len(order)) if m >> i & 1]
        if len(sub) > cfg["max_batch"] or sum(order[i][3] for i in sub) > budget:
            continue
        # rank-closed: no lower-ranked admitted while a higher-ranked waits
        if sub != list(range(len(sub))):
            continue
        if len(sub) > len(best):
            best = tuple(sub)
    return order, [order[i] for i in best], pinned


@pytest.mark.parametrize("seed", range(40))
def test_full_step_brute_force(seed):
    rng = random.Random(100 + seed)
    n = rng.randrange(0, 8)
    cfg = cfgd(block_tokens=rng.choice([1, 4, 16]), tau=rng.randrange(1, 50),
               A1=rng.randrange(0, 1 << 10), A2=rng.randrange(0, 8), S0=rng.randrange(0, 1 << 12),
               S1=rng.randrange(0, 1 << 9), SH=rng.randrange(0, 6), c_other=rng.randrange(0, 500),
               starvation_threshold=rng.randrange(1, 6), max_batch=rng.randrange(1, 6),
               score_bits=rng.choice([12, 20, 40]))
    recs = []
    for i in range(n):
        st = rng.choice([O.READY] * 4 + [O.PAUSED_P, O.PAUSED_D, O.PAUSED_S])
        ha = rng.randrange(2)
        recs.append(dict(id=1000 + i, state=st, has_api=ha, ctx=rng.randrange(0, 200),
                         pre_rem=rng.randrange(0, 40), api_ticks=rng.randrange(0, 3000) * ha,
                         resp_len=rng.randrange(0, 30) * ha, post_len=rng.randrange(0, 40) * ha,
                         pending=rng.randrange(0, 500), cnt=rng.randrange(0, 8),
                         starving=int(rng.random() < 0.2),
                         strategy=(st - O.PAUSED_P) if st >= O.PAUSED_P else O.NONE))
        if rng.random() < 0.3 and i:
            recs[-1]["pre_rem"] = recs[0]["pre_rem"]; recs[-1]["ctx"] = recs[0]["ctx"]  # ties
    kv = rng.randrange(0, 60)
    cfg["capacity"] = 16
    p = pool_of(cfg, recs, next_id=1000 + n)
    out = p.step(kv_total=kv)
    order, adm, pinned = _brute_step(cfg, recs, kv)
    assert out["pinned"] == pinned
    assert list(out["ranked_id"]) == [e[0] for e in order]
    assert list(out["ranked_score"]) == [e[1] for e in order]
    assert list(out["admitted_id"]) == [e[0] for e in adm]
    assert list(out["admitted_strategy"]) == [e[4] for e in adm]


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("cname,seed", [("C1", 0), ("C2", 1), ("C3", 2), ("C2", 3)])
def test_step_invariants_on_generated_pools(cname, seed):
    cfg = gen.lib_config(cname)
    snap = gen.snapshot(cname, seed=seed, id_base=seed * 5000 + 3)
    p = O.OraclePool(cfg)
    p.load(snap, snap["next_id"])
    kv = gen.CONFIGS[cname]["kv_total"]
    for _ in range(3):
        before = p.pool.copy()
        out = p.step(kv_total=kv, debug=True)
        ready = before["state"] == O.READY
        # the ranking is a permutation of the waiting queue
        assert sorted(out["ranked_id"].tolist()) == sorted(before["id"][ready].tolist())
        keys = list(zip(-out["ranked_starving"].astype(np.int64), out["ranked_score"], out["ranked_id"]))
        assert keys == sorted(keys) and len(set(keys)) == len(keys)
        # the chosen strategy's waste is at most the other two
        for s in np.nonzero(p.pool["state"] == O.READY)[0]:
            if p.pool["has_api"][s]:
                W = [out["W_P"][s], out["W_D"][s], out["W_S"][s]]
                assert W[out["strategy"][s]] == min(W)
        # admitted blocks are at most the budget; admitted is a prefix; the next does not fit
        B = cfg["block_tokens"]
        slot = {int(i): k for k, i in enumerate(p.pool["id"])}
        dem = [-(-(int(p.pool["ctx"][slot[int(i)]]) + 1) // B) for i in out["ranked_id"]]
        na = out["n_admitted"]
        assert list(out["admitted_id"]) == list(out["ranked_id"][:na])
        assert sum(dem[:na]) == out["budget_used"] <= out["budget"]
        if na < len(dem) and na < cfg["max_batch"]:
            assert sum(dem[:na + 1]) > out["budget"]
        pinned = sum(-(-int(c) // B) for c, s in zip(p.pool["ctx"], p.pool["state"]) if s == O.PAUSED_P)
        assert out["pinned"] == pinned


def test_table1_fixture_step_order(golden):
    # Table 1 under fixture a as a pool: strategies = paper labels, ranked by the
    # literal integral R2 < R3 < R1 (reading R16)
    t1 = golden["table1"]
    f = t1["fixtures"]["a"]
    cfg = cfgd(block_tokens=1, tau=f["tau"], A2=f["A2"], S1=f["S1"], max_batch=1)
    recs = []
    for i, (name, r) in enumerate(t1["requests"].items()):
        recs.append(dict(id=i, ctx=0, pre_rem=r["api_after"], has_api=1,
                         api_ticks=r["api_iters"] * f["tau"], post_len=r["post"]))
    p = pool_of(cfg, recs)
    out = p.step(kv_total=6, debug=True)
    assert "".join("PDS"[s] for s in out["strategy"][:3]) == "PDS"
    assert list(out["ranked_id"]) == [1, 2, 0]
    assert [int(x) for x in out["score"][:3]] == [2790, 297, 700]
