"""lamps_iterate (one engine iteration in one call: API returns, arrivals, the step with its
events) against the oracle running the same iteration as three separate calls, on closed
loops -- every step's outputs and, periodically, the whole pool state bit-exact -- on the
fused path (returns, arrivals and events applied in the kernel's prologue) and the 3-kernel
path."""
import numpy as np
import pytest

import gen
import oracle as O
from parity_util import PATH_FLAGS, compare_outputs, compare_state, make_pair, seg_rows_to_arrays

pytestmark = pytest.mark.gpu


def loop(cname, n_req, steps, initial, per_step, path="fused", seed=0, state_every=10, **over):
    cfg = gen.lib_config(cname, **over)
    kv = gen.CONFIGS[cname]["kv_total"]
    s, o = make_pair(cfg, debug=False, path=path)
    reqs = gen.requests(cname, n_req, seed=seed)
    drv = gen.ClosedLoop(reqs, gen.PROFILES[gen.CONFIGS[cname]["profile"]]["tau"], initial, per_step, seed)
    prev = []
    seen = dict(ret=0, ev=0, arr=0)
    for t in range(steps):
        rids, resp, rrows = drv.api_returns(t)
        idx, arows = drv.arrivals(t)
        ev = drv.events(t, prev)
        ra, rb = seg_rows_to_arrays(rrows)
        aa, ab = seg_rows_to_arrays(arows)
        g, gids = s.iterate(events=ev, ret_ids=rids, ret_resp=resp, ret_next=ra, arrivals=aa, kv_total=kv)
        # the oracle runs the same iteration as three calls
        if rids:
            assert o.api_return(rids, resp, rb) == 0
        if len(arows):
            rc, oids = o.submit(ab)
            assert rc == 0 and np.array_equal(gids, oids), t
            drv.on_submitted(idx, gids)
        r = o.step(ev, kv)
        compare_outputs(s, g, r, where=f"{cname} t={t}")
        if t % state_every == 0 or t == steps - 1:
            compare_state(s, o, where=f"{cname} t={t}")
        prev = g["admitted_id"]
        seen["ret"] += len(rids); seen["ev"] += len(ev); seen["arr"] += len(arows)
    s.close()
    return seen


@pytest.mark.parametrize("path", ["fused", "multi"])
def test_iterate_closed_loop_c3(path):
    seen = loop("C3", 1500, 150, 600, 6.0, path=path)
    assert seen["ret"] > 0 and seen["ev"] > 0 and seen["arr"] > 0


def test_iterate_closed_loop_c1_starvation():
    loop("C1", 16, 300, 16, 0, starvation_threshold=20)


def test_iterate_rejects_atomically():
    """A bad part (unknown returning id, bad arrival) rejects the whole call; nothing applied."""
    from paper_2410_18248_b200.lamps import SEGMENT_DTYPE, LAMPS_ENOENT, LAMPS_EINVAL
    cfg = gen.lib_config("C2")
    s, o = make_pair(cfg, debug=False)
    snap = gen.snapshot("C2", seed=1, id_base=5)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    before = s.export_pool()
    nxt = np.zeros(1, SEGMENT_DTYPE); nxt["pre_len"] = 5
    rc, _, _ = s.iterate_rc(ret_ids=[snap["next_id"] + 5], ret_resp=[1], ret_next=nxt, kv_total=3000)
    assert rc == LAMPS_ENOENT
    bad = np.zeros(1, SEGMENT_DTYPE); bad["has_api"] = 2
    rc, _, _ = s.iterate_rc(arrivals=bad, kv_total=3000)
    assert rc == LAMPS_EINVAL
    after = s.export_pool()
    for f in ("state", "ctx", "pre_rem", "cnt", "pending"):
        assert np.array_equal(before[f], after[f]), f
    s.close()


def _segs(n, has_api=1, seed=0):
    """n arrival segments in both record types (library, oracle), lengths varied by seed."""
    rows = [dict(prompt_len=60 + (7 * k + seed) % 90, pre_len=3 + (5 * k + seed) % 11, has_api=has_api,
                 api_seconds=0.25 + 0.125 * ((k + seed) % 5), resp_len=4 + k % 9, post_len=2 + (3 * k) % 7)
            for k in range(n)]
    return seg_rows_to_arrays(rows)


# (API returns, arrivals, events) around the 2 KB staging carried in the kernel's parameter
# block (32 B per return / arrival, 16 B per event): exactly 2048 B and one record more
# (the copy path), each kind alone and mixed
@pytest.mark.parametrize("n_ret,n_arr,n_ev", [(0, 64, 0), (0, 65, 0), (0, 0, 128), (0, 0, 129),
                                              (30, 30, 8), (30, 30, 9), (64, 0, 0), (65, 0, 0), (1, 1, 1)])
def test_iterate_staging_sizes(n_ret, n_arr, n_ev):
    from paper_2410_18248_b200.lamps import EVENT_DTYPE
    cfg = gen.lib_config("C3")
    kv = 1 << 19  # every eligible request fits: admitted lists of up to max_batch (256)
    s, o = make_pair(cfg, debug=False)
    # 300 requests that call an API after a few tokens
    a, b = _segs(300)
    g, gids = s.iterate(arrivals=a, kv_total=kv)
    rc, oids = o.submit(b)
    assert rc == 0 and np.array_equal(gids, oids)
    compare_outputs(s, g, o.step(None, kv), where="t0")
    prev = g["admitted_id"]
    # the first 100 admitted call their API (paused), the rest keep decoding
    ev = np.zeros(100, EVENT_DTYPE)
    ev["id"], ev["kind"] = prev[:100], 1
    g, _ = s.iterate(events=ev, kv_total=kv)
    compare_outputs(s, g, o.step(ev, kv), where="t1")
    paused = [int(x) for x in ev["id"]]
    prev = g["admitted_id"]
    assert len(prev) >= n_ev
    # the iteration under test: n_ret returns (next segment without an API), n_arr
    # arrivals, n_ev finished requests of the previous batch
    ret_ids = np.asarray(paused[:n_ret], np.uint64)
    ra, rb = _segs(n_ret, has_api=0, seed=3)
    resp = np.full(n_ret, 6, np.uint32)
    aa, ab = _segs(n_arr, seed=5)
    ev = np.zeros(n_ev, EVENT_DTYPE)
    ev["id"], ev["kind"] = prev[:n_ev], 2
    g, gids = s.iterate(events=ev, ret_ids=ret_ids, ret_resp=resp, ret_next=ra, arrivals=aa, kv_total=kv)
    if n_ret:
        assert o.api_return(ret_ids, resp, rb) == 0
    if n_arr:
        rc, oids = o.submit(ab)
        assert rc == 0 and np.array_equal(gids, oids)
    compare_outputs(s, g, o.step(ev, kv), where="t2")
    compare_state(s, o, where="t2")
    # and a plain step with events of the same size class (lamps_schedule_step)
    ev2 = np.zeros(min(n_ev, len(g["admitted_id"])), EVENT_DTYPE)
    ev2["id"], ev2["kind"] = g["admitted_id"][:len(ev2)], 2
    compare_outputs(s, s.step(ev2, kv), o.step(ev2, kv), where="t3")
    compare_state(s, o, where="t3")
    s.close()


def test_rejected_step_leaves_handle_unchanged():
    """A step refused for its own preconditions (here: the timing ring is full) is refused
    before anything is staged: the pool and the host shadow are unchanged, and the same
    iteration then runs exactly as on a twin handle that never saw the refusal (the inline
    staging of the refused call must not leak into the next one)."""
    from paper_2410_18248_b200 import LAMPS_TIMING, Scheduler
    from paper_2410_18248_b200.lamps import EVENT_DTYPE, LAMPS_EINVAL
    cfg = gen.lib_config("C2")
    snap = gen.snapshot("C2", seed=4, id_base=11)
    kv = 1 << 19  # full batches (max_batch admitted), so 200 events exceed the 2 KB inline staging
    s, t = Scheduler(cfg, flags=LAMPS_TIMING), Scheduler(cfg)
    for h in (s, t):
        h.import_pool(snap, snap["id_base"], snap["next_id"])
    g = s.step(kv_total=kv)
    assert np.array_equal(g["admitted_id"], t.step(kv_total=kv)["admitted_id"])
    for _ in range(4095):  # fill the timing ring (4096 entries)
        s.step_async(kv)
        t.step_async(kv)
    gs, gt = s.result(), t.result()
    assert np.array_equal(gs["admitted_id"], gt["admitted_id"])
    before = s.export_pool()
    small = np.zeros(2, EVENT_DTYPE)
    small["id"], small["kind"] = gs["admitted_id"][:2], 2
    assert s.step_rc(small, kv) == LAMPS_EINVAL  # ring full
    rc, _, _ = s.iterate_rc(events=small, kv_total=kv)
    assert rc == LAMPS_EINVAL
    after = s.export_pool()
    for f in ("state", "ctx", "pre_rem", "cnt", "pending"):
        assert np.array_equal(before[f], after[f]), f
    s.timing()  # drain
    assert len(gs["admitted_id"]) >= 200
    big = np.zeros(200, EVENT_DTYPE)  # 3200 B > 2 KB: the copy path
    big["id"], big["kind"] = gs["admitted_id"][:len(big)], 1
    a, b = s.step(big, kv), t.step(big, kv)
    for k in ("n_eligible", "n_admitted", "n_preempted", "budget_used"):
        assert a[k] == b[k], k
    assert np.array_equal(a["admitted_id"], b["admitted_id"])
    s.close(); t.close()
