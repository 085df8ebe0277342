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
