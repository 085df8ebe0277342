"""GPU <-> oracle parity for SURVEY row F1: the baseline rank keys (FCFS, SJF, SJF
by total length; R25) and LAMPS's selective score update (R26), on every path of
the CUDA pass (fused step kernel, 3-kernel path, global-LSD fallback)."""
import numpy as np
import pytest

import gen
import oracle as O
from parity_util import PATH_FLAGS, compare_outputs, compare_state, make_pair, snapshot_step_parity
from test_parity_gpu import closed_loop

pytestmark = pytest.mark.gpu
PATHS = list(PATH_FLAGS)
POLICIES = [O.POL_FCFS, O.POL_SJF, O.POL_SJF_TOTAL]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("cname", ["C2", "C3"])
def test_policy_snapshot_parity(cname, policy, path):
    snapshot_step_parity(cname, seed=policy, id_base=31, steps=3, path=path, policy=policy)


@pytest.mark.parametrize("policy", POLICIES)
def test_policy_c4_snapshot_parity(policy):
    snapshot_step_parity("C4", seed=1, id_base=1000, steps=2, policy=policy)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("interval", [1, 2, 10])
def test_selective_update_snapshot_parity(interval, path):
    snapshot_step_parity("C3", seed=4, id_base=3, steps=12, path=path, score_interval=interval)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("policy,interval", [(O.POL_LAMPS, 10), (O.POL_LAMPS, 3), (O.POL_FCFS, 10),
                                             (O.POL_SJF, 1), (O.POL_SJF_TOTAL, 10)])
def test_policy_closed_loop(policy, interval, path):
    """Submissions, API calls / returns (which mark segments dirty) and finishes."""
    st = closed_loop("C3", 1200, 120, 500, 5.0, path=path, state_every=5, policy=policy, score_interval=interval)
    assert st["api"] > 0 and st["adm"] > 0


def test_selective_update_c4_toolbench_interval_10():
    """The paper's configuration: ToolBench-shaped pool, interval 10."""
    snapshot_step_parity("C4", seed=2, id_base=77, steps=12, score_interval=10)


def test_cached_state_roundtrip_through_import():
    """Export / import of the selective-update state (age, dirty, cached score)
    resumes exactly where the oracle is."""
    from paper_2410_18248_b200 import Scheduler
    cfg = gen.lib_config("C2", score_interval=5)
    snap = gen.snapshot("C2", seed=9, id_base=40)
    s, o = make_pair(cfg, debug=False)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    o.load(snap, snap["next_id"])
    kv = gen.CONFIGS["C2"]["kv_total"]
    for t in range(3):
        g, r = s.step(kv_total=kv), o.step(kv_total=kv)
        compare_outputs(s, g, r, where=f"t={t}")
    e = s.export_pool()
    s2 = Scheduler(cfg)
    e2 = dict(e); e2["id"] = e["id"]
    s2.import_pool(e2, snap["id_base"], snap["next_id"])
    # the importing handle has no previous admitted list: give the oracle the same
    o.prev_adm = np.zeros(0, np.uint64)
    for t in range(3, 8):
        g, r = s2.step(kv_total=kv), o.step(kv_total=kv)
        compare_outputs(s2, g, r, where=f"t={t}")
        compare_state(s2, o, where=f"t={t}")
    s.close(); s2.close()


def test_policy_config_validation():
    from paper_2410_18248_b200 import Scheduler, LampsError
    for bad in (dict(policy=4), dict(policy=O.POL_SJF_TOTAL, tau=0), dict(policy=O.POL_SJF, tau=0),
                dict(score_interval=128)):
        cfg = gen.lib_config("C1")
        cfg.update(bad)
        with pytest.raises(LampsError):
            Scheduler(cfg)
