"""SURVEY row F2 on the GPU: the simulators driven by the CUDA pass produce exactly the
schedules the oracle-driven runs produce (worked example unit model; workload-scale
engine with error injection)."""
import pytest

import gen
from sim import PassRanker, StaticRanker, average_jct, simulate_unit
from sim import engine
from sim_util import OracleBackend, OracleRanker, table1_cfg, table1_specs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fx", ["a", "b"])
@pytest.mark.parametrize("policy", [0, 1, 2, 3, "pref"])
def test_unit_model_pass_equals_oracle(golden, fx, policy):
    pol = 0 if policy == "pref" else policy
    cfg = table1_cfg(golden, fx, pol)
    runs = []
    for rk in (PassRanker(cfg), OracleRanker(cfg)):
        if policy == "pref":
            rk = StaticRanker([2, 1, 0], rk)
        reqs, tl = simulate_unit(table1_specs(golden), rk, tau=cfg["tau"])
        runs.append((tl, [r.done_at for r in reqs], [r.api_label for r in reqs], average_jct(reqs)))
    assert runs[0] == runs[1]
    expect = {0: 29 / 3, 1: 35 / 3, 2: 31 / 3, 3: 11, "pref": 10}[policy]
    assert abs(float(runs[0][3]) - expect) < 1e-12


@pytest.mark.parametrize("cname,n,rate,T,p", [("C3", 200, 4.0, 100, 0), ("C3", 200, 4.0, 20, 300_000),
                                              ("C2", 300, 6.0, 100, 500_000)])
def test_engine_pass_equals_oracle(cname, n, rate, T, p):
    cfg = gen.lib_config(cname, starvation_threshold=T)
    be = engine.SchedulerBackend(cfg)
    g = engine.run(cname, n, rate, be, seed=3, len_error_ppm=p, api_error_ppm=p)
    be.close()
    o = engine.run(cname, n, rate, OracleBackend(cfg), seed=3, len_error_ppm=p, api_error_ppm=p)
    assert g == o
    assert g["finished"] == n
