"""SURVEY row F2 trends, on the GPU pass: the paper's starvation-threshold study
(Multi-API with GPT-J) and prediction-error study, as
simulated completion-time statistics of the iteration-level engine (sim/engine.py).
Writes one JSON document to stdout.  Trend only: the engine, not a serving system."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from sim import engine  # noqa: E402

N = int(os.environ.get("N", "600"))
RATE = float(os.environ.get("RATE", "4.0"))
KV = int(os.environ.get("KV", "1000"))
SEEDS = [int(x) for x in os.environ.get("SEEDS", "0,1,2").split(",")]


def avg(rows):
    keys = ("jct_mean_s", "jct_median_s", "jct_p99_s", "throughput_rps", "preempted_total")
    return {k: sum(r[k] for r in rows) / len(rows) for k in keys}


def sweep(cname, profile, kv, label, cases, **fixed):
    out = []
    for case in cases:
        rows = []
        t0 = time.time()
        for sd in SEEDS:
            cfg = gen.lib_config(cname, profile=profile, starvation_threshold=case.get("T", 100), kv_total=kv)
            be = engine.SchedulerBackend(cfg)
            m = engine.run(cname, N, RATE, be, seed=sd, kv_total=kv, profile=profile,
                           len_error_ppm=case.get("p", 0), api_error_ppm=case.get("p", 0))
            be.close()
            m.pop("done_step")
            rows.append(m)
        r = dict(case, **avg(rows), wall_s=round(time.time() - t0, 1))
        print(label, r, file=sys.stderr)
        out.append(r)
    return out


res = {
    "workload": f"{N} requests per run, Poisson {RATE} req/s, seeds {SEEDS}; Multi-API classes (gen.requests C3), "
                f"GPT-J profile, KV budget {KV} blocks; one step = one decode iteration (tau = 12 ms)",
    "starvation": sweep("C3", "gptj", KV, "T", [{"T": t} for t in (10, 50, 100, 200, 1000, 65535)]),
    "error_injection": sweep("C3", "gptj", KV, "p", [{"p": p} for p in (0, 50_000, 100_000, 300_000, 500_000)]),
}
print(json.dumps(res, indent=1))
