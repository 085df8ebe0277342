"""where does the starvation threshold matter?  Sweeps of the load (arrival
rate), KV budget and API-duration scale x threshold T on the GPU pass (sim/engine.py), the
paper's Multi-API classes with GPT-J and Single-API for contrast.  Prints one
JSON document: per regime, per T, completion-time statistics averaged over seeds."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from sim import engine  # noqa: E402

N = int(os.environ.get("N", "600"))
TS = [int(x) for x in os.environ.get("TS", "10,50,100,200,1000,65535").split(",")]
SEEDS = [int(x) for x in os.environ.get("SEEDS", "0,1").split(",")]
# (config, KV budget blocks, API-duration scale, arrival rates req/s)
REGIMES = json.loads(os.environ.get("REGIMES", json.dumps([
    ["C3", 1000, 1.0, [1.6, 2.5]],
    ["C3", 1000, 0.1, [2.0, 3.0, 4.0]],
    ["C3", 500, 0.1, [1.5, 2.0, 3.0]],
    ["C2", 1000, 0.1, [3.0, 4.0, 6.0]],
])))


res = {"workload": f"{N} requests per run, seeds {SEEDS}; gen.requests classes (Table 2), GPT-J profile; "
                   f"tau = 12 ms per step; API durations scaled as listed", "regimes": []}
for cname, kv, scale, rates in REGIMES:
    for rate in rates:
        rows = []
        for T in TS:
            ms = []
            t0 = time.time()
            for sd in SEEDS:
                cfg = gen.lib_config(cname, profile="gptj", starvation_threshold=T, kv_total=kv)
                be = engine.SchedulerBackend(cfg)
                m = engine.run(cname, N, rate, be, seed=sd, kv_total=kv, profile="gptj", api_scale=scale)
                be.close()
                m.pop("done_step")
                ms.append(m)
            r = {"T": T, **{k: sum(m[k] for m in ms) / len(ms) for k in
                            ("jct_mean_s", "jct_median_s", "jct_p99_s", "throughput_rps", "preempted_total")},
                 "wall_s": round(time.time() - t0, 1)}
            print(cname, kv, scale, rate, r, file=sys.stderr, flush=True)
            rows.append(r)
        res["regimes"].append({"config": cname, "kv": kv, "api_scale": scale, "rate": rate, "rows": rows})
print(json.dumps(res, indent=1))
