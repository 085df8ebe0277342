"""Which binned-R paths the stress pools of tests/test_binned_gpu.py reach: per step, the largest
hint-miss count and overflow-list length over the CTAs (trace slots 16 / 17) and the fallbacks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gen
from paper_2410_18248_b200 import Scheduler, LAMPS_TRACE

CONTENT = ("state", "has_api", "starving", "strategy", "cnt", "ctx", "pre_rem", "api_ticks", "resp_len",
           "post_len", "pending")


def run(name, cname, snap, steps):
    s = Scheduler(gen.lib_config(cname), flags=LAMPS_TRACE)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    for t in range(steps):
        s.step(kv_total=gen.CONFIGS[cname]["kv_total"])
        tr = s.trace().astype(np.int64)
        print(f"{name} step {t}: max hint misses {tr[:, 16].max()}, max overflow keys {tr[:, 17].max()}, stats {s.stats()}")
    s.close()


snap = gen.snapshot("C4", seed=0, id_base=0)
live = np.flatnonzero(snap["state"] != 0)
order = live[np.argsort((snap["ctx"] + snap["pre_rem"])[live], kind="stable")]
for f in CONTENT:
    v = snap[f].copy(); v[live] = snap[f][order]; snap[f] = v
run("C4 sorted layout", "C4", snap, 5)
cfg = gen.lib_config("C5")
snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99)
ready = snap["state"] == 1
snap["cnt"] = np.where(ready, cfg["starvation_threshold"] - 2, snap["cnt"])
snap["starving"] = np.where(ready, 0, snap["starving"])
run("C5 mass flip", "C5", snap, 4)
