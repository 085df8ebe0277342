"""e2e per engine iteration, same box, same pool: three separate calls vs lamps_iterate."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2410_18248_b200 import Scheduler
from paper_2410_18248_b200.lamps import EVENT_DTYPE, SEGMENT_DTYPE

cfg = gen.lib_config("C5"); cap = cfg["capacity"]
snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99, n=cap - 8192)
kv = gen.CONFIGS["C5"]["kv_total"]
N = int(os.environ.get("N", "200"))


def run(mode):
    s = Scheduler(cfg)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    prev = s.step(kv_total=kv)["admitted_id"]
    paused = []
    T = {"build": 0.0, "call": 0.0}
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    for k in range(N):
        t0 = time.perf_counter()
        ev = np.zeros(min(4, len(prev)), EVENT_DTYPE)
        for j in range(len(ev)):
            ev[j]["id"], ev[j]["kind"] = prev[j], 2 if j < 2 else 1
        ids = np.asarray(paused[:2], np.uint64)
        nxt = np.zeros(len(ids), SEGMENT_DTYPE); nxt["pre_len"], nxt["has_api"] = 50, 0
        resp = np.full(len(ids), 16, np.uint32)
        paused = paused[2:]
        segs = np.zeros(2, SEGMENT_DTYPE)
        segs["prompt_len"], segs["pre_len"], segs["has_api"], segs["api_seconds"] = 300, 100, 1, 1.5
        segs["resp_len"], segs["post_len"] = 64, 50
        t1 = time.perf_counter()
        if mode == "iterate":
            out, _ = s.iterate(events=ev, ret_ids=ids, ret_resp=resp, ret_next=nxt, arrivals=segs, kv_total=kv)
        else:
            if len(ids):
                s.api_return(ids, resp, nxt)
            s.submit_rc(segs)
            out = s.step(ev, kv)
        t2 = time.perf_counter()
        T["build"] += t1 - t0; T["call"] += t2 - t1
        paused += [int(x) for x in ev["id"][2:]]
        prev = out["admitted_id"]
    torch.cuda.synchronize()
    tot = time.perf_counter() - t_all
    s.close()
    print(f"{mode:9s} total {1e6 * tot / N:6.1f} us/iter  (build {1e6 * T['build'] / N:5.1f}, calls {1e6 * T['call'] / N:6.1f})")


for rnd in range(2):
    run("separate")
    run("iterate")
