"""Host-side cost of the public API calls of one e2e step (bench.py's e2e loop), C5 pool."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen
from paper_2410_18248_b200 import Scheduler
from paper_2410_18248_b200.lamps import EVENT_DTYPE, SEGMENT_DTYPE

cfg = gen.lib_config("C5")
cap = cfg["capacity"]
snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99, n=cap - 8192)
s = Scheduler(cfg)
s.import_pool(snap, snap["id_base"], snap["next_id"])
kv = gen.CONFIGS["C5"]["kv_total"]
prev = s.step(kv_total=kv)["admitted_id"]
paused = []
T = {"api_return": 0.0, "step": 0.0, "submit": 0.0, "py": 0.0}
N = int(os.environ.get("N", "200"))
torch.cuda.synchronize()
t_all = time.perf_counter()
for k in range(N):
    t0 = time.perf_counter()
    ev = np.zeros(min(4, len(prev)), EVENT_DTYPE)
    for j in range(len(ev)):
        ev[j]["id"], ev[j]["kind"] = prev[j], 2 if j < 2 else 1
    t1 = time.perf_counter(); T["py"] += t1 - t0
    if paused:
        ids = np.asarray(paused[:2], np.uint64)
        nxt = np.zeros(len(ids), SEGMENT_DTYPE)
        nxt["pre_len"], nxt["has_api"] = 50, 0
        s.api_return(ids, np.full(len(ids), 16, np.uint32), nxt)
        paused = paused[2:]
    t2 = time.perf_counter(); T["api_return"] += t2 - t1
    out = s.step(ev, kv)
    t3 = time.perf_counter(); T["step"] += t3 - t2
    paused += [int(x) for x in ev["id"][2:]]
    segs = np.zeros(2, SEGMENT_DTYPE)
    segs["prompt_len"], segs["pre_len"], segs["has_api"], segs["api_seconds"] = 300, 100, 1, 1.5
    segs["resp_len"], segs["post_len"] = 64, 50
    t4 = time.perf_counter(); T["py"] += t4 - t3
    s.submit_rc(segs)
    t5 = time.perf_counter(); T["submit"] += t5 - t4
    prev = out["admitted_id"]
torch.cuda.synchronize()
tot = time.perf_counter() - t_all
print({k: round(v / N * 1e6, 1) for k, v in T.items()}, "total us/step", round(tot / N * 1e6, 1))
# the step alone, async + result, and the bare kernel via events
st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
for k in range(N):
    s.step_async(kv)
torch.cuda.synchronize()
print("step_async back-to-back us/step", round((time.perf_counter() - t0) / N * 1e6, 1))
t0 = time.perf_counter()
for k in range(N):
    s.step(None, kv)
print("step (sync, no events) us/step", round((time.perf_counter() - t0) / N * 1e6, 1))
