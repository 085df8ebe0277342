import os, sys, time, ctypes
sys.path.insert(0, "/root/repo")
import numpy as np, torch, gen
from paper_2410_18248_b200 import Scheduler
from paper_2410_18248_b200.lamps import EVENT_DTYPE, lib, lamps_step_out
cfg = gen.lib_config("C5"); cap = cfg["capacity"]
snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99, n=cap - 8192)
s = Scheduler(cfg); s.import_pool(snap, snap["id_base"], snap["next_id"])
kv = gen.CONFIGS["C5"]["kv_total"]
N = 300
L = lib(); out = lamps_step_out()
ev = np.zeros(0, EVENT_DTYPE)
for name, fn in [
    ("raw ctypes step (no events)", lambda: L.lamps_schedule_step(s.h, None, 0, kv, ctypes.byref(out))),
    ("s.step(None)", lambda: s.step(None, kv)),
    ("_result only", lambda: s._result(s._out)),
    ("async + step_result raw", lambda: (L.lamps_schedule_step_async(s.h, kv), L.lamps_step_result(s.h, ctypes.byref(out)))),
    ("async only + cuda sync", lambda: (L.lamps_schedule_step_async(s.h, kv), torch.cuda.synchronize())),
]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N): fn()
    torch.cuda.synchronize()
    print(f"{name:32s} {1e6*(time.perf_counter()-t0)/N:7.1f} us")
