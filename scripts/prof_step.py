"""Run a few async scheduling steps over the C5 pool (for ncu / nsys-less profiling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2410_18248_b200 import Scheduler, LAMPS_TIMING

cname = os.environ.get("CFG", "C5")
steps = int(os.environ.get("STEPS", "6"))
cfg = gen.lib_config(cname)
snap = gen.snapshot(cname, seed=0, id_base=(1 << 20) * 7 + 99)
s = Scheduler(cfg, flags=LAMPS_TIMING if os.environ.get("TIMING") else 0)
s.import_pool(snap, snap["id_base"], snap["next_id"])
kv = gen.CONFIGS[cname]["kv_total"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(steps):
    flush.zero_()
    s.step_async(kv)
r = s.result()
print("n_eligible", r["n_eligible"], "admitted", r["n_admitted"], "stats", s.stats())
if os.environ.get("TIMING"):
    ms, n = s.timing()
    print("phase ms/step", [x / n for x in ms])
