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
if os.environ.get("TRACE"):
    import numpy as np
    from paper_2410_18248_b200 import LAMPS_TRACE
    st = Scheduler(cfg, flags=LAMPS_TRACE)
    st.import_pool(snap, snap["id_base"], snap["next_id"])
    names = ["score", "publish", "barrier1", "exchange", "barrier2", "scatter", "barrier3", "sort", "admit"]
    acc = []
    for it in range(10):
        flush.zero_()
        st.step_async(kv)
        t = st.trace().astype(np.int64)
        if it >= 3:
            acc.append(t)
    t = np.stack(acc)  # steps x cta x 16
    d = np.diff(t[:, :, :10], axis=2) / 1.965e3  # us at max clock
    print("phase durations us (median over steps; max over CTAs / mean over CTAs):")
    for k, nm in enumerate(names):
        col = d[:, :, k] if k < 8 else d[:, :1, k]
        print(f"  {nm:10s} max {np.median(col.max(axis=1)):7.2f}  mean {np.median(col.mean(axis=1)):7.2f}")
    tot = (t[:, 0, 9] - t[:, :, 0].min(axis=1)) / 1.965e3
    print("  CTA0 start->admit done (us, median):", float(np.median(tot)))
