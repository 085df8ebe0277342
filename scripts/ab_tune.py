"""A/B of the fused kernel's LAMPS_TUNE knobs on one box: for each setting, a fresh handle
(the knobs are read at init), 300 burn-in steps (range weights converge), then 40 timed
steps with the L2 flushed; repeated in rounds so box drift hits every setting alike."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2410_18248_b200 import Scheduler

CN = os.environ.get("CFG", "C5")
cfg = gen.lib_config(CN)
snap = gen.snapshot(CN, seed=0, id_base=(1 << 20) * 7 + 99)
kv = gen.CONFIGS[CN]["kv_total"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
settings = [int(x, 0) for x in os.environ.get("TUNES", "0,1,2,3").split(",")]
res = {t: [] for t in settings}
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
    for t in settings:
        os.environ["LAMPS_TUNE"] = str(t)
        s = Scheduler(cfg)
        s.import_pool(snap, snap["id_base"], snap["next_id"])
        for _ in range(300):
            s.step_async(kv)
        s.import_pool(snap, snap["id_base"], snap["next_id"])
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(int(os.environ.get("STEPS", "40")))]
        for a, b in ev:
            flush.zero_()
            a.record()
            s.step_async(kv)
            b.record()
        torch.cuda.synchronize()
        res[t].append(sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3)
        s.close()
for t in settings:
    v = sorted(res[t])
    print(f"tune {t}: us/step {['%.2f' % x for x in res[t]]}  median {v[len(v) // 2]:.2f}")
