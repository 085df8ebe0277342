"""Phase clock trace of the one-CTA small-pool kernel (k_small) on C1-C3: score+compaction,
grid+sort, admission (trace slots 0..3, SM clocks)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import gen
from paper_2410_18248_b200 import Scheduler, LAMPS_TRACE
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cname in ("C1", "C2", "C3"):
    cfg = gen.lib_config(cname)
    snap = gen.snapshot(cname, seed=0, id_base=(1 << 20) * 7 + 99)
    kv = gen.CONFIGS[cname]["kv_total"]
    s = Scheduler(cfg, flags=LAMPS_TRACE)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    acc = []
    for it in range(20):
        flush.zero_()
        s.step_async(kv)
        t = s.trace().astype(np.int64)
        if it >= 3:
            acc.append(t[0, :4])
    t = np.median(np.stack(acc), axis=0)
    d = np.diff(t) / 1965.0
    print(cname, "score+compact %.2f  grid+sort %.2f  admit %.2f us" % tuple(d))
    s.close()
