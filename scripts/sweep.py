"""Pool-size sweep (BASELINE config C5: 2^10 .. 2^23 slots, GPT-J profile): device time per
scheduling step (CUDA events, L2 flushed before every step) and the path taken (the one-CTA
kernel up to 4096 slots, the fused cooperative kernel up to #SM * 10240, the large-pool path above;
the untimed first step after the import builds the range grid).  JSON to stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2410_18248_b200 import Scheduler  # noqa: E402

lo, hi = int(os.environ.get("LO", "10")), int(os.environ.get("HI", "23"))
STEPS = int(os.environ.get("STEPS", "10"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for lg in range(lo, hi + 1):
    cap = 1 << lg
    ib = max(20, lg)
    cfg = gen.lib_config("C5", capacity=cap, id_bits=ib, score_bits=min(35, 63 - ib))
    snap = gen.snapshot("C5", seed=1, id_base=cap * 3 + 5, n=cap, capacity=cap)
    s = Scheduler(cfg)
    kv = gen.CONFIGS["C5"]["kv_total"]
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    for _ in range(3):
        flush.zero_()
        s.step_async(kv)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    flush.zero_()
    s.step_async(kv)  # the cold step after the import (builds the range grid), untimed
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(STEPS)]
    for a, b in ev:
        flush.zero_()
        a.record()
        s.step_async(kv)
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    ms = sum(ts) / STEPS
    r = s.result()
    k, _ = s.stats()
    row = {"slots": cap, "eligible": r["n_eligible"], "us_per_step": round(ms * 1e3, 2),
           "us_median": round(ts[len(ts) // 2] * 1e3, 2), "decisions_per_s": r["n_eligible"] / (ms / 1e3),
           "path": ("k_small" if cap <= 4096 else "k_fused") if k == 1 else ("big (k_big_score + k_big_sort)"
                                                                           if k == 2 else "3-kernel")}
    print(row, file=sys.stderr, flush=True)
    rows.append(row)
    s.close()
print(json.dumps({"sweep": rows, "l2": "flushed before every step (256 MiB write)", "config": "C5 (GPT-J)"}, indent=1))
