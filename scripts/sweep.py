"""Pool-size sweep (BASELINE config C5: 2^10 .. 2^23 slots, GPT-J profile): device time per
scheduling step (CUDA events, L2 flushed before every step) and the path taken (fused
cooperative kernel up to #SM * 10240 slots, the 3-kernel path above).  JSON to stdout."""
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
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(STEPS)]
    for a, b in ev:
        flush.zero_()
        a.record()
        s.step_async(kv)
        b.record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / STEPS
    r = s.result()
    k, _ = s.stats()
    row = {"slots": cap, "eligible": r["n_eligible"], "us_per_step": round(ms * 1e3, 2),
           "decisions_per_s": r["n_eligible"] / (ms / 1e3), "path": "fused" if k == 1 else "3-kernel"}
    print(row, file=sys.stderr, flush=True)
    rows.append(row)
    s.close()
print(json.dumps({"sweep": rows, "l2": "flushed before every step (256 MiB write)", "config": "C5 (GPT-J)"}, indent=1))
