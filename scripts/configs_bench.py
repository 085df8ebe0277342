"""Step time on each BASELINE.json config (C1-C5 pools from gen.snapshot, the config's own
KV budget and cost profile), L2 flushed before every timed step, 100 burn-in steps (range
weights), 50 timed steps from the snapshot.  Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2410_18248_b200 import Scheduler  # noqa: E402
from paper_2410_18248_b200.lamps import LAMPS_GRID_STEP  # noqa: E402

flush = torch.empty(256 << 20 if not os.environ.get("NOFLUSH") else 16, dtype=torch.uint8, device="cuda")
out = []
runs = [(c, 0) for c in ("C1", "C2", "C3", "C4", "C5")]
runs += [(c, LAMPS_GRID_STEP) for c in ("C1", "C2", "C3")]  # small pools on the grid-wide kernel
for cname, flags in runs:
    cfg = gen.lib_config(cname)
    snap = gen.snapshot(cname, seed=0, id_base=(1 << 20) * 7 + 99)
    kv = gen.CONFIGS[cname]["kv_total"]
    s = Scheduler(cfg, flags=flags)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    for _ in range(100):
        flush.zero_()
        s.step_async(kv)
    s.import_pool(snap, snap["id_base"], snap["next_id"])
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in ev:
        flush.zero_()
        a.record()
        s.step_async(kv)
        b.record()
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    r = s.result()
    k, _ = s.stats()
    med = us[len(us) // 2]
    out.append({"config": cname, "kernel": "k_fused (grid)" if flags or cfg["capacity"] > 4096 else "k_small (one CTA)",
                "slots": cfg["capacity"], "live": int((snap["state"] != 0).sum()),
                "eligible": r["n_eligible"], "admitted": r["n_admitted"], "kernels_per_step": k,
                "us_median": round(med, 2), "us_min": round(us[0], 2), "us_max": round(us[-1], 2),
                "decisions_per_s": r["n_eligible"] / (med * 1e-6)})
    s.close()
print(json.dumps({"configs": out}, indent=1))
