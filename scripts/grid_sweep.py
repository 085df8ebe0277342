"""Step time of small pools vs the fused kernel's grid size (LAMPS_FUSED_GRID), L2 flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2410_18248_b200 import Scheduler
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cname in ("C2", "C4"):
    cfg = gen.lib_config(cname)
    snap = gen.snapshot(cname, seed=0, id_base=77)
    kv = gen.CONFIGS[cname]["kv_total"]
    for G in (1, 2, 4, 8, 16, 32, 64, 148):
        os.environ["LAMPS_FUSED_GRID"] = str(G)
        try:
            s = Scheduler(cfg)
        except Exception as e:
            print(cname, G, "n/a", e); continue
        s.import_pool(snap, snap["id_base"], snap["next_id"])
        for _ in range(50):
            s.step_async(kv)
        s.import_pool(snap, snap["id_base"], snap["next_id"])
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
        for a, b in ev:
            flush.zero_(); a.record(); s.step_async(kv); b.record()
        torch.cuda.synchronize()
        k, _ = s.stats()
        print(cname, "G", G, "us/step %.2f" % (sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3), "kernels", k)
        s.close()
