"""A few steps of the large-pool path (for an ncu launch list): CAP_LG slots, FLAGS (512 =
LAMPS_BIG_STEP to force it below the fused kernel's capacity)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import gen
from paper_2410_18248_b200 import Scheduler
lg = int(os.environ.get("CAP_LG", "21"))
cap = 1 << lg
cfg = gen.lib_config("C5", capacity=cap, id_bits=max(20, lg), score_bits=35)
snap = gen.snapshot("C5", seed=1, id_base=cap * 3 + 5, n=cap, capacity=cap)
s = Scheduler(cfg, flags=int(os.environ.get("FLAGS", "0")))
s.import_pool(snap, snap["id_base"], snap["next_id"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(6):
    flush.zero_()
    s.step_async(gen.CONFIGS["C5"]["kv_total"])
torch.cuda.synchronize()
print(s.result()["n_admitted"])
