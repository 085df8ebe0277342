"""CTA 0's timeline on the multi-shard path with one rank (P2P self-exchange or NCCL): head
sort end -> exchange done -> admission end, from the fused kernel's SM-clock trace."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2410_18248_b200 import Scheduler, LAMPS_TRACE, LAMPS_MERGE
from paper_2410_18248_b200.lamps import LAMPS_XPORT_P2P
cfg = gen.lib_config("C5")
snap = gen.snapshot("C5", seed=0, id_base=(1 << 20) * 7 + 99)
s = Scheduler(cfg, flags=LAMPS_TRACE | LAMPS_MERGE, transport=LAMPS_XPORT_P2P)
s.import_pool(snap, snap["id_base"], snap["next_id"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
acc = []
for it in range(8):
    flush.zero_()
    s.step_async(20000)
    t = s.trace().astype(np.int64)
    if it >= 3:
        acc.append(t)
t = np.stack(acc)
f = lambda a, b: np.median(t[:, 0, b] - t[:, 0, a]) / 1965
print("CTA0: L(7->8) %.2f  exchange(8->15) %.2f  merge+admit(15->9) %.2f us" % (f(7, 8), f(8, 15), f(15, 9)))
g = lambda a, b: np.median(t[:, 0, b] - t[:, 0, a]) / 1965
print("  stores(8->48) %.2f fence+flags(48->49) %.2f wait(49->15) %.2f load(15->50) %.2f merge(50->51) %.2f cut(51->52) %.2f admit(52->53) %.2f" %
      (g(8, 48), g(48, 49), g(49, 15), g(15, 50), g(50, 51), g(51, 52), g(52, 53)))
print("others L max %.2f" % (np.median((t[:, 1:, 8] - t[:, 1:, 7]).max(axis=1)) / 1965))
