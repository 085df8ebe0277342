"""Strong-scaling diagnosis at N = 1: 8 co-resident shard kernels (131072 slots each).  Per
shard: kernel start (CTA 0, global clock) relative to the earliest shard, its L phase start /
end, and the admission (CTA 0 SM clocks), median over steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import gen
from paper_2410_18248_b200 import Scheduler, LAMPS_TRACE
from paper_2410_18248_b200.lamps import LAMPS_SHARE_DEVICE, LAMPS_XPORT_P2P
W = 8
cfg = gen.lib_config("C5")
cap = cfg["capacity"] // W
cfg["capacity"] = cap
kv = gen.CONFIGS["C5"]["kv_total"] // W
streams = [torch.cuda.Stream() for _ in range(W)]
S = [Scheduler(cfg, flags=LAMPS_SHARE_DEVICE | LAMPS_TRACE, stream=streams[g], world=W, rank=g,
               transport=LAMPS_XPORT_P2P, local_ranks=W) for g in range(W)]
hs = [s.p2p_handle() for s in S]
for s in S:
    s.p2p_connect(hs)
for g, s in enumerate(S):
    sn = gen.snapshot("C5", seed=g, n=cap, capacity=cap, id_base=1000, kv_total=kv)
    s.import_pool(sn, sn["id_base"], sn["next_id"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()
rows = []
for it in range(12):
    flush.zero_()
    torch.cuda._sleep(200_000)
    e0 = torch.cuda.Event(); e0.record(main)
    for st in streams:
        st.wait_event(e0)
    Scheduler.group_step_async(S, [kv] * W)
    torch.cuda.synchronize()
    for s in S:
        s.result()
    if it >= 4:
        tr = [s.trace().astype(np.int64) for s in S]
        rows.append(tr)
t0s = np.array([[tr[g][0, 29] for g in range(W)] for tr in rows])  # steps x shards
base = t0s.min(axis=1, keepdims=True)
print("kernel start of each shard after the first, us (median over steps):", np.round(np.median((t0s - base) / 1e3, axis=0), 2))
lend = np.array([[tr[g][:, 27].max() for g in range(W)] for tr in rows])
print("last range sort end per shard after the first start, us:", np.round(np.median((lend - base) / 1e3, axis=0), 2))
for g in range(W):
    t = np.stack([tr[g] for tr in rows])  # steps x cta x slots
    d = lambda a, b: np.median((t[:, 0, b] - t[:, 0, a]) / 1965.0)
    dm = lambda a, b: np.median(((t[:, :, b] - t[:, :, a]) / 1965.0).max(axis=1))
    print(f"shard {g}: score {dm(0,1):5.1f} R {dm(1,6):5.1f} barrier {dm(6,7):5.1f} L(max) {dm(13,14):5.1f} "
          f"cta0: L {d(13,14):5.1f} store {d(14,8):4.1f} exchange+merge {d(8,9):5.1f}")
print("CTA 0 exchange / merge timeline (us from TRACE 8): records stored, flags raised -> wait done (TRACE 15), staged, merged, cut, admitted")
for g in range(W):
    t = np.stack([tr[g] for tr in rows])[:, 0, :]
    rel = lambda k: np.median((t[:, k] - t[:, 8]) / 1965.0)
    print(f"shard {g}: loop start {rel(58):6.1f} head key {rel(60):6.1f} rec1024 built {rel(59):6.1f} records(t0) {rel(48):6.1f} flags {rel(49):6.1f}  wait-done {rel(15):6.1f}  staged {rel(50):6.1f}  merged {rel(51):6.1f}  "
          f"cut {rel(52):6.1f}  admitted {rel(53):6.1f}  head keys {int(np.median(t[:, 56]))} wait {int(np.median(t[:, 57]))}")
