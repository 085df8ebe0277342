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
if os.environ.get("NOFLUSH"):
    flush = torch.empty(16, dtype=torch.uint8, device="cuda")
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
    from paper_2410_18248_b200 import LAMPS_HEAD_ONLY
    st = Scheduler(cfg, flags=LAMPS_TRACE | (LAMPS_HEAD_ONLY if os.environ.get("HEAD") else 0))
    st.import_pool(snap, snap["id_base"], snap["next_id"])
    acc = []
    for it in range(10):
        flush.zero_()
        st.step_async(kv)
        t = st.trace().astype(np.int64)
        if it >= 3:
            acc.append(t)
    t = np.stack(acc)  # steps x cta x 16
    # warm steps: S, R (range counting sort + run stores), barrier, L, A
    segs = [("score", 0, 1), ("R search+count", 1, 4), ("R run offsets", 4, 5), ("R local place", 5, 12),
            ("R store", 12, 6), ("barrier", 6, 7),
            ("L prep", 7, 13), ("L sort", 13, 14), ("L store+spl", 14, 8),
            ("A wait/pinned", 8, 15), ("A admit", 15, 9)]
    print("phase durations us (median over steps of max / mean over CTAs):")
    for nm, a0, a1 in segs:
        d = (t[:, :, a1] - t[:, :, a0]) / 1.965e3
        if a0 >= 8 and a1 in (15, 9):
            d = d[:, :1]
        print(f"  {nm:12s} max {np.median(d.max(axis=1)):7.2f}  mean {np.median(d.mean(axis=1)):7.2f}")
    # critical path: every CTA leaves the barrier at about the same time, so the step is
    # max(pre-barrier) + barrier + max(post-barrier); CTA 0's post includes the admission
    pre = (t[:, :, 6] - t[:, :, 0]) / 1.965e3
    post = (t[:, :, 8] - t[:, :, 7]) / 1.965e3
    post[:, 0] = (t[:, 0, 9] - t[:, 0, 7]) / 1.965e3
    print(f"  pre-barrier max {np.median(pre.max(axis=1)):6.2f} (cta {int(np.median(pre.argmax(axis=1)))})  "
          f"post-barrier max {np.median(post.max(axis=1)):6.2f} (cta {int(np.median(post.argmax(axis=1)))}), "
          f"cta0 post {np.median(post[:, 0]):6.2f}, others' mean {np.median(post[:, 1:].mean(axis=1)):6.2f}")
    lp = (t[:, 0, 13] - t[:, 0, 7]) / 1.965e3
    print(f"  cta0: L prep {np.median(lp):5.2f} sort {np.median((t[:, 0, 14] - t[:, 0, 13]) / 1.965e3):5.2f} "
          f"store {np.median((t[:, 0, 8] - t[:, 0, 14]) / 1.965e3):5.2f} admit {np.median((t[:, 0, 9] - t[:, 0, 8]) / 1.965e3):5.2f}")
    for base, part in ((16, "starving"), (24, "nonstarv")):
        for nm, a0, a1 in (("bucket starts", 0, 1), ("rank level1", 1, 2), ("refine", 2, 3), ("lsd fallback", 3, 4)):
            d = (t[:, :, base + a1] - t[:, :, base + a0]) / 1.965e3
            ok = (t[:, :, base + a0] > 0) & (t[:, :, base + a1] >= t[:, :, base + a0])
            d = np.where(ok, d, 0)
            print(f"  L.{part}.{nm:14s} max {np.median(d.max(axis=1)):7.2f}  mean {np.median(d.mean(axis=1)):7.2f}")
        nb = t[:, :, base + 5]
        print(f"  L.{part}.big groups   max {int(nb.max())} mean {nb.mean():.2f}")
    for nm, a0, a1 in (("sort end -> gf sync", 14, 10), ("grid entries", 10, 11), ("-> A", 11, 8)):
        d0 = (t[:, 0, a1] - t[:, 0, a0]) / 1.965e3
        d1 = (t[:, 1:, a1] - t[:, 1:, a0]) / 1.965e3
        print(f"  store.{nm:20s} cta0 {np.median(d0):6.2f}  others max {np.median(d1.max(axis=1)):6.2f} mean {np.median(d1.mean(axis=1)):6.2f}")
    nmiss, novf = t[:, 1:, 16], t[:, 1:, 17]
    print(f"  binned R: hint misses per CTA median {np.median(nmiss):.0f} max {nmiss.max()}, overflow keys median {np.median(novf):.0f} max {novf.max()}")
    ms, nst = st.timing() if False else (None, None)
    if os.environ.get("PERCTA"):
        t0 = acc[-1]
        print("cta  sm  keys  score  R   barr  Lsort [load+minmax zero count scan place rank final]  store")
        for cta in range(t0.shape[0]):
            r = t0[cta]
            d = lambda a, b: (r[b] - r[a]) / 1965
            sub = [(r[33 + i] - r[32 + i]) / 1965 if r[32 + i] and r[33 + i] else 0.0 for i in range(7)]
            print(f"{cta:3d} {r[28]:4d} {r[30]:6d} {d(0,1):6.2f} {d(1,6):5.2f} {d(6,7):5.2f} {d(13,14):6.2f} [" +
                  " ".join(f"{x:5.2f}" for x in sub) + f"] {d(14,8):5.2f}")
    if os.environ.get("LEVELS"):
        t0 = acc[-1]
        print("cta  keys  per-level (us, groups) of the non-starving part; level-0 substeps or/and,count,scan,scatter,final")
        for cta in range(t0.shape[0]):
            r = t0[cta, 32:]
            lv = []
            for k in range(7):
                if r[2 * k] == 0:
                    break
                nxt = r[2 * k + 2] if k < 6 and r[2 * k + 2] else r[14]
                lv.append(f"L{k}:{(nxt - r[2*k]) / 1965:.2f}us/{r[2*k+1]}g")
            ss = ""
            if r[16]:
                b = [r[0], r[16], r[17], r[18], r[19], r[20]]
                ss = " sub " + ",".join(f"{(b[i+1]-b[i]) / 1965:.2f}" for i in range(5)) + f" cut {r[21]} keys {r[22]}"
            print(f"{cta:3d} {t0[cta,30]:6d} " + " ".join(lv) + ss)
    if os.environ.get("ADMIT"):
        r = acc[-1][0, 40:45]
        print("admit substeps us (init+loads, scan+count, writes+hash, preempted):",
              [round((r[i + 1] - r[i]) / 1965, 2) for i in range(4)])
