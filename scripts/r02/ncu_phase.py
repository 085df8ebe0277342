"""Aggregate an ncu source page (cuda,sass) of k_fused by source line ranges (phases):
warp-stall samples, executed warp instructions and the stall mix per phase."""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, line = "?", None, None
per = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] == "Function Name" or hdr is None:
        continue
    if r[0] not in ("",):
        line = int(r[0]) if r[0].isdigit() else line
        continue
    if r[2] in ("...", "") or r[4] == "-":
        continue
    try:
        samp = int(r[6] or 0); inst = int(r[7] or 0)
    except ValueError:
        continue
    d = per[(fname, line)]
    d[0] += samp; d[1] += inst
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("", "-", "0"):
            d[2][h[6:]] += int(r[i])
spec = sys.argv[2] if len(sys.argv) > 2 else None
phases = []  # (name, file, lo, hi)
if spec:
    for ln in open(spec):
        ln = ln.split("#")[0].strip()
        if ln:
            nm, f, lo, hi = ln.split()
            phases.append((nm, f, int(lo), int(hi)))
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for (f, l), d in per.items():
    nm = f"{f}:other"
    for p in phases:
        if p[1] == f and p[2] <= (l or 0) <= p[3]:
            nm = p[0]; break
    a = agg[nm]
    a[0] += d[0]; a[1] += d[1]; a[2].update(d[2])
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"total samples {ts}, warp instructions {ti}")
for nm, a in sorted(agg.items(), key=lambda x: -x[1][0]):
    top = ", ".join(f"{k} {100*v/max(a[0],1):.0f}%" for k, v in a[2].most_common(4))
    print(f"{nm:28s} {100*a[0]/ts:5.1f}% smp {100*a[1]/ti:5.1f}% inst ({a[1]:9d})  {top}")
if "--lines" in sys.argv:
    for (f, l), d in sorted(per.items(), key=lambda x: -x[1][0])[:40]:
        print(f"{f}:{l} {100*d[0]/ts:5.1f}% {d[1]}")
if "--stalls" in sys.argv:
    for (f, l), d in sorted(per.items(), key=lambda x: -x[1][0])[:25]:
        top = ", ".join(f"{k} {100*v/max(d[0],1):.0f}%" for k, v in d[2].most_common(4))
        print(f"{f}:{l} {100*d[0]/ts:5.1f}% inst {d[1]:8d}  {top}")
if "--range" in sys.argv:  # per-line instructions / samples of file:lo-hi
    spec_r = sys.argv[sys.argv.index("--range") + 1]
    f0, rng = spec_r.split(":")
    lo, hi = map(int, rng.split("-"))
    for (f, l), d in sorted(per.items(), key=lambda x: (x[0][0], x[0][1] or 0)):
        if f == f0 and l is not None and lo <= l <= hi and (d[0] or d[1]):
            top = ", ".join(f"{k} {100*v/max(d[0],1):.0f}%" for k, v in d[2].most_common(3))
            print(f"{f}:{l:5d} smp {d[0]:5d} inst {d[1]:9d}  {top}")
