"""Summarise an ncu report's source page: top CUDA source lines by warp-stall samples."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kid = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"]
if kid:
    cmd += ["--print-kernel-base", "function", "-k", kid]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
res = []
for r in rows:
    if r and r[0] == "#":
        hdr = r
        continue
    if len(r) > 3 and r[0] == "Line":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        res.append((s, d.get("#", d.get("Line", "")), d.get("Source", "")[:110]))
tot = sum(x[0] for x in res) or 1
for s, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}%  L{ln:>4}  {src}")
