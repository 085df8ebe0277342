"""Top CUDA source lines of an ncu report by warp-stall samples and executed instructions
(needs -lineinfo and --import-source on)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, res = "?", None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            samp = int(r[4] or 0); inst = int(r[7] or 0)
        except (ValueError, IndexError):
            continue
        res.append((samp, inst, f"{fname}:{r[0]}", r[1][:100]))
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
print(f"total samples {ts}, warp instructions {ti}")
for s, i, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {loc:22s} {src}")
