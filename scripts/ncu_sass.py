"""Top SASS instructions of an ncu report by warp-stall samples (with stall reason columns)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur); continue
    if r and r[0] == "Address":
        if cur is None:
            cur = {"name": "?", "rows": []}; blocks.append(cur)
        cur["hdr"] = r; continue
    if cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(dict(zip(cur["hdr"], r)))
b = blocks[0]
res = []
for i, d in enumerate(b["rows"]):
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    res.append((s, i, d["Source"]))
tot = sum(x[0] for x in res) or 1
print(b["name"][:80], "total samples", tot)
for s, i, src in sorted(res, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}%  #{i:<5} {src}")
