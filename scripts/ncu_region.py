"""Warp-stall samples of an ncu report's SASS, cut into regions at the kernel's trace points
(the clock reads S2UR/CS2R SR_CLOCK... of TRACE(k)): per region the samples, the executed
instructions and the top stall reasons; with an address range, the instructions inside it."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; R = []
for r in rows:
    if r and r[0] == "Address": hdr = r; continue
    if hdr and len(r) == len(hdr): R.append(dict(zip(hdr, r)))
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in R) or 1
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
    for d in R:
        a = int(d["Address"], 16)
        if lo <= a < hi:
            s = int(d["Warp Stall Sampling (All Samples)"] or 0)
            top = sorted(((float(d[k] or 0), k[6:]) for k in st), reverse=True)[:2]
            print(f"{a:6x} {100*s/tot:5.2f}% {int(d['Instructions Executed'] or 0):8d}  {d['Source'][:60]:60s} " +
                  " ".join(f"{k}:{v:.0f}" for v, k in top if v))
    sys.exit()
# regions between clock reads
cut = [i for i, d in enumerate(R) if "SR_CLOCK" in d["Source"] or "CLOCK" in d["Source"].upper()]
print("total samples", tot, "clock reads at", [R[i]["Address"] for i in cut][:40])
edges = [0] + cut + [len(R)]
for a, b in zip(edges, edges[1:]):
    seg = R[a:b]
    s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in seg)
    if s < tot * 0.01: continue
    ins = sum(int(d["Instructions Executed"] or 0) for d in seg)
    agg = {k: sum(float(d[k] or 0) for d in seg) for k in st}
    top = sorted(((v, k[6:]) for k, v in agg.items()), reverse=True)[:4]
    print(f"{R[a]['Address']}-{R[b-1]['Address']}: {100*s/tot:5.1f}% samples, {ins} warp-inst; " +
          ", ".join(f"{k} {100*v/max(s,1):.0f}%" for v, k in top))
