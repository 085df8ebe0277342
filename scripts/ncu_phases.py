"""Per-phase breakdown of the fused step kernel from an ncu source page (samples + instructions)."""
import csv, io, subprocess, sys, os
rep = sys.argv[1]
src_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_18248_b200", "csrc", "kernels_fused.cu")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, res = "?", None, []
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try: res.append((int(r[7] or 0), int(r[4] or 0), fname, int(r[0]), r[1][:100]))
        except: pass
ti = sum(x[0] for x in res) or 1; ts = sum(x[1] for x in res) or 1
src = open(src_path).read().split("\n")
keys = ["uint32_t bucket_of", "uint64_t* local_lsd", "uint64_t* local_sort", "k_fused(Bufs", "// ---------------- S:",
        "// ---------------- H:", "// ---------------- T:", "// ---------------- X:", "// CTA r sorts",
        "// ---------------- L:", "// ---------------- A:"]
marks = sorted([(i, k) for i, l in enumerate(src, 1) for k in keys if k in l])
agg = {}
for i, s, f, ln, txt in res:
    if f == "kernels_fused.cu":
        k = "header"
        for at, name in marks:
            if ln >= at: k = name
    else:
        k = f
    a = agg.setdefault(k, [0, 0]); a[0] += i; a[1] += s
print(f"total samples {ts}, warp instructions {ti/1e6:.1f}M")
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:28s} samples {100*s/ts:5.1f}%  inst {100*i/ti:5.1f}%")
print("top lines:")
for i, s, f, ln, txt in sorted(res, key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {100*s/ts:5.1f}% {f}:{ln} {txt}")
