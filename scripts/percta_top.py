"""Slowest CTAs of the fused kernel's range sort from gpurun_out/percta.txt (prof_step PERCTA=1)."""
import sys
import numpy as np
rows = [[float(x) for x in l.split()] for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/percta.txt")
        if len(l.split()) >= 10 and l.split()[0].isdigit()]
a = np.array(rows)
print("cta keys buckets Lsort | P+zero count+scan place+rank refine | big score Xscatter")
for i in np.argsort(-a[:, 3])[:6]:
    print(" ".join(f"{x:7.2f}" for x in a[i]))
print("mean", " ".join(f"{x:7.2f}" for x in a.mean(axis=0)))
