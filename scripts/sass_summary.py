"""SASS evidence for the fused step kernel: opcode histogram of k_fused<false, false> from
cuobjdump of liblamps.so, and the instructions that prove the design (TMA bulk copies
UBLKCP + mbarrier SYNCS in the score phase, shared-memory atomics, no tensor-core
instructions).  Usage: python scripts/sass_summary.py [out.sass.gz]"""
import collections
import gzip
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2410_18248_b200", "liblamps.so")
syms = subprocess.run(["cuobjdump", "-symbols", lib], capture_output=True, text=True).stdout
fn = [l.split()[-1] for l in syms.splitlines() if "k_fusedILb0ELb0E" in l][0]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
if len(sys.argv) > 1:
    with gzip.open(sys.argv[1], "wt") as f:
        f.write(sass)
ops = collections.Counter()
for line in sass.splitlines():
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m:
        ops[m.group(2).split(".")[0]] += 1
total = sum(ops.values())
print(f"k_fused<false, false> ({fn}): {total} SASS instructions (static)")
for k in ("UBLKCP", "SYNCS", "ATOMS", "ATOMG", "RED", "BAR", "VOTE", "SHFL", "IMAD", "LDS", "STS", "LDG", "STG",
          "HMMA", "UTCMMA", "UTCHMMA", "UTCQMMA"):
    print(f"  {k:8s} {ops.get(k, 0)}")
print("top opcodes:")
for k, v in ops.most_common(25):
    print(f"  {k:10s} {v:6d}  {100 * v / total:5.1f}%")
