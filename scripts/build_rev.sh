#!/bin/bash
# Build liblamps.so of git revision $1 into $2 (A/B measurements: LAMPS_LIB=$2 python ...).
set -e
rev=$1; out=$2
tmp=$(mktemp -d)
git archive "$rev" paper_2410_18248_b200/csrc include | tar -x -C "$tmp"
objs=""
for f in "$tmp"/paper_2410_18248_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-ffp-contract=off,-O2 --expt-relaxed-constexpr -I "$tmp/include" \
    -I "$tmp/paper_2410_18248_b200/csrc" -c "$f" -o "$o" &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs -lcudart
rm -rf "$tmp"
