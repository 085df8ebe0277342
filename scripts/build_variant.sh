#!/bin/bash
# Build liblamps.so of the working tree with extra nvcc flags into $1 (A/B: LAMPS_LIB=$1 ...).
set -e
out=$1; shift
tmp=$(mktemp -d)
objs=""
for f in paper_2410_18248_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-ffp-contract=off,-O2 --expt-relaxed-constexpr -I include \
    -I paper_2410_18248_b200/csrc "$@" -c "$f" -o "$o" &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs -lcudart
rm -rf "$tmp"
