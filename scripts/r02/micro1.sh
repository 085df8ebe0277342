set -x
mkdir -p gpurun_out/r02
cd scripts/micro
for f in smem_atomics multisplit barrier; do nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/$f $f.cu && /tmp/$f; done > ../../gpurun_out/r02/micro1.txt 2>&1
cd ../..
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02/bench_base.json 2> gpurun_out/r02/bench_base.err
TRACE=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/r02/trace_base.txt 2>&1
