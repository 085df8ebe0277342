# build, bench + trace, then the ncu full capture of k_fused (TAG names the outputs)
set -x
TAG=${TAG:-p}
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_$TAG.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-variants > gpurun_out/r02/bench_$TAG.json 2> gpurun_out/r02/bench_$TAG.err
TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/r02/trace_$TAG.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/r02/prof_$TAG -f python scripts/prof_step.py > gpurun_out/r02/ncu_$TAG.log 2>&1
