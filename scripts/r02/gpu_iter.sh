# build + GPU tests (fast) + bench + per-phase trace; TAG names the outputs
set -x
TAG=${TAG:-it}
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r02/gputest_$TAG.txt 2>&1
tail -3 gpurun_out/r02/gputest_$TAG.txt
timeout 600 python bench.py --no-cpu-baseline --no-variants > gpurun_out/r02/bench_$TAG.json 2> gpurun_out/r02/bench_$TAG.err
TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/r02/trace_$TAG.txt 2>&1
