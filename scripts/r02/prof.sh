# ncu full capture (source counters) of the fused step kernel: gpurun_out/r02/prof_${TAG}.ncu-rep
set -x
mkdir -p gpurun_out/r02
TAG=${TAG:-cur}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_$TAG.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o gpurun_out/r02/prof_$TAG -f python scripts/prof_step.py > gpurun_out/r02/ncu_$TAG.log 2>&1
