# ncu full captures (source counters) of k_fused: the working tree's build and each .so given
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/r02/prof_cur -f python scripts/prof_step.py > gpurun_out/r02/ncu_cur.log 2>&1
for so in "$@"; do
  LAMPS_LIB=$so ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/r02/prof_$(basename $so .so) -f python scripts/prof_step.py > gpurun_out/r02/ncu_$(basename $so .so).log 2>&1
done
