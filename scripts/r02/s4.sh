# ncu source-level capture of the current k_fused + the phase trace with hint stats
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/s4/trace.txt 2>&1
grep binned gpurun_out/s4/trace.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o gpurun_out/s4/prof -f python scripts/prof_step.py > gpurun_out/s4/ncu.log 2>&1
python scripts/ncu_lines.py gpurun_out/s4/prof.ncu-rep 60 > gpurun_out/s4/lines.txt 2>&1
python scripts/ncu_summary.py gpurun_out/s4/prof.ncu-rep > gpurun_out/s4/summary.txt 2>&1
head -5 gpurun_out/s4/summary.txt
