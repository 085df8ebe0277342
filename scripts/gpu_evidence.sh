# Round evidence: bench JSON, reference arm, ncu launch list + full capture of the fused
# kernel, per-phase trace.  Outputs under gpurun_out/evidence/.
set -x
mkdir -p gpurun_out/evidence
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/evidence/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/evidence/bench.json 2> gpurun_out/evidence/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/evidence/bench_reference.json 2>> gpurun_out/evidence/bench.err
TRACE=1 STEPS=3 python scripts/prof_step.py > gpurun_out/evidence/trace.txt 2>&1
STEPS=6 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/evidence/launches.csv python scripts/prof_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o gpurun_out/evidence/prof_fused -f python scripts/prof_step.py > /dev/null 2>&1
cuobjdump -sass paper_2410_18248_b200/liblamps.so > gpurun_out/evidence/sass_full.txt 2>&1
timeout 600 python bench.py --merge --steps 30 --no-cpu-baseline > gpurun_out/evidence/bench_merge.json 2>> gpurun_out/evidence/bench.err
python scripts/ncu_summary.py gpurun_out/evidence/prof_fused.ncu-rep > gpurun_out/evidence/ncu_fused.txt 2>&1
