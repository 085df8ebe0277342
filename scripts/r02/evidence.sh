# Round-2 evidence: smoke, bench (N=1), reference arm, strong-scaling line, configs, sweep,
# launch list + ncu full capture of k_fused and k_small, SASS, sanitizers.  gpurun_out/r02ev/.
set -x
O=gpurun_out/r02ev; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>> $O/bench.err
timeout 600 python bench.py --scaling strong --steps 30 --warmup 5 > $O/bench_strong.json 2>> $O/bench.err
timeout 900 python scripts/configs_bench.py > $O/configs.json 2>&1
timeout 900 python scripts/sweep.py > $O/sweep.json 2>&1
TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py > $O/trace.txt 2>&1
HEAD=1 TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py > $O/trace_head.txt 2>&1
python scripts/r02/small_trace.py > $O/small_trace.txt 2>&1
STEPS=6 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python scripts/prof_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o $O/prof_fused -f python scripts/prof_step.py > /dev/null 2>&1
CFG=C2 ncu --set full --clock-control none --import-source on -k regex:k_small -s 3 -c 1 -o $O/prof_small -f python scripts/prof_step.py > /dev/null 2>&1
python scripts/ncu_summary.py $O/prof_fused.ncu-rep > $O/ncu_fused.txt 2>&1
python scripts/ncu_summary.py $O/prof_small.ncu-rep > $O/ncu_small.txt 2>&1
cuobjdump -sass paper_2410_18248_b200/liblamps.so > $O/sass_full.txt 2>&1
