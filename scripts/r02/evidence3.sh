# Round-2 final evidence (after the TMA range sort / binned R): bench (N=1), reference arm,
# strong-scaling line, configs, sweep, traces, the bench command's launch list, ncu full
# captures of k_fused (C5) and k_small (C2), SASS.  Output: gpurun_out/r02ev2/.
O=gpurun_out/r02ev3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>> $O/bench.err
timeout 600 python bench.py --scaling strong --steps 30 --warmup 5 > $O/bench_strong.json 2>> $O/bench.err
LAMPS_BENCH_OVERSUBSCRIBE=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_n2_oversubscribed.json 2>> $O/bench.err
timeout 900 python scripts/configs_bench.py > $O/configs.json 2>&1
timeout 900 python scripts/sweep.py > $O/sweep.json 2>&1
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py > $O/trace.txt 2>&1
HEAD=1 ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py > $O/trace_head.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o $O/prof_fused -f python scripts/prof_step.py > /dev/null 2>&1
CFG=C2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 3 -c 1 -o $O/prof_small -f python scripts/prof_step.py > /dev/null 2>&1
python scripts/ncu_summary.py $O/prof_fused.ncu-rep > $O/ncu_fused.txt 2>&1
python scripts/ncu_summary.py $O/prof_small.ncu-rep > $O/ncu_small.txt 2>&1
python scripts/ncu_lines.py $O/prof_fused.ncu-rep 40 > $O/ncu_fused_lines.txt 2>&1
python scripts/ncu_region.py $O/prof_fused.ncu-rep > $O/ncu_fused_regions.txt 2>&1
python scripts/sass_summary.py $O/sass_full.txt.gz > $O/sass_summary.txt 2>&1
head -12 $O/ncu_fused.txt
ls -la $O
python scripts/r02/small_trace.py > $O/small_trace.txt 2>&1
cat $O/small_trace.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_full.txt 2>&1
tail -3 $O/gpu_tests_full.txt
