# final refresh: the bench line, configs, traces, full GPU test suite of the last build
O=gpurun_out/r02final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 200 $O/bench.json; echo
timeout 900 python scripts/configs_bench.py > $O/configs.json 2>&1
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py > $O/trace.txt 2>&1
HEAD=1 ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py > $O/trace_head.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o $O/prof_fused -f python scripts/prof_step.py > /dev/null 2>&1
python scripts/ncu_summary.py $O/prof_fused.ncu-rep > $O/ncu_fused.txt 2>&1
python scripts/ncu_lines.py $O/prof_fused.ncu-rep 40 > $O/ncu_fused_lines.txt 2>&1
python scripts/ncu_region.py $O/prof_fused.ncu-rep > $O/ncu_fused_regions.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/sass_summary.py $O/sass_full.txt.gz > $O/sass_summary.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_full.txt 2>&1
tail -3 $O/gpu_tests_full.txt
