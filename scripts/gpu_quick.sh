# build, smoke, fast GPU tests, bench (phases), per-phase trace
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_q.json"))
print("us/step", round(d["us_per_step"], 2), "frac", round(d["roofline"]["frac"], 4), d["kernels"]["k_fused"]["phase_us"])
print("variants", [(v["name"], round(v["us_per_step"], 1)) for v in d.get("variants", [])])
PY
TRACE=1 STEPS=3 python scripts/prof_step.py 2>&1 | sed -n 2,20p
if [ "$PERCTA" = "1" ]; then TRACE=1 PERCTA=1 STEPS=3 python scripts/prof_step.py 2>&1 | tail -150 > gpurun_out/percta.txt; fi
