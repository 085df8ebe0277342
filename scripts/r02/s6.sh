# small-pool kernel A/B: fast GPU tests, then C1-C5 step times and k_small phases of the working
# tree vs ab/*.so (two alternating rounds)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s6
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/s6/tests.txt 2>&1
tail -2 gpurun_out/s6/tests.txt; grep -m2 -A12 "Error" gpurun_out/s6/tests.txt
for rnd in 1 2; do
  for so in "" "$@"; do
    echo "== ${so:-current}"
    LAMPS_LIB=$so timeout 600 python scripts/configs_bench.py 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
print(' '.join(f\"{c['config']}:{c['us_median']}\" for c in d['configs'] if 'small' in c['kernel'] or c['config'] in ('C4','C5')))"
    LAMPS_LIB=$so python scripts/r02/small_trace.py 2>/dev/null
  done
done
