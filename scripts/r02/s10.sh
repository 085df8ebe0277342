# head-only (F3) change: the head-path parity tests, then the bench's head_only variant of the
# working tree vs ab/*.so (alternating, 3 rounds)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "head" 2>&1 | tail -2
for rnd in 1 2 3; do
  for so in "" "$@"; do
    LAMPS_LIB=$so timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${so:-current}', round(d['us_per_step'],2), [(v['name'], round(v['us_per_step'],2)) for v in d['variants'] if 'head' in v['name']])"
  done
done
