# large-pool kernel with the shared-memory range sort: parity of the big paths (incl. the slow
# 2^21 case), then 2^21..2^23 step times of the working tree vs ab/*.so (alternating, 2 rounds)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "above_fused_capacity" 2>&1 | tail -2
for rnd in 1 2; do
  for so in "" "$@"; do
    echo "== ${so:-current}"
    LAMPS_LIB=$so LO=21 HI=23 STEPS=20 timeout 600 python scripts/sweep.py 2>&1 >/dev/null | python -c "
import sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{') and 'slots' in l and 'path' in l:
        try:
            d=eval(l); print(d['slots'], d['us_per_step'])
        except Exception: pass
"
  done
done
