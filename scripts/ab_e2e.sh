for r in 1 2 3; do
  for lib in ab/head.so ""; do
    echo "lib=${lib:-new} run $r: $(LAMPS_LIB=$lib N=400 python scripts/e2e_iterate.py 2>&1 | grep '^iterate' | tail -1)"
  done
done
for lib in ab/head.so "" ab/head.so ""; do
  echo "lib=${lib:-new} bench e2e: $(LAMPS_LIB=$lib python bench.py --steps 20 --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(round(d["e2e"]["ms_per_step"]*1e3,1), round(d["us_per_step"],1))')"
done
