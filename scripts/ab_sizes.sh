# step time at several pool sizes for the current build and the given .so files (same box)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for so in "" "$@"; do
  echo "== ${so:-current}"
  LAMPS_LIB=$so LO=11 HI=20 STEPS=20 python scripts/sweep.py 2>&1 >/dev/null | awk -F"'us_per_step': " '{split($2,a,","); printf "%s ", a[1]} END {print ""}'
done
