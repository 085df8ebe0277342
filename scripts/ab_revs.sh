# A/B of builds on one box: current tree vs the .so files given as arguments (ab/*.so).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rnd in 1 2; do
  echo "== current"; TUNES=0 ROUNDS=2 python scripts/ab_tune.py
  for so in "$@"; do echo "== $so"; LAMPS_LIB=$so TUNES=0 ROUNDS=2 python scripts/ab_tune.py; done
done
