# same-box A/B: the working tree's build vs the .so files given (ab/*.so); then a phase trace of each
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/r02
for rnd in 1 2 3; do
  echo "== current"; TUNES=0 ROUNDS=1 python scripts/ab_tune.py
  for so in "$@"; do echo "== $so"; LAMPS_LIB=$so TUNES=0 ROUNDS=1 python scripts/ab_tune.py; done
done
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/r02/ab_trace_cur.txt 2>&1
for so in "$@"; do ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 LAMPS_LIB=$so timeout 300 python scripts/prof_step.py > gpurun_out/r02/ab_trace_$(basename $so .so).txt 2>&1; done
