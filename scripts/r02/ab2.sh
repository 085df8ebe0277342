# longer same-box A/B: the working tree's build vs ab/*.so, 200 timed steps per round, 6 rounds;
# then the bench line of each (LAMPS_LIB)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/ab2
for rnd in 1 2 3 4 5 6; do
  echo "== current"; STEPS=200 TUNES=0 ROUNDS=1 python scripts/ab_tune.py
  for so in "$@"; do echo "== $so"; LAMPS_LIB=$so STEPS=200 TUNES=0 ROUNDS=1 python scripts/ab_tune.py; done
done > gpurun_out/ab2/ab.txt 2>&1
python - <<'PY'
import re
cur=None; res={}
for line in open("gpurun_out/ab2/ab.txt"):
    if line.startswith("=="): cur=line[3:].strip()
    m=re.search(r"median ([0-9.]+)", line)
    if m: res.setdefault(cur,[]).append(float(m.group(1)))
for k,v in res.items(): print(k, sorted(v), "median", sorted(v)[len(v)//2])
PY
for so in "" ${NOBENCH:+} $([ -z "$NOBENCH" ] && echo "$@"); do
  LAMPS_LIB=$so timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', '${so:-current}', round(d['us_per_step'],2), d['step_us'], d['clocks'])"
done
