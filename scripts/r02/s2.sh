# parity (fast GPU tests) of the working tree, then same-box A/B vs ab/*.so, then a phase trace
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s2/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/s2/tests.txt 2>&1
tail -3 gpurun_out/s2/tests.txt
bash scripts/r02/ab.sh "$@" > gpurun_out/s2/ab.txt 2>&1
cat gpurun_out/s2/ab.txt | grep tune
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/s2/trace.txt 2>&1
head -16 gpurun_out/s2/trace.txt
