# parity (fast GPU tests); on failure a memcheck of the strong-scaling bench; A/B vs ab/*.so; trace
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3/smoke.txt 2>&1
tail -1 gpurun_out/s3/smoke.txt
timeout 900 python -m pytest tests -m gpu -q -k "not slow" > gpurun_out/s3/tests.txt 2>&1
tail -3 gpurun_out/s3/tests.txt
if grep -q "failed" gpurun_out/s3/tests.txt; then
  true
  grep -m3 -B2 -A12 "Error" gpurun_out/s3/tests.txt
fi
bash scripts/r02/ab.sh "$@" > gpurun_out/s3/ab.txt 2>&1
grep tune gpurun_out/s3/ab.txt
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/s3/trace.txt 2>&1
head -16 gpurun_out/s3/trace.txt
