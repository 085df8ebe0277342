# fast GPU tests, long same-box A/B vs ab/*.so (scripts/r02/ab2.sh), phase trace of the working tree
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s5
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/s5/tests.txt 2>&1
tail -2 gpurun_out/s5/tests.txt
grep -m2 -A12 "Error" gpurun_out/s5/tests.txt
bash scripts/r02/ab2.sh "$@"
ADMIT=1 TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/s5/trace.txt 2>&1
head -16 gpurun_out/s5/trace.txt; grep "store\.\|binned\|substeps" gpurun_out/s5/trace.txt
