mkdir -p gpurun_out/sanitize2
CS=/usr/local/cuda/bin/compute-sanitizer
STEPS=3 timeout 1500 $CS --tool racecheck --error-exitcode 9 --print-limit 50 python scripts/sanitize.py > gpurun_out/sanitize2/racecheck.txt 2>&1
echo "racecheck rc=$?" > gpurun_out/sanitize2/summary.txt
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/sanitize2/gputest.txt 2>&1
