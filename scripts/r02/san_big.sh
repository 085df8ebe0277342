mkdir -p gpurun_out/sanitize3
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  STEPS=4 timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 30 python scripts/sanitize.py big big_fallback > gpurun_out/sanitize3/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize3/summary.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sanitize3/gputest.txt 2>&1
