# compute-sanitizer over every step path (scripts/sanitize.py): the closed-loop modes on
# C3 and the 2^20-slot bench pool.  Reports under gpurun_out/sanitize/; each tool bounded
# by its own timeout.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  steps=6; [ $tool = racecheck ] && steps=3
  STEPS=$steps timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
     python scripts/sanitize.py > gpurun_out/sanitize/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  tail -3 gpurun_out/sanitize/$tool.txt
done
# negative controls: the tools must flag these
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sanitizer_control scripts/micro/sanitizer_control.cu
$CS --tool memcheck --error-exitcode 9 /tmp/sanitizer_control o > gpurun_out/sanitize/control_memcheck.txt 2>&1
echo "control memcheck rc=$? (expect 9)" | tee -a gpurun_out/sanitize/summary.txt
$CS --tool racecheck --error-exitcode 9 /tmp/sanitizer_control r > gpurun_out/sanitize/control_racecheck.txt 2>&1
echo "control racecheck rc=$? (expect 9)" | tee -a gpurun_out/sanitize/summary.txt
