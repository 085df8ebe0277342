mkdir -p gpurun_out/r02
TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/r02/trace_${TAG:-t}.txt 2>&1
NOFLUSH=1 TRACE=1 PERCTA=1 STEPS=3 timeout 300 python scripts/prof_step.py > gpurun_out/r02/trace_${TAG:-t}_noflush.txt 2>&1
