set -x
python -c "import __graft_entry__ as g; g.build()"
STEPS=4 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_step.py
ncu --set full --clock-control none --import-source on -k regex:k_sort -s 1 -c 1 -o gpurun_out/prof_sort -f python scripts/prof_step.py
ncu --set full --clock-control none --import-source on -k regex:k_score -s 1 -c 1 -o gpurun_out/prof_score -f python scripts/prof_step.py
ncu --set full --clock-control none --import-source on -k regex:k_admit -s 1 -c 1 -o gpurun_out/prof_admit -f python scripts/prof_step.py
