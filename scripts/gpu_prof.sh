set -x
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o gpurun_out/prof_fused -f python scripts/prof_step.py
