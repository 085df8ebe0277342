# tune-knob A/B in one binary (LAMPS_TUNE values), 6 rounds x 200 steps; fast tests with the knob on
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
LAMPS_TUNE=16 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_binned_gpu.py -m gpu -x -q -k "not slow" 2>&1 | tail -2
STEPS=200 TUNES=0,16 ROUNDS=6 python scripts/ab_tune.py
