python -c "import __graft_entry__ as g; g.build()" > /dev/null
TRACE=1 STEPS=3 python scripts/prof_step.py
