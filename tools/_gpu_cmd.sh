mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/ab_knobs.py gather_ws 0,1 5,3,4 2>&1 | tail -8
