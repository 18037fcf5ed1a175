mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/ab_gather.py 0,4 5,3 2>&1 | tail -4
