mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MN_BENCH_STEPS=1 python bench.py 2>&1 >/dev/null | grep steps
MN_BENCH_STEPS=1 python bench.py --config 3 2>&1 >/dev/null | grep steps
MN_BENCH_STEPS=1 python bench.py --config 1 2>&1 >/dev/null | grep steps
