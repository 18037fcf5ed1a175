mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r2l.log 2>&1; tail -3 gpurun_out/pytest_gpu_r2l.log
MN_BENCH_STEPS=1 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], {e['name']: round(e['ms_per_step'],3) for e in l['kernels'][:6]})"
