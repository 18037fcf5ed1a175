# scratch command for one gpurun call (edited per experiment)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu_r2a.log 2>&1; tail -22 gpurun_out/pytest_gpu_r2a.log
python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -3 gpurun_out/bench_r2a.err; cut -c1-600 gpurun_out/bench_r2a.json
