mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "workspace or chunked" --durations=8 > gpurun_out/pytest_mem_r2c.log 2>&1; tail -15 gpurun_out/pytest_mem_r2c.log
python bench.py --max-workspace-gb 2 --no-e2e --cpu-seconds 4 --steps 5 > gpurun_out/bench_r2c_cfg5_chunked_2gb.json 2>/dev/null; cut -c1-300 gpurun_out/bench_r2c_cfg5_chunked_2gb.json
