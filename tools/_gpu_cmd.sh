mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "transpose or auto or capacity or full_size" > gpurun_out/pytest_pack.log 2>&1; tail -3 gpurun_out/pytest_pack.log
python tools/ab_knobs.py small_path 8192 5,3 2>&1 | tail -2
