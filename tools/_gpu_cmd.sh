mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/pytest_dist3.log 2>&1; tail -20 gpurun_out/pytest_dist3.log
python tools/dist_world1.py 5 > gpurun_out/dist_world1_cfg5.json 2> gpurun_out/dw1.err; tail -2 gpurun_out/dw1.err; cat gpurun_out/dist_world1_cfg5.json
