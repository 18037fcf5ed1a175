mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -k "edge or nccl or real_kernels" > gpurun_out/pytest_dist_edge.log 2>&1; tail -25 gpurun_out/pytest_dist_edge.log
