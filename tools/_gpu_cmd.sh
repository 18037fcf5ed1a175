mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -k "nccl or real_kernels" > gpurun_out/pytest_p2p_r2h.log 2>&1; tail -30 gpurun_out/pytest_p2p_r2h.log
