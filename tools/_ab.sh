python tools/dist_world1.py 5 2>/dev/null | tail -1 | cut -c1-700; timeout 1500 python -m pytest tests/test_gpu_dist.py -q -m gpu -x 2>&1 | tail -2
