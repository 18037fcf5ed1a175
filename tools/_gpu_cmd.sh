python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_poly.py tests/test_gpu_dist.py -q -m gpu -x 2>&1 | tail -1
bash tools/_quick.sh 2>&1 | tail -4
