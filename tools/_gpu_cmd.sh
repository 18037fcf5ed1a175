# scratch command for one gpurun call (edited per experiment); default: build, GPU parity, quick bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
bash tools/_quick.sh 2>&1 | tail -4
