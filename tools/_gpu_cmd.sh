python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
for a in "--config 5" "--config 3" "--config 5 --outputs shared"; do
python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', round(l['ms_per_step'],3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:4]])"
done
