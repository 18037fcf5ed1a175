python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in 512 148 96 64 40; do
MN_XV=$v python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('grid $v', round(l['ms_per_step'],3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:3]])"
done
MN_XV=64 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "msd" 2>&1 | tail -2
