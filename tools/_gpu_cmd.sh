python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in 0 1 2 3; do
for c in 5 3; do
MN_XV=$v python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('var $v cfg $c', ' '.join('%s %.3f' % (n, k[n]) for n in ('node_gather','node_giant') if n in k), 'step %.3f' % l['ms_per_step'])"
done; done
MN_XV=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "whole_path or full_size or fans" 2>&1 | tail -2
