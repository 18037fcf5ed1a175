# quick: node/elem parity subset + kernel times on configs 5/4/3 (EXTRA env passes through)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for v in ""; do
for c in 5 3; do
 env $v python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('$v cfg $c', ' '.join('%s %.3f' % (n, k[n]) for n in ('node_gather','elem_scatter','elem_segsort','elem_count') if n in k), 'step %.3f' % l['ms_per_step'])"
done; done
