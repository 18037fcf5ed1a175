# quick: GPU parity (parity file) + node_gather / step times on configs 5, 3, 4 and shared 4
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for a in "--config 5" "--config 3" "--config 4" "--config 4 --outputs shared"; do
 python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('$a'.ljust(28), ' '.join('%s %.3f' % (n, k[n]) for n in ('node_gather','elem_scatter','elem_segsort','elem_count','scan_counts') if n in k), 'step %.3f' % l['ms_per_step'])"
done
