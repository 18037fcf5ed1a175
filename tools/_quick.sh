# quick: node parity subset + node_gather times on configs 5/4/3 and shared 4
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "node or shared or whole or fan" 2>&1 | tail -2
for c in 5 4 3; do
 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 ${EXTRA} 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('cfg $c node_gather %.3f step %.3f' % (k['node_gather'], l['ms_per_step']))"
done
python bench.py --config 4 --outputs shared --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('shared cfg 4 node_gather %.3f step %.3f' % (k['node_gather'], l['ms_per_step']))"
