mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_poly.py -q -m gpu -x 2>&1 | tail -2
for a in "--config 2" "--config 1" "--config 6 --outputs shared"; do
 python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('$a'.ljust(34), ' '.join('%s %.3f' % (n, v) for n, v in k.items() if v > 0.005), 'step %.3f' % l['ms_per_step'])"
done
