mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests -q -m gpu -x -k "chunk" 2>&1 | tail -2
for w in 2 6 12; do
 python bench.py --config 5 --max-workspace-gb $w --no-cpu-baseline --steps 5 2>/dev/null > gpurun_out/bench_chunked_$w.json
 python -c "
import json,sys; l=json.loads(open('gpurun_out/bench_chunked_$w.json').read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('ws $w GB ranges', l['config'].get('node_ranges'), 'G tets/s %.3f' % (l['value']/1e9), 'ms/step %.3f' % l['ms_per_step'], ' '.join('%s %.3f' % (n, v) for n, v in k.items() if v > 0.05))"
done
for a in "--config 5" "--config 6"; do
 python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={e['name']:e['ms_per_step'] for e in l['kernels']}
print('$a'.ljust(12), ' '.join('%s %.3f' % (n, v) for n, v in k.items() if v > 0.05), 'step %.3f' % l['ms_per_step'])"
done
timeout 900 python -m pytest tests/test_gpu_poly.py tests/test_gpu_dist.py -q -m gpu -x 2>&1 | tail -1
