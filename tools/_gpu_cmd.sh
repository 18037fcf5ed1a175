python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in 5 3; do
python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$c', round(l['ms_per_step'],3), round(l['value']/1e9,3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:5]])"
done
