python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for a in "--config 5" "--config 3" "--config 6"; do
python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c7 $a', round(l['ms_per_step'],3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:4]])"
done
cp paper_1604_04689_b200/libmeshnbr.so /tmp/c7.so; cp paper_1604_04689_b200/libmeshnbr_c8.so paper_1604_04689_b200/libmeshnbr.so; touch paper_1604_04689_b200/libmeshnbr.so
for a in "--config 5" "--config 3" "--config 6"; do
python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c8 $a', round(l['ms_per_step'],3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:4]])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "transpose" 2>&1 | tail -1
