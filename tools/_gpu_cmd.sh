for v in m6 m5; do
cp paper_1604_04689_b200/libmeshnbr_$v.so paper_1604_04689_b200/libmeshnbr.so; touch paper_1604_04689_b200/libmeshnbr.so
for a in "--config 5" "--config 3"; do
python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $a', round(l['ms_per_step'],3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:4]])"
done; done
