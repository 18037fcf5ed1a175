python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_poly.py -q -m gpu -x 2>&1 | tail -1
for a in "--config 5 --outputs shared" "--config 5"; do
python bench.py $a --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', round(l['ms_per_step'],3), [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels'][:4]])"
done
python - <<'PY'
import torch, time, meshgen, paper_1604_04689_b200 as mn
conn, N = meshgen.kuhn_tets(320, device="cuda")
for f in (mn.find_node_neighbors, mn.find_elem_neighbors):
    f(conn, "tet4", N); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): f(conn, "tet4", N)
    torch.cuda.synchronize(); print(f.__name__, round((time.perf_counter() - t) / 5 * 1e3, 3), "ms (wall, config 5)")
PY
