bash tools/gpu_round.sh r1t
python bench.py --config 4 --elem-path transpose --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 transpose', l['ms_per_step'], [(e['name'], round(e['ms_per_step'],3)) for e in l['kernels']])"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_chunk_scatter_fixed|k_chunk_sort|k_node_gather_t|k_node_compact" -c 4 \
    -o gpurun_out/full_r1t python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_r1t.log 2>&1; tail -1 gpurun_out/ncu_full_r1t.log
