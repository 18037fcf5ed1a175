mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fixed or whole_path_both or full_size" 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench_t1.json 2>/dev/null; python -c "
import json; l=json.loads(open('gpurun_out/bench_t1.json').read().strip().splitlines()[-1]); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel'], l['roofline']['frac']); [print(k['name'], round(k['ms_per_step'],3)) for k in l['kernels']]"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_t1.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_chunk_scatter_fixed|k_chunk_sort|k_node_gather_t" -c 3 \
    -o gpurun_out/full_t1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_t1.log 2>&1; tail -2 gpurun_out/ncu_full_t1.log
