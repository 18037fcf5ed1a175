bash tools/gpu_round.sh r1v
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_chunk_scatter_fixed|k_chunk_sort|k_node_gather_t|k_node_compact" -c 4 \
    -o gpurun_out/full_r1v python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_r1v.log 2>&1; tail -1 gpurun_out/ncu_full_r1v.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_poly_gather|k_poly_chunk_scatter|k_chunk_sort" -c 3 \
    -o gpurun_out/full_r1v_cfg6 python bench.py --config 6 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_r1v_cfg6.log 2>&1; tail -1 gpurun_out/ncu_full_r1v_cfg6.log
