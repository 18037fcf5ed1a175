bash tools/gpu_round.sh r1w
python bench.py --outputs shared --no-cpu-baseline --no-e2e > gpurun_out/bench_r1w_cfg5_shared.json 2>/dev/null
