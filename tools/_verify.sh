# verify HEAD: smoke, all GPU tests, default bench, launch list of config 5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_v.log 2>&1; tail -1 gpurun_out/smoke_v.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu_v.log 2>&1; tail -3 gpurun_out/pytest_gpu_v.log
python bench.py > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err; tail -1 gpurun_out/bench_v.err; cut -c1-600 gpurun_out/bench_v.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_v_cfg5.csv python bench.py --config 5 --steps 1 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-parity > /dev/null 2>&1
echo done
