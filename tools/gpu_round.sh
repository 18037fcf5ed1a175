#!/bin/bash
# One GPU session: tests, smoke, bench (JSON line), ncu launch list of the bench command, and the
# secondary workloads (config 4 hex, config 6 polygons, element-sharing adjacency).
# Usage (under gpurun): bash tools/gpu_round.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.err
python bench.py --config 6 --cpu-seconds 5 > gpurun_out/bench_${TAG}_cfg6.json 2>/dev/null
python bench.py --config 4 --cpu-seconds 5 > gpurun_out/bench_${TAG}_cfg4.json 2>/dev/null
python bench.py --config 4 --outputs shared --cpu-seconds 5 > gpurun_out/bench_${TAG}_cfg4_shared.json 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_cfg6.csv python bench.py --config 6 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
