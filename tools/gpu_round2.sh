#!/bin/bash
# Round-2 measurement campaign (under gpurun): bench lines for every config, the memory-bounded mode,
# emulated 2-rank runs of both exchange modes, ncu launch lists (time + DRAM bytes per launch).
# Usage: bash tools/gpu_round2.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.log
python tools/dist_world1.py 5 > gpurun_out/dist_world1_${TAG}_cfg5.json 2>/dev/null
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.err
for c in 1 2 3 4 6; do
  python bench.py --config $c --cpu-seconds 6 > gpurun_out/bench_${TAG}_cfg$c.json 2>/dev/null
done
python bench.py --config 4 --outputs shared --cpu-seconds 5 --no-e2e > gpurun_out/bench_${TAG}_cfg4_shared.json 2>/dev/null
python bench.py --config 5 --outputs shared --cpu-seconds 5 --no-e2e > gpurun_out/bench_${TAG}_cfg5_shared.json 2>/dev/null
for gb in 2 6 12; do
  python bench.py --max-workspace-gb $gb --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bench_${TAG}_cfg5_chunked_${gb}gb.json 2>/dev/null
done
for ex in p2p a2a; do
  MN_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 1 --config 3 --exchange $ex --no-cpu-baseline \
    > gpurun_out/bench_${TAG}_n2_emulated_cfg3_$ex.json 2>/dev/null
done
for c in 5 4 6 1; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}_cfg$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e \
      --no-cpu-baseline --no-parity > /dev/null 2>&1
done
echo done
