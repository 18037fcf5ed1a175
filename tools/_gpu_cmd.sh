mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "small_path or auto" > gpurun_out/pytest_small_r2f.log 2>&1; tail -3 gpurun_out/pytest_small_r2f.log
for c in 1 2 3; do python bench.py --config $c --no-e2e --cpu-seconds 3 --steps 20 > gpurun_out/bench_r2f_cfg$c.json 2>gpurun_out/bench_r2f_cfg$c.err; python -c "
import json; l=json.loads(open('gpurun_out/bench_r2f_cfg$c.json').read().strip().splitlines()[-1]); print($c, round(l['ms_per_step'],4), {k: v for k, v in l.get('latency', {}).items() if k != 'what'}, l['parity']['ok'])"; done
