# scratch command for one gpurun call (edited per experiment)
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket|NUMA node\(s\)"; nvidia-smi -L) > gpurun_out/host_info.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
bash tools/_quick.sh 2>&1 | tail -6
