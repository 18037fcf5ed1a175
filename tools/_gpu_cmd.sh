mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_property.py -q -m gpu > gpurun_out/pytest_property_r2k.log 2>&1; tail -3 gpurun_out/pytest_property_r2k.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_r2k.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/sanitizer_racecheck_r2k.txt
