mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_property.py -q -m gpu > gpurun_out/pytest_property_r2k.log 2>&1; tail -3 gpurun_out/pytest_property_r2k.log
