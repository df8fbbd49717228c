python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_nonfinite.py -q -s > gpurun_out/nonfinite.log 2>&1; echo "nonfinite rc=$?"
tail -3 gpurun_out/nonfinite.log
timeout 1500 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_reservoir.py -k "1000" -q -s > gpurun_out/slow.log 2>&1; echo "slow rc=$?"
grep -E "R=|medium fp32|passed|failed|Error" gpurun_out/slow.log | tail -20
