python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -s > gpurun_out/virt.log 2>&1; echo "virt rc=$?"
grep -E "steps|passed|failed|Error|error" gpurun_out/virt.log | tail -30
