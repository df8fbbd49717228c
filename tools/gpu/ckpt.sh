python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_checkpoint.py -q -x > gpurun_out/ckpt.log 2>&1; echo "ckpt rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/ckpt.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
