python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_virtual.py -k "independent_of_grid" -q > gpurun_out/vcanary.log 2>&1; echo "vcanary rc=$?"; tail -3 gpurun_out/vcanary.log
grep -E "Error|assert" gpurun_out/vcanary.log | head -5
