# round-2 re-entry: HEAD build on the box -- GPU tests, 20-step and 50-step bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/v_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/v_tests.log
timeout 300 python bench.py > gpurun_out/v_bench20.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/v_bench20.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v_bench50.log 2>&1; echo "bench50 rc=$?"; tail -c 1500 gpurun_out/v_bench50.log
