# what the driver runs at round end, on the final build
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 3000 python -m pytest tests/ -x -q -m gpu > gpurun_out/d_tests.log 2>&1; echo "pytest -m gpu rc=$?"; tail -2 gpurun_out/d_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/d_smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/d_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/d_bench.log | tail -1 | cut -c1-600
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/d_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/d_ref.log | tail -1 | cut -c1-400
