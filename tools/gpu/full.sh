python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -rs > gpurun_out/full.log 2>&1; echo "full rc=$?"
tail -5 gpurun_out/full.log
timeout 900 python tools/vr_seed_spread.py 4 bf16 1 2 3 4 2>&1 | tail -4
timeout 900 python tools/vr_seed_spread.py 4 bf16-fp32x 1 2 3 4 2>&1 | tail -4
