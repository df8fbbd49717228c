python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_virtual.py -k "1000" -q -s > gpurun_out/slow.log 2>&1; echo "slow rc=$?"
grep -E "R=|passed|failed|Error" gpurun_out/slow.log | tail -8
WL=n=100,sims=1100,C=6000,theta=1000,B=64,k=100 timeout 1200 python tools/vr_seed_spread.py 8 bf16 2 3 2>&1 | tail -2
