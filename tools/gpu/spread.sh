python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/vr_seed_spread.py 1 bf16 1 2 3 4 2>&1 | tail -4
WL=n=100,sims=1100,C=6000,theta=1000,B=64,k=100 timeout 1200 python tools/vr_seed_spread.py 4 bf16 1 2 3 4 2>&1 | tail -4
WL=n=100,sims=1100,C=6000,theta=1000,B=256,k=100 timeout 600 python tools/vr_seed_spread.py 1 bf16 1 2 2>&1 | tail -4
