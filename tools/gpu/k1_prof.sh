# K1 per-role wait counters + CTA-0 tile timeline, overlapped vs staged variant
python -c "import __graft_entry__ as g; g.build()"
free -g | head -2; nproc
timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/prof_ov.log 2>&1; echo "ov rc=$?"
MEL_K1_STAGED=1 timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/prof_staged.log 2>&1; echo "staged rc=$?"
head -c 1500 gpurun_out/prof_ov.log; echo; head -c 1200 gpurun_out/prof_staged.log
