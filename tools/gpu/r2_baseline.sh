set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench0.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench0.log
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw -c 1 -o gpurun_out/r2_k1_base $CMD > gpurun_out/r2_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2_ncu.log
