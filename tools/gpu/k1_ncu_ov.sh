# one steady-state K1 launch (inside the timed NVTX range) under ncu --set full
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
export MEL_K1_ADAM_FRAC=${FRAC:-0.4}
$CMD > gpurun_out/ncu_ov_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw -c 1 -o gpurun_out/r2_k1_ov $CMD > gpurun_out/ncu_ov.log 2>&1; echo "ncu rc=$?"
grep -o '"out_fwd_dw": {"ms_per_step": [0-9.]*' gpurun_out/ncu_ov_plain.log
