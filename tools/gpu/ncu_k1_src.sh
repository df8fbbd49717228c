# K1 steady-state launch under ncu --set full with source correlation; per-source-line stall summary
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw -c 1 -o gpurun_out/k1src $CMD > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/k1src.ncu-rep --page source --csv --print-source cuda 2>/dev/null > gpurun_out/k1src_cuda.csv
ncu -i gpurun_out/k1src.ncu-rep --page source --csv 2>/dev/null > gpurun_out/k1src_sass.csv
ls -la gpurun_out/k1src*
rm -f gpurun_out/k1src.ncu-rep
