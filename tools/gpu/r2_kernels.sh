# final per-kernel ncu evidence: K2 (tensor), commit_copy (HBM), the separate Adam over all 257M params (HBM, --flags 8)
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --nvtx --nvtx-include "timed/" -k regex:"out_dh|commit_copy" -c 2 -o gpurun_out/k_a $CMD > /dev/null 2>&1; echo "ncu a rc=$?"
$CMD --flags 8 > /dev/null 2>&1 && ncu --set full --clock-control none --nvtx --nvtx-include "timed/" -k regex:"adam_kernel" -c 1 -o gpurun_out/k_b $CMD --flags 8 > /dev/null 2>&1; echo "ncu b rc=$?"
for f in k_a k_b; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/${f}_raw.csv
  python3 - gpurun_out/${f}_raw.csv <<'P'
import csv, sys
r = list(csv.reader(open(sys.argv[1]))); h = r[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__cycles_active.avg.pct_of_peak_sustained_elapsed', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__registers_per_thread']
for row in r[2:]:
    d = dict(zip(h, row))
    print(d.get('Kernel Name', '')[:40], {k.split('.')[0].replace('__', '.') + ('' if k.endswith('.sum') or k.startswith('launch') else '%'): d.get(k) for k in keys})
P
  rm -f gpurun_out/$f.ncu-rep
done
