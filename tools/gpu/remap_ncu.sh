# K1 duration A/B under ncu (timed region, 5 steps, clock-control none): target-ring fix alone vs + REMAP
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in fixonly base fixonly base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw --csv $CMD > gpurun_out/rn_$v.csv 2>/dev/null
  python3 - gpurun_out/rn_$v.csv $v <<'P'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; mi = h.index("Metric Name"); vi = h.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
print(sys.argv[2], "K1 us per launch:", [round(x / 1e3, 1) for x in t] if max(t) > 1e5 else t)
P
done
