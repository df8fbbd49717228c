# K1 A/B under ncu: with / without the L2 prefetch of the next W tile (duration, DRAM bytes)
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in base nopf base nopf; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw --csv $CMD > gpurun_out/pf_$v.csv 2>/dev/null
  python3 - gpurun_out/pf_$v.csv $v <<'P'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if "Metric Name" in r); h = rows[i0]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[i0 + 1:]:
    if len(r) > vi: out.setdefault(r[mi], []).append(float(r[vi].replace(",", "")))
t = out["gpu__time_duration.sum"]; rd = out["dram__bytes_read.sum"]; wr = out["dram__bytes_write.sum"]
print(sys.argv[2], "K1 ms mean %.4f" % (sum(t) / len(t) / 1e6), "read GB %.3f" % (sum(rd) / len(rd) / 1e9), "write GB %.3f" % (sum(wr) / len(wr) / 1e9))
P
done
