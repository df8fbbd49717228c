# REMAP: second slabs pre-issued (base) vs first slabs only (prev): tests, tile budget, K1 under ncu
timeout 900 python -m pytest tests/test_gpu_train.py -k "grid or fused_adam_bit or reanchored" -q -x > gpurun_out/p2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/p2_tests.log
R=2 bash tools/gpu/tile_ab.sh prev base
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in prev base prev base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw --csv $CMD > gpurun_out/p2_$v.csv 2>/dev/null
  python3 - gpurun_out/p2_$v.csv $v <<'P'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if "Metric Name" in r); h = rows[i0]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows[i0 + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
print(sys.argv[2], "K1 ms mean %.4f" % (sum(t) / len(t) / 1e6))
P
done
