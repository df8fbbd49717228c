# H5 (W in TMEM, 5-slot H ring over the W tile's SMEM) vs wt (W in TMEM, 3 slots) vs base: tests, tile budget, K1 ncu
MEL_LIB=libmel_h5.so timeout 900 python -m pytest tests/test_gpu_train.py -k "grid or fused_adam_bit or reanchored" -q -x > gpurun_out/h5_tests.log 2>&1; echo "h5 tests rc=$?"; tail -2 gpurun_out/h5_tests.log
grep -E "Error|assert" gpurun_out/h5_tests.log | head -3
R=1 bash tools/gpu/tile_ab.sh base h5 wt
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in base h5 wt base h5; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw --csv $CMD > gpurun_out/h5_$v.csv 2>/dev/null
  python3 - gpurun_out/h5_$v.csv $v <<'P'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if "Metric Name" in r); h = rows[i0]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows[i0 + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
print(sys.argv[2], "K1 ms mean %.4f" % (sum(t) / len(t) / 1e6))
P
done
