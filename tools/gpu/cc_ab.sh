# commit_copy entry grouping A/B (MEL_CC_GROUP 1 / 2 / 4): ncu launch list of the timed region per build
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in g1 g2 base g1 g2 base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:"commit" --csv $CMD > gpurun_out/cc_$v.csv 2>/dev/null
  echo "== $v"; python tools/ncu_launches.py gpurun_out/cc_$v.csv 5 | grep commit
done
