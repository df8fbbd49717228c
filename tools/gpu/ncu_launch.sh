# per-kernel durations (ncu launch list, timed region) for variant builds: bash ncu_launch.sh base v1 ...
for v in "$@"; do
  if [ "$v" = base ]; then lib=libmel.so; else lib=libmel_$v.so; fi
  MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch > gpurun_out/nl_$v.csv 2>/dev/null
  echo "== $v"; python3 tools/ncu_launches.py gpurun_out/nl_$v.csv 3 2>/dev/null | head -20
done
