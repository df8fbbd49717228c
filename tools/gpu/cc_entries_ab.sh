# commit_copy: 1 / 2 / 4 entries in flight (2D grid) -- ncu at the bench's 4 puts, microbench at 128-put bursts
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in base ce2 ce4 base ce2 ce4; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:"commit_copy" --csv $CMD > gpurun_out/ce_$v.csv 2>/dev/null
  echo -n "$v "; python tools/ncu_launches.py gpurun_out/ce_$v.csv 5 | grep commit_copy
done
for v in base ce2 ce4; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  echo -n "$v "; MEL_LIB=$lib timeout 300 python tools/microbench.py 2>&1 | grep commit
done
timeout 900 python -m pytest tests/test_gpu_reservoir.py tests/test_gpu_buffers.py tests/test_gpu_nonfinite.py -q -m "gpu and not slow" > gpurun_out/ce_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ce_tests.log
