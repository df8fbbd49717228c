# commit + sample control CTA: 1024 / 512 / 256 threads -- ncu launch times at the bench's 4 puts; reservoir tests per build
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in base t512 t256 base t512 t256; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:"commit_sample" --csv $CMD > gpurun_out/ct_$v.csv 2>/dev/null
  echo -n "$v "; python tools/ncu_launches.py gpurun_out/ct_$v.csv 5 | grep commit_sample
done
for v in t512 t256; do
  MEL_LIB=libmel_$v.so timeout 900 python -m pytest tests/test_gpu_reservoir.py tests/test_gpu_buffers.py tests/test_gpu_virtual.py -q -m "gpu and not slow" > gpurun_out/ct_tests_$v.log 2>&1; echo "$v tests rc=$?"; tail -1 gpurun_out/ct_tests_$v.log
done
