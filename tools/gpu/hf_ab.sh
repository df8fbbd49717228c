# head forward 256 vs 512 threads per CTA: ncu launch list of the timed region (interleaved), then the train tests
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
for v in hf256 base hf256 base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib $CMD > /dev/null 2>&1 && MEL_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k regex:"head_" --csv $CMD > gpurun_out/hf_$v.csv 2>/dev/null
  echo "== $v"; python tools/ncu_launches.py gpurun_out/hf_$v.csv 5 | grep head
done
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_reservoir.py -m "gpu and not slow" -q > gpurun_out/hf_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/hf_tests.log
