# (1) the 5-chunk grid canary on the build before the target-ring fix (expected to fail),
# (2) the fix alone (K1_REMAP=0), (3) the fix + REMAP staging: K1 GPU tests, then per-tile cycle budget A/B
for v in prefix fixonly base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib timeout 600 python -m pytest tests/test_gpu_train.py -k "grid or fused_adam_bit" -q -x > gpurun_out/ra_$v.log 2>&1; echo "$v tests rc=$?"; tail -2 gpurun_out/ra_$v.log
done
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/ra_all.log 2>&1; echo "all rc=$?"; tail -2 gpurun_out/ra_all.log
R=2 bash tools/gpu/tile_ab.sh fixonly base
for v in fixonly base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-paper-batch > gpurun_out/ra_b_$v.log 2>&1
  python3 -c "
import json; l=[x for x in open('gpurun_out/ra_b_$v.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$v', round(d['value']), round(d['ms_per_step'],4), 'K1', round(d['kernels']['out_fwd_dw']['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
