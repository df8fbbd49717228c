P='import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]); print("%.4f ms/step  K1 %.4f  K2 %.4f adam %.4f %.0f samples/s" % (d["ms_per_step"], d["kernels"]["out_fwd_dw"]["ms_per_step"], d["kernels"]["out_dh"]["ms_per_step"], d["kernels"]["adam"]["ms_per_step"], d["value"]))'
for i in 1 2 3; do for lib in libmel.so libmel_ng.so; do
  echo -n "$lib: "; MEL_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-paper-batch 2>&1 | python -c "$P"
done; done
for B in 128 192; do for fl in 0 8; do
  echo -n "B=$B flags $fl: "; timeout 300 python bench.py --steps 20 --warmup 3 --batch $B --flags $fl --no-cpu-baseline --no-e2e --no-paper-batch 2>&1 | python -c "$P"
done; done
