# K1 experiment builds (MEL_LIB=libmel_<v>.so, built with MEL_NVCC_DEFS): K1 / step time and per-role waits
P='import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]); k=d["kernels"]; print("%.4f ms/step  K1 %.4f  K2 %.4f  head %.4f %.0f samples/s" % (d["ms_per_step"], k["out_fwd_dw"]["ms_per_step"], k["out_dh"]["ms_per_step"], k["head_fwd"]["ms_per_step"]+k["head_bwd"]["ms_per_step"], d["value"]))'
for v in "$@"; do
  if [ "$v" = base ]; then lib=libmel.so; else lib=libmel_$v.so; fi
  echo -n "== $v: "; MEL_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-paper-batch 2>&1 | python -c "$P"
  MEL_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/exp_$v.log 2>&1
  python - "$v" <<'P'
import json,sys
v=sys.argv[1]
l=[x for x in open("gpurun_out/exp_%s.log"%v) if x.startswith("{")][0]
d=json.loads(l); k=d["k1_wait_cycles_mean_per_cta"]
print("   %s prof ms/step %.4f | %s" % (v, d["ms_per_step"], " ".join("%s=%.0fk"%(a,b/1e3) for a,b in k.items() if b)))
P
  grep -E "^tile  [5-8]|^chunk  [0-4]" gpurun_out/exp_$v.log
done
