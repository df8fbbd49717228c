# A/B over variant builds (MEL_LIB=libmel_<v>.so; "base" = libmel.so), R interleaved rounds
# usage: R=2 bash tools/gpu/ab_multi.sh base v1 env:VAR=value ...
P='import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]); k=d["kernels"]; print("%.4f ms/step  K1 %.4f  K2 %.4f  head %.4f  other %.4f  %.0f samples/s" % (d["ms_per_step"], k["out_fwd_dw"]["ms_per_step"], k["out_dh"]["ms_per_step"], k["head_fwd"]["ms_per_step"]+k["head_bwd"]["ms_per_step"], d["ms_per_step"]-k["out_fwd_dw"]["ms_per_step"]-k["out_dh"]["ms_per_step"]-k["head_fwd"]["ms_per_step"]-k["head_bwd"]["ms_per_step"], d["value"]))'
for r in $(seq ${R:-2}); do
for v in "$@"; do
  envs=""; lib=libmel.so
  case "$v" in base) ;; env:*) envs="${v#env:}" ;; *) lib=libmel_$v.so ;; esac
  echo -n "$r $v: "; env $envs MEL_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-paper-batch ${BENCH_ARGS} 2>&1 | python -c "$P"
done; done
