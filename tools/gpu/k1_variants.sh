# K1 variant builds (MEL_LIB=libmel_<v>.so): per-role wait counters + step time
for v in "$@"; do
  if [ "$v" = base ]; then lib=libmel.so; else lib=libmel_$v.so; fi
  MEL_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/var_$v.log 2>&1
  echo "== $v rc=$?"
  python - "$v" <<'P'
import json,sys
v=sys.argv[1]
l=[x for x in open("gpurun_out/var_%s.log"%v) if x.startswith("{")][0]
d=json.loads(l); k=d["k1_wait_cycles_mean_per_cta"]
print("%s ms/step %.4f | %s" % (v, d["ms_per_step"], " ".join("%s=%.0fk"%(a,b/1e3) for a,b in k.items() if b)))
P
done
