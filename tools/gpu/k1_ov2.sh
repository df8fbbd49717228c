# overlapped K1 (MMA CTAs + Adam CTAs): parity, then the Adam-CTA share sweep
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_train.py -q -x > gpurun_out/ov2_test.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/ov2_test.log
for f in 0.25 0.35 0.45; do
  MEL_K1_ADAM_FRAC=$f timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/ov2_$f.log 2>&1
  echo "== frac $f rc=$?"
  python - $f <<'P'
import json,sys
v=sys.argv[1]
l=[x for x in open("gpurun_out/ov2_%s.log"%v) if x.startswith("{")][0]
d=json.loads(l); k=d["k1_wait_cycles_mean_per_cta"]
print("%s ms/step %.4f | %s" % (v, d["ms_per_step"], " ".join("%s=%.0fk"%(a,b/1e3) for a,b in k.items() if b)))
P
done
