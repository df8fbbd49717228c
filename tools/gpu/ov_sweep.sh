# overlapped K1: bit-identity tests, then the Adam-CTA share sweep (K1 time + per-role waits)
timeout 600 python -m pytest tests/test_gpu_train.py -q -x -k "bit_identical" 2>&1 | tail -2
for f in ${FRACS:-0.35 0.4 0.45 0.5}; do
  echo -n "frac $f: "; MEL_K1_OVERLAP=1 MEL_K1_ADAM_FRAC=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-paper-batch 2>&1 | grep -o "\"out_fwd_dw\": {\"ms_per_step\": [0-9.]*"
  MEL_K1_OVERLAP=1 MEL_K1_ADAM_FRAC=$f timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/ovs_$f.log 2>&1
  python - $f <<'P'
import json,sys
f=float(sys.argv[1])
l=[x for x in open("gpurun_out/ovs_%s.log"%sys.argv[1]) if x.startswith("{")][0]
d=json.loads(l); k=d["k1_wait_cycles_mean_per_cta"]
na=round(148*f); nm=148-na
mm=lambda key: k[key]*148/nm/1e3
aa=lambda key: k[key]*148/na/1e3
print("   ms %.4f | MMA CTAs(%d): total %.0fk dy_full %.0fk h_full %.0fk dw_readout %.0fk ring_wait %.0fk | Adam CTAs(%d): total %.0fk queue_wait %.0fk done_wait %.0fk" % (
  d["ms_per_step"], nm, mm("mma_total"), mm("mma_dy_full"), mm("mma_h_full"), mm("epi_dw_readout"), mm("epi_adam_load_wait"), na, aa("adam_total"), aa("adam_ring_wait"), aa("adam_loop")))
P
done
