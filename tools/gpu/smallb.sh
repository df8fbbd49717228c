# fused vs separate Adam of W_L at small batches (the policy threshold)
for b in 10 64 128 192 256; do
  for f in 100000 1; do
    MEL_FUSED_MIN_B=$f timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-paper-batch > gpurun_out/sb_${b}_$f.log 2>&1
    python3 -c "
import json; l=[x for x in open('gpurun_out/sb_${b}_$f.log') if x.startswith('{')][-1]; d=json.loads(l)
print('B=$b', 'fused' if $f == 1 else 'unfused', round(d['value']), round(d['ms_per_step'],4), 'K1', round(d['kernels']['out_fwd_dw']['ms_per_step'],4), 'adam', round(d['kernels']['adam']['ms_per_step'],4))"
  done
done
