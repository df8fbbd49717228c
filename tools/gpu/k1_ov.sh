# K1 overlapped-Adam variant: parity + A/B bench against the staged variant
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_fullsize.py -q -x > gpurun_out/ov_test.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/ov_test.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ov_bench.log 2>&1; echo "bench rc=$?"
python - <<'P'
import json
for f in ["gpurun_out/ov_bench.log"]:
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["ms_per_step"], {k:round(v["ms_per_step"],4) for k,v in d["kernels"].items()}, d["roofline"]["frac"], d.get("clocks"))
P
MEL_K1_STAGED=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ov_bench_staged.log 2>&1; echo "bench staged rc=$?"
grep -o '"out_fwd_dw": {"ms_per_step": [0-9.]*' gpurun_out/ov_bench_staged.log
