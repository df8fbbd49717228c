python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/head.log 2>&1; echo "full rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/head.log | tail -3
P='import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]); k=d["kernels"]; print("%.4f ms/step  K1 %.4f  K2 %.4f hf %.4f hb %.4f loss %.4f adam %.4f commit %.4f %.0f samples/s launches %d" % (d["ms_per_step"], k["out_fwd_dw"]["ms_per_step"], k["out_dh"]["ms_per_step"], k["head_fwd"]["ms_per_step"], k["head_bwd"]["ms_per_step"], k["loss"]["ms_per_step"], k["adam"]["ms_per_step"], k["commit"]["ms_per_step"], d["value"], d["gpu_launches"]))'
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-paper-batch 2>&1 | python -c "$P"; done
