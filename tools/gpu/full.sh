python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rs > gpurun_out/full.log 2>&1; echo "full rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/full.log | tail -8
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.log 2>&1; echo "bench rc=$?"
python - <<'P'
import json
l=[x for x in open("gpurun_out/bench_r2b.log") if x.startswith("{")][-1]
d=json.loads(l)
print("value", d["value"], "ms", d["ms_per_step"], "K1", d["kernels"]["out_fwd_dw"]["ms_per_step"], "frac", d["roofline"]["frac"], "traffic", d["roofline"]["traffic"])
print("windows", d["windows_samples_per_s"]); print("cpu", d["cpu_baseline"]); print("e2e", d["e2e"]["value"]); print("b10", d["paper_batch_b10"]); print("clocks", d["clocks"])
P
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.log
