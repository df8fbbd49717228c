# build, GPU tests (not slow), bench, launch list of the timed region
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c_tests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c_bench.log 2>&1; echo "bench rc=$?"
python3 - <<'P'
import json
l=[x for x in open("gpurun_out/c_bench.log") if x.startswith("{")][-1]; d=json.loads(l)
print(d["value"], d["ms_per_step"], d["gpu_launches"], d["roofline"]["frac"], {k:round(v["ms_per_step"]*1e3,1) for k,v in d["kernels"].items()}, d["clocks"]["sm_mhz"], d["e2e"]["value"])
P
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv $CMD > gpurun_out/c_launches.csv 2>/dev/null; echo "ncu launches rc=$?"
python tools/ncu_launches.py gpurun_out/c_launches.csv 5
