python -c "import __graft_entry__ as g; g.build()"
nvidia-smi -L
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_validation.py -q -x -rs > gpurun_out/mgpu.log 2>&1; echo "mgpu rc=$?"
grep -E "passed|failed|FAILED|SKIPPED" gpurun_out/mgpu.log | tail -5
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
python - $N <<'P'
import json,sys
l=[x for x in open("gpurun_out/bench_n%s.log"%sys.argv[1]) if x.startswith("{")][-1]
d=json.loads(l); print("N", d["n_gpus"], "value", d["value"], "ms", d["ms_per_step"], "K1", d["kernels"]["out_fwd_dw"]["ms_per_step"], "e2e", (d.get("e2e") or {}).get("value"), d["clocks"])
P
