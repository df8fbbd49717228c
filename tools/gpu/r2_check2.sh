python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/c2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c2_tests.log
timeout 300 python bench.py > gpurun_out/c2_bench.log 2>&1; echo "bench rc=$?"
python3 -c "
import json; l=[x for x in open('gpurun_out/c2_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']), d['ms_per_step'], d['gpu_launches'], round(d['roofline']['frac'],3), d['e2e']['value'], d['paper_batch_b10']['samples_per_s'], d['paper_batch_b10']['ms_per_step'], d['clocks'])"
