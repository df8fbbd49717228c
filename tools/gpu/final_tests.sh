python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/ft_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ft_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/ft_bench.log 2>&1; echo "bench rc=$?"
python3 -c "
import json; l=[x for x in open('gpurun_out/ft_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']), d['ms_per_step'], d['gpu_launches'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], round(d['kernels']['commit']['ms_per_step']*1e3,1))"
timeout 300 python tools/microbench.py 2>&1 | grep commit
