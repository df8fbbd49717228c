python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_nonfinite.py tests/test_gpu_reservoir.py tests/test_gpu_buffers.py tests/test_gpu_checkpoint.py -q -x > gpurun_out/fs_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fs_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/fs_bench.log 2>&1; echo "bench rc=$?"
python3 -c "
import json; l=[x for x in open('gpurun_out/fs_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']), d['ms_per_step'], d['paper_batch_b10'])"
