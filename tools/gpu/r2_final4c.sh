# final tree, 4 GPUs: multi-rank tests + 4-rank bench; then a 200-step 1-GPU bench (power-cap behaviour)
bash tools/gpu/mgpu.sh
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-paper-batch > gpurun_out/b200.log 2>&1; echo "b200 rc=$?"
python3 -c "
import json; l=[x for x in open('gpurun_out/b200.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']), d['ms_per_step'], d['clocks'], d['windows_samples_per_s'])"
