# 2 ranks: L2 prefetch of the next W tile under the in-kernel exchange, on (ppf) / off (base), interleaved
for v in base ppf base ppf base ppf; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  MEL_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ppf_$v.log 2>&1
  python3 -c "
import json; l=[x for x in open('gpurun_out/ppf_$v.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$v', round(d['value']), round(d['ms_per_step'],4), 'K1', round(d['kernels']['out_fwd_dw']['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
