for cfg in "0 1" "0 4" "16 1" "16 4" "8 4" "24 8"; do
  set -- $cfg
  MEL_SM_RESERVE=$1 MEL_BUCKETS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e > gpurun_out/sw_$1_$2.log 2>&1
done
