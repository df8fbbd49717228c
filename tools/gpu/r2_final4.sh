# final build on 4 GPUs: multi-rank tests (incl. the 4-rank ones) + 4-rank bench, 2-rank bench, grid-independence canary
bash tools/gpu/mgpu.sh
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2b.log 2>&1; echo "bench N=2 rc=$?"
grep '^{' gpurun_out/bench_n2b.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N2', d['value'], d['ms_per_step'])"
timeout 600 python -m pytest tests/test_gpu_train.py -k grid -q > gpurun_out/grid.log 2>&1; echo "grid rc=$?"; tail -3 gpurun_out/grid.log
