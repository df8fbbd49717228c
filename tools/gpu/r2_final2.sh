# final build on 2 GPUs: multi-rank tests + 2-rank bench, then every slow GPU test
bash tools/gpu/mgpu.sh
timeout 3000 python -m pytest tests -m "gpu and slow" -q -s > gpurun_out/f_slow.log 2>&1; echo "slow rc=$?"
grep -E "err|R=|passed|failed|Error" gpurun_out/f_slow.log | tail -20
