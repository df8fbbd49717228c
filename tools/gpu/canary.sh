timeout 900 python -m pytest tests/test_gpu_train.py -k "grid" -q > gpurun_out/canary.log 2>&1; echo "canary rc=$?"; tail -3 gpurun_out/canary.log
