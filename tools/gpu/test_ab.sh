# GPU tests (not slow) of the working build, then A/B: working build vs libmel_ab.so (HEAD)
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/t.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/t.log | tail -5
bash tools/gpu/k1_exp.sh base ab "$@"
