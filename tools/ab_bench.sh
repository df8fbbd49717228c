#!/bin/bash
# Alternate bench runs of the working build (A) and libmel_ab.so (B) on the same box.
# Usage: bash tools/ab_bench.sh [rounds] [gpus] [extra bench args]
R=${1:-3}; N=${2:-1}; shift 2 || shift $#
P='import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]); print("%.4f ms/step  K1 %.4f  K2 %.4f  %.0f samples/s" % (d["ms_per_step"], d["kernels"]["out_fwd_dw"]["ms_per_step"], d["kernels"]["out_dh"]["ms_per_step"], d["value"]))'
run() {
  if [ "$N" -gt 1 ]; then
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus "$N" --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | python -c "$P"
  else
    python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | python -c "$P"
  fi
}
for i in $(seq "$R"); do
  echo -n "A: "; run "$@"
  echo -n "B: "; MEL_LIB=libmel_ab.so run "$@"
done
