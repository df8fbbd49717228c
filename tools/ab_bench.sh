#!/bin/bash
# Alternate bench runs of the working build (A) and libmel_ab.so (B) on the same box.
# Usage: bash tools/ab_bench.sh [rounds] [extra bench args]
R=${1:-3}; shift || true
P='import json,sys; d=json.loads(sys.stdin.read()); print("%.4f ms/step  K1 %.4f  K2 %.4f" % (d["ms_per_step"], d["kernels"]["out_fwd_dw"]["ms_per_step"], d["kernels"]["out_dh"]["ms_per_step"]))'
for i in $(seq "$R"); do
  echo -n "A: "; python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "$P"
  echo -n "B: "; MEL_LIB=libmel_ab.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "$P"
done
