# final build, 4 GPUs: multi-rank tests + 4-rank and 2-rank benches
bash tools/gpu/mgpu.sh
