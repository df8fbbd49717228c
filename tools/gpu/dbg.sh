python -c "import __graft_entry__ as g; g.build()"
export CUDA_LAUNCH_BLOCKING=1
for lib in libmel.so libmel_ae790a7.so libmel_73bc5fc.so libmel_0b775fb.so; do
 echo "== $lib"; MEL_LIB=$lib NG=24 CAP=48 timeout 120 python tools/gpu/dbg_k64.py 256 2>&1 | tail -2
done
MEL_LIB=libmel.so timeout 600 python -m pytest tests/test_gpu_train.py -q -x -k "N1369" 2>&1 | tail -3
