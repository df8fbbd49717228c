for lib in libmel.so libmel_noremap.so; do
  echo "== $lib"
  for bf in "10 0" "10 8" "64 0" "64 8" "128 0"; do
    MEL_LIB=$lib timeout 300 python tools/diag_grid.py $bf 25 0,29,7,1 2>&1 | grep "^B="
  done
done
