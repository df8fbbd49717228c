# K1 per-tile cycle budget (CTA 0 timeline from bench.py --profile), clock-independent A/B of
# variant builds: mean over tiles 3..40 of the tile period, MMA phase (W ready -> dW done) and
# Adam phase (dW done -> Adam done); R interleaved rounds
for r in $(seq ${R:-2}); do
for v in "$@"; do
  envs=""; lib=libmel.so
  case "$v" in base) ;; env:*) envs="${v#env:}" ;; *) lib=libmel_$v.so ;; esac
  env $envs MEL_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/tp_$v.log 2>&1
  python - "$r $v" gpurun_out/tp_$v.log <<'P'
import sys, json, re
name, path = sys.argv[1], sys.argv[2]
rows = []
for l in open(path):
    if l.startswith("tile"):
        f = l.split(); per = re.search(r"period (\d+)", l)
        if per: rows.append((int(f[1].rstrip(":")), [int(x) for x in f[2:14]], int(per.group(1))))
    elif l.startswith("{"): ms = json.loads(l)["ms_per_step"]
rows = [r for r in rows if 3 <= r[0] <= 40]
n = len(rows)
per = sum(r[2] for r in rows) / n; mma = sum(r[1][4] for r in rows) / n; adam = sum(r[1][5] - r[1][4] for r in rows) / n
print("%-12s tiles %d  period %6.0f  MMA %6.0f  Adam %6.0f  gap %6.0f  (ms/step %.4f)" % (name, n, per, mma, adam, per - mma - adam, ms))
P
done; done
