# drain-phase sample cost, parallel draws (base) vs one thread (prev), interleaved
for v in prev base prev base; do
  lib=libmel.so; [ "$v" != base ] && lib=libmel_$v.so
  echo -n "$v: "; MEL_LIB=$lib python - <<'P' 2>&1 | tail -1
import numpy as np, torch
from paper_2309_16743_b200 import mel
cfg = mel.Config(n_field=1000 * 1000, hidden=(256, 256), capacity=6000, threshold=1000, batch=1024, steps_per_sim=100,
                 precision=1, storage=1, seed=1, staging_entries=64)
ctx = mel.Context(cfg)
f = torch.rand(1000 * 1000, device="cuda", dtype=torch.float32) * 400 + 100
X = np.array([300, 200, 400, 250, 350], dtype=np.float32)
for i in range(6000):
    while ctx.put(i // 100, i % 100, X, f) != 0:
        ctx.sample()
ctx.close()
ctx.sample()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize(); ev[0].record()
for _ in range(4):
    ctx.sample()
ev[1].record(); torch.cuda.synchronize()
print("%.1f us per drain-phase sample call (1024 draws)" % (ev[0].elapsed_time(ev[1]) * 1e3 / 4))
P
done
