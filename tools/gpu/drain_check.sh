python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/dr_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/dr_tests.log
grep -E "^FAILED|Error" gpurun_out/dr_tests.log | head -5
# drain-phase step cost: paper-shape reservoir closed and drained, commit + sample launches timed by CUDA events
python - <<'P'
import time, numpy as np, torch
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
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize(); ev[0].record()
n = 0
for _ in range(5):
    st, _, k = ctx.sample(); n += 1
ev[1].record(); torch.cuda.synchronize()
print("drain: %d sample calls (1024 draws each), %.1f us per call (commit + draws, incl. host overhead)" % (n, ev[0].elapsed_time(ev[1]) * 1e3 / n))
P
