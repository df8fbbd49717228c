"""Free-running bf16 loss gap at training step 1000 through virtual ranks, over seeds
(the chaotic-drift error bar of DESIGN.md section 3 at R ranks).  GPU box:
    python tools/vr_seed_spread.py R mode seed..."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
from harness import FieldTable, make_config  # noqa: E402
from mel_inputs import design  # noqa: E402
from oracle import trainer as otr  # noqa: E402
from paper_2309_16743_b200 import mel  # noqa: E402

R, mode = int(sys.argv[1]), sys.argv[2]
for seed in [int(x) for x in sys.argv[3:]]:
    g = {k: int(v) for k, v in (kv.split("=") for kv in os.environ.get("WL", "").split(",") if kv)}
    wl = replace(design.MEDIUM, name="vr-1k", n=g.get("n", 48), sims=g.get("sims", 150), capacity=g.get("C", 600),
                 threshold=g.get("theta", 100), batch=g.get("B", 64), puts_per_step=g.get("k", 12), world=R)
    flags = mel.FLAG_FP32_EXCHANGE if mode.endswith("-fp32x") else 0
    table = FieldTable(wl, seed=seed)
    if R == 1:
        class _One:                                       # world 1: the plain context
            def __init__(self, cfg):
                self.ctx = [mel.Context(cfg)]
            def step(self, want_loss=True):
                return self.ctx[0].step(want_loss=want_loss)
            def close(self):
                self.ctx[0].close_ctx()
        vg = _One(make_config(wl, precision=1, storage=1, flags=flags, seed=seed))
    else:
        vg = mel.VirtualGroup(make_config(wl, precision=1, storage=1, flags=flags, seed=seed), R)
    tr = otr.Trainer(wl.n_field, wl.hidden, wl.tau, wl.capacity, wl.threshold, wl.batch, world=R, seed=seed, storage=1)
    lg, lo = [], []
    for op in design.build_oplog(wl):
        if op[0] == "PUT":
            _, r, s, t = op
            vg.ctx[r].put(s, t, table.Xs(s), table.field(s, t)); tr.put(r, s, t, table.Xs(s), table.field(s, t))
        elif op[0] == "CLOSE":
            vg.ctx[op[1]].close(); tr.close(op[1])
        elif op[0] == "SAMPLE":
            vg.ctx[op[1]].sample(); tr.sample(op[1])
        elif op[0] == "STEP":
            a, l1 = vg.step(want_loss=True)
            b, l2 = tr.step()
            if a == 0:
                lg.append(l1); lo.append(l2)
                if len(lg) == 1000:
                    break
    vg.close()
    lg, lo = np.array(lg), np.array(lo)
    e = (lg - lo) / lo
    print("%s R=%d %s seed %d: signed rel gap at step 1000 %+.3e, mean over 951-1000 %+.3e, over 501-1000 %+.3e" %
          (os.environ.get("WL", "n=48"), R, mode, seed, e[-1], e[-50:].mean(), e[-500:].mean()), flush=True)
