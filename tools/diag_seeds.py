"""Diagnostic: bf16 free-running step-1000 loss gap vs the fp64 oracle over seeds."""
import os, sys
from dataclasses import replace
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
from harness import FieldTable, make_config
from mel_inputs import design
from oracle import trainer as otr
from paper_2309_16743_b200 import mel

for seed in [int(x) for x in sys.argv[1:]]:
    wl = replace(design.MEDIUM, name="m1k", capacity=6000, threshold=1000, sims=1100)
    table = FieldTable(wl, seed=seed)
    ctx = mel.Context(make_config(wl, precision=1, storage=1, seed=seed))
    tr = otr.Trainer(wl.n_field, wl.hidden, wl.tau, wl.capacity, wl.threshold, wl.batch, seed=seed, storage=1)
    lg, lo = [], []
    for op in design.build_oplog(wl):
        if op[0] == "PUT":
            _, r, s, t = op
            ctx.put(s, t, table.Xs(s), table.field(s, t)); tr.put(0, s, t, table.Xs(s), table.field(s, t))
        elif op[0] == "SAMPLE":
            ctx.sample(); tr.sample(0)
        elif op[0] == "STEP":
            a, l1 = ctx.step(want_loss=True); b, l2 = tr.step()
            if a == 0:
                lg.append(l1); lo.append(l2)
                if len(lg) == 1000: break
    e = (np.array(lg) - np.array(lo)) / np.array(lo)
    print("seed %d: signed rel err step1000 %+.2e | mean|e| 951-1000 %.2e | mean signed 951-1000 %+.2e | loss %.3e" %
          (seed, e[-1], np.abs(e[-50:]).mean(), e[-50:].mean(), lo[-1]), flush=True)
    print("   rel err at steps 100..1000:", " ".join("%+.1e" % e[i - 1] for i in range(100, 1001, 100)), flush=True)
