"""Diagnostic: K1 grid independence at one workload (B, hidden, flags) over grids; prints
per grid the steps completed, the first error and a hash of p, m, v (MEL_LIB picks the build)."""
import hashlib
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import FieldTable, make_config  # noqa: E402
from mel_inputs import design  # noqa: E402
from paper_2309_16743_b200 import mel  # noqa: E402

B, flags, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
grids = [int(x) for x in sys.argv[4].split(",")]
wl = replace(design.MEDIUM, name="medium-bf16", capacity=600, threshold=100, sims=40, puts_per_step=40, n=101, batch=B)
table = FieldTable(wl)
for g in grids:
    if g:
        os.environ["MEL_K1_CTAS"] = str(g)
    else:
        os.environ.pop("MEL_K1_CTAS", None)
    ctx = mel.Context(make_config(wl, precision=1, storage=1, flags=flags))
    n, err, losses = 0, None, []
    try:
        for op in design.build_oplog(wl):
            if op[0] == "PUT":
                _, r, s, t = op
                ctx.put(s, t, table.Xs(s), table.field(s, t))
            elif op[0] == "CLOSE":
                ctx.close()
            elif op[0] == "SAMPLE":
                ctx.sample()
            elif op[0] == "STEP":
                st, loss = ctx.step(want_loss=True)
                if st == 0:
                    n += 1
                    losses.append(loss)
                    if n == steps:
                        break
    except Exception as e:  # noqa: BLE001
        err = str(e)[:80]
    h = hashlib.sha1()
    try:
        stt = ctx.get_state()
        for k in ("p", "m", "v"):
            for x in stt[k]:
                h.update(x.tobytes())
    except Exception as e:  # noqa: BLE001
        err = (err or "") + " | state: " + str(e)[:40]
    print("B=%d flags=%d grid=%3d steps=%d err=%s hash=%s losses=%s" % (B, flags, g, n, err, h.hexdigest()[:12],
                                                                     ["%.4g" % l for l in losses[:3]] + ["..."] + ["%.4g" % l for l in losses[-2:]]), flush=True)
    del ctx
