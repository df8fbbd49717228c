"""Checkpoint / resume of a rank (include/mel.h reservoir_save / reservoir_load with
mel_get_state / mel_set_state; SPEC's ServerCheckpoint): a context restored
mid-run -- puts pending in the staging ring, evictions done, Philox counters advanced --
continues exactly as the original: the same sampled slots on every SAMPLE, bitwise the same
losses and final parameters, moments and buffer contents."""
from dataclasses import replace

import numpy as np
import pytest

from harness import FieldTable, make_config
from mel_inputs import design

pytestmark = pytest.mark.gpu


def _gpu():
    import torch
    return torch.cuda.is_available()


@pytest.mark.parametrize("prec,policy", [(0, 0), (1, 0), (0, 2)], ids=["fp32-reservoir", "bf16-reservoir", "fp32-firo"])
def test_resume_from_checkpoint_is_bit_identical(prec, policy):
    if not _gpu():
        pytest.skip("needs a GPU")
    from paper_2309_16743_b200 import mel
    if prec == 0:
        wl = replace(design.TINY_EVICT, puts_per_step=7)
    else:
        wl = replace(design.MEDIUM, n=24, sims=12, capacity=120, threshold=20, batch=256, puts_per_step=40)
    table = FieldTable(wl)
    cfg = make_config(wl, precision=prec, storage=prec, policy=policy)
    ops = design.build_oplog(wl)
    # cut right after some puts of a step, before its SAMPLE: puts are pending
    cut = [i for i, op in enumerate(ops) if op[0] == "PUT" and ops[i + 1][0] == "PUT"][len(ops) // 6]
    a = mel.Context(cfg)

    def run(ctx, lo, hi):
        out = []
        for op in ops[lo:hi]:
            if op[0] == "PUT":
                _, r, s, t = op
                assert ctx.put(s, t, table.Xs(s), table.field(s, t)) == 0
            elif op[0] == "CLOSE":
                ctx.close()
            elif op[0] == "SAMPLE":
                out.append(("S", tuple(ctx.sample(want_slots=True)[1].tolist())))
            elif op[0] == "STEP":
                st, loss = ctx.step(want_loss=True)
                out.append(("T", st, loss))
                if st == 2:
                    break
        return out

    run(a, 0, cut)
    assert a.stats()["pending"] > 0
    blob = a.save_reservoir()
    state = a.get_state()
    b = mel.Context(cfg)
    b.load_reservoir(blob)
    b.set_state(state)
    ra = run(a, cut, len(ops))
    rb = run(b, cut, len(ops))
    assert ra == rb
    assert any(x[0] == "T" and x[1] == 0 for x in ra)
    sa, sb = a.get_state(), b.get_state()
    for k in ("p", "m", "v"):
        for x, y in zip(sa[k], sb[k]):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), k
    da, db = a.dump(), b.dump()
    for k in da:
        assert np.array_equal(da[k], db[k]), k
    st_a, st_b = a.stats(), b.stats()
    for k in ("population", "unseen", "seen", "puts", "committed", "draws", "evictions", "pending"):
        assert st_a[k] == st_b[k], k
    assert np.array_equal(st_a["hist"], st_b["hist"])


def test_load_rejects_another_configuration():
    if not _gpu():
        pytest.skip("needs a GPU")
    from paper_2309_16743_b200 import mel
    wl = design.TINY_EVICT
    a = mel.Context(make_config(wl))
    blob = a.save_reservoir()
    b = mel.Context(make_config(replace(wl, capacity=40)))
    with pytest.raises(mel.MelError) as e:
        b.load_reservoir(blob)
    assert e.value.code == mel.EINVAL
