"""Non-finite inputs (include/mel.h surrogate_step, MEL_ENONFINITE): a put whose field holds
a NaN marks its slot; a step whose batch draws that slot updates nothing -- every parameter,
moment and the step / sample counters stay bitwise unchanged -- returns MEL_ENONFINITE and
records status 3 for surrogate_step_result; the next batch without it trains normally.
Covered on the fp32 path, the bf16 path with the Adam of W_L fused into K1, and two
virtual ranks (the skip decided collectively: a NaN on rank 1 stops rank 0's update too)."""
from dataclasses import replace

import numpy as np
import pytest

from harness import FieldTable, make_config
from mel_inputs import design

pytestmark = pytest.mark.gpu


def _gpu():
    import torch
    return torch.cuda.is_available()


def _flat(st):
    return np.concatenate([x.reshape(-1).view(np.uint32) for k in ("p", "m", "v") for x in st[k]])


def _fill(ctxs, wl, table, bad_put, bad_rank=0):
    """C puts per rank (fill phase: put i -> slot i); put `bad_put` of `bad_rank` has a NaN."""
    for r, ctx in enumerate(ctxs):
        for i in range(wl.capacity):
            s, t = i % wl.sims, (i // wl.sims) % wl.tau
            f = np.array(table.field(s, t), dtype=np.float32)
            if r == bad_rank and i == bad_put:
                f[len(f) // 3] = np.nan
            assert ctx.put(s, t, table.Xs(s), f) == 0


@pytest.mark.parametrize("prec", [0, 1], ids=["fp32", "bf16-fused"])
def test_nan_field_skips_the_step_state_unchanged(prec):
    if not _gpu():
        pytest.skip("needs a GPU")
    from paper_2309_16743_b200 import mel
    if prec == 0:
        wl = replace(design.TINY_EVICT, capacity=24, threshold=4)
    else:
        wl = replace(design.MEDIUM, n=24, sims=8, hidden=(64, 64), capacity=48, threshold=8, batch=64)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=prec, storage=prec, staging=wl.capacity + 4))
    bad = 5
    _fill([ctx], wl, table, bad)
    skipped = trained_after = 0
    for _ in range(60):
        st, slots, n = ctx.sample(want_slots=True)
        before = ctx.get_state()
        call = ctx.step_calls if hasattr(ctx, "step_calls") else 0
        if bad in set(int(x) for x in slots):
            with pytest.raises(mel.MelError) as e:
                ctx.step(want_loss=True)
            assert e.value.code == -7
            after = ctx.get_state()
            assert np.array_equal(_flat(before), _flat(after))
            assert (after["k"], after["S"]) == (before["k"], before["S"])
            assert ctx.step_result(call)[0] == 3
            skipped += 1
        else:
            r, loss = ctx.step(want_loss=True)
            assert r == 0 and np.isfinite(loss)
            after = ctx.get_state()
            assert after["k"] == before["k"] + 1
            trained_after += skipped > 0
        if skipped and trained_after >= 2:
            break
    assert skipped >= 1 and trained_after >= 2, (skipped, trained_after)


def test_nan_on_one_virtual_rank_skips_every_rank():
    if not _gpu():
        pytest.skip("needs a GPU")
    from paper_2309_16743_b200 import mel
    wl = replace(design.MEDIUM, n=24, sims=8, hidden=(128, 128), capacity=48, threshold=8, batch=64, world=2)
    table = FieldTable(wl)
    vg = mel.VirtualGroup(make_config(wl, precision=1, storage=1, staging=wl.capacity + 4), 2)
    bad = 7
    _fill(vg.ctx, wl, table, bad, bad_rank=1)
    skipped = trained = 0
    for _ in range(60):
        slots1 = None
        for r in range(2):
            st, sl, n = vg.ctx[r].sample(want_slots=True)
            if r == 1:
                slots1 = set(int(x) for x in sl)
        before = [c.get_state() for c in vg.ctx]
        if bad in slots1:
            with pytest.raises(mel.MelError) as e:
                vg.step(want_loss=True)
            assert e.value.code == -7
            after = [c.get_state() for c in vg.ctx]
            for b, a in zip(before, after):
                assert np.array_equal(_flat(b), _flat(a)) and a["k"] == b["k"]
            skipped += 1
        else:
            r, loss = vg.step(want_loss=True)
            assert r == 0 and np.isfinite(loss)
            trained += 1
        if skipped and trained >= 2:
            break
    vg.close()
    assert skipped >= 1 and trained >= 2, (skipped, trained)
