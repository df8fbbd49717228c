"""Validation on a dedicated GPU: mel_params_copy moves the
trainer's parameters to a context on another GPU, whose surrogate_eval then matches the
trainer's own evaluation bit for bit, and the trainer can keep stepping meanwhile."""
from dataclasses import replace

import numpy as np
import pytest

from harness import FieldTable, make_config
from mel_inputs import design, heat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mel():
    from paper_2309_16743_b200 import build, mel as m
    build.build()
    return m


def test_params_copy_to_a_second_gpu(mel):
    """On a 1-GPU box the validation context shares the trainer's GPU: the same copy, the
    same cross-stream event ordering and the same bit-exact evaluation, through the copy
    engine instead of NVLink."""
    import torch
    dev_val = 1 if torch.cuda.device_count() >= 2 else 0
    wl = replace(design.MEDIUM, n=32, sims=12, capacity=400, threshold=60, batch=64, puts_per_step=40)
    table = FieldTable(wl)
    cfg = make_config(wl, precision=mel.BF16, storage=mel.STORE_BF16)
    trainer = mel.Context(cfg, device=0)
    val = mel.Context(cfg, device=dev_val)
    order = design.stream_order(wl.sims, wl.tau)
    pos = [0]

    def train(k):
        for _ in range(k):
            for s, t in order[pos[0]:pos[0] + wl.puts_per_step]:
                trainer.put(s, t, table.Xs(s), table.field(s, t))
            pos[0] += wl.puts_per_step
            trainer.sample()
            trainer.step(want_loss=False)

    Xv = design.draw_design(3, seed=1, validation=True)
    X = np.repeat(Xv, wl.tau, 0).astype(np.float32)
    t = np.tile(np.arange(wl.tau), 3).astype(np.uint32)
    F = np.concatenate([heat.simulate(Xv[s], wl.n, wl.tau) for s in range(3)])
    train(8)
    val.copy_params_from(trainer)
    train(3)                                   # the copy does not block the trainer's queue
    assert np.isfinite(val.eval(X, t, F)[0])
    val.copy_params_from(trainer)
    a, b = trainer.get_params(), val.get_params()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert trainer.eval(X, t, F)[0] == val.eval(X, t, F)[0]


def test_eval_reads_device_fields_in_place(mel):
    """surrogate_eval with the held-out fields already on the GPU (unified addressing)
    gives the same MSE as with the fields in host memory."""
    import torch
    wl = replace(design.MEDIUM, n=32, sims=12, capacity=400, threshold=60, batch=64, puts_per_step=40)
    table = FieldTable(wl)
    ctx = mel.Context(make_config(wl, precision=mel.BF16, storage=mel.STORE_BF16), device=0)
    for s, t in design.stream_order(wl.sims, wl.tau)[:200]:
        ctx.put(s, t, table.Xs(s), table.field(s, t))
    ctx.sample()
    ctx.step(want_loss=False)
    Xv = design.draw_design(3, seed=1, validation=True)
    X = np.repeat(Xv, wl.tau, 0).astype(np.float32)
    t = np.tile(np.arange(wl.tau), 3).astype(np.uint32)
    F = np.concatenate([heat.simulate(Xv[s], wl.n, wl.tau) for s in range(3)])
    m_host, _ = ctx.eval(X, t, F)
    m_dev, _ = ctx.eval(X, t, torch.from_numpy(F).cuda(0))
    assert m_host == m_dev and np.isfinite(m_host)
