"""GPU parity of the on-device heat-equation client (include/mel_heat.h)
against the pinned input generator mel_inputs/heat.py (fp64 DST-I solve of the same
implicit scheme, rounded to fp32; pinned by closed forms in test_oracle_heat.py).
Both solve the scheme exactly in fp64 by different routes (dense DST GEMMs on the GPU,
scipy's fast sine transform on the host), so the fp32 fields agree to within one ulp."""
import numpy as np
import pytest

from harness import compare_reservoir  # noqa: F401  (shared test helpers)
from mel_inputs import design, heat
from oracle import reservoir as ores
from paper_2309_16743_b200 import mel

pytestmark = pytest.mark.gpu


def _ulps(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(a - b)                      # fields are positive kelvin: ordered bit patterns


@pytest.mark.parametrize("n,tau", [(3, 3), (5, 1), (12, 6), (41, 10), (100, 5)])
def test_fields_match_the_scheme(n, tau):
    gen = mel.Heat(n, tau)
    assert gen.basis_bytes == 5 * tau * n * n * 8
    X = design.draw_design(7, seed=4)
    got = gen.fields(np.repeat(X, tau, 0), np.tile(np.arange(tau), 7)).cpu().numpy().reshape(7, tau, n * n)
    for s in range(7):
        ref = heat.simulate(X[s], n, tau)
        u = _ulps(got[s], ref)
        assert u.max() <= 1 and (u == 0).mean() >= 0.99, (n, tau, s, u.max(), (u == 0).mean())
    gen.destroy()


def test_paper_shape_sampled_fields():
    """1000 x 1000 grid, 100 steps (the 4 GB basis): sampled (X, t) against the host solve."""
    n, tau = 1000, 100
    gen = mel.Heat(n, tau)
    X = design.draw_design(2, seed=8)
    ts = np.array([1, 99])
    got = gen.fields(X, ts).cpu().numpy()
    for j in range(2):
        ref = heat.simulate(X[j], n, tau)[ts[j]]
        u = _ulps(got[j], ref)
        assert u.max() <= 1 and (u == 0).mean() >= 0.99
    gen.destroy()


def test_put_generated_into_the_reservoir():
    """Generated puts land in the buffer exactly like host puts of the same fields: slots,
    metadata and counters bit-exact, payload within one fp32 ulp of the host solve."""
    n, tau, sims = 16, 10, 30
    C, theta, B = 64, 8, 8
    gen = mel.Heat(n, tau)
    cfg = mel.Config(n_field=n * n, hidden=(32,), capacity=C, threshold=theta, batch=B, steps_per_sim=tau, seed=2,
                     staging_entries=40)
    ctx = mel.Context(cfg)
    res = ores.Reservoir(C, theta, n * n, seed=2)
    X = design.draw_design(sims, seed=2)
    order = design.stream_order(sims, tau)
    fields = {s: heat.simulate(X[s], n, tau) for s in range(sims)}
    i = 0
    while i < len(order):
        chunk = order[i:i + 30]
        s_ = np.array([p[0] for p in chunk]); t_ = np.array([p[1] for p in chunk])
        st, k = ctx.put_generated(gen, s_, X[s_], t_)
        assert st in (mel.OK, mel.EAGAIN) and (st == mel.EAGAIN or k == len(chunk))
        for s, t in chunk[:k]:                        # a full staging ring (back-pressure,
            res.put(s, t, X[s], fields[s][t])        # P:264) leaves the rest for later
        i += k
        a, sa, _ = ctx.sample(want_slots=True)
        b, sb = res.sample(B)
        assert a == b and list(sa) == list(sb)
    ctx.close(); res.close()
    d = ctx.dump(payload=True)
    occ = res.sim >= 0
    assert np.array_equal(d["sim"][occ].astype(np.int64), res.sim[occ])
    assert np.array_equal(d["t"][occ].astype(np.int64), res.t[occ])
    assert np.array_equal(d["seen"][occ].astype(np.int64), res.seen[occ])
    u = _ulps(d["payload"][occ], res.payload[occ])
    assert u.max() <= 1
    gen.destroy()
