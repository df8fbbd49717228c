"""The on-device heat-equation client at paper shape on one B200:
basis build time (5 x 100 implicit-Euler steps on the 1000 x 1000 grid, fp64 DST GEMMs),
field generation throughput (reservoir-bound fp32 fields from the basis), and generation +
training sharing the GPU: each training step also generates and puts --puts-per-step new
time steps (reservoir_put_generated) from a stream of simulations.  One JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from mel_inputs import design
    from paper_2309_16743_b200 import mel

    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=1000)
    ap.add_argument("--tau", type=int, default=100)
    ap.add_argument("--puts-per-step", type=int, default=64)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    n, tau, N = a.grid, a.tau, a.grid * a.grid
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gen = mel.Heat(n, tau)
    t_basis = time.perf_counter() - t0

    # generation alone: 64 fields per call, all t of a simulation range
    X = torch.from_numpy(design.draw_design(64, seed=3)).cuda()
    ts = torch.arange(64, device="cuda", dtype=torch.int32) % tau
    for _ in range(3):
        gen.fields(X, ts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        out = gen.fields(X, ts)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fields_per_s = 64 / (ms / 1e3)

    # generation + training in one allocation (paper-shaped trainer, Reservoir C=6000, theta=1000)
    cfg = mel.Config(n_field=N, hidden=(256, 256), capacity=6000, threshold=1000, batch=1024, steps_per_sim=tau,
                     precision=mel.BF16, storage=mel.STORE_BF16, seed=1, staging_entries=a.puts_per_step + 16)
    ctx = mel.Context(cfg)
    sims = 1 + (a.steps * a.puts_per_step + 1000) // tau
    Xd = design.draw_design(sims, seed=1)
    order = design.stream_order(sims, tau)
    sent = steps = 0
    # fill to the watermark first (not timed)
    while sent <= 1000:
        k = min(a.puts_per_step, len(order) - sent)
        s_ = np.array([p[0] for p in order[sent:sent + k]]); t_ = np.array([p[1] for p in order[sent:sent + k]])
        st, m = ctx.put_generated(gen, s_, Xd[s_], t_)
        sent += m
        ctx.sample()
    ctx.sync()
    t0 = time.perf_counter()
    put_timed = 0
    while steps < a.steps:
        k = min(a.puts_per_step, len(order) - sent)
        if k:
            s_ = np.array([p[0] for p in order[sent:sent + k]]); t_ = np.array([p[1] for p in order[sent:sent + k]])
            st, m = ctx.put_generated(gen, s_, Xd[s_], t_)
            sent += m
            put_timed += m
        r, _, _ = ctx.sample()
        if r == mel.OK:
            ctx.step(want_loss=False)
            steps += 1
    ctx.sync()
    dt = time.perf_counter() - t0
    print(json.dumps({
        "grid": n, "tau": tau, "basis_GB": round(gen.basis_bytes / 1e9, 2), "basis_build_s": round(t_basis, 2),
        "generate_ms_per_64_fields": round(ms, 3), "fields_per_s": round(fields_per_s, 1),
        # algorithmic bytes per field: 5 fp64 basis rows read + the fp32 field written
        "generate_hbm_GB_per_s": round(fields_per_s * 44 * N / 1e9, 1),
        "train_with_generation": {"steps": steps, "puts_per_step": a.puts_per_step, "generated": put_timed,
                                  "seconds": round(dt, 3), "samples_per_s": round(steps * 1024 / dt, 1),
                                  "generated_per_s": round(put_timed / dt, 1)}}))


if __name__ == "__main__":
    main()
