"""Online (Reservoir) versus multi-epoch offline training on one B200, the paper's
§4.4 comparison (Table 2) scaled to one GPU: the offline run trains for E
epochs on a fixed dataset of S_off simulations written to a file beforehand (read back by
the dataset's loader threads, surrogate_train_offline, FIFO batches in epoch order), the
online run streams S_on = 10 x S_off fresh simulations through the Reservoir for the same
number of training steps.  Same trainer, same shapes, same batch; validation MSE on the 10
held-out simulations at the end; throughput = samples trained per second of the
training loop (file reads included for offline, puts included for online).
    python tools/offline_compare.py [--grid 200] [--sims 250] [--epochs 20]
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from mel_inputs import design, heat_torch
    from paper_2309_16743_b200 import mel

    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=200)
    ap.add_argument("--sims", type=int, default=250)
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--dir", default=tempfile.gettempdir())
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n_field, tau = a.grid * a.grid, 100
    phi = heat_torch.basis(a.grid, tau, device=dev)
    Xv = torch.from_numpy(design.draw_design(10, seed=1, validation=True)).to(dev)
    tv = torch.arange(tau, device=dev).repeat(10)
    Xv_rep = Xv.repeat_interleave(tau, 0)
    Fv = heat_torch.fields(phi, Xv_rep, tv).cpu().numpy()
    Xv_np, tv_np = Xv_rep.cpu().numpy(), tv.cpu().numpy().astype(np.uint32)

    def config(policy, capacity, threshold, staging):
        return mel.Config(n_field=n_field, hidden=(256, 256), capacity=capacity, threshold=threshold, batch=a.batch,
                          steps_per_sim=tau, precision=mel.BF16, storage=mel.STORE_BF16, seed=1,
                          staging_entries=staging, policy=policy)

    # ---- offline: write the dataset of a.sims simulations, then E epochs from the file
    Xd = torch.from_numpy(design.draw_design(a.sims, seed=1)).to(dev)
    path = os.path.join(a.dir, "mel_offline_%d.bin" % os.getpid())

    def records():
        for s in range(a.sims):
            F = heat_torch.fields(phi, Xd[s].expand(tau, 5), torch.arange(tau, device=dev)).cpu().numpy()
            Xs = Xd[s].cpu().numpy()
            for t in range(tau):
                yield s, t, Xs, F[t]
    t0 = time.perf_counter()
    n_rec = mel.write_dataset(path, n_field, records())
    t_write = time.perf_counter() - t0
    ds = mel.Dataset(path, threads=a.threads)
    ctx = mel.Context(config(mel.FIFO, 2 * a.batch, 0, 2 * a.batch))
    steps_off = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for e in range(a.epochs):
        st, _ = ctx.train_offline(ds, seed=1, epoch=e, want_losses=False)
        steps_off += st
    ctx.sync()
    dt_off = time.perf_counter() - t0
    mse_off, _ = ctx.eval(Xv_np, tv_np, Fv)
    ds.close()
    os.remove(path)
    del ctx

    # ---- online: 10x the simulations streamed through the Reservoir, same step count
    sims_on = 10 * a.sims
    Xo = torch.from_numpy(design.draw_design(sims_on, seed=2)).to(dev)
    order = design.stream_order(sims_on, tau)
    per_step = -(-len(order) // steps_off)
    ctx = mel.Context(config(mel.RESERVOIR, 6000, 1000, per_step + 16))
    sent = steps_on = 0
    keep = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while steps_on < steps_off:
        k = min(per_step, len(order) - sent)
        if k:
            pairs = order[sent:sent + k]
            s = torch.tensor([p[0] for p in pairs], device=dev)
            t = torch.tensor([p[1] for p in pairs], device=dev)
            F = heat_torch.fields(phi, Xo[s], t)
            keep = [F]
            Xh = Xo[s].cpu().numpy()
            for j, (ss, tt) in enumerate(pairs):
                assert ctx.put(ss, tt, Xh[j], F[j]) == mel.OK
            sent += k
        r, _, _ = ctx.sample()
        if r == mel.OK:
            ctx.step(want_loss=False)
            steps_on += 1
    ctx.sync()
    dt_on = time.perf_counter() - t0
    mse_on, _ = ctx.eval(Xv_np, tv_np, Fv)
    out = {
        "grid": a.grid, "n_field": n_field, "batch": a.batch, "steps": steps_off,
        "offline": {"sims": a.sims, "records": n_rec, "epochs": a.epochs, "dataset_GB": round(n_rec * 4 * n_field / 1e9, 2),
                    "write_s": round(t_write, 1), "train_s": round(dt_off, 2),
                    "samples_per_s": round(steps_off * a.batch / dt_off, 1), "val_mse": mse_off,
                    "loader_threads": a.threads},
        "online": {"sims": sims_on, "unique_samples": sent, "train_s": round(dt_on, 2),
                   "samples_per_s": round(steps_on * a.batch / dt_on, 1), "val_mse": mse_on},
        "val_mse_online_vs_offline": round(mse_on / mse_off - 1.0, 3),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
