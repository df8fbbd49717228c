"""Validation on a dedicated GPU ("validation stalls the consumption"; SURVEY §8(f)
f4), paper shape: train S steps with a validation pass on the 10 held-out simulations
every V steps, (a) inline on the training GPU, (b) offloaded: mel_params_copy to a second
GPU's context and surrogate_eval there from a helper thread while training continues.
One JSON line per placement of the held-out fields (host memory, or resident on the GPU
that evaluates): wall time and training samples/s of both, validation MSEs."""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from mel_inputs import design, heat_torch
    from paper_2309_16743_b200 import mel

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--every", type=int, default=100)
    a = ap.parse_args()
    grid, tau, B = 1000, 100, 1024
    N = grid * grid
    cfg = mel.Config(n_field=N, hidden=(256, 256), capacity=6000, threshold=1000, batch=B, steps_per_sim=tau,
                     precision=mel.BF16, storage=mel.STORE_BF16, seed=1, staging_entries=64)
    dev = torch.device("cuda", 0)
    phi = heat_torch.basis(grid, tau, device=dev)
    Xv = torch.from_numpy(design.draw_design(10, seed=1, validation=True)).to(dev)
    tv = torch.arange(tau, device=dev).repeat(10)
    Fv_dev = heat_torch.fields(phi, Xv.repeat_interleave(tau, 0), tv)        # held-out fields, GPU 0
    Fv = Fv_dev.cpu().numpy()
    Xv_np, tv_np = Xv.repeat_interleave(tau, 0).cpu().numpy(), tv.cpu().numpy().astype(np.uint32)
    sims = 200
    Xd = torch.from_numpy(design.draw_design(sims, seed=1)).to(dev)
    order = design.stream_order(sims, tau)

    Fv_dev1 = Fv_dev.to(torch.device("cuda", 1))                             # ... and on GPU 1

    def run(offload, device_fields):
        ctx = mel.Context(cfg, device=0)
        val = mel.Context(cfg, device=1) if offload else None
        sent = 0
        pool = []
        while sent < 6000:                          # fill the buffer (not timed)
            pairs = order[sent:sent + 64]
            s = torch.tensor([p[0] for p in pairs], device=dev); t = torch.tensor([p[1] for p in pairs], device=dev)
            F = heat_torch.fields(phi, Xd[s], t)
            pool.append(F)
            Xh = Xd[s].cpu().numpy()
            for j, (ss, tt) in enumerate(pairs):
                ctx.put(ss, tt, Xh[j], F[j])
            sent += len(pairs)
            ctx.sample()
        ctx.sync()
        mses, threads = [], []
        t0 = time.perf_counter()
        for k in range(a.steps):
            ctx.sample()
            ctx.step(want_loss=False)
            if (k + 1) % a.every == 0:
                if offload:
                    val.copy_params_from(ctx)
                    fv = Fv_dev1 if device_fields else Fv
                    th = threading.Thread(target=lambda: mses.append(val.eval(Xv_np, tv_np, fv)[0]))
                    th.start()
                    threads.append(th)
                else:
                    mses.append(ctx.eval(Xv_np, tv_np, Fv_dev if device_fields else Fv)[0])
        ctx.sync()
        dt = time.perf_counter() - t0
        for th in threads:
            th.join()
        return {"seconds": round(dt, 3), "train_samples_per_s": round(a.steps * B / dt, 1),
                "validations": len(mses), "val_mse_last": mses[-1] if mses else None}

    for dev_fields in (False, True):
        inline = run(False, dev_fields)
        offl = run(True, dev_fields)
        print(json.dumps({"steps": a.steps, "every": a.every, "heldout_fields": "device" if dev_fields else "host",
                          "inline": inline, "offloaded": offl,
                          "speedup": round(inline["seconds"] / offl["seconds"], 3)}), flush=True)


if __name__ == "__main__":
    main()
