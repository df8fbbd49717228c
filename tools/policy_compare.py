"""The paper's buffer comparison (Fig. 2 / Table 1) on one B200, paper
shape (1000x1000 field, 6-256-256-10^6 MLP, B = 1024, C = 6000, theta = 1000):
a wall-clock producer streams fields at a fixed rate with a production gap in the
middle, the consumer loop samples and trains whenever its buffer gives a batch.
Reported per policy: training throughput (samples consumed / s), steps, GPU time
fraction spent training, unique samples ingested, repeats per unique sample, the
population at the end, and the validation MSE on the 10 held-out simulations
 after the same wall-clock budget (the paper's Table 1 comparison).  Usage:
    python tools/policy_compare.py [--rate 2000] [--seconds 6] [--gap 2,4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(policy, args):
    import torch
    from mel_inputs import design, heat_torch
    from paper_2309_16743_b200 import mel

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    n_field, tau, sims = args.grid * args.grid, 100, 10000
    cfg = mel.Config(n_field=n_field, hidden=(256, 256), capacity=6000, threshold=1000, batch=1024,
                     steps_per_sim=tau, precision=mel.BF16, storage=mel.STORE_BF16, seed=1,
                     staging_entries=64, policy=policy)
    ctx = mel.Context(cfg, stream=stream.cuda_stream)
    phi = heat_torch.basis(args.grid, tau, device=dev)
    Xd = torch.from_numpy(design.draw_design(sims, seed=1)).to(dev)
    order = design.stream_order(sims, tau)
    gap0, gap1 = args.gap
    sent = steps = 0
    busy = 0.0
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    keep = []
    while True:
        now = time.perf_counter() - t0
        if now >= args.seconds:
            break
        produce_t = now if now < gap0 else (gap0 if now < gap1 else now - (gap1 - gap0))
        due = min(int(args.rate * produce_t), len(order))
        while sent < due:                           # producer: device-resident exact fields
            k = min(due - sent, 16)
            pairs = order[sent:sent + k]
            s = torch.tensor([p[0] for p in pairs], device=dev)
            t = torch.tensor([p[1] for p in pairs], device=dev)
            F = heat_torch.fields(phi, Xd[s], t)
            keep = [F]
            Xh = Xd[s].cpu().numpy()
            for j, (ss, tt) in enumerate(pairs):
                if ctx.put(ss, tt, Xh[j], F[j]) != 0:
                    k = j
                    break
            sent += k
            if k < len(pairs):
                break                               # staging ring full: production suspended
        st, _, _ = ctx.sample()
        if st == 0:
            ev0.record(stream)
            ctx.step(want_loss=False)
            ev1.record(stream)
            ev1.synchronize()
            busy += ev0.elapsed_time(ev1) / 1e3
            steps += 1
        else:
            stream.synchronize()
            time.sleep(0.0005)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st = ctx.stats()
    # validation MSE on the 10 held-out simulations, after the same wall-clock budget
    import numpy as np
    Xv = torch.from_numpy(design.draw_design(10, seed=1, validation=True)).to(dev)
    tv = torch.arange(tau, device=dev)
    sse = 0.0
    for i in range(10):
        Fv = heat_torch.fields(phi, Xv[i:i + 1].repeat(tau, 1), tv).cpu().numpy()
        mse, _ = ctx.eval(Xv[i:i + 1].repeat(tau, 1).cpu().numpy(), tv.cpu().numpy().astype(np.uint32), Fv)
        sse += mse
    val_mse = sse / 10
    uniq = st["committed"]
    name = {0: "reservoir", 1: "fifo", 2: "firo"}[policy]
    return {"policy": name, "steps": steps, "samples_per_s": steps * 1024 / wall, "gpu_busy_frac": busy / wall,
            "produced": sent, "unique_ingested": int(uniq), "repeats_per_unique": st["draws"] / max(1, uniq),
            "population_end": int(st["population"]), "pending_end": int(st["pending"]), "wall_s": wall,
            "val_mse_normalised": val_mse, "val_mse_K2": val_mse * 400.0 ** 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=2000.0, help="producer samples/s (SURVEY §8(d) default)")
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--gap", type=lambda s: tuple(float(x) for x in s.split(",")), default=(2.0, 4.0),
                    help="production pause [t0, t1) in seconds")
    ap.add_argument("--grid", type=int, default=1000)
    args = ap.parse_args()
    rows = [run(p, args) for p in (0, 1, 2)]
    for r in rows:
        print(json.dumps(r), flush=True)
    print("\n| policy | steps | training samples/s | GPU busy | unique ingested | repeats / unique | population at end | val MSE (K²) |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        print("| %s | %d | %.0f | %.1f%% | %d | %.1f | %d | %.1f |" % (
            r["policy"], r["steps"], r["samples_per_s"], 100 * r["gpu_busy_frac"], r["unique_ingested"],
            r["repeats_per_unique"], r["population_end"], r["val_mse_K2"]))


if __name__ == "__main__":
    main()
