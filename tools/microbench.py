"""Per-kernel microbenchmarks of SURVEY §8(d) item 9 at paper shape (1000x1000 field,
C = 6000), timed with the library's per-kernel CUDA events (MEL_FLAG_TIMING):

* commit: a burst of device-resident puts committed at once (commit_ctrl + commit_copy:
  staging fp32 read + normalised bf16 slot write, 2*N*4 + N*2 algorithmic bytes per put);
* Adam (unfused kernel, MEL_FLAG_UNFUSED_ADAM) over all 257M parameters: 28 B/param +
  2 B/param of W_L bf16 shadow;
* sample: B = 1024 Philox draws with seen counters.
Prints one JSON line per kernel with achieved GB/s against MEASURED_PEAKS.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from mel_inputs import design, heat_torch
    from paper_2309_16743_b200 import mel

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    hbm = peaks["hbm_gbs"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    grid, tau, C, B = 1000, 100, 6000, 1024
    N = grid * grid
    cfg = mel.Config(n_field=N, hidden=(256, 256), capacity=C, threshold=1000, batch=B, steps_per_sim=tau,
                     precision=mel.BF16, storage=mel.STORE_BF16, seed=1, staging_entries=256,
                     flags=mel.FLAG_UNFUSED_ADAM)
    ctx = mel.Context(cfg, stream=stream.cuda_stream)
    phi = heat_torch.basis(grid, tau, device=dev)
    Xd = torch.from_numpy(design.draw_design(200, seed=1)).to(dev)
    order = design.stream_order(200, tau)
    cur = [0]

    def puts(n):
        pairs = order[cur[0]:cur[0] + n]
        cur[0] += n
        s = torch.tensor([p[0] for p in pairs], device=dev)
        t = torch.tensor([p[1] for p in pairs], device=dev)
        F = heat_torch.fields(phi, Xd[s], t)
        Xh = Xd[s].cpu().numpy()
        torch.cuda.synchronize()
        for j, (ss, tt) in enumerate(pairs):
            ctx.put(ss, tt, Xh[j], F[j])
        return F

    # fill the reservoir, then time commits of bursts of 128 puts (fill + evict phases)
    keep = []
    for _ in range(C // 200):
        keep.append(puts(200))
        ctx.sample()
    ctx.sync()
    ctx.set_flags(mel.FLAG_TIMING | mel.FLAG_UNFUSED_ADAM)
    ctx.kernel_time_reset()
    nb, burst = 4, 128
    for _ in range(nb):
        keep.append(puts(burst))
        ctx.sample()                       # commit point
    ctx.sync()
    ms, _ = ctx.kernel_time(mel.K_COMMIT)
    per_put = (2 * N * 4 + N * 2)
    gbs = nb * burst * per_put / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": "commit (ctrl + copy)", "puts": nb * burst, "ms": ms, "bytes_per_put": per_put,
                      "achieved_GBs": gbs, "frac_hbm": gbs / hbm}))
    ms_s, n_s = ctx.kernel_time(mel.K_SAMPLE)
    print(json.dumps({"kernel": "sample", "launches": n_s, "us_per_launch": 1e3 * ms_s / max(1, n_s),
                      "draws_per_launch": B}))
    # unfused Adam over every parameter: a few training steps
    ctx.kernel_time_reset()
    steps = 10
    for _ in range(steps):
        keep = keep[-4:]
        keep.append(puts(4))
        ctx.sample()
        ctx.step(want_loss=False)
    ctx.sync()
    ms, n = ctx.kernel_time(mel.K_ADAM)
    P = ctx.n_params
    bytes_ = 28.0 * P + 2.0 * N * 256
    gbs = steps * bytes_ / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": "adam (unfused, 257M params)", "ms_per_step": ms / steps, "bytes_per_step": bytes_,
                      "achieved_GBs": gbs, "frac_hbm": gbs / hbm}))


if __name__ == "__main__":
    main()
