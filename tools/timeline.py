"""GPU timeline of a few paper-shape training steps through CUPTI (torch.profiler):
every kernel / memcpy of the library with its start, duration and the idle gap before
it, so the step's non-kernel time can be attributed.  Usage: python tools/timeline.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from mel_inputs import design, heat_torch
    from paper_2309_16743_b200 import mel

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    grid, tau, C, B = 1000, 100, 6000, 1024
    N = grid * grid
    cfg = mel.Config(n_field=N, hidden=(256, 256), capacity=C, threshold=1000, batch=B, steps_per_sim=tau,
                     precision=mel.BF16, storage=mel.STORE_BF16, seed=1, staging_entries=64)
    ctx = mel.Context(cfg, stream=stream.cuda_stream)
    phi = heat_torch.basis(grid, tau, device=dev)
    Xd = torch.from_numpy(design.draw_design(200, seed=1)).to(dev)
    order = design.stream_order(200, tau)
    cur = [0]

    def fields(n):
        pairs = order[cur[0]:cur[0] + n]
        cur[0] += n
        s = torch.tensor([p[0] for p in pairs], device=dev)
        t = torch.tensor([p[1] for p in pairs], device=dev)
        return pairs, Xd[s].cpu().numpy(), heat_torch.fields(phi, Xd[s], t)

    keep = []
    while ctx.stats()["population"] < C:
        pairs, Xh, F = fields(200)
        keep.append(F)
        torch.cuda.synchronize()
        for j, (s, t) in enumerate(pairs):
            ctx.put(s, t, Xh[j], F[j])
        ctx.sample()
        ctx.step(want_loss=False)
    pool = [fields(4) for _ in range(8)]
    torch.cuda.synchronize()

    def one(i):
        pairs, Xh, F = pool[i]
        for j, (s, t) in enumerate(pairs):
            ctx.put(s, t, Xh[j], F[j])
        ctx.sample()
        ctx.step(want_loss=False)

    for i in range(3):
        one(i)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(3, 8):
            one(i)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev_end = None
    total_gap = 0.0
    rows = []
    for e in evs:
        st, en = e.time_range.start, e.time_range.end
        gap = (st - prev_end) if prev_end is not None else 0.0
        prev_end = max(prev_end or 0, en)
        total_gap += max(gap, 0)
        rows.append((st - t0, en - st, gap, e.name[:60]))
    span = evs[-1].time_range.end - t0
    print("5 steps: span %.1f us, idle gaps %.1f us (%.1f%%), %d GPU activities" % (span, total_gap,
                                                                                   100 * total_gap / span, len(evs)))
    n_step = len(rows) // 5
    print("%10s %9s %8s  %s" % ("start us", "dur us", "gap us", "activity"))
    for r in rows[-n_step:]:
        print("%10.1f %9.1f %8.1f  %s" % r)


if __name__ == "__main__":
    main()
