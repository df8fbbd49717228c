#!/usr/bin/env python
"""bench.py -- reservoir-fed online training of the paper-shaped heat-equation
MLP surrogate (arXiv 2309.16743; BASELINE.json configs[2], and configs[3] per
rank under torchrun) on B200.

One timed step = the whole hot path of SURVEY §8(a) for one batch per rank:
k device-resident reservoir_put calls (the streamed clients' time steps), one
reservoir_sample_batch (commit with eviction, watermark gate, Philox sampling),
one surrogate_step (gather, head fwd, tcgen05 output layer fwd+MSE+dW, split-K
dH, head bwd, NCCL gradient all-reduce when N > 1, Adam + LR schedule).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "surrogate training samples/sec at 1/2/4/8 B200; % tensor-core roofline; val MSE"
UNIT = "samples/s"
N_GRID, TAU, SIMS = 1000, 100, 10000
HIDDEN = (256, 256)
CAP, THETA, BATCH = 6000, 1000, 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--puts-per-step", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-paper-batch", action="store_true", help="skip the secondary B=10 (P:317) measurement")
    ap.add_argument("--grid", type=int, default=N_GRID)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--profile", action="store_true", help="timed region only (for ncu)")
    ap.add_argument("--flags", type=int, default=0, help="MEL_FLAG_* bits (e.g. 8 = Adam of W_L as a separate kernel)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


def config_block(args, world):
    return {"workload": "paper-shaped (BASELINE configs[%d])" % (2 if world == 1 else 3),
            "field": "%dx%d" % (args.grid, args.grid), "tau": TAU, "sims_streamed": SIMS,
            "mlp": "6-256-256-%d" % (args.grid * args.grid), "capacity": CAP, "threshold": THETA,
            "batch_per_rank": args.batch, "global_batch": args.batch * world, "puts_per_step": args.puts_per_step,
            "routing": "(sim + t) mod R", "precision": "bf16 tcgen05 output layer, fp32 master/Adam",
            "target_storage": "bf16", "l2": "inputs larger than L2 (W 0.5 GB, Adam state 3 GB, targets 2 GB / step)",
            "parallelism": "dp%d" % world,
            "exchange": ("none" if world == 1 else
                         "NCCL reduce-scatter + sharded Adam + shadow all-gather" if args.flags & 16 else
                         "in-kernel over NVLink: dW tiles (%s) TMA-stored/reduce-added into the owner rank, fused Adam "
                         "at the owner, bf16 shadow rows pushed to every rank; NCCL for the 1.3 MB head + biases"
                         % ("fp32" if args.flags & 32 else "bf16"))}


# ------------------------------------------------------------------------------------
# oracle timing (cpu_baseline and --impl reference): the oracle as it stands
# ------------------------------------------------------------------------------------
def oracle_paper_rate(n_full: int, budget_s: float, batch: int = 8, fields=None, modes=("all_cores", "single_thread"),
                      max_steps: int = 1000):
    """The oracle as it stands (numpy fp64, oracle.trainer) running REAL paper-shape
    training steps (6-256-256-N, N = n_full) at a small batch ("paper shape:
    1 step at B = 8"), timed on the host cores in two modes: BLAS over every core and
    single-threaded.  Each timed step = sample B slots from an oracle reservoir + fp64
    forward/backward + Adam over all 257M parameters.  The reservoir holds 4B streamed
    fields (heat solutions when `fields` is given, else uniform in [100, 500) K: the
    arithmetic does not depend on the values); the weights are seeded uniform(-a, a),
    a = 1/sqrt(fan_in) (input generation, not the oracle's Philox init, which would
    cost minutes at this size).  Returns {mode: (samples_per_s, steps_timed, threads)}."""
    import numpy as np
    from threadpoolctl import threadpool_info, threadpool_limits
    from mel_inputs import design
    from oracle import mlp as omlp
    from oracle import trainer as otr
    rng = np.random.default_rng(7)
    dims = omlp.layer_dims(n_full, HIDDEN)
    params = []
    for i, o in zip(dims[:-1], dims[1:]):
        a = 1.0 / np.sqrt(i)
        params.append((((rng.random((o, i), dtype=np.float32) * 2 - 1) * a).astype(np.float32),
                       ((rng.random(o, dtype=np.float32) * 2 - 1) * a).astype(np.float32)))
    cap = 4 * batch
    tr = otr.Trainer(n_full, HIDDEN, TAU, cap, batch, batch, seed=1, storage=1, params=params)
    del params
    X = design.draw_design(cap, seed=1)
    for i in range(cap):
        f = fields[i % len(fields)] if fields is not None else (100.0 + 400.0 * rng.random(n_full)).astype(np.float32)
        tr.put(0, i, i % TAU, X[i], f)
    all_threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    out = {}
    tr.sample(0); tr.step()                                             # warm-up step
    for mode in modes:
        with threadpool_limits(limits=1 if mode == "single_thread" else None):
            ts = []
            t0 = time.perf_counter()
            while not ts or (len(ts) < max_steps and time.perf_counter() - t0 < budget_s):
                a = time.perf_counter()
                tr.sample(0); tr.step()
                ts.append(time.perf_counter() - a)
        out[mode] = (batch / statistics.median(ts), len(ts), 1 if mode == "single_thread" else all_threads)
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cores = len(os.sched_getaffinity(0))
    n_full = args.grid * args.grid
    # each reference step is one real paper-shape oracle step at B = 8 (all cores); the
    # run is bounded to a few minutes (at least one timed step)
    budget = min(90.0, 6.0 * args.steps)
    r = oracle_paper_rate(n_full, budget, modes=("all_cores",), max_steps=args.steps)
    rate, n_steps, threads = r["all_cores"]
    desc = ("%d real paper-shape oracle steps (fp64 numpy, 6-256-256-%d, Adam over all parameters) at B=8, "
            "after 1 warm-up step, median step time" % (n_steps, n_full))
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
            "steps": n_steps, "warmup": 1, "ms_per_step": 8 / rate * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, world),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "host_cores": cores, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------
class Clocks:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region: NVML
    (what nvidia-smi reads) polled every 2 ms from a thread, only samples taken between
    __enter__ and __exit__ kept; nvidia-smi -lms 20 as the fallback without pynvml."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap")]

    def __init__(self, idx):
        self.idx, self.p, self.path = idx, None, "/tmp/mel_clocks_%d.csv" % os.getpid()
        self.nv, self.rows, self.err = None, [], None

    def __enter__(self):
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.nv, self.stop = nv, threading.Event()
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((sm, mx, rs))
                    except Exception as e:          # keep sampling; report the last error
                        self.err = str(e)
                    self.stop.wait(0.002)

            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
            return self
        except Exception:
            self.nv = None
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                       "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.5)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.th.join()
            return
        if self.p:
            time.sleep(0.05)
            self.p.terminate()
            self.p.wait()
            self.f.close()

    def summary(self):
        if self.nv is not None:
            if not self.rows:
                return {"error": "no NVML sample inside the timed region" + (": " + self.err if self.err else "")}
            sm = [float(r[0]) for r in self.rows]
            mx = float(max(r[1] for r in self.rows))
            reasons = set()
            for _, _, rs in self.rows:
                for name, attr in self.REASONS:
                    if rs & getattr(self.nv, attr, 0):
                        reasons.add(name)
            loaded = [s for s in sm if s > 0.5 * mx] or sm
            return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "nvml, 2 ms"}
        try:
            rows = [[x.strip() for x in l.split(",")] for l in open(self.path).read().strip().splitlines()]
            rows = [r for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
            if not rows:
                return {"error": "no nvidia-smi sample inside the timed region"}
            sm = [float(r[1]) for r in rows]
            mx = max(float(r[2]) for r in rows)
            reasons = set()
            for r in rows:
                for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(name)
            loaded = [s for s in sm if s > 0.5 * mx] or sm
            return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "nvidia-smi -lms 20"}
        except Exception as e:
            return {"error": str(e)}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    from mel_inputs import design, heat_torch
    from paper_2309_16743_b200 import mel

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [mel.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    n_field = args.grid * args.grid
    B, k = args.batch, args.puts_per_step
    cfg = mel.Config(n_field=n_field, hidden=HIDDEN, capacity=CAP, threshold=THETA, batch=B, steps_per_sim=TAU,
                     precision=mel.BF16, storage=mel.STORE_BF16, seed=1, staging_entries=32, flags=args.flags)
    # a dedicated stream shared by torch (events, data generation) and libmel, so
    # that CUDA events bracket exactly the library's work
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = mel.Context(cfg, rank=rank, world=world, nccl_id=nccl_id, device=local, stream=stream.cuda_stream)

    # synthetic ensemble: exact heat solutions by linearity from a GPU-generated basis
    phi = heat_torch.basis(args.grid, TAU, device=dev)                       # (5, tau, N) fp32
    Xd = torch.from_numpy(design.draw_design(SIMS, seed=1)).to(dev)
    order = design.routed_stream(SIMS, TAU, rank, world)
    cursor = [0]

    def next_batch(n):
        pairs = order[cursor[0]:cursor[0] + n]
        cursor[0] += n
        s = torch.tensor([p[0] for p in pairs], device=dev)
        t = torch.tensor([p[1] for p in pairs], device=dev)
        return pairs, Xd[s], heat_torch.fields(phi, Xd[s], t)

    def put_many(pairs, Xs, F):
        Xh = Xs.cpu().numpy()
        for i, (s, t) in enumerate(pairs):
            r = ctx.put(s, t, Xh[i], F[i])
            assert r == 0, "staging ring full"

    # warm-up phase 1: stream until the reservoir is full (P:321 C = 6000)
    filled = 0
    while filled < CAP:
        pairs, Xs, F = next_batch(16)
        put_many(pairs, Xs, F)
        filled += len(pairs)
        st, _, _ = ctx.sample()
        ctx.step(want_loss=False)
        torch.cuda.current_stream(dev).synchronize()
    # device-resident pool of the timed steps' streamed fields
    total_steps = args.warmup + args.steps
    pool = [next_batch(k) for _ in range(total_steps + 12)]
    torch.cuda.synchronize()

    def one_step(i, want_loss=False):
        pairs, Xs, F = pool[i]
        Xh = pool_X[i]
        for j, (s, t) in enumerate(pairs):
            ctx.put(s, t, Xh[j], F[j], zero_copy=True)   # the pool outlives the run
        ctx.sample()
        return ctx.step(want_loss=want_loss)

    pool_X = [p[1].cpu().numpy() for p in pool]
    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        if world == 1:
            return v
        tt = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return tt.item()

    # ---- timed region (device-resident inputs) ----
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.nvtx.range_push("timed")
        ev0.record(stream)
        win_ev = [ev0]                              # throughput over windows of 10 steps
        for i in range(args.warmup, total_steps):
            if (i - args.warmup) % 10 == 0 and i > args.warmup:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                win_ev.append(e)
            one_step(i)
        ev1.record(stream)
        if args.steps % 10 == 0:
            win_ev.append(ev1)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launch_count() - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / args.steps
    value = B * world * args.steps / (ms / 1e3)

    if args.profile:
        if rank == 0:
            allc = ctx.debug_counters()
            raw = allc[:160 * 32].reshape(160, 32)
            prof = raw[:148].astype(np.float64)
            tl = allc[160 * 32:160 * 32 + 768].reshape(64, 12).astype(np.int64)
            tl2 = allc[160 * 32 + 768:].reshape(17, 8).astype(np.int64)
            names = {0: "mma_total", 1: "mma_w_full", 2: "mma_h_full", 3: "mma_y_empty", 4: "mma_dy_full",
                     5: "mma_dw_empty", 6: "mma_fwd_issue", 7: "mma_dw_issue", 8: "epi_total", 9: "epi_t_full", 10: "epi_y_full", 11: "epi_dy_empty",
                     12: "epi_adam_load_wait", 13: "epi_dw_readout", 14: "epi_db_bar", 16: "tma_total", 17: "tma_w_empty",
                     18: "tma_h_empty", 24: "ld_total", 25: "ld_t_empty",
                     26: "adam_total", 27: "adam_ring_wait", 28: "adam_loop"}
            k1 = {v: float(prof[:, k].mean()) for k, v in names.items()}
            print(json.dumps({"ms_per_step": ms_step, "value": value, "k1_wait_cycles_mean_per_cta": k1}), flush=True)
            # CTA 0 timeline of the last launch, cycles relative to the MMA warp's tile start
            # (0 W ready, 1 H chunk 0 ready, 2 targets chunk 0, 3 Y chunk 0, 4 dW done,
            #  5 Adam / send done, 6 producer resumes, 7 loader resumes, 8 peers' dW arrived,
            #  9 send performed at the owner, 10 send issued, 11 overlapped Adam of the tile done)
            nt = int(np.count_nonzero(tl[:, 0]))
            for t in range(min(nt, 60)):
                print("tile %2d: " % t + " ".join("%8d" % (tl[t, k] - tl[t, 0] if tl[t, k] else 0) for k in range(12)) +
                      ("  period %d" % (tl[t + 1, 0] - tl[t, 0]) if t + 1 < nt else ""))
            # tile 5 per chunk: 0 fwd issue, 1 dW issue, 2 epilogue has Y, 3 dY in TMEM, 4 epilogue done
            for c in range(16):
                print("chunk %2d: " % c + " ".join("%8d" % (tl2[c, k] - tl[5, 0]) for k in range(5)))
        return 0
    # ---- per-kernel timing pass (CUDA events around each kernel class) ----
    ctx.set_flags(mel.FLAG_TIMING | args.flags)
    ctx.kernel_time_reset()
    n_kt = min(args.steps, 10)
    extra = [next_batch(k) for _ in range(n_kt)]
    extra_X = [e[1].cpu().numpy() for e in extra]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(n_kt):
        pairs, Xs, F = extra[i]
        for j, (s, t) in enumerate(pairs):
            ctx.put(s, t, extra_X[i][j], F[j], zero_copy=True)
        ctx.sample()
        ctx.step(want_loss=False)
    e1.record(stream)
    torch.cuda.synchronize()
    kt_total = e0.elapsed_time(e1)
    kernels = {}
    for kid, name in enumerate(mel.KERNEL_NAMES):
        tms, nl = ctx.kernel_time(kid)
        kernels[name] = {"ms_per_step": tms / n_kt, "share": tms / kt_total if kt_total else None}
    ctx.set_flags(args.flags)
    P = peaks()
    K = HIDDEN[-1]
    n_params = ctx.n_params
    # algorithmic work per launch (SURVEY §8(d) per-unit figures x units):
    # flops of the GEMMs; bytes the algorithm must move (not this design's dY^T round trip)
    # fused: the Adam of W_L runs inside K1 (world 1, or the in-kernel NVLink exchange at
    # world > 1, where each rank updates the 1/R of the rows it owns)
    fused = (not (args.flags & mel.FLAG_UNFUSED_ADAM)) if world == 1 else not (args.flags & mel.FLAG_NCCL_EXCHANGE)
    n_small = n_params - n_field * K                                    # head + biases
    k1_bytes = n_field * (2.0 * K + 2.0 * B + (26.0 * K / world if fused else 4.0 * K))
    alg = {   # name: (flops, bytes)
        "out_fwd_dw": (4.0 * B * n_field * K, k1_bytes),                # Y = H W^T, dW = dY^T H (+ Adam of W_L if fused)
        "out_dh": (2.0 * B * n_field * K, 2.0 * n_field * K),           # dH = dY W
        "adam": (0.0, 28.0 * (n_small if fused else n_params) + (0.0 if fused else 2.0 * n_field * K)),
    }
    tpeak = P.get("bf16_tflops_sustained", P.get("bf16_tflops"))

    def fracs(name):
        f_, b_ = alg[name]
        d = kernels[name]["ms_per_step"] / 1e3
        if d <= 0:
            return None
        return {"tensor": (f_ / d / 1e12, tpeak, "TFLOP/s"), "hbm": (b_ / d / 1e9, P["hbm_gbs"], "GB/s")}

    dom = max(alg, key=lambda n: kernels[n]["ms_per_step"])
    fr = fracs(dom)
    bound = max(fr, key=lambda k: fr[k][0] / fr[k][1])
    achieved, peak, unit_r = fr[bound]
    other = "tensor" if bound == "hbm" else "hbm"
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        ent = prof.get(dom) or prof.get(dom + "_kernel") or {}
        traffic = ent.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"kernel": dom, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit_r,
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json %s" % ("bf16_tflops_sustained" if bound == "tensor" else "hbm_gbs"),
                "secondary": {"bound": other, "achieved": fr[other][0], "unit": fr[other][2],
                              "frac": fr[other][0] / fr[other][1]},
                "algorithmic_bytes": alg[dom][1], "algorithmic_flops": alg[dom][0], "fused_adam": fused}
    if world > 1 and fused and dom == "out_fwd_dw":
        # bytes each rank must push over NVLink per launch: its dW of the rows other ranks own
        # (fp32) and the new bf16 shadow of its own rows to every other rank
        nv_bytes = ((world - 1) / world * n_field * K * (4.0 if args.flags & mel.FLAG_FP32_EXCHANGE else 2.0) +
                    (world - 1) / world * n_field * K * 2.0)
        nv_peak = P.get("nvlink_gbs", 770.0)
        nv_ach = nv_bytes / (kernels[dom]["ms_per_step"] / 1e3) / 1e9
        roofline["nvlink"] = {"bytes_per_launch": nv_bytes, "achieved": nv_ach, "peak": nv_peak, "unit": "GB/s",
                              "frac": nv_ach / nv_peak,
                              "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}
    for name in alg:
        f2 = fracs(name)
        if f2:
            b2 = max(f2, key=lambda k: f2[k][0] / f2[k][1])
            kernels[name]["achieved"] = f2[b2][0]
            kernels[name]["unit"] = f2[b2][2]
            kernels[name]["frac"] = f2[b2][0] / f2[b2][1]
    step_flops = (6.0 * B * n_field * K + 6.0 * B * K * K + 4.0 * B * 6 * K)
    tensor_frac_step = step_flops / (ms_step / 1e3) / 1e12 / P["bf16_tflops"]
    # the step's tensor fraction vs the burst and the sustained peak,
    # and vs the attainable min(peak, I x HBM) of the ideal fused step (I = FLOP / ideal bytes:
    # bf16 targets B*N*2, two reads of the bf16 W_L shadow, 26 B/param of fused Adam)
    ideal_bytes = B * n_field * 2.0 + 2.0 * (K * n_field * 2.0) + 26.0 * n_params
    intensity = step_flops / ideal_bytes
    attainable = min(P["bf16_tflops"], intensity * P["hbm_gbs"] / 1e3)
    step_tflops = step_flops / (ms_step / 1e3) / 1e12
    tensor_roofline = {"step_tflops": step_tflops, "frac_burst": tensor_frac_step,
                       "frac_sustained": step_tflops / P.get("bf16_tflops_sustained", P["bf16_tflops"]),
                       "intensity_flop_per_byte": intensity, "attainable_tflops": attainable,
                       "frac_attainable": step_tflops / attainable}
    windows = None
    if len(win_ev) >= 2:
        w = [win_ev[j].elapsed_time(win_ev[j + 1]) for j in range(len(win_ev) - 1)]
        w = [B * world * 10 / (x / 1e3) for x in w]
        windows = {"steps_per_window": 10, "n": len(w), "mean": float(np.mean(w)), "median": float(np.median(w))}

    # ---- end-to-end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        n_e2e = min(args.steps, 50)
        host = [next_batch(k) for _ in range(n_e2e)]
        host = [(p, Xs.cpu().numpy(), F.cpu().pin_memory()) for p, Xs, F in host]
        torch.cuda.synchronize()
        barrier()
        base = ctx.step_calls
        losses = []
        t0 = time.perf_counter()
        for i, (pairs, Xh, Fh) in enumerate(host):
            for j, (s, t) in enumerate(pairs):
                ctx.put(s, t, Xh[j], Fh[j])          # pinned host -> device (copy stream)
            ctx.sample()
            ctx.step(want_loss=False)
            if i >= 1:                               # device -> host loss of step i-1 while step i runs
                losses.append(ctx.step_result(base + i - 1)[1])
        losses.append(ctx.step_result(base + n_e2e - 1)[1])
        torch.cuda.synchronize()
        wall = max_over_ranks(time.perf_counter() - t0)
        assert len(losses) == n_e2e and all(np.isfinite(losses))
        e2e = {"value": B * world * n_e2e / wall, "unit": UNIT, "h2d_bytes_per_step": k * (4 * n_field + 32),
               "d2h_bytes_per_step": 8, "steps": n_e2e,
               "timing": "host wall clock, max over ranks; each step's loss is read back (mapped pinned "
                         "memory, surrogate_step_result) while the next step runs",
               "last_loss": losses[-1]}

    # ---- validation MSE on 10 held-out simulations (the validation design stream) ----
    val = None
    try:
        n_val = 10
        Xv = torch.from_numpy(design.draw_design(n_val, seed=1, validation=True)).to(dev)
        tv = torch.arange(TAU, device=dev)
        sse, cnt = 0.0, 0
        for i in range(n_val):                       # one simulation (100 time steps, 400 MB) at a time
            Fv = heat_torch.fields(phi, Xv[i:i + 1].repeat(TAU, 1), tv).cpu().numpy()
            mse, _ = ctx.eval(Xv[i:i + 1].repeat(TAU, 1).cpu().numpy(), tv.cpu().numpy().astype(np.uint32), Fv)
            sse += mse * TAU
            cnt += TAU
        mse = sse / cnt
        val = {"mse_normalised": mse, "mse_K2": mse * 400.0 ** 2, "samples": cnt, "simulations": n_val}
    except Exception as e:
        val = {"error": str(e)}
    stats = ctx.stats()

    # ---- secondary line: the paper's own per-GPU batch b = 10, world 1 ----
    # the step is then bound by the Adam over all 257M parameters (7.75 GB of
    # HBM per step -> <= 8.4k samples/s); a second context, the same kernels (the batch runs
    # padded to one 64-row chunk, rows >= 10 masked), C = 1200 so the fill is short
    paper_b = None
    if world == 1 and not args.no_paper_batch:
        try:
            cfg10 = mel.Config(n_field=n_field, hidden=HIDDEN, capacity=1200, threshold=THETA, batch=10,
                               steps_per_sim=TAU, precision=mel.BF16, storage=mel.STORE_BF16, seed=1,
                               staging_entries=32, flags=args.flags)
            c10 = mel.Context(cfg10, device=local, stream=stream.cuda_stream)
            filled = 0
            while filled < 1200:
                pairs, Xs, F = next_batch(16)
                Xh = Xs.cpu().numpy()
                for j, (s_, t_) in enumerate(pairs):
                    assert c10.put(s_, t_, Xh[j], F[j]) == 0
                filled += len(pairs)
                c10.sample(); c10.step(want_loss=False)
                torch.cuda.current_stream(dev).synchronize()
            n10 = 30
            for _ in range(3):
                c10.sample(); c10.step(want_loss=False)
            torch.cuda.synchronize()
            a10, b10 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a10.record(stream)
            for _ in range(n10):
                c10.sample(); c10.step(want_loss=False)
            b10.record(stream)
            torch.cuda.synchronize()
            ms10 = a10.elapsed_time(b10) / n10
            K_ = HIDDEN[-1]
            bytes10 = 26.0 * c10.n_params + n_field * (2.0 * K_ + 2.0 * 10)   # fused Adam + W shadow + targets
            paper_b = {"batch": 10, "samples_per_s": 10 / (ms10 / 1e3), "ms_per_step": ms10, "steps": n10,
                       "ideal_hbm_bytes": bytes10, "hbm_gbs": bytes10 / (ms10 / 1e3) / 1e9,
                       "hbm_frac": bytes10 / (ms10 / 1e3) / 1e9 / peaks()["hbm_gbs"],
                       "note": "P:317 per-GPU batch; optimizer-bound (SURVEY 8(d): <= 8.4k samples/s per GPU)"}
            c10.close_ctx()
        except Exception as e:  # secondary measurement only
            paper_b = {"error": str(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # real paper-shape oracle steps at B = 8 on the host cores, all-core
        # BLAS and single-threaded; the reservoir holds heat solutions of this run's design
        Fh = heat_torch.fields(phi, Xd[:8], torch.arange(8, device=dev) * 12).cpu().numpy()
        r = oracle_paper_rate(n_field, 10.0, fields=list(Fh), max_steps=1)
        (v_all, n_all, th_all), (v_one, n_one, _) = r["all_cores"], r["single_thread"]
        cpu = {"value": v_all, "unit": UNIT, "cores": th_all, "host_cores": len(os.sched_getaffinity(0)),
               "kind": "oracle", "single_thread": {"value": v_one, "cores": 1, "steps": n_one},
               "sample": "real paper-shape oracle training steps (fp64 numpy, 6-256-256-%d, Adam over all "
                         "257M parameters) at B=8: %d timed steps with BLAS on all cores (value) and %d "
                         "single-threaded, after 1 warm-up step, median" % (n_field, n_all, n_one)}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (exact heat-equation solutions, seeded)",
            "config": config_block(args, world), "gpu_launches": launches, "clocks": clk.summary(),
            "roofline": roofline, "tensor_frac_step": tensor_frac_step, "tensor_roofline": tensor_roofline,
            "windows_samples_per_s": windows, "kernels": kernels, "paper_batch_b10": paper_b,
            "cpu_baseline": cpu, "e2e": e2e, "val_mse": val,
            "reservoir": {"population": stats["population"], "unseen": stats["unseen"],
                          "evictions": stats["evictions"], "puts": stats["puts"], "draws": stats["draws"],
                          "repeats_per_unique": stats["draws"] / max(1, stats["committed"]),
                          # how many times the evicted items had been seen (retired-count
                          # histogram, last bin saturates), as {seen_count: items}
                          "evicted_seen_hist": {int(i): int(v) for i, v in enumerate(stats["hist"]) if v}}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close_ctx()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
