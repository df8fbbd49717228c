"""CPU emulation (not a test): which bf16 operand of the output layer drives the
free-running drift from the fp64 trajectory?  Variants round W3, H2 and/or dY to
bf16 (RNE) inside an otherwise fp64 oracle step; same op-log as the GPU test."""
import os, sys, time
from dataclasses import replace
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from mel_inputs import design, heat
from oracle import mlp, reservoir as ores

def rne(x):
    return ores.bf16_bits_to_f64(ores.f32_to_bf16_bits(np.asarray(x, np.float32)))

def run(variant, steps=1000):
    wl = replace(design.MEDIUM, name="m1k", capacity=6000, threshold=1000, sims=1100)
    X = design.draw_design(wl.sims, seed=1)
    phi = heat.basis(wl.n, wl.tau)
    res = ores.Reservoir(wl.capacity, wl.threshold, wl.n_field, seed=1, storage=1)
    tens = [x.astype(np.float64) for x in mlp.flatten(mlp.init_params(mlp.layer_dims(wl.n_field, wl.hidden), 1))]
    opt = mlp.Adam(tens); S = 0; losses = []
    for op in design.build_oplog(wl):
        if op[0] == "PUT":
            _, r, s, t = op; res.put(s, t, X[s], heat.fields_from_basis(phi, X[s], t))
        elif op[0] == "SAMPLE":
            st, sl = res.sample(wl.batch)
        elif op[0] == "STEP":
            if st != 0: continue
            sl_ = np.asarray(sl)
            xn = mlp.normalise_inputs(res.X[sl_], res.t[sl_], wl.tau); tn = ores.stored_to_f64(res.payload[sl_], 1)
            W1, b1, W2, b2, W3, b3 = tens
            Z1 = xn @ W1.T + b1; H1 = np.maximum(Z1, 0); Z2 = H1 @ W2.T + b2; H2 = np.maximum(Z2, 0)
            H2q = rne(H2) if "H" in variant else H2
            W3q = rne(W3) if "W" in variant else W3
            Y = H2q @ W3q.T + b3; R = Y - tn; N = R.size
            losses.append(float(np.mean(R * R)))
            dY = 2 * R / N
            dYq = rne(dY * N) / N if "D" in variant else dY
            gW3 = dYq.T @ H2q; gb3 = dY.sum(0); dH2 = dYq @ W3q
            dZ2 = dH2 * (Z2 > 0); gW2 = dZ2.T @ H1; gb2 = dZ2.sum(0); dZ1 = (dZ2 @ W2) * (Z1 > 0)
            gW1 = dZ1.T @ xn; gb1 = dZ1.sum(0)
            tens = opt.step(tens, [gW1, gb1, gW2, gb2, gW3, gb3], mlp.lr_schedule(S)); S += len(sl_)
            if len(losses) == steps: break
    return np.array(losses)

if __name__ == "__main__":
    t0 = time.time()
    base = run("")
    np.save("/tmp/emu_base.npy", base)
    for v in sys.argv[1:]:
        l = run(v)
        e = np.abs(l - base) / base
        print("variant %-4s step1000 rel err %.2e  mean(951-1000) %.2e  (%.0fs)" % (v, e[-1], e[-50:].mean(), time.time() - t0), flush=True)
