"""Grid Monte Carlo at BASELINE config 4 (2048 x 2048 Ackley, 20 members, 10k samples).

Prints one JSON line per model: joint draws per second (device time, CUDA
events around cpb_classify_mc on a resident field), the closed-form check
(fraction of vertices within 4 binomial SE, test_acceptance.py:75-97) and the
ncu-free pipe story is left to profiles/.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2407_18015_b200 as cpb
    from oracle import critprob_oracle as orc

    H = W = int(os.environ.get("MC_SIZE", 2048))
    n = int(os.environ.get("MC_N", 10_000))
    vals = orc.ackley_ensemble(W, H, 20, noise_amp=0.3, seed=0)
    stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
    for kind in ("uniform", "epanechnikov", "histogram"):
        field = cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec(kind))
        for rng in ("splitmix64", "philox"):
            est = cpb.EstimatorSpec("monte_carlo", n_samples=n, seed=0, rng=rng)
            cpb.classify_field(field, cpb.EstimatorSpec("monte_carlo", n_samples=64, seed=0, rng=rng),
                               output="device")
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            prob = cpb.classify_field(field, est, output="device")
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1)
            closed = cpb.classify_field(field, output="device")
            frac = {}
            for ch in ("min", "max", "saddle"):
                p = closed.channel(ch)[1:-1, 1:-1]
                q = prob.channel(ch)[1:-1, 1:-1]
                se = torch.sqrt(p * (1 - p) / n)
                frac[ch] = round(float(((q - p).abs() <= 4 * se + 1e-15).double().mean()), 5)
            draws = (H - 2) * (W - 2) * n
            print(json.dumps({"model": kind, "rng": rng, "n": n, "grid": [H, W], "ms": round(ms, 2),
                              "gdraws_per_s": round(draws / ms / 1e6, 2), "within_4se": frac}))


if __name__ == "__main__":
    main()
