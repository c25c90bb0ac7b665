import sys, time, json, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_18015_b200 as cpb
from oracle import critprob_oracle as orc
vals = orc.ackley_ensemble(64, 64, 50, noise_amp=0.3, seed=0)
f = cpb.UncertainField.from_ensemble(cpb.EnsembleStack(vals), cpb.ModelSpec("uniform"))
for est in (cpb.EstimatorSpec("monte_carlo", n_samples=2000, seed=0), cpb.EstimatorSpec("closed_form")):
    for ch in (("min",), ("saddle",)):
        cpb.classify_field(f, est, channels=ch)
        ts = []
        for _ in range(20):
            t = time.perf_counter(); cpb.classify_field(f, est, channels=ch); ts.append(time.perf_counter() - t)
        print(json.dumps({"method": est.method, "ch": ch, "median_us": round(statistics.median(ts) * 1e6, 1)}))
