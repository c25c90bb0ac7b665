import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2407_18015_b200 as cpb
from oracle import critprob_oracle as orc
vals = orc.ackley_ensemble(1024, 1024, 20, noise_amp=0.3, seed=0)
stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
for kind in ("epanechnikov", "histogram"):
    f = cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec(kind))
    cpb.classify_field(f, cpb.EstimatorSpec("monte_carlo", n_samples=2000, seed=0), output="device")
torch.cuda.synchronize()
print("ok")
