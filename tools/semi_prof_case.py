"""Small semianalytical run for ncu (1024^2 histogram(5) field, c = 2000)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402

vals = orc.ackley_ensemble(1024, 1024, 20, noise_amp=0.3, seed=0)
stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
f = cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec("histogram", bins=5))
cpb.classify_field(f, cpb.EstimatorSpec("semianalytical", c=2000, seed=0), output="device")
torch.cuda.synchronize()
print("ok")
