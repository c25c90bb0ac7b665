import sys, os, subprocess
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
shape = tuple(int(x) for x in sys.argv[1].split(","))
import numpy as np, torch
sys.path.insert(0, "tests")
os.environ["CUDA_LAUNCH_BLOCKING"] = "1"
import test_gpu_parity as T
from oracle import critprob_oracle as orc
M, H, W = shape
vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=1)
try:
    dev, out, counts, rng = T._fused_uniform(vals)
    import paper_2407_18015_b200 as cpb
    ref = cpb.classify_field(T._fit(vals, "uniform"))
    print(shape, "ok", [float(np.max(np.abs(out[c] - ref.channel(ch)))) for c, ch in enumerate(("min","max","saddle"))])
except Exception as e:
    print(shape, "ERR", repr(e)[:300])
