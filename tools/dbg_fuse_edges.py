"""Which (shape, degenerate pixels) make the fused uniform kernel fail? One case per process."""
import subprocess, sys, json
cases = [((9, h, w), []) for h, w in ((200, 390), (200, 392), (200, 394), (200, 391), (200, 393), (200, 130), (200, 131), (200, 258), (40, 390), (8, 390))]
code = r'''
import sys, json, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch
from oracle import critprob_oracle as orc
import test_gpu_parity as T
(M, H, W), degs = json.loads(sys.argv[1])
vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=11)
for r, c in degs:
    vals[:, r, c] = vals[0, r, c]
try:
    T._fused_uniform(vals)
    print("ok")
except Exception as e:
    print("FAIL", str(e)[:120])
'''
import os
for shape, degs in cases:
    r = subprocess.run([sys.executable, "-c", code, json.dumps([shape, degs])], capture_output=True, text=True, timeout=300)
    print(shape, degs, (r.stdout.strip().splitlines() or [r.stderr.strip()[-200:]])[-1])
