import numpy as np, sys
sys.path.insert(0, '.')
import paper_2407_18015_b200 as cpb
from oracle import critprob_oracle as orc
rng = np.random.default_rng(12)
tiny = np.float32(1e-45)
special = np.array([-0.0, 0.0, tiny, -tiny, -1.0, 1.0, 0.5, -0.5, 1e-38, -1e-38], dtype=np.float32)
H, W, M = 6, 40, 23
vals = rng.choice(special, size=(M, H, W)).astype(np.float32)
vals[0] = -1.0
vals[1] = 1.0
vals[:, 5, :20] = rng.uniform(-1, 1, (M, 20)).astype(np.float32)
for bins in (2, 3, 4, 5, 8, 9):
    got = cpb.UncertainField.from_ensemble(cpb.EnsembleStack(vals), cpb.ModelSpec("histogram", bins=bins)).params
    ref = orc.fit(vals, "histogram", bins)
    for k in ref:
        bad = np.argwhere(got[k] != ref[k])
        if len(bad):
            r, c = bad[0][:2]
            print(bins, k, len(bad), (r, c), got[k][r, c], ref[k][r, c], sorted(vals[:, r, c].tolist()))
