import sys, json, torch
sys.path.insert(0, '.')
import paper_2407_18015_b200 as cpb
from oracle import critprob_oracle as orc
vals = orc.ackley_ensemble(2048, 2048, 20, noise_amp=0.3, seed=0)
stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
for bins in (5, 8):
    f = cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec("histogram", bins=bins))
    for est in (cpb.EstimatorSpec("semianalytical", c=10000, seed=0), cpb.EstimatorSpec("combinatorial"), cpb.EstimatorSpec()):
        cpb.classify_field(f, est, output="device"); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); cpb.classify_field(f, est, output="device"); b.record(); torch.cuda.synchronize()
        print(json.dumps({"bins": bins, "method": est.method, "ms": round(a.elapsed_time(b), 2),
                          "mvert_s": round(2046 * 2046 / a.elapsed_time(b) / 1e3, 1)}))
