"""Small invocations of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: the fits (single-model TMA ring per kind, the fused multi-model fit),
the closed-form stencils (uniform, Epanechnikov piece-parallel, histogram
state tables at bins 5 / 8 / 16, the bins > 16 fallback), the mixed-precision
variants, Monte Carlo (both RNGs, all kinds: the two-stage candidate ring of
Epanechnikov / histogram), semianalytical, combinatorial, the per-case
batches and the host pipeline (cpb_run_host_models).  Sizes are small
(sanitizers replay every access) but larger than one tile in both axes, with
ragged edges.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402


def main():
    torch.cuda.set_device(0)
    vals = orc.ackley_ensemble(70, 21, 20, noise_amp=0.3, seed=0)
    vals[:, 3, 4] = vals[0, 3, 4]  # one degenerate pixel (eps widening, exact mode)
    stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
    for kind, bins in (("uniform", 5), ("epanechnikov", 5), ("histogram", 5), ("histogram", 8),
                       ("histogram", 16), ("histogram", 24), ("gaussian", 5)):
        f = cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec(kind, bins=bins))
        _ = f.params
        if kind != "gaussian":
            cpb.classify_field(f)
            if kind != "histogram":
                cpb.classify_field(f, cpb.EstimatorSpec(precision="mixed"))
        for rng in ("splitmix64", "philox"):
            cpb.classify_field(f, cpb.EstimatorSpec("monte_carlo", n_samples=300, seed=2, rng=rng))
        if kind == "histogram":
            cpb.classify_field(f, cpb.EstimatorSpec("semianalytical", c=200, seed=1))
            if bins <= 8:
                cpb.classify_field(f, cpb.EstimatorSpec("combinatorial"))
    models = [cpb.ModelSpec("uniform"), cpb.ModelSpec("epanechnikov"), cpb.ModelSpec("histogram", bins=5)]
    fs = cpb.UncertainField.from_ensemble_models(stack, models)
    for f in fs:
        cpb.classify_field(f)
    cases = [cpb.random_case(s, model=m) for s in range(6) for m in ("uniform", "epanechnikov", "histogram")]
    cpb.closed_form_triples(cases)
    cpb.mc_all_patterns_batch(cases, 3000, seed=3)
    # host pipeline: two models over one upload
    from paper_2407_18015_b200 import _lib
    import ctypes

    lib = _lib.load()
    M, H, W = vals.shape
    host = np.ascontiguousarray(vals)
    outs = [np.zeros((H, W)) for _ in range(6)]
    valid = np.zeros((H, W), dtype=np.uint8)
    ptrs = (ctypes.c_void_p * 6)(*[o.ctypes.data for o in outs])
    kinds = (ctypes.c_int32 * 2)(0, 2)
    bins = (ctypes.c_int32 * 2)(5, 5)
    ks = (ctypes.c_double * 2)(1.0, 1.0)
    _lib.check(lib.cpb_run_host_models(host.ctypes.data, M, H, W, 2, kinds, bins, ks, 0, 0, 0, 7, ptrs,
                                       valid.ctypes.data))
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
