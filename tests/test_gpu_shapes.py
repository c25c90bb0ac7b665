"""Odd shapes through every entry point of the grid path (GPU).

Widths that are not multiples of 4 / 32 / 128, odd member counts, grids of
one band or one segment, member strides that are or are not 16-byte aligned:
the TMA paths (fits, fused fit + stencil) and their fallbacks must agree with
the oracle / with each other on all of them.  A width not divisible by 4 once
faulted the fused kernel (misaligned per-row TMA boxes); these shapes pin
that class of bug across the fit, fused, host-streaming and per-model paths.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402

CLOSED_TOL = 1e-12
# (members, height, width): H W and W modulo 4 both ways, one band (W <= 128),
# a partial last band, a single segment row, odd member counts
SHAPES = [(3, 5, 7), (9, 12, 130), (7, 64, 131), (16, 33, 128), (5, 20, 257), (11, 140, 260),
          (4, 3, 390), (13, 131, 64), (2, 9, 1001)]


def _vals(M, H, W, seed):
    v = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=seed)
    if H > 4 and W > 4:
        v[:, H // 2, W - 2] = v[0, H // 2, W - 2]  # a degenerate pixel near the right edge
    return np.ascontiguousarray(v)


@pytest.mark.parametrize("shape", SHAPES)
def test_fit_and_closed_form_all_models(shape):
    M, H, W = shape
    vals = _vals(M, H, W, seed=M + H + W)
    stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
    for kind, bins in (("uniform", 5), ("epanechnikov", 5), ("histogram", 5), ("histogram", 12)):
        if kind != "uniform" and M < 2:
            continue
        field = cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec(kind, bins=bins))
        ref_params = orc.fit(vals, kind, bins)
        for k, v in ref_params.items():
            assert np.array_equal(field.params[k], v), (shape, kind, k)
        prob = cpb.classify_field(field)
        ref = orc.classify(ref_params, kind)
        for ch in ("min", "max", "saddle"):
            assert np.max(np.abs(prob.channel(ch) - ref[ch])) <= CLOSED_TOL, (shape, kind, ch)


@pytest.mark.parametrize("shape", SHAPES)
def test_multi_model_fit_matches_single(shape):
    M, H, W = shape
    if M < 2:
        pytest.skip("epanechnikov needs two members")
    vals = _vals(M, H, W, seed=2 * M + W)
    stack = cpb.EnsembleStack(torch.as_tensor(vals, device="cuda"))
    models = [cpb.ModelSpec("uniform"), cpb.ModelSpec("epanechnikov"), cpb.ModelSpec("histogram", bins=5)]
    for m, f in zip(models, cpb.UncertainField.from_ensemble_models(stack, models)):
        for k, v in orc.fit(vals, m.kind, m.bins).items():
            assert np.array_equal(f.params[k], v), (shape, m.kind, k)


@pytest.mark.parametrize("shape", SHAPES)
def test_fused_uniform_matches_separate(shape):
    """cpb_fit_classify (fused where the layout allows, else fit + finish) ==
    cpb_fit + the closed form, bit for bit."""
    from test_gpu_parity import _fused_uniform, _fit

    M, H, W = shape
    if H < 3 or W < 3:
        pytest.skip("no interior")
    vals = _vals(M, H, W, seed=3 * M + H)
    dev, out, counts, _ = _fused_uniform(vals)
    ref = cpb.classify_field(_fit(vals, "uniform"))
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(out[c], ref.channel(ch)), (shape, ch)


@pytest.mark.parametrize("shape", SHAPES)
def test_run_host_models_matches_oracle(shape):
    from paper_2407_18015_b200 import _lib

    M, H, W = shape
    if M < 2:
        pytest.skip("epanechnikov needs two members")
    vals = _vals(M, H, W, seed=5 * M + W)
    lib = _lib.load()
    models = [("uniform", 5), ("epanechnikov", 5), ("histogram", 4)]
    outs = [np.full((H, W), np.nan) for _ in range(3 * len(models))]
    valid = np.zeros((H, W), dtype=np.uint8)
    kinds = (ctypes.c_int32 * 3)(*[_lib.KIND_CODES[k] for k, _ in models])
    bins = (ctypes.c_int32 * 3)(*[b for _, b in models])
    ks = (ctypes.c_double * 3)(*[float(cpb.ModelSpec(k).k) for k, _ in models])
    ptrs = (ctypes.c_void_p * 9)(*[o.ctypes.data for o in outs])
    _lib.check(lib.cpb_run_host_models(vals.ctypes.data, M, H, W, 3, kinds, bins, ks, 0, 0, 0, 7,
                                       ptrs, valid.ctypes.data))
    for i, (kind, b) in enumerate(models):
        ref = orc.classify(orc.fit(vals, kind, b), kind)
        for c, ch in enumerate(("min", "max", "saddle")):
            assert np.max(np.abs(outs[3 * i + c] - ref[ch])) <= CLOSED_TOL, (shape, kind, ch)
