"""BASELINE.json configs 1-4 at their full sizes on the GPU (config 5 is bench.py's).

Full-size checks use what the domain offers beyond the oracle's reach:
rows re-computed by the CPU oracle (spot rows), probability bounds, the
min+max+saddle <= 1 identity, and the MC-vs-closed-form binomial bound of
test_acceptance.py:75-97.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402


def _field(vals, kind, bins=5):
    return cpb.UncertainField.from_ensemble(cpb.EnsembleStack(torch.as_tensor(vals, device="cuda")),
                                            cpb.ModelSpec(kind=kind, bins=bins))


def _spot_rows(vals, field, kind, bins, rows, prob):
    """Re-run the oracle on a 3-row window around each spot row; compare."""
    eps = field.device_field().eps
    for r in rows:
        win = vals[:, r - 1:r + 2]
        ref = orc.classify(orc.fit(win, kind, bins, eps=eps), kind)
        for ch in ("min", "max", "saddle"):
            err = np.max(np.abs(prob.channel(ch)[r, 1:-1] - ref[ch][1, 1:-1]))
            assert err <= 1e-12, (kind, bins, r, ch, err)


def _bounds(prob):
    pm, pM, ps = prob.p_min, prob.p_max, prob.p_saddle
    for a in (pm, pM, ps):
        assert a.min() >= -1e-15 and a.max() <= 1 + 1e-12
    assert (pm + pM + ps).max() <= 1 + 1e-12


def test_config1_uniform_64x64x20():
    vals = orc.ackley_ensemble(64, 64, 20, noise_amp=0.3, seed=0)
    prob = cpb.classify_field(_field(vals, "uniform"))
    ref = orc.classify(orc.fit(vals, "uniform"), "uniform")
    for ch in ("min", "max", "saddle"):
        assert np.max(np.abs(prob.channel(ch) - ref[ch])) <= 1e-12


@pytest.mark.parametrize("kind", ["uniform", "epanechnikov"])
def test_config2_500x500x20(kind):
    vals = orc.ackley_ensemble(500, 500, 20, noise_amp=0.3, seed=0)
    field = _field(vals, kind)
    prob = cpb.classify_field(field)
    _bounds(prob)
    _spot_rows(vals, field, kind, 5, (1, 250, 498), prob)
    if kind == "uniform":  # the whole grid is cheap enough for the oracle
        ref = orc.classify(orc.fit(vals, kind), kind)
        for ch in ("min", "max", "saddle"):
            assert np.max(np.abs(prob.channel(ch) - ref[ch])) <= 1e-12


@pytest.mark.parametrize("bins", [8, 16, 32])
def test_config3_histogram_2048x2048x40(bins):
    vals = orc.ackley_ensemble(2048, 2048, 40, noise_amp=0.3, seed=0)
    field = _field(vals, "histogram", bins)
    prob = cpb.classify_field(field)
    _bounds(prob)
    _spot_rows(vals, field, "histogram", bins, (1, 1024, 2046), prob)
    # fit bit-exact on a row band
    band = vals[:, 700:704]
    ref = orc.fit(band, "histogram", bins, eps=field.device_field().eps)
    got = field.params
    for k in ("lo", "hi", "weights"):
        assert np.array_equal(got[k][700:704], ref[k])


@pytest.mark.parametrize("kind", ["uniform", "epanechnikov"])
def test_config4_monte_carlo_2048x2048x20_1e4(kind):
    vals = orc.ackley_ensemble(2048, 2048, 20, noise_amp=0.3, seed=0)
    field = _field(vals, kind)
    n = 10_000
    closed = cpb.classify_field(field)
    holder = {}
    mc = cpb.classify_field(field, cpb.EstimatorSpec(method="monte_carlo", n_samples=n, seed=0),
                            counts_out=holder)
    # binomial bound against the closed form (test_acceptance.py:75-97)
    for ch in ("min", "max", "saddle"):
        p = closed.channel(ch)[1:-1, 1:-1]
        q = mc.channel(ch)[1:-1, 1:-1]
        se = np.sqrt(np.maximum(p * (1 - p), 1e-12) / n)
        assert (np.abs(q - p) <= 4 * se + 1e-12).mean() >= 0.99, ch
    # the reference stream: counts of a few rows equal the oracle's (bit-exact draws)
    counts = holder["counts"].cpu().numpy()
    r = 1234
    win = vals[:, r - 1:r + 2]
    ref_counts = {}
    orc.classify(orc.fit(win, kind, eps=field.device_field().eps), kind, method="monte_carlo",
                 n_samples=n, seed=0, counts_out=ref_counts, row0=r - 1, global_width=2048,
                 block=64)
    for i, ch in enumerate(("min", "max", "saddle")):
        d = np.abs(counts[i, r, 1:-1] - ref_counts[ch][1, 1:-1])
        if kind == "uniform":
            assert d.max() == 0, ch
        else:
            assert d.max() <= 1, ch
