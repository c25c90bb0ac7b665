"""The reference's ten acceptance gates (pkg/tests/test_acceptance.py), run on
the B200 path with the same thresholds.

Gate 2 (closed form vs MC(1e6), 1500 cases) lives in test_gpu_cases.py
(test_acceptance_closed_vs_mc_1e6).  Timing gates compare this path's own
estimators (closed form vs Monte Carlo, 1x vs 2x pixels) on the GPU.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402

BOUNDED = ("uniform", "epanechnikov", "histogram")


def _iid_dist(kind):  # test_acceptance.py:36-41
    if kind == "uniform":
        return cpb.uniform(-0.7, 1.1)
    if kind == "epanechnikov":
        return cpb.epanechnikov(0.2, 0.9)
    return cpb.histogram(-1.0, 1.0, [0.1, 0.3, 0.25, 0.2, 0.15])


def _uniform_ackley_field(width, height, members=50, seed=0):  # test_acceptance.py:44-46
    vals = orc.ackley_ensemble(width, height, members, noise_amp=0.3, seed=seed)
    return cpb.UncertainField.from_ensemble(cpb.EnsembleStack(vals), cpb.ModelSpec("uniform"))


def test_01_symmetry_exactness():
    five = [cpb.NeighborhoodCase(_iid_dist(k), tuple(_iid_dist(k) for _ in range(4))) for k in BOUNDED]
    three = [cpb.NeighborhoodCase(_iid_dist(k), tuple(_iid_dist(k) for _ in range(2))) for k in BOUNDED]
    t5 = cpb.closed_form_triples(five)
    t3 = cpb.closed_form_triples(three)
    worst = max(np.max(np.abs(t5 - [0.2, 0.2, 1.0 / 15.0])), np.max(np.abs(t3 - 1.0 / 3.0)),
                np.max(np.abs(t3.sum(axis=1) - 1.0)))
    assert worst <= 1e-9, worst


def test_03_histogram_combinatorial_equivalence():
    cases = [cpb.random_case(3000 + i, model="histogram", bins=1 + i % 4) for i in range(200)]
    fast = cpb.closed_form_triples(cases)[:, 0]
    direct = cpb.combinatorial_batch(cases)[:, 0]
    assert np.max(np.abs(fast - direct)) <= 1e-9


def test_04_mc_convergence_toward_closed_form():
    """convergence_study(field, "min", [100, 2000], seed=1): RMSE ratio in [2, 7]."""
    field = _uniform_ackley_field(64, 64)
    ref = cpb.classify_field(field)
    rmse = []
    for n in (100, 2000):
        est = cpb.classify_field(field, cpb.EstimatorSpec("monte_carlo", n_samples=n, seed=1))
        d = ref.p_min[ref.valid] - est.p_min[ref.valid]
        rmse.append(math.sqrt(float(np.mean(d * d))))
    coarse, fine = rmse
    assert fine < coarse and 2.0 <= coarse / fine <= 7.0, (coarse, fine)


def test_05_closed_form_faster_than_mc():
    """closed form >= 10x faster than MC(2000) (device time, warm, 1024^2 grid)."""
    vals = orc.ackley_ensemble(1024, 1024, 20, noise_amp=0.3, seed=0)
    field = cpb.UncertainField.from_ensemble(cpb.EnsembleStack(torch.as_tensor(vals, device="cuda")),
                                             cpb.ModelSpec("uniform"))

    def timed(est, channels):
        cpb.classify_field(field, est, channels=channels, output="device")
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cpb.classify_field(field, est, channels=channels, output="device")
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    for channel in ("min", "saddle"):
        t_mc = timed(cpb.EstimatorSpec("monte_carlo", n_samples=2000, seed=0), (channel,))
        t_cf = timed(cpb.EstimatorSpec("closed_form"), (channel,))
        assert t_mc >= 10.0 * t_cf, (channel, t_mc, t_cf)


def _window_mean(prob, peaks):  # bench.py:175-182
    vals = []
    for r, c in peaks:
        assert prob.valid[r - 1:r + 2, c - 1:c + 2].all()
        vals.append(prob.p_max[r - 1:r + 2, c - 1:c + 2])
    return float(np.mean(vals))


def test_06_outlier_robustness_ordering():
    """robustness_ratio (bench.py:185-212) on gaussian_mixture_ensemble(128, 128, 40, 10, 0):
    histogram > uniform and Epanechnikov >= uniform."""
    vals, peaks, outliers = orc.gaussian_mixture_ensemble(128, 128, 40, 10, 0)
    stack = cpb.EnsembleStack(vals)
    ratios = {}
    for label, model in (("uniform", cpb.ModelSpec("uniform")),
                         ("epanechnikov", cpb.ModelSpec("epanechnikov")),
                         ("histogram", cpb.ModelSpec("histogram", bins=5))):
        prob = cpb.classify_field(cpb.UncertainField.from_ensemble(stack, model), channels=("max",))
        num, den = _window_mean(prob, peaks), _window_mean(prob, outliers)
        ratios[label] = math.inf if den == 0.0 and num > 0.0 else num / den
    assert ratios["histogram"] > ratios["uniform"] and ratios["epanechnikov"] >= ratios["uniform"], ratios


def test_07_affine_invariance():
    cases = [cpb.random_case(5000 + i, model=BOUNDED[i % 3]) for i in range(100)]
    base = cpb.closed_form_triples(cases)
    worst = 0.0
    for alpha in (1e-3, 1.0, 1e3):
        for beta in (-10.0, 0.0, 10.0):
            moved = cpb.closed_form_triples([c.affine(alpha, beta) for c in cases])
            worst = max(worst, float(np.max(np.abs(moved - base))))
    assert worst < 1e-9, worst


def test_08_semianalytical_convergence():
    cases = [cpb.random_case(7000 + i, model="histogram", bins=5) for i in range(100)]
    closed = cpb.closed_form_triples(cases)
    px = np.arange(100, dtype=np.uint64)
    est = cpb.semianalytical_batch(cases, 10_000, seed=11, pixels=px)
    again = cpb.semianalytical_batch(cases, 10_000, seed=11, pixels=px)
    assert np.array_equal(est, again)
    assert math.sqrt(float(np.mean((est - closed) ** 2))) < 0.01
    vals = orc.ackley_ensemble(16, 16, 12, noise_amp=0.3, seed=2)
    field = cpb.UncertainField.from_ensemble(cpb.EnsembleStack(vals), cpb.ModelSpec("histogram", bins=4))
    spec = cpb.EstimatorSpec("semianalytical", c=10_000, seed=3)
    one = cpb.classify_field(field, spec, workers=1)
    two = cpb.classify_field(field, spec, workers=2)
    assert all(np.array_equal(one.channel(ch), two.channel(ch)) for ch in ("min", "max", "saddle"))


def test_09_parallel_determinism_and_pixel_scaling():
    field = _uniform_ackley_field(48, 48, members=12, seed=4)
    for spec in (cpb.EstimatorSpec("closed_form"), cpb.EstimatorSpec("monte_carlo", n_samples=400, seed=7)):
        one = cpb.classify_field(field, spec, workers=1)
        two = cpb.classify_field(field, spec, workers=2)
        assert all(np.array_equal(one.channel(ch), two.channel(ch)) for ch in ("min", "max", "saddle"))
        assert np.array_equal(one.valid, two.valid)
    # device time of the closed form at 1x and 2x pixels (large enough to be work-bound)
    small = _uniform_ackley_field(1024, 1024, members=12, seed=5)
    large = _uniform_ackley_field(2048, 1024, members=12, seed=5)

    def t(f):
        cpb.classify_field(f, output="device")
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            cpb.classify_field(f, output="device")
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    assert t(large) / t(small) <= 2.5


def test_10_two_neighborhood_completeness():
    cases = [cpb.random_case(9000 + i, model=BOUNDED[i % 3], neighborhood=2) for i in range(500)]
    totals = cpb.closed_form_triples(cases).sum(axis=1)
    assert np.max(np.abs(totals - 1.0)) <= 1e-9
