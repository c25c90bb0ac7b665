"""Pin the CPU oracle to the reference's own outputs (golden fixtures).

The fixtures come from running /root/reference's critprob package
(tests/golden/make_golden.py).  Fit and Monte Carlo must match bit for bit;
the closed form within 1e-13 absolute (the oracle re-associates nothing but
numpy's BLAS dot may; observed 0).
"""

import numpy as np
import pytest

from oracle import critprob_oracle as orc

FIT_PARAMS = {"uniform": ("lo", "hi"), "histogram": ("lo", "hi", "weights"),
              "epanechnikov": ("mean", "halfwidth"), "gaussian": ("mean", "stddev")}


def _cases(gold, prefix_filter=None):
    tags = sorted({k.rsplit("/", 1)[0] for k in gold if k.count("/") == 3})
    return tags


def test_fit_bitexact(golden):
    fit = golden["fit"]
    seen = 0
    for key in fit:
        if not key.startswith("ens/"):
            continue
        name = key.split("/", 1)[1]
        ens = fit[key]
        for k2 in fit:
            parts = k2.split("/")
            if len(parts) != 4 or parts[0] != name:
                continue
            _, kind, bins, pname = parts
            got = orc.fit(ens, kind, bins=int(bins))
            assert np.array_equal(got[pname], fit[k2]), k2
            seen += 1
    assert seen > 40


def test_from_scalar_bitexact(golden):
    fit = golden["fit"]
    for eb in (0.5, 0.0):
        got = orc.from_scalar(fit["scalar/raster"], eb)
        assert np.array_equal(got["lo"], fit[f"scalar/{eb}/lo"])
        assert np.array_equal(got["hi"], fit[f"scalar/{eb}/hi"])


def test_closed_form_matches_reference(golden):
    fit, closed = golden["fit"], golden["closed"]
    seen = 0
    for key in closed:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "min":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        params = orc.fit(fit[f"ens/{name}"], kind, bins=bins)
        got = orc.classify(params, kind)
        for ch in ("min", "max", "saddle"):
            ref = closed[f"{name}/{kind}/{bins}/{ch}"]
            assert np.max(np.abs(got[ch] - ref)) <= 1e-13, (key, ch)
        seen += 1
    assert seen >= 30


def test_closed_form_known_answer(golden):
    closed = golden["closed"]
    got = orc.classify({"lo": closed["kat3x3/lo"], "hi": closed["kat3x3/hi"]}, "uniform")
    # test_engine.py:161-163 pins
    assert got["min"][1, 1] == pytest.approx(0.41865234375, abs=1e-12)
    assert got["max"][1, 1] == pytest.approx(0.008170572916666667, abs=1e-12)
    assert got["saddle"][1, 1] == pytest.approx(0.1377604166666667, abs=1e-12)
    for ch in ("min", "max", "saddle"):
        assert np.max(np.abs(got[ch] - closed[f"kat3x3/{ch}"])) <= 1e-15


def test_iid_symmetry():
    # test_engine.py:85-111: i.i.d. neighbourhoods give (0.2, 0.2, 1/15)
    for kind, params in (
        ("uniform", {"lo": np.zeros((3, 3)), "hi": np.ones((3, 3))}),
        ("epanechnikov", {"mean": np.full((3, 3), 2.0), "halfwidth": np.full((3, 3), 0.7)}),
        ("histogram", {"lo": np.zeros((3, 3)), "hi": np.ones((3, 3)),
                       "weights": np.tile([0.1, 0.3, 0.25, 0.2, 0.15], (3, 3, 1))}),
    ):
        got = orc.classify(params, kind)
        assert got["min"][1, 1] == pytest.approx(0.2, abs=1e-12)
        assert got["max"][1, 1] == pytest.approx(0.2, abs=1e-12)
        assert got["saddle"][1, 1] == pytest.approx(1.0 / 15.0, abs=1e-12)


def test_from_scalar_closed(golden):
    fit, closed = golden["fit"], golden["closed"]
    for eb in (0.5, 0.0):
        got = orc.classify(orc.from_scalar(fit["scalar/raster"], eb), "uniform")
        for ch in ("min", "max", "saddle"):
            assert np.max(np.abs(got[ch] - closed[f"scalar/{eb}/{ch}"])) <= 1e-13


def test_monte_carlo_bitexact(golden):
    fit, mc = golden["fit"], golden["mc"]
    seen = 0
    for key in mc:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "n":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        n = int(mc[key])
        params = orc.fit(fit[f"ens/{name}"], kind, bins=bins)
        got = orc.classify(params, kind, method="monte_carlo", n_samples=n, seed=9)
        for ch in ("min", "max", "saddle"):
            assert np.array_equal(got[ch], mc[f"{name}/{kind}/{bins}/{ch}"]), (key, ch)
        seen += 1
    assert seen >= 12


def test_rng_bitexact(golden):
    rng = golden["rng"]
    px = rng["pixels"]
    for seed in (0, 7, -1, 2**64 - 2, 123456789):
        assert np.array_equal(orc.uniforms(seed, px, 3, 11), rng[f"{seed}"])


def test_rng_prefix_and_offset():
    a = orc.uniforms(5, np.arange(3), 2, 50)
    b = orc.uniforms(5, np.arange(3), 2, 20, start=30)
    assert np.array_equal(a[:, :, 30:], b)


def test_synthetic_rows_consistent():
    full = orc.synthetic_rows(0, 12, 10, 12, 6)
    part = orc.synthetic_rows(5, 4, 10, 12, 6)
    assert full.dtype == np.float32 and full.shape == (6, 12, 10)
    assert np.array_equal(full[:, 5:9], part)


def test_semianalytical_bitexact(golden):
    fit, semi = golden["fit"], golden["semi"]
    seen = 0
    for key in semi:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "c":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        c = int(semi[key])
        params = orc.fit(fit[f"ens/{name}"], kind, bins=bins)
        got = orc.classify(params, kind, method="semianalytical", n_samples=c, seed=2)
        for ch in ("min", "max", "saddle"):
            assert np.array_equal(got[ch], semi[f"{name}/{kind}/{bins}/{ch}"]), (key, ch)
        seen += 1
    assert seen >= 6


def test_synthetic_generators_match_reference(golden):
    """The oracle's ackley_ensemble and gaussian_mixture_ensemble (synth.py:54-121)
    reproduce the reference's bytes (used to build the acceptance-gate inputs)."""
    g = golden["synth"]
    vals, peaks, outliers = orc.gaussian_mixture_ensemble(32, 32, 6, 3, 4)
    assert np.array_equal(vals, g["mixture"])
    assert [tuple(p) for p in g["peaks"]] == peaks and [tuple(p) for p in g["outlier_peaks"]] == outliers
    assert np.array_equal(orc.ackley_ensemble(20, 12, 5, noise_amp=0.3, seed=7), g["ackley"])
