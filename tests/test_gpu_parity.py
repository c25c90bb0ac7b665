"""GPU parity: the sm_100a path through the C ABI against the reference.

Every test calls the product package (ctypes -> libcritprob_b200.so) and
checks it against the golden fixtures produced by the reference itself
(tests/golden/make_golden.py) and against the pinned CPU oracle on seeded
inputs.  Bars (from SURVEY.md section 8 / the north_star):

- fit (lo/hi, counts->weights, mean, std, halfwidth): bit-exact
- closed form (float64): |gpu - ref| <= 1e-12 absolute
- Monte Carlo, splitmix64 stream: uniform/histogram identical counts;
  epanechnikov/gaussian identical except where libm ulps flip an exact tie
  (<= 1 count per channel per pixel, and in practice none)
- keyed uniform stream: bit-exact
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402

CLOSED_TOL = 1e-12


def _fit(vals, kind, bins=5, k=None):
    model = cpb.ModelSpec(kind=kind, bins=bins) if k is None else cpb.ModelSpec(kind=kind, bins=bins, k=k)
    return cpb.UncertainField.from_ensemble(cpb.EnsembleStack(vals), model)


def _models_in(fit):
    out = []
    for key in fit:
        parts = key.split("/")
        if len(parts) == 4 and parts[0] != "scalar":
            out.append((parts[0], parts[1], int(parts[2]), parts[3]))
    return out


# ---------------------------------------------------------------- fit
def test_fit_bitexact_against_reference(golden):
    fit = golden["fit"]
    seen = 0
    cache = {}
    for name, kind, bins, pname in _models_in(fit):
        key = (name, kind, bins)
        if key not in cache:
            cache[key] = _fit(fit[f"ens/{name}"], kind, bins).params
        got = cache[key][pname]
        ref = fit[f"{name}/{kind}/{bins}/{pname}"]
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), (name, kind, bins, pname, np.max(np.abs(got - ref)))
        seen += 1
    assert seen > 40


def test_fit_device_resident_stack_matches_host(golden):
    vals = golden["fit"]["ens/ackley"]
    host = _fit(vals, "histogram", 8).params
    dev = _fit(torch.as_tensor(vals, device="cuda"), "histogram", 8).params
    for k in host:
        assert np.array_equal(host[k], dev[k])


def test_fit_large_members_loop_path():
    rng = np.random.default_rng(5)
    vals = (rng.uniform(-1, 1, (9, 11)) + rng.uniform(-0.3, 0.3, (300, 9, 11))).astype(np.float32)
    for kind, bins in (("uniform", 5), ("epanechnikov", 5), ("gaussian", 5), ("histogram", 7)):
        got = _fit(vals, kind, bins).params
        ref = orc.fit(vals, kind, bins)
        for k in ref:
            assert np.array_equal(got[k], ref[k]), (kind, k)


def test_fit_k_parameter_and_errors():
    rng = np.random.default_rng(6)
    vals = rng.uniform(0, 1, (12, 5, 6)).astype(np.float32)
    got = _fit(vals, "epanechnikov", k=1.0).params["halfwidth"]
    assert np.array_equal(got, orc.fit(vals, "epanechnikov", k=1.0)["halfwidth"])
    single = np.ones((1, 4, 4), dtype=np.float32)
    for kind in ("epanechnikov", "gaussian"):
        with pytest.raises(ValueError):
            _fit(single, kind)
    bad = torch.zeros((3, 4, 4), device="cuda")
    bad[1, 2, 2] = float("nan")
    with pytest.raises(ValueError):
        _fit(bad, "uniform")
    with pytest.raises(ValueError):
        cpb.EnsembleStack(np.full((2, 3, 3), np.inf, dtype=np.float32))


def test_from_scalar_bitexact(golden):
    fit = golden["fit"]
    for eb in (0.5, 0.0):
        f = cpb.UncertainField.from_scalar(fit["scalar/raster"], eb)
        assert np.array_equal(f.params["lo"], fit[f"scalar/{eb}/lo"])
        assert np.array_equal(f.params["hi"], fit[f"scalar/{eb}/hi"])
    with pytest.raises(ValueError):
        cpb.UncertainField.from_scalar(np.ones((3, 3)), -0.1)


# ---------------------------------------------------------------- closed form
def test_closed_form_against_reference(golden):
    fit, closed = golden["fit"], golden["closed"]
    seen = 0
    for key in closed:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "min":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        prob = cpb.classify_field(_fit(fit[f"ens/{name}"], kind, bins))
        for ch in ("min", "max", "saddle"):
            ref = closed[f"{name}/{kind}/{bins}/{ch}"]
            err = np.max(np.abs(prob.channel(ch) - ref))
            assert err <= CLOSED_TOL, (name, kind, bins, ch, err)
        assert not prob.valid[0].any() and prob.valid[1:-1, 1:-1].all()
        seen += 1
    assert seen >= 30


def test_closed_form_user_built_fields(golden):
    closed = golden["closed"]
    f = cpb.UncertainField(cpb.ModelSpec("uniform"), {"lo": closed["kat3x3/lo"], "hi": closed["kat3x3/hi"]})
    prob = cpb.classify_field(f)
    assert prob.p_min[1, 1] == pytest.approx(0.41865234375, abs=1e-12)
    assert prob.p_max[1, 1] == pytest.approx(0.008170572916666667, abs=1e-12)
    assert prob.p_saddle[1, 1] == pytest.approx(0.1377604166666667, abs=1e-12)
    for kind, params in (
        ("uniform", {"lo": np.zeros((3, 3)), "hi": np.ones((3, 3))}),
        ("epanechnikov", {"mean": np.full((3, 3), 2.0), "halfwidth": np.full((3, 3), 0.7)}),
        ("histogram", {"lo": np.zeros((3, 3)), "hi": np.ones((3, 3)),
                       "weights": np.tile([0.1, 0.3, 0.25, 0.2, 0.15], (3, 3, 1))}),
    ):
        prob = cpb.classify_field(cpb.UncertainField(cpb.ModelSpec(kind, bins=5), params))
        assert prob.p_min[1, 1] == pytest.approx(0.2, abs=1e-12), kind
        assert prob.p_max[1, 1] == pytest.approx(0.2, abs=1e-12), kind
        assert prob.p_saddle[1, 1] == pytest.approx(1.0 / 15.0, abs=1e-12), kind


def test_closed_form_disjoint_supports():
    # test_engine.py:114-143: certain minimum / maximum
    lo = np.full((3, 3), 2.0)
    hi = np.full((3, 3), 3.0)
    lo[1, 1], hi[1, 1] = 0.0, 1.0
    prob = cpb.classify_field(cpb.UncertainField(cpb.ModelSpec("uniform"), {"lo": lo, "hi": hi}))
    # the reference grid path gives 1.0000000000000002 here (3-node GL weights sum to 2 + 4e-16)
    assert prob.p_min[1, 1] == pytest.approx(1.0, abs=1e-15)
    assert prob.p_max[1, 1] == 0.0 and prob.p_saddle[1, 1] == 0.0
    prob = cpb.classify_field(cpb.UncertainField(cpb.ModelSpec("uniform"), {"lo": -hi, "hi": -lo}))
    assert prob.p_max[1, 1] == pytest.approx(1.0, abs=1e-15) and prob.p_min[1, 1] == 0.0


def test_from_scalar_closed(golden):
    fit, closed = golden["fit"], golden["closed"]
    for eb in (0.5, 0.0):
        prob = cpb.classify_field(cpb.UncertainField.from_scalar(fit["scalar/raster"], eb))
        for ch in ("min", "max", "saddle"):
            assert np.max(np.abs(prob.channel(ch) - closed[f"scalar/{eb}/{ch}"])) <= CLOSED_TOL


@pytest.mark.parametrize("kind,bins,shape,members", [
    ("uniform", 5, (64, 64), 20),          # BASELINE config 1
    ("epanechnikov", 5, (70, 90), 20),     # config 2 model, reduced grid
    ("histogram", 8, (40, 52), 40),        # config 3 bins, reduced grid
    ("histogram", 16, (30, 33), 40),
    ("histogram", 32, (20, 24), 40),
])
def test_closed_form_against_oracle_ackley(kind, bins, shape, members):
    vals = orc.ackley_ensemble(shape[1], shape[0], members, noise_amp=0.3, seed=0)
    field = _fit(vals, kind, bins)
    ref = orc.classify(orc.fit(vals, kind, bins), kind)
    prob = cpb.classify_field(field)
    for ch in ("min", "max", "saddle"):
        err = np.max(np.abs(prob.channel(ch) - ref[ch]))
        assert err <= CLOSED_TOL, (ch, err)


def test_closed_form_offsets_and_degenerate(golden):
    # far-from-origin supports and degenerate pixels mixed into a wide range
    fit = golden["fit"]
    for name in ("offset", "degenerate", "constant", "wide"):
        vals = fit[f"ens/{name}"]
        for kind, bins in (("uniform", 5), ("epanechnikov", 5), ("histogram", 3), ("histogram", 8)):
            ref = orc.classify(orc.fit(vals, kind, bins), kind)
            prob = cpb.classify_field(_fit(vals, kind, bins))
            for ch in ("min", "max", "saddle"):
                err = np.max(np.abs(prob.channel(ch) - ref[ch]))
                assert err <= CLOSED_TOL, (name, kind, bins, ch, err)


@pytest.mark.parametrize("bins", [9, 16, 32, 64])
def test_closed_form_many_bins(golden, bins):
    """bins > 8 (closed_hist_otf_kernel: states derived on the fly from cumulative
    counts): far-offset, degenerate, constant and random stacks against the oracle."""
    fit = golden["fit"]
    for name in ("offset", "degenerate", "constant", "wide", "rand"):
        vals = fit[f"ens/{name}"]
        ref = orc.classify(orc.fit(vals, "histogram", bins), "histogram")
        prob = cpb.classify_field(_fit(vals, "histogram", bins))
        for ch in ("min", "max", "saddle"):
            err = np.max(np.abs(prob.channel(ch) - ref[ch]))
            assert err <= CLOSED_TOL, (name, bins, ch, err)


def test_channel_subset_and_validation(golden):
    vals = golden["fit"]["ens/rand"]
    field = _fit(vals, "uniform")
    full = cpb.classify_field(field)
    only = cpb.classify_field(field, channels="min")
    assert np.array_equal(only.p_min, full.p_min)
    assert np.all(only.p_max == 0.0) and np.all(only.p_saddle == 0.0)
    with pytest.raises(ValueError):
        cpb.classify_field(field, channels=("min", "ridge"))
    with pytest.raises(ValueError):
        cpb.classify_field(field, workers=0)
    with pytest.raises(ValueError):
        cpb.classify_field(_fit(vals, "gaussian"))
    with pytest.raises(ValueError):
        cpb.classify_field(field, cpb.EstimatorSpec(method="semianalytical"))
    tiny = _fit(np.random.default_rng(0).uniform(0, 1, (4, 2, 3)).astype(np.float32), "uniform")
    with pytest.raises(ValueError):
        cpb.classify_field(tiny)


def test_workers_do_not_change_results(golden):
    field = _fit(golden["fit"]["ens/rand"], "histogram", 5)
    one = cpb.classify_field(field, workers=1)
    two = cpb.classify_field(field, workers=4)
    for ch in ("min", "max", "saddle"):
        assert np.array_equal(one.channel(ch), two.channel(ch))


# ---------------------------------------------------------------- Monte Carlo
def test_monte_carlo_bitexact_against_reference(golden):
    fit, mc = golden["fit"], golden["mc"]
    seen = 0
    for key in mc:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "n":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        n = int(mc[key])
        est = cpb.EstimatorSpec(method="monte_carlo", n_samples=n, seed=9)
        prob = cpb.classify_field(_fit(fit[f"ens/{name}"], kind, bins), est)
        for ch in ("min", "max", "saddle"):
            ref = mc[f"{name}/{kind}/{bins}/{ch}"]
            got = prob.channel(ch)
            if kind in ("uniform", "histogram"):
                assert np.array_equal(got, ref), (name, kind, bins, ch)
            else:
                assert np.max(np.abs(got - ref)) <= 1.0 / n + 1e-15, (name, kind, ch)
        seen += 1
    assert seen >= 12


@pytest.mark.parametrize("kind,bins", [("uniform", 5), ("histogram", 5), ("histogram", 9),
                                       ("epanechnikov", 5), ("gaussian", 5)])
def test_monte_carlo_counts_against_oracle(kind, bins):
    vals = orc.ackley_ensemble(23, 17, 20, noise_amp=0.3, seed=1)
    n = 3001
    ref_counts = {}
    orc.classify(orc.fit(vals, kind, bins), kind, method="monte_carlo", n_samples=n, seed=77,
                 counts_out=ref_counts)
    holder = {}
    cpb.classify_field(_fit(vals, kind, bins),
                       cpb.EstimatorSpec(method="monte_carlo", n_samples=n, seed=77),
                       counts_out=holder)
    got = holder["counts"].cpu().numpy()
    for i, ch in enumerate(("min", "max", "saddle")):
        diff = np.abs(got[i] - ref_counts[ch])
        if kind in ("uniform", "histogram"):
            assert diff.max() == 0, (kind, ch)
        else:
            assert diff.max() <= 1 and diff.sum() <= 3, (kind, ch, diff.max(), diff.sum())


@pytest.mark.parametrize("n", [1, 5, 31, 32, 33, 64, 95])
def test_monte_carlo_two_stage_small_n(n):
    """Histogram MC (two-stage draws, warp-compacted candidates) at sample
    counts around the warp width, and on a constant field (ties everywhere):
    counts bit-identical to the oracle's."""
    vals = orc.ackley_ensemble(19, 13, 20, noise_amp=0.3, seed=5)
    flat = np.repeat(vals[:, :1, :1], 13, axis=1).repeat(19, axis=2)
    for v in (vals, flat):
        ref_counts = {}
        orc.classify(orc.fit(v, "histogram", 4), "histogram", method="monte_carlo", n_samples=n,
                     seed=31, counts_out=ref_counts)
        holder = {}
        cpb.classify_field(_fit(v, "histogram", 4),
                           cpb.EstimatorSpec(method="monte_carlo", n_samples=n, seed=31),
                           counts_out=holder)
        got = holder["counts"].cpu().numpy()
        for i, ch in enumerate(("min", "max", "saddle")):
            assert np.array_equal(got[i], ref_counts[ch]), (n, ch)


def test_monte_carlo_vs_closed_form_binomial_bound():
    # test_acceptance.py:75-97 style: |p_mc - p_closed| <= 4 SE for >= 99% of vertices
    vals = orc.ackley_ensemble(64, 64, 20, noise_amp=0.3, seed=0)
    for kind in ("uniform", "epanechnikov"):
        field = _fit(vals, kind)
        closed = cpb.classify_field(field)
        n = 20000
        for rng in ("splitmix64", "philox"):
            mc = cpb.classify_field(field, cpb.EstimatorSpec(method="monte_carlo", n_samples=n,
                                                             seed=3, rng=rng))
            for ch in ("min", "max", "saddle"):
                p = closed.channel(ch)[1:-1, 1:-1]
                q = mc.channel(ch)[1:-1, 1:-1]
                se = np.sqrt(np.maximum(p * (1 - p), 1e-12) / n)
                ok = np.abs(q - p) <= 4 * se + 1e-12
                assert ok.mean() >= 0.99, (kind, rng, ch, ok.mean())


def test_monte_carlo_chunking_boundary(golden):
    # test_engine.py:642-651: large n, the per-lane split must not matter
    vals = golden["fit"]["ens/rand"]
    field = _fit(vals, "uniform")
    a = cpb.classify_field(field, cpb.EstimatorSpec(method="monte_carlo", n_samples=150_000, seed=3))
    ref = orc.classify(orc.fit(vals, "uniform"), "uniform", method="monte_carlo", n_samples=150_000,
                       seed=3, block=8)
    for ch in ("min", "max", "saddle"):
        assert np.array_equal(a.channel(ch), ref[ch])


# ---------------------------------------------------------------- RNG + synth
def test_unit_block_bitexact(golden):
    rng = golden["rng"]
    for seed in (0, 7, -1, 2**64 - 2, 123456789):
        assert np.array_equal(cpb.unit_block(seed, rng["pixels"], 3, 11), rng[f"{seed}"])
    a = cpb.unit_block(5, np.arange(4), 2, 40)
    assert np.array_equal(a, orc.uniforms(5, np.arange(4), 2, 40))


def test_synthetic_rows_match_host_twin():
    dev = cpb.synthetic_rows(0, 40, 33, 40, 7, seed=4).cpu().numpy()
    host = orc.synthetic_rows(0, 40, 33, 40, 7, seed=4)
    assert np.array_equal(dev, host)
    part = cpb.synthetic_rows(13, 5, 33, 40, 7, seed=4).cpu().numpy()
    assert np.array_equal(part, host[:, 13:18])


# ---------------------------------------------------------------- semianalytical
SEMI_TOL = 1e-13  # the mean is numpy's pairwise sum; the neighbour CDFs multiply by 1/binw


def test_semianalytical_against_reference(golden):
    fit, semi = golden["fit"], golden["semi"]
    seen = 0
    for key in semi:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "c":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        c = int(semi[key])
        prob = cpb.classify_field(_fit(fit[f"ens/{name}"], kind, bins),
                                  cpb.EstimatorSpec(method="semianalytical", c=c, seed=2))
        for ch in ("min", "max", "saddle"):
            err = np.max(np.abs(prob.channel(ch) - semi[f"{name}/{kind}/{bins}/{ch}"]))
            assert err <= SEMI_TOL, (key, ch, err)
        seen += 1
    assert seen >= 6


def test_semianalytical_close_to_closed_form():
    # test_acceptance.py:185-216: RMSE < 0.01 against the closed form
    vals = orc.ackley_ensemble(40, 36, 20, noise_amp=0.3, seed=2)
    field = _fit(vals, "histogram", 5)
    closed = cpb.classify_field(field)
    semi = cpb.classify_field(field, cpb.EstimatorSpec(method="semianalytical", c=10000, seed=0))
    ref = orc.classify(orc.fit(vals, "histogram", 5), "histogram", method="semianalytical",
                       n_samples=10000, seed=0)
    for ch in ("min", "max", "saddle"):
        d = semi.channel(ch)[1:-1, 1:-1] - closed.channel(ch)[1:-1, 1:-1]
        assert np.sqrt(np.mean(d * d)) < 0.01
        assert np.max(np.abs(semi.channel(ch) - ref[ch])) <= SEMI_TOL
    with pytest.raises(ValueError):
        cpb.classify_field(_fit(vals, "uniform"), cpb.EstimatorSpec(method="semianalytical"))


# ---------------------------------------------------------------- one-call host path
def test_run_host_models_matches_oracle():
    """cpb_run_host_models / cpb_run_host: host buffers in, host planes out (C ABI)."""
    import ctypes

    from paper_2407_18015_b200 import _lib

    lib = _lib.load()
    # conftest sets CPB_HOST_CHUNK_BYTES small: the row-chunked H2D + chunk views path
    vals = np.ascontiguousarray(orc.ackley_ensemble(37, 4099, 6, noise_amp=0.3, seed=3))
    M, H, W = vals.shape
    models = [("uniform", 5), ("epanechnikov", 5), ("histogram", 4)]
    outs = [np.full((H, W), np.nan) for _ in range(3 * len(models))]  # every element is written
    valid = np.full((H, W), 7, dtype=np.uint8)
    kinds = (ctypes.c_int32 * 3)(*[_lib.KIND_CODES[k] for k, _ in models])
    bins = (ctypes.c_int32 * 3)(*[b for _, b in models])
    ks = (ctypes.c_double * 3)(*[float(cpb.ModelSpec(k).k) for k, _ in models])
    ptrs = (ctypes.c_void_p * 9)(*[o.ctypes.data for o in outs])
    _lib.check(lib.cpb_run_host_models(vals.ctypes.data, M, H, W, 3, kinds, bins, ks, 0, 0, 0, 7,
                                       ptrs, valid.ctypes.data))
    assert valid[1:-1, 1:-1].all() and not valid[0].any() and not valid[:, -1].any()
    for i, (kind, b) in enumerate(models):
        ref = orc.classify(orc.fit(vals, kind, b), kind)
        for c, ch in enumerate(("min", "max", "saddle")):
            assert np.max(np.abs(outs[3 * i + c] - ref[ch])) <= CLOSED_TOL, (kind, ch)
    # single-model entry point, Monte Carlo
    o = [np.full((H, W), np.nan) for _ in range(3)]
    _lib.check(lib.cpb_run_host(vals.ctypes.data, M, H, W, 0, 5, 1.0, 1, 11, 300, 7,
                                o[0].ctypes.data, o[1].ctypes.data, o[2].ctypes.data, None))
    ref = orc.classify(orc.fit(vals, "uniform"), "uniform", method="monte_carlo", n_samples=300,
                       seed=11)
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(o[c], ref[ch])
    bad = vals.copy()
    bad[2, 7, 7] = np.nan
    with pytest.raises(ValueError):
        _lib.check(lib.cpb_run_host(bad.ctypes.data, M, H, W, 0, 5, 1.0, 0, 0, 0, 7,
                                    o[0].ctypes.data, None, None, None))


def test_run_host_partial_channels_and_per_member_copies(monkeypatch):
    """Unrequested channels come back exactly 0.0 even with a non-NULL host plane
    (test_engine.py:616-623), and the per-member H2D path (member planes wider
    than the driver's maximum 2-D copy pitch) gives the same result."""
    import ctypes

    from paper_2407_18015_b200 import _lib

    lib = _lib.load()
    vals = np.ascontiguousarray(orc.ackley_ensemble(41, 57, 7, noise_amp=0.3, seed=4))
    M, H, W = vals.shape
    ref = orc.classify(orc.fit(vals, "uniform"), "uniform")
    for pitch in (None, "64"):
        if pitch:
            monkeypatch.setenv("CPB_HOST_MAX_PITCH", pitch)
        o = [np.full((H, W), np.nan) for _ in range(3)]
        _lib.check(lib.cpb_run_host(vals.ctypes.data, M, H, W, 0, 5, 1.0, 0, 0, 0, _lib.CH_MIN,
                                    o[0].ctypes.data, o[1].ctypes.data, o[2].ctypes.data, None))
        assert np.max(np.abs(o[0] - ref["min"])) <= CLOSED_TOL
        assert np.array_equal(o[1], np.zeros((H, W))) and np.array_equal(o[2], np.zeros((H, W)))


# ---------------------------------------------------------------- combinatorial (Eq. 5)
COMB_TOL = 1e-12  # the reference evaluates each all-uniform term exactly; we use 3-node GL


def test_combinatorial_against_reference(golden):
    fit, comb = golden["fit"], golden["comb"]
    seen = 0
    for key in comb:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "done":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        field = _fit(fit[f"ens/{name}"], kind, bins)
        prob = cpb.classify_field(field, cpb.EstimatorSpec(method="combinatorial"))
        closed = cpb.classify_field(field)
        for ch in ("min", "max", "saddle"):
            ref = comb[f"{name}/{kind}/{bins}/{ch}"]
            assert np.max(np.abs(prob.channel(ch) - ref)) <= COMB_TOL, (key, ch)
            # test_acceptance.py:100-108: Eq. 5 agrees with the factorised form (on
            # non-degenerate fields; eps-wide supports far from the origin are rounding
            # noise in both of the reference's methods)
            if name in ("rand", "ackley"):
                assert np.max(np.abs(prob.channel(ch) - closed.channel(ch))) <= 1e-9, (key, ch)
        seen += 1
    assert seen >= 8
    with pytest.raises(ValueError):
        cpb.classify_field(_fit(fit["ens/rand"], "histogram", 9), cpb.EstimatorSpec(method="combinatorial"))


def test_run_host_streaming_eps_fixup():
    """Chunks are stencilled with a provisional eps; rows whose pixels depend on
    eps (degenerate / clamped) are redone once the last chunk sets the global eps."""
    import ctypes

    from paper_2407_18015_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(8)
    M, H, W = 6, 300, 20
    vals = (rng.uniform(-1, 1, (H, W)) + rng.uniform(-0.3, 0.3, (M, H, W))).astype(np.float32)
    vals[:, 5, 7] = 0.25          # degenerate pixel in the first chunk
    vals[:, 6, 3] = vals[0, 6, 3]  # and another (epanechnikov: std == 0 -> clamped to eps/2)
    vals[2, 280, 11] = 1000.0     # the last chunk widens the global range, hence eps
    vals = np.ascontiguousarray(vals)
    models = [("uniform", 5), ("epanechnikov", 5), ("histogram", 3)]
    outs = [np.full((H, W), np.nan) for _ in range(9)]  # the library must write every element
    kinds = (ctypes.c_int32 * 3)(*[_lib.KIND_CODES[k] for k, _ in models])
    bins = (ctypes.c_int32 * 3)(*[b for _, b in models])
    ks = (ctypes.c_double * 3)(*[float(cpb.ModelSpec(k).k) for k, _ in models])
    ptrs = (ctypes.c_void_p * 9)(*[o.ctypes.data for o in outs])
    _lib.check(lib.cpb_run_host_models(vals.ctypes.data, M, H, W, 3, kinds, bins, ks, 0, 0, 0, 7,
                                       ptrs, None))
    for i, (kind, b) in enumerate(models):
        ref = orc.classify(orc.fit(vals, kind, b), kind)
        for c, ch in enumerate(("min", "max", "saddle")):
            assert np.max(np.abs(outs[3 * i + c] - ref[ch])) <= CLOSED_TOL, (kind, ch)


def test_release_workspace_returns_cached_scratch():
    import ctypes

    from paper_2407_18015_b200 import _lib

    lib = _lib.load()
    vals = np.ascontiguousarray(orc.ackley_ensemble(40, 30, 8, noise_amp=0.3, seed=0))
    outs = [np.zeros((30, 40)) for _ in range(3)]
    _lib.check(lib.cpb_run_host(vals.ctypes.data, 8, 30, 40, _lib.KIND_CODES["uniform"], 5, 1.0, 0, 0,
                                0, 7, *[o.ctypes.data for o in outs], None))
    released = ctypes.c_size_t(0)
    _lib.check(lib.cpb_release_workspace(ctypes.byref(released)))
    assert released.value > 0
    _lib.check(lib.cpb_release_workspace(ctypes.byref(released)))
    assert released.value == 0


def test_fit_histogram_threshold_edges():
    """Members at +-0, subnormals and exact bin edges: the exact threshold binning
    (fields.py:146-152) including thresholds at zero."""
    rng = np.random.default_rng(12)
    tiny = np.float32(1e-45)
    special = np.array([-0.0, 0.0, tiny, -tiny, -1.0, 1.0, 0.5, -0.5, 1e-38, -1e-38], dtype=np.float32)
    H, W, M = 6, 40, 23
    vals = rng.choice(special, size=(M, H, W)).astype(np.float32)
    vals[0] = -1.0
    vals[1] = 1.0
    vals[:, 5, :20] = rng.uniform(-1, 1, (M, 20)).astype(np.float32)
    for bins in (2, 3, 4, 5, 8, 9):
        got = _fit(vals, "histogram", bins).params
        ref = orc.fit(vals, "histogram", bins)
        for k in ref:
            assert np.array_equal(got[k], ref[k]), (bins, k)


def test_fit_multi_matches_separate_fits():
    """cpb_fit_multi (one pass, all models) writes exactly the planes of separate fits."""
    rng = np.random.default_rng(21)
    vals = (rng.uniform(-1, 1, (37, 53)) + rng.uniform(-0.3, 0.3, (17, 37, 53))).astype(np.float32)
    vals[:, 4, 4] = 0.125  # degenerate pixel
    stack = cpb.EnsembleStack(vals)
    for models in ([cpb.ModelSpec("uniform"), cpb.ModelSpec("epanechnikov"), cpb.ModelSpec("histogram", bins=5)],
                   [cpb.ModelSpec("histogram", bins=8), cpb.ModelSpec("gaussian")],
                   [cpb.ModelSpec("histogram", bins=12), cpb.ModelSpec("uniform")],   # > 8 bins: separate
                   [cpb.ModelSpec("histogram", bins=3), cpb.ModelSpec("histogram", bins=4)]):
        fused = cpb.UncertainField.from_ensemble_models(stack, models)
        for m, f in zip(models, fused):
            ref = orc.fit(vals, m.kind, m.bins)
            got = f.params
            for k in ref:
                assert np.array_equal(got[k], ref[k]), (m, k)
            if m.kind != "gaussian":
                p = cpb.classify_field(f)
                q = cpb.classify_field(cpb.UncertainField.from_ensemble(stack, m))
                assert np.array_equal(p.p_min, q.p_min) and np.array_equal(p.p_saddle, q.p_saddle)


def test_row_slabs_on_device_match_single_gpu():
    """The multi-GPU path's device side (SlabField views, fused slab fit, the
    {-min, max} pair -> global eps, halo rows, stencil rows, global pixel keys)
    for G = 3 slabs run one after another on this GPU.  The two collectives are
    emulated in-process: the MAX of the slabs' pairs and copies of the boundary
    rows between the slabs' planes (what NCCL does across ranks)."""
    from paper_2407_18015_b200 import distributed as D

    H, W, M, G = 23, 31, 12, 3
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=4)
    vals[:, 11, 7] = 0.5  # a degenerate pixel: needs the GLOBAL eps
    dev = torch.device("cuda")
    models = [cpb.ModelSpec("uniform"), cpb.ModelSpec("epanechnikov"), cpb.ModelSpec("histogram", bins=5)]
    slabs = [D.slab_rows(H, r, G) for r in range(G)]
    fields = [[D.SlabField(m, s, W, M, dev) for m in models] for s in slabs]
    for s, fs in zip(slabs, fields):
        ens = torch.as_tensor(np.ascontiguousarray(vals[:, s.row_begin:s.row_end]), device=dev)
        D.fit_slab_fields(fs, ens, finish=False)
    pair = torch.stack([fs[0].pair for fs in fields]).max(dim=0).values  # NCCL MAX all-reduce
    for fs in fields:
        fs[0].pair.copy_(pair)
        D.finish_slab_fields(fs)  # world 1 here: eps only
    for r in range(G - 1):  # halo rows: last owned row down, first owned row up
        lo_s, hi_s = slabs[r], slabs[r + 1]
        for fa, fb in zip(fields[r], fields[r + 1]):
            for pa, pb in zip(D._plane_views(fa.dev), D._plane_views(fb.dev)):
                last = lo_s.halo_top + lo_s.owned - 1
                pb[..., 0, :].copy_(pa[..., last, :])
                pa[..., last + 1, :].copy_(pb[..., hi_s.halo_top, :])
    torch.cuda.synchronize()
    stack = cpb.EnsembleStack(vals)
    for i, m in enumerate(models):
        full = cpb.UncertainField.from_ensemble(stack, m)
        ref_c = cpb.classify_field(full)
        est = cpb.EstimatorSpec("monte_carlo", n_samples=300, seed=6)
        ref_m = cpb.classify_field(full, est)
        for s, fs in zip(slabs, fields):
            a, b = s.stencil_rows()
            g0 = s.local_row0
            out, _ = D.classify_slab(fs[i].dev, s, cpb.EstimatorSpec())
            outm, _ = D.classify_slab(fs[i].dev, s, est)
            for c, ch in enumerate(("min", "max", "saddle")):
                got = out[c, a:b].cpu().numpy()
                assert np.array_equal(got, ref_c.channel(ch)[g0 + a:g0 + b]), (m.kind, ch)
                assert np.array_equal(outm[c, a:b].cpu().numpy(), ref_m.channel(ch)[g0 + a:g0 + b]), (m.kind, ch)


def test_closed_counts_fused_match_plane_sums():
    """cpb_classify_closed_counts: the per-type sums fused into the stencils equal
    the sums of the written planes (to rounding) for every model and kernel."""
    from paper_2407_18015_b200 import _lib
    from paper_2407_18015_b200.engine import run_rows

    vals = orc.ackley_ensemble(70, 45, 12, noise_amp=0.3, seed=2)
    for kind, bins in (("uniform", 5), ("epanechnikov", 5), ("histogram", 5), ("histogram", 12),
                       ("histogram", 30)):
        field = _fit(vals, kind, bins)
        dev = field.device_field()
        out = torch.zeros((3, 45, 70), dtype=torch.float64, device="cuda")
        sums = torch.zeros(3, dtype=torch.float64, device="cuda")
        run_rows(dev, cpb.EstimatorSpec(), ("min", "max", "saddle"), 1, 44,
                 {"min": out[0], "max": out[1], "saddle": out[2]}, type_sums=sums)
        ref = out[:, 1:44, 1:69].sum(dim=(1, 2))
        assert torch.allclose(sums, ref, rtol=1e-13, atol=0), (kind, bins, sums, ref)
        prob = cpb.classify_field(field)
        assert np.array_equal(out[0].cpu().numpy(), prob.p_min), kind
    with pytest.raises(ValueError):
        _lib.check(_lib.load().cpb_classify_closed_counts(dev.ref(), 1, 44, None, None, None, None, 0))


def test_closed_mixed_precision_within_stated_bound(golden):
    """EstimatorSpec(precision="mixed"): FP32 Gauss-Legendre evaluation for the
    uniform and Epanechnikov stencils within the north_star's 1e-6 absolute
    bound of the reference (goldens incl. degenerate / far-offset stacks, and a
    config-2-shaped field); histogram fields stay fp64 (identical results)."""
    fit, closed = golden["fit"], golden["closed"]
    mixed = cpb.EstimatorSpec(precision="mixed")
    worst = 0.0
    for key in closed:
        parts = key.split("/")
        if len(parts) != 4 or parts[3] != "min":
            continue
        name, kind, bins = parts[0], parts[1], int(parts[2])
        field = _fit(fit[f"ens/{name}"], kind, bins)
        prob = cpb.classify_field(field, mixed)
        for ch in ("min", "max", "saddle"):
            err = float(np.max(np.abs(prob.channel(ch) - closed[f"{name}/{kind}/{bins}/{ch}"])))
            if kind == "histogram":
                assert err <= CLOSED_TOL, (name, ch, err)
            else:
                assert err <= 1e-6, (name, kind, ch, err)
                worst = max(worst, err)
    vals = orc.ackley_ensemble(200, 150, 20, noise_amp=0.3, seed=0)
    for kind in ("uniform", "epanechnikov"):
        ref = orc.classify(orc.fit(vals, kind), kind)
        prob = cpb.classify_field(_fit(vals, kind), mixed)
        for ch in ("min", "max", "saddle"):
            err = float(np.max(np.abs(prob.channel(ch) - ref[ch])))
            assert err <= 1e-6, (kind, ch, err)
            worst = max(worst, err)
    print("mixed-precision max |error|", worst)
    with pytest.raises(ValueError):
        cpb.EstimatorSpec(precision="fp16")


# ---------------------------------------------------------------- fused fit + uniform stencil
def _fused_uniform(vals, row_begin=None, row_end=None):
    """cpb_fit_classify + cpb_fit_classify_finish on a (M, H, W) stack."""
    import ctypes

    from paper_2407_18015_b200 import _lib
    from paper_2407_18015_b200.fields import DeviceField

    lib = _lib.load()
    M, H, W = vals.shape
    rb = 1 if row_begin is None else row_begin
    re_ = H - 1 if row_end is None else row_end
    ens = torch.as_tensor(np.ascontiguousarray(vals), device="cuda")
    dev = DeviceField("uniform", 5, M, H, W)
    dev.allocate_fitted()
    out = torch.full((3, H, W), -7.0, dtype=torch.float64, device="cuda")
    out[:, [0, -1], :] = 0.0
    out[:, :, [0, -1]] = 0.0
    nb = ctypes.c_size_t()
    _lib.check(lib.cpb_fit_classify_work_bytes(W, rb, re_, ctypes.byref(nb)))
    work = torch.empty(max(1, nb.value), dtype=torch.uint8, device="cuda")
    s = _lib.stream_ptr()
    rng = dev.tensors["range"].data_ptr()
    _lib.check(lib.cpb_fit_classify(ens.data_ptr(), H * W, dev.ref(), rng, 0, rb, re_,
                                    out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
                                    work.data_ptr(), s))
    gmin, gmax = ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.cpb_read_range(rng, ctypes.byref(gmin), ctypes.byref(gmax), s))
    dev.eps = lib.cpb_epsilon(gmin.value, gmax.value)
    counts = torch.zeros(3, dtype=torch.float64, device="cuda")
    _lib.check(lib.cpb_fit_classify_finish(dev.ref(), rb, re_, out[0].data_ptr(), out[1].data_ptr(),
                                           out[2].data_ptr(), counts.data_ptr(), work.data_ptr(), s))
    torch.cuda.synchronize()
    return dev, out.cpu().numpy(), counts.cpu().numpy(), (gmin.value, gmax.value)


@pytest.mark.parametrize("shape", [(20, 3, 3), (20, 37, 130), (7, 131, 127), (64, 259, 253), (1, 5, 129),
                                   (256, 9, 300), (33, 140, 128)])
def test_fused_fit_classify_uniform_bitexact(shape):
    """One-pass fit + stencil (cpb_fit_classify) == cpb_fit + cpb_classify_closed,
    bit for bit: planes, range, every probability; expected counts = plane sums."""
    M, H, W = shape
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=H + W)
    if H > 4 and W > 4:
        vals[:, H // 2, W // 3] = 0.125  # degenerate pixels: rows queued for the final eps
        vals[:, 1, 1] = vals[0, 1, 1]
    dev, out, counts, rng = _fused_uniform(vals)
    field = _fit(vals, "uniform")
    ref = cpb.classify_field(field)
    params = field.params
    from paper_2407_18015_b200.fields import UncertainField

    got = UncertainField(cpb.ModelSpec("uniform"), _device_field=dev).params
    for k in ("lo", "hi"):
        assert np.array_equal(got[k], params[k]), k
    assert rng == (float(vals.min()), float(vals.max()))
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(out[c], ref.channel(ch)), (shape, ch, np.max(np.abs(out[c] - ref.channel(ch))))
        assert abs(counts[c] - ref.channel(ch).sum()) <= 1e-9 * max(1.0, abs(counts[c]))
    oref = orc.classify(orc.fit(vals, "uniform"), "uniform")
    assert max(np.max(np.abs(out[c] - oref[ch])) for c, ch in enumerate(("min", "max", "saddle"))) <= CLOSED_TOL


def test_fused_fit_classify_band_edges_and_degenerate_edges():
    """The fused kernel reads only its own 128-column band and computes the band
    edge columns (127 / 128, 255 / 256, ...) in-kernel once both bands around a
    boundary are done; an edge vertex touching a degenerate pixel is flagged and
    redone with the final eps by the finish pass.  Degenerate pixels right at
    the band boundaries and at a row-segment boundary (row 128), bit-exact
    against fit + classify and within tolerance of the oracle."""
    M, H, W = 9, 300, 392  # W % 4 == 0 and H W % 4 == 0: the TMA-streamed path
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=11)
    for r, c in ((40, 127), (41, 128), (90, 255), (90, 256), (128, 200), (129, 128), (200, 383), (250, 1)):
        vals[:, r, c] = vals[0, r, c]  # lo == hi: widened by the global eps at use
    dev, out, counts, _ = _fused_uniform(vals)
    ref = cpb.classify_field(_fit(vals, "uniform"))
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(out[c], ref.channel(ch)), (ch, np.max(np.abs(out[c] - ref.channel(ch))))
        assert abs(counts[c] - ref.channel(ch).sum()) <= 1e-9 * max(1.0, abs(counts[c]))
    oref = orc.classify(orc.fit(vals, "uniform"), "uniform")
    assert max(np.max(np.abs(out[c] - oref[ch])) for c, ch in enumerate(("min", "max", "saddle"))) <= CLOSED_TOL
    # partial row range starting inside a segment, band edges included (no
    # degenerate pixels here: a partial range sees only its rows' eps)
    plain = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=11)
    dev, out, counts, _ = _fused_uniform(plain, 100, 260)
    pref = cpb.classify_field(_fit(plain, "uniform"))
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(out[c][100:260], pref.channel(ch)[100:260]), ch


@pytest.mark.parametrize("shape", [(9, 200, 390), (9, 200, 391), (5, 40, 130)])
def test_fused_fit_classify_unaligned_rows(shape):
    """Widths that are not a multiple of 4 with a 16-byte member stride: the
    per-row TMA box would start misaligned (an illegal-instruction fault), so
    the fused call takes the plain fit + finish path -- same results."""
    M, H, W = shape
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=W)
    dev, out, counts, _ = _fused_uniform(vals)
    ref = cpb.classify_field(_fit(vals, "uniform"))
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(out[c], ref.channel(ch)), ch


def test_fused_fit_classify_partial_rows_and_nonfinite():
    M, H, W = 12, 50, 140
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=1)
    dev, out, counts, _ = _fused_uniform(vals, 5, 31)
    ref = cpb.classify_field(_fit(vals, "uniform"))
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(out[c][5:31], ref.channel(ch)[5:31])
        assert np.all(out[c][1:5, 1:-1] == -7.0) and np.all(out[c][31:-1, 1:-1] == -7.0)
    bad = vals.copy()
    bad[3, 20, 20] = np.nan
    import ctypes

    from paper_2407_18015_b200 import _lib

    dev, out, counts, rng = None, None, None, None
    with pytest.raises(ValueError):
        _fused_uniform(bad)


def test_fused_uniform_slab_path_matches_classify_field():
    """distributed.fit_classify_uniform (the bench's uniform step) at G = 1."""
    from paper_2407_18015_b200 import distributed as D

    M, H, W = 16, 45, 263
    vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=2)
    vals[:, 10, 10] = 0.5
    slab = D.slab_rows(H, 0, 1)
    dev = torch.device("cuda")
    f = D.SlabField(cpb.ModelSpec("uniform"), slab, W, M, dev)
    out = torch.zeros((3, H, W), dtype=torch.float64, device=dev)
    total, _ = D.fit_classify_uniform(f, torch.as_tensor(vals, device=dev), slab, out)
    ref = cpb.classify_field(_fit(vals, "uniform"))
    o = out.cpu().numpy()
    for c, ch in enumerate(("min", "max", "saddle")):
        assert np.array_equal(o[c], ref.channel(ch)), ch
    assert np.allclose(total.cpu().numpy(), [ref.channel(ch).sum() for ch in ("min", "max", "saddle")],
                       rtol=1e-12)


def test_fused_multi_fit_classify_matches_separate():
    """cpb_fit_multi_classify (distributed.fit_classify): one pass fits uniform,
    Epanechnikov and histogram fields and stencils the uniform one -- planes
    bit-identical to separate fits, uniform probabilities to classify_field."""
    from paper_2407_18015_b200 import distributed as D

    dev = torch.device("cuda")
    for (M, H, W), bins in (((16, 45, 263), 5), ((40, 131, 256), 8), ((12, 30, 200), 3)):
        vals = orc.ackley_ensemble(W, H, M, noise_amp=0.3, seed=H)
        vals[:, 10, 10] = 0.5
        slab = D.slab_rows(H, 0, 1)
        models = [cpb.ModelSpec("histogram", bins=bins), cpb.ModelSpec("uniform"), cpb.ModelSpec("epanechnikov")]
        fields = [D.SlabField(m, slab, W, M, dev) for m in models]
        out = torch.zeros((3, H, W), dtype=torch.float64, device=dev)
        total, _ = D.fit_classify(fields, torch.as_tensor(vals, device=dev), slab, out)
        stack = cpb.EnsembleStack(vals)
        from paper_2407_18015_b200.fields import UncertainField

        for m, f in zip(models, fields):
            ref = cpb.UncertainField.from_ensemble(stack, m)
            got = UncertainField(m, _device_field=f.dev)
            for k, v in ref.params.items():
                assert np.array_equal(got.params[k], v), (M, H, W, m.kind, k)
        ref = cpb.classify_field(cpb.UncertainField.from_ensemble(stack, cpb.ModelSpec("uniform")))
        o = out.cpu().numpy()
        for c, ch in enumerate(("min", "max", "saddle")):
            assert np.array_equal(o[c], ref.channel(ch)), ch
        assert np.allclose(total.cpu().numpy(), [ref.channel(ch).sum() for ch in ("min", "max", "saddle")],
                           rtol=1e-12)


@pytest.mark.parametrize("members", [49, 93, 211, 255])
def test_histogram_fitted_weights_not_renormalised(members):
    """The table stencil uses the fitted weights count / M as they are; the
    reference renormalises w / sum(w) first (engine.py:538-540).  For count
    weights the sum is 1 to within an ulp (at most 2.2e-16 away over all
    compositions of M <= 255 into 5 bins), so the skipped division moves the
    probabilities by ~1e-16.  Pinned against the renormalising oracle at 1e-13
    on member counts whose weight sums are furthest from 1 (5 and 7 bins: the
    table kernels; 12 bins: states from cumulative counts)."""
    vals = orc.ackley_ensemble(26, 22, members, noise_amp=0.3, seed=members)
    for bins in (5, 7, 12):
        ref = orc.classify(orc.fit(vals, "histogram", bins), "histogram")
        prob = cpb.classify_field(_fit(vals, "histogram", bins))
        for ch in ("min", "max", "saddle"):
            err = np.max(np.abs(prob.channel(ch) - ref[ch]))
            assert err <= 1e-13, (members, bins, ch, err)
