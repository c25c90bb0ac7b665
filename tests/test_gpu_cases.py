"""GPU parity of the batched per-case API (cpb_cases_* through paper_2407_18015_b200.cases).

Bars: closed form within 1e-12 of the reference (its own grid-vs-case
tolerance, test_engine.py:548-559; observed ~1e-16), Monte Carlo bit-exact for
uniform / histogram draws (transcendental kinds: <= 1 flipped draw per
channel), semianalytical within 1e-13 (reciprocal-multiply CDFs; numpy's pairwise mean), combinatorial
within 1e-12.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2407_18015_b200 as cpb  # noqa: E402
from oracle import cases_oracle as co  # noqa: E402
from oracle import critprob_oracle as orc  # noqa: E402
from paper_2407_18015_b200.cases import CaseBatch  # noqa: E402


def _batch(g, k):
    return CaseBatch.from_arrays(k, g[f"k{k}/kind"], g[f"k{k}/a"], g[f"k{k}/b"], g[f"k{k}/bins"],
                                 g[f"k{k}/weights"])


@pytest.mark.parametrize("k", [4, 2])
def test_closed_against_reference(golden, k):
    g = golden["cases"]
    bounded = ~np.any(g[f"k{k}/kind"] == 3, axis=1)
    kind, a, b, bins, w = (g[f"k{k}/{x}"][bounded] for x in ("kind", "a", "b", "bins", "weights"))
    got = CaseBatch.from_arrays(k, kind, a, b, bins, w).closed()
    err = np.max(np.abs(got - g[f"k{k}/closed"][bounded]))
    assert err <= 1e-12, err


@pytest.mark.parametrize("k", [4, 2])
def test_mc_against_reference(golden, k):
    g = golden["cases"]
    n, seed = int(g["mc/n"]), int(g["mc/seed"])
    got = _batch(g, k).monte_carlo(n, seed, g[f"k{k}/pixels"])
    ref = g[f"k{k}/mc"]
    exact_kind = np.all(np.isin(g[f"k{k}/kind"], (0, 2)), axis=1)
    assert np.array_equal(got[exact_kind], ref[exact_kind])
    assert np.max(np.abs(got - ref)) * n <= 1.0 + 1e-9


@pytest.mark.parametrize("k", [4, 2])
def test_semi_and_combinatorial_against_reference(golden, k):
    g = golden["cases"]
    hist = np.all(g[f"k{k}/kind"] == 2, axis=1)
    sel = {x: g[f"k{k}/{x}"][hist] for x in ("kind", "a", "b", "bins", "weights", "pixels")}
    batch = CaseBatch.from_arrays(k, sel["kind"], sel["a"], sel["b"], sel["bins"], sel["weights"])
    semi = batch.semianalytical(int(g["semi/c"]), int(g["semi/seed"]), sel["pixels"])
    # the neighbour CDFs multiply by 1/binw (cpb_sample.cuh hist_cdf_fast): 1e-13;
    # the mean itself is numpy's pairwise sum (grid == per case bitwise, test_gpu_engine)
    assert np.max(np.abs(semi - g[f"k{k}/semi"][hist])) <= 1e-13
    small = np.max(sel["bins"], axis=1) <= 5
    sb = CaseBatch.from_arrays(k, *(sel[x][small] for x in ("kind", "a", "b", "bins", "weights")))
    comb = sb.combinatorial()
    assert np.max(np.abs(comb - g[f"k{k}/comb"][hist][small])) <= 1e-12


def test_known_answers():
    # test_engine.py:147-169 (all-uniform) and 171-191 (mixed kinds)
    kat = cpb.NeighborhoodCase(cpb.uniform(0.0, 2.0), (cpb.uniform(1.0, 3.0), cpb.uniform(0.5, 2.5),
                                                       cpb.uniform(1.5, 3.5), cpb.uniform(0.0, 2.0)))
    t = cpb.closed_form_triple(kat)
    assert t.p_min == pytest.approx(0.41865234375, abs=1e-12)
    assert t.p_max == pytest.approx(0.008170572916666667, abs=1e-12)
    assert t.p_saddle == pytest.approx(0.1377604166666667, abs=1e-12)
    mixed = cpb.NeighborhoodCase(
        cpb.epanechnikov(1.0, 0.9),
        (cpb.histogram(0.2, 2.2, [0.3, 0.5, 0.2]), cpb.uniform(0.5, 2.5), cpb.epanechnikov(1.4, 1.0),
         cpb.histogram(-0.2, 1.8, [0.25, 0.25, 0.5])))
    t = cpb.closed_form_triple(mixed)
    assert t.p_min == pytest.approx(0.2680767777717538, abs=1e-12)
    assert t.p_max == pytest.approx(0.0594104715257872, abs=1e-12)
    assert t.p_saddle == pytest.approx(0.06347446822834163, abs=1e-12)
    assert cpb.local_min_prob(mixed) == t.p_min and cpb.saddle_prob(mixed) == t.p_saddle


def test_iid_symmetry_and_disjoint():
    # test_engine.py:85-143: five i.i.d. -> 1/5, 1/5, 1/15 (2 neighbours: 1/3, 1/3, 1/3)
    for f in (lambda: cpb.uniform(0, 1), lambda: cpb.epanechnikov(0.0, 1.0),
              lambda: cpb.histogram(0.0, 1.0, [0.2, 0.5, 0.3])):
        t = cpb.closed_form_triple(cpb.NeighborhoodCase(f(), tuple(f() for _ in range(4))))
        assert t.p_min == pytest.approx(0.2, abs=1e-12) and t.p_max == pytest.approx(0.2, abs=1e-12)
        assert t.p_saddle == pytest.approx(1.0 / 15.0, abs=1e-12)
        t = cpb.closed_form_triple(cpb.NeighborhoodCase(f(), (f(), f())))
        assert t.p_min == pytest.approx(1 / 3, abs=1e-12) and t.p_saddle == pytest.approx(1 / 3, abs=1e-12)
    d = cpb.NeighborhoodCase(cpb.uniform(0.0, 1.0), tuple(cpb.uniform(2.0, 3.0) for _ in range(4)))
    t = cpb.closed_form_triple(d)
    assert t.p_min == pytest.approx(1.0, abs=1e-14) and t.p_max == 0.0 and t.p_saddle == 0.0
    for n in (1, 10, 1000):
        assert cpb.mc_pattern_prob(d, "min", n) == 1.0


def test_random_cases_against_oracle():
    rng = np.random.default_rng(3)
    cases = []
    for i in range(60):
        model = ("uniform", "epanechnikov", "histogram")[i % 3]
        case = cpb.random_case(1000 + i, model=model, neighborhood=4 if i % 5 else 2, bins=int(rng.integers(1, 12)))
        cases.append(case.affine(float(rng.uniform(0.1, 50)), float(rng.uniform(-1e3, 1e3))) if i % 7 == 0 else case)
    got = cpb.closed_form_triples(cases)
    for i, c in enumerate(cases):
        k, kind, a, b, bins, w = cpb.cases.pack_arrays([c])
        ref = co.closed_triple(co.unpack(kind, a, b, bins, w)[0])
        assert np.max(np.abs(got[i] - np.array(ref))) <= 1e-12, i


def test_negation_affine_and_saddle_swap():
    # test_engine.py:201-262: negation swaps min/max, affine maps leave triples unchanged
    cases = [cpb.random_case(s, model=m) for s in range(10) for m in ("uniform", "epanechnikov", "histogram")]
    base = cpb.closed_form_triples(cases)
    neg = cpb.closed_form_triples([c.negate() for c in cases])
    aff = cpb.closed_form_triples([c.affine(3.5, -2.0) for c in cases])
    assert np.max(np.abs(neg[:, [1, 0, 2]] - base)) <= 1e-12
    assert np.max(np.abs(aff - base)) <= 1e-12


def test_grid_case_consistency():
    # test_engine.py:548-572: grid == per-case (closed 1e-12, MC bitwise with pixel_index)
    vals = orc.ackley_ensemble(12, 10, 16, noise_amp=0.3, seed=0)
    for kind in ("uniform", "histogram", "epanechnikov"):
        field = cpb.UncertainField.from_ensemble(cpb.EnsembleStack(vals), cpb.ModelSpec(kind))
        closed = cpb.classify_field(field)
        mc = cpb.classify_field(field, cpb.EstimatorSpec("monte_carlo", n_samples=777, seed=4))
        rc = [(r, c) for r in range(1, 9) for c in range(1, 11)]
        cases = [cpb.case_at(field, r, c) for r, c in rc]
        got = cpb.closed_form_triples(cases)
        px = np.array([cpb.pixel_index(field, r, c) for r, c in rc], dtype=np.uint64)
        gmc = cpb.mc_all_patterns_batch(cases, 777, seed=4, pixels=px)
        for i, (r, c) in enumerate(rc):
            ref = [closed.channel(ch)[r, c] for ch in ("min", "max", "saddle")]
            assert np.max(np.abs(got[i] - ref)) <= 1e-12, (kind, r, c)
            refm = [mc.channel(ch)[r, c] for ch in ("min", "max", "saddle")]
            if kind != "epanechnikov":
                assert np.array_equal(gmc[i], refm), (kind, r, c)


def test_errors_match_reference():
    g = cpb.NeighborhoodCase(cpb.GaussianSampler(0, 1), tuple(cpb.GaussianSampler(0, 1) for _ in range(4)))
    with pytest.raises(TypeError):
        cpb.closed_form_triple(g)
    u = cpb.random_case(1, model="uniform")
    with pytest.raises(ValueError):
        cpb.semianalytical_prob(u, "min", 10)
    with pytest.raises(ValueError):
        cpb.combinatorial_triple(cpb.random_case(1, model="histogram", bins=9))
    with pytest.raises(ValueError):
        cpb.mc_pattern_prob(u, "min", 0)
    with pytest.raises(ValueError):
        cpb.mc_pattern_prob(u, "ridge", 10)
    p = cpb.mc_pattern_prob(g, "min", 10 ** 5, seed=0)  # test_engine.py:360-365
    assert abs(p - 0.2) <= 0.006
    t = cpb.mc_all_patterns(cpb.random_case(11, model="uniform", neighborhood=2), 50000, seed=0)
    assert t.total == pytest.approx(1.0, abs=1e-12)


def test_acceptance_closed_vs_mc_1e6():
    """test_acceptance.py:75-97 as one batch per model: 500 cases x 1e6 joint draws,
    >= 99 % of (case, pattern) checks within 4 binomial standard errors."""
    n = 1_000_000
    for offset, kind in enumerate(("uniform", "epanechnikov", "histogram")):
        cases = [cpb.random_case(1000 * offset + i, model=kind, neighborhood=4) for i in range(500)]
        batch = CaseBatch.pack(cases)
        closed = batch.closed()
        mc = batch.monte_carlo(n, seed=0, pixels=np.arange(500, dtype=np.uint64))
        se = np.sqrt(closed * (1.0 - closed) / n)
        within = np.abs(closed - mc) <= 4.0 * se
        assert within.mean(axis=0).min() >= 0.99, (kind, within.mean(axis=0))


def test_validate_random_cases():
    s = cpb.validate_random_cases(200, model="histogram", samples=200_000, seed=3)
    assert s.cases == 200 and s.within_4se >= 0.97 and s.max_abs_dev < 0.01
    assert "validate model=histogram" in s.to_text()
