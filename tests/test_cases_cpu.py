"""Per-case API on the CPU: the oracle against the reference's goldens, and the
package's host-side case construction (random_case, packing) against the
reference's own objects (tests/golden/cases.npz, make_golden.case_fixtures)."""

import numpy as np
import pytest

from oracle import cases_oracle as co


def _group(golden, k):
    g = golden["cases"]
    return g, co.unpack(g[f"k{k}/kind"], g[f"k{k}/a"], g[f"k{k}/b"], g[f"k{k}/bins"], g[f"k{k}/weights"])


@pytest.mark.parametrize("k", [4, 2])
def test_oracle_closed_matches_reference(golden, k):
    g, cases = _group(golden, k)
    ref = g[f"k{k}/closed"]
    seen = 0
    for i, c in enumerate(cases):
        if np.isnan(ref[i, 0]):
            continue
        assert np.max(np.abs(np.array(co.closed_triple(c)) - ref[i])) <= 1e-14, i
        seen += 1
    assert seen >= 30


@pytest.mark.parametrize("k", [4, 2])
def test_oracle_mc_and_semi_bitexact(golden, k):
    g, cases = _group(golden, k)
    n, seed = int(g["mc/n"]), int(g["mc/seed"])
    c, sseed = int(g["semi/c"]), int(g["semi/seed"])
    px = g[f"k{k}/pixels"]
    for i, case in enumerate(cases):
        assert np.array_equal(np.array(co.mc_triple(case, n, seed, int(px[i]))), g[f"k{k}/mc"][i]), i
        if not np.isnan(g[f"k{k}/semi"][i, 0]):
            got = np.array(co.semi_triple(case, c, sseed, int(px[i])))
            assert np.array_equal(got, g[f"k{k}/semi"][i]), i


def test_oracle_combinatorial_matches_reference(golden):
    for k in (4, 2):
        g, cases = _group(golden, k)
        ref = g[f"k{k}/comb"]
        for i, case in enumerate(cases):
            small = all(d["kind"] == "histogram" and d["w"].size <= 3 for d in (case[0], *case[1]))
            if np.isnan(ref[i, 0]) or (k == 4 and not small):
                continue
            assert np.max(np.abs(np.array(co.comb_triple(case)) - ref[i])) <= 1e-14, (k, i)


def test_random_case_and_packing_match_reference(golden):
    """The package's random_case (synth.py:124-151) and its cpb_case_batch packing
    rebuild the reference's objects exactly (pure host code, no device)."""
    import paper_2407_18015_b200 as cpb
    from paper_2407_18015_b200.cases import pack_arrays

    models = ("uniform", "epanechnikov", "histogram", "gaussian")
    for k in (4, 2):
        g = golden["cases"]
        spec = g[f"k{k}/random_spec"]
        cases = [cpb.random_case(int(s), model=models[int(m)], neighborhood=k, bins=int(b)) for s, m, b in spec]
        kk, kind, a, b, bins, w = pack_arrays(cases)
        n = len(cases)
        assert kk == k
        assert np.array_equal(kind, g[f"k{k}/kind"][:n])
        assert np.array_equal(a, g[f"k{k}/a"][:n]) and np.array_equal(b, g[f"k{k}/b"][:n])
        hist = kind == 2
        assert np.array_equal(bins[hist], g[f"k{k}/bins"][:n][hist])
        mb = w.shape[2]
        assert np.array_equal(w, g[f"k{k}/weights"][:n, :, :mb])


def test_case_objects_validate_like_reference():
    import paper_2407_18015_b200 as cpb

    with pytest.raises(ValueError):
        cpb.uniform(1.0, 1.0)
    with pytest.raises(ValueError):
        cpb.epanechnikov(0.0, 0.0)
    with pytest.raises(ValueError):
        cpb.histogram(0.0, 1.0, [0.0, 0.0])
    with pytest.raises(ValueError):
        cpb.NeighborhoodCase(cpb.uniform(0, 1), (cpb.uniform(0, 1),) * 3)
    with pytest.raises(ValueError):
        cpb.random_case(0, model="cauchy")
    h = cpb.histogram(0.0, 2.0, [1.0, 3.0])
    assert np.array_equal(h.bin_weights, [0.25, 0.75])
    assert np.array_equal(h.negate().bin_weights, [0.75, 0.25]) and h.negate().support.lo == -2.0
    trip = cpb.ProbabilityTriple(0.1, 0.2, 0.3)
    assert list(trip) == [0.1, 0.2, 0.3] and trip.total == pytest.approx(0.6)
