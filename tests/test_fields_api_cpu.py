"""Host-side types of the reference API (pkg/tests/test_fields.py:25-60, 185-210),
restated for paper_2407_18015_b200: no device needed."""

import math

import numpy as np
import pytest

import paper_2407_18015_b200 as cpb


def sample_stack(seed=0, shape=(30, 6, 7)):
    rng = np.random.default_rng(seed)
    return cpb.EnsembleStack(rng.uniform(-2.0, 3.0, shape).astype(np.float32))


class TestModelSpec:
    def test_defaults(self):
        spec = cpb.ModelSpec(kind="histogram")
        assert spec.bins == 5 and spec.k == pytest.approx(math.sqrt(5.0))

    def test_validation(self):
        for kw in ({"kind": "cauchy"}, {"kind": "histogram", "bins": 0}, {"kind": "epanechnikov", "k": 0.0}):
            with pytest.raises(ValueError):
                cpb.ModelSpec(**kw)


class TestEnsembleStack:
    def test_shape_properties(self):
        stack = sample_stack()
        assert (stack.members, stack.height, stack.width) == (30, 6, 7)
        assert stack.values.dtype == np.float32

    def test_validation(self):
        with pytest.raises(ValueError):
            cpb.EnsembleStack(np.zeros((4, 5)))
        with pytest.raises(ValueError):
            cpb.EnsembleStack(np.zeros((0, 4, 5)))
        bad = np.zeros((2, 3, 3))
        bad[1, 1, 1] = np.nan
        with pytest.raises(ValueError):
            cpb.EnsembleStack(bad)

    def test_normalized_range_and_map(self):
        stack = sample_stack(3)
        norm, scale, offset = stack.normalized()
        assert norm.values.min() == pytest.approx(0.0, abs=1e-7)
        assert norm.values.max() == pytest.approx(1.0, abs=1e-7)
        assert norm.values == pytest.approx(scale * stack.values.astype(np.float64) + offset, abs=1e-6)

    def test_normalized_degenerate(self):
        stack = cpb.EnsembleStack(np.full((3, 4, 4), 2.5, dtype=np.float32))
        norm, scale, offset = stack.normalized()
        assert scale == 1.0 and offset == 0.0 and np.array_equal(norm.values, stack.values)


class TestProbabilityField:
    def test_empty(self):
        prob = cpb.ProbabilityField.empty(4, 5)
        assert prob.shape == (4, 5) and not prob.valid.any() and prob.p_min.sum() == 0.0

    def test_channel_lookup(self):
        prob = cpb.ProbabilityField.empty(3, 3)
        assert prob.channel("min") is prob.p_min and prob.channel("max") is prob.p_max
        assert prob.channel("saddle") is prob.p_saddle
        with pytest.raises(ValueError):
            prob.channel("ridge")

    def test_shape_mismatch_rejected(self):
        with pytest.raises(ValueError):
            cpb.ProbabilityField(np.zeros((3, 3)), np.zeros((3, 3)), np.zeros((3, 4)),
                                 np.zeros((3, 3), dtype=bool))
