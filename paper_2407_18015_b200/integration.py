"""Swap the reference package's hot-path entry points for the GPU path.

    import critprob
    from paper_2407_18015_b200.integration import patch_reference
    patch_reference(critprob)          # critprob.classify_field & co. now run on the B200

This is the drop-in proof at the reference's own boundary (its Python API;
the reference has no FFI): after the patch, code written against ``critprob``
-- including the reference's own unmodified test suite
(tools/run_reference_tests.py) -- calls the sm_100a kernels for

- ``UncertainField.from_ensemble`` / ``from_scalar``   fields.py:125-178
- ``classify_field`` (every estimator)                 engine.py:716-787
- per case (``patch_cases=True``): ``closed_form_triple``, ``local_min_prob``,
  ``local_max_prob``, ``saddle_prob``, ``closed_pattern_prob``,
  ``mc_all_patterns``, ``mc_pattern_prob``, ``semianalytical_prob``,
  ``combinatorial_triple``, ``histogram_min_prob_combinatorial``
                                                       engine.py:127-441

Inputs and results stay the reference's own types (its ``UncertainField``
with the float64 ``params`` dict, ``ProbabilityField``, ``ProbabilityTriple``),
so everything downstream of the call is untouched.  The reference module is
passed in by the caller: this package never imports it.
"""

from __future__ import annotations

import functools

import numpy as np

_PATCHED_ATTR = "__cpb_patched__"


def _model(m):
    from .fields import ModelSpec

    return ModelSpec(kind=m.kind, bins=m.bins, k=m.k)


def _estimator(e):
    from .engine import EstimatorSpec

    if e is None:
        return None
    return EstimatorSpec(method=e.method, n_samples=e.n_samples, c=e.c, seed=e.seed)


def patch_reference(critprob, patch_cases: bool = True) -> dict:
    """Replace the reference's entry points (in every loaded critprob module
    that bound them) with GPU-backed wrappers.  Returns {name: original}."""
    import sys

    from . import cases as C
    from . import engine as E
    from . import fields as F

    rf = sys.modules[critprob.__name__ + ".fields"]
    re_ = sys.modules[critprob.__name__ + ".engine"]
    originals = {}

    # ---- fit (classmethods: patched on the class itself)
    RefField = rf.UncertainField
    if not getattr(RefField.from_ensemble, _PATCHED_ATTR, False):
        originals["from_ensemble"] = RefField.__dict__["from_ensemble"]
        originals["from_scalar"] = RefField.__dict__["from_scalar"]

        def from_ensemble(cls, stack, model):
            vals = np.asarray(stack.values)
            if vals.shape[0] < 2 and model.kind in ("epanechnikov", "gaussian"):
                raise ValueError(f"{model.kind} fit needs at least two members")
            ours = F.UncertainField.from_ensemble(F.EnsembleStack(vals), _model(model))
            return cls(model, ours.params)

        def from_scalar(cls, values, error_bound):
            ours = F.UncertainField.from_scalar(values, error_bound)
            return cls(rf.ModelSpec("uniform"), ours.params)

        from_ensemble.__cpb_patched__ = True
        RefField.from_ensemble = classmethod(from_ensemble)
        RefField.from_scalar = classmethod(from_scalar)

    # ---- grid classification
    RefProb = rf.ProbabilityField

    def classify_field(field, estimator=None, workers=1, channels=F.CHANNELS):
        ours = F.UncertainField(_model(field.model), field.params)
        res = E.classify_field(ours, _estimator(estimator), workers, channels)
        return RefProb(res.p_min, res.p_max, res.p_saddle, res.valid)

    repl = {"classify_field": classify_field}

    # ---- per case
    if patch_cases:
        Triple = re_.ProbabilityTriple

        def triple(fn):
            @functools.wraps(fn)
            def w(*a, **k):
                return Triple(*fn(*a, **k))
            return w

        repl.update({
            "closed_form_triple": triple(C.closed_form_triple),
            "local_min_prob": C.local_min_prob,
            "local_max_prob": C.local_max_prob,
            "saddle_prob": C.saddle_prob,
            "closed_pattern_prob": C.closed_pattern_prob,
            "mc_all_patterns": triple(C.mc_all_patterns),
            "mc_pattern_prob": C.mc_pattern_prob,
            "semianalytical_prob": C.semianalytical_prob,
            "combinatorial_triple": triple(C.combinatorial_triple),
            "histogram_min_prob_combinatorial": C.histogram_min_prob_combinatorial,
        })
    for name, fn in repl.items():
        orig = getattr(re_, name)
        if getattr(orig, _PATCHED_ATTR, False):
            continue
        originals[name] = orig
        setattr(fn, _PATCHED_ATTR, True)
        # every loaded critprob module that imported the name (from .engine import ...)
        for mname, mod in list(sys.modules.items()):
            if (mname == critprob.__name__ or mname.startswith(critprob.__name__ + ".")) and \
                    getattr(mod, name, None) is orig:
                setattr(mod, name, fn)
    return originals
