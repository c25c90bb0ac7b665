"""B200-native critical-point probabilities for uncertain 2-D ensembles (arXiv 2407.18015).

Drop-in for the grid hot path of the reference ``critprob`` package: the
noise-model fit (``UncertainField.from_ensemble`` / ``from_scalar``), the
closed-form min/max/saddle stencil and the Monte Carlo estimator
(``classify_field``), computed by hand-written sm_100a CUDA kernels behind
the C ABI in include/critprob_b200.h.  There is no CPU fallback.
"""

from .cases import (
    CaseBatch,
    FiniteDistribution,
    GaussianSampler,
    NeighborhoodCase,
    ProbabilityTriple,
    Support,
    ValidationSummary,
    case_at,
    closed_form_triple,
    closed_form_triples,
    closed_pattern_prob,
    combinatorial_batch,
    combinatorial_triple,
    epanechnikov,
    histogram,
    histogram_min_prob_combinatorial,
    local_max_prob,
    local_min_prob,
    mc_all_patterns,
    mc_all_patterns_batch,
    mc_pattern_prob,
    random_case,
    saddle_prob,
    semianalytical_batch,
    semianalytical_prob,
    uniform,
    validate_random_cases,
)
from .engine import (
    COMBINATORIAL_MAX_BINS,
    ESTIMATOR_METHODS,
    PATTERNS,
    EstimatorSpec,
    classify_field,
    pixel_index,
)
from .fields import (
    CHANNELS,
    MODEL_KINDS,
    EnsembleStack,
    ModelSpec,
    ProbabilityField,
    UncertainField,
    pinned_empty,
    set_device,
)
from .field_io import (
    UcvfError,
    UcvfFormatError,
    UcvfPayloadError,
    UcvfValueError,
    export_heatmap,
    load_ensemble,
    load_probability_field,
    load_scalar_field,
    save_ensemble,
    save_probability_field,
    save_scalar_field,
    uniform_field_from_scalar,
)
from .rngstream import unit_block, unit_planes
from .synth import synthetic_ensemble, synthetic_rows

__all__ = [
    "CHANNELS", "COMBINATORIAL_MAX_BINS", "ESTIMATOR_METHODS", "MODEL_KINDS", "PATTERNS",
    "EnsembleStack", "EstimatorSpec", "ModelSpec", "ProbabilityField", "UncertainField",
    "classify_field", "pinned_empty", "pixel_index", "set_device", "synthetic_ensemble", "synthetic_rows",
    "unit_block", "unit_planes", "UcvfError", "UcvfFormatError", "UcvfPayloadError",
    "UcvfValueError", "export_heatmap", "load_ensemble", "load_probability_field",
    "load_scalar_field", "save_ensemble", "save_probability_field", "save_scalar_field",
    "uniform_field_from_scalar",
    # per-case API (engine.py:50-459) as GPU batches
    "CaseBatch", "FiniteDistribution", "GaussianSampler", "NeighborhoodCase", "ProbabilityTriple",
    "Support", "ValidationSummary", "case_at", "closed_form_triple", "closed_form_triples",
    "closed_pattern_prob", "combinatorial_batch", "combinatorial_triple", "epanechnikov", "histogram",
    "histogram_min_prob_combinatorial", "local_max_prob", "local_min_prob", "mc_all_patterns",
    "mc_all_patterns_batch", "mc_pattern_prob", "random_case", "saddle_prob", "semianalytical_batch",
    "semianalytical_prob", "uniform", "validate_random_cases",
]
