"""Grid classification with the reference's API, computed by the sm_100a kernels.

Mirrors the grid entry points of critprob.engine
(/root/reference/pkg/src/critprob/engine.py):

- ``EstimatorSpec``   engine.py:88-105 (same fields, defaults, ValueErrors)
- ``classify_field``  engine.py:716-787 (same signature, validation order and
                      ProbabilityField result; ``workers`` is accepted and,
                      as in the reference, never changes the result)
- ``pixel_index``     engine.py:482-484

Closed form runs ``cpb_classify_closed``, Monte Carlo ``cpb_classify_mc``,
the semianalytical estimator ``cpb_classify_semi`` and the combinatorial
(Eq. 5) cross-check ``cpb_classify_combinatorial`` (include/critprob_b200.h).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fields import CHANNELS, ProbabilityField, UncertainField

PATTERNS = ("min", "max", "saddle")
ESTIMATOR_METHODS = ("closed_form", "monte_carlo", "semianalytical", "combinatorial")
# closed form: "fp64" (parity with the reference to ~1e-15) or "mixed": float64
# partition and accumulation, single-precision Gauss-Legendre evaluation for the
# uniform and Epanechnikov stencils (north_star bound 1e-6 absolute, measured
# ~1.5e-7); histogram fields stay fp64 (24-bit positions cannot resolve bin
# edges several bins away to 1e-6)
PRECISIONS = ("fp64", "mixed")
COMBINATORIAL_MAX_BINS = 8


@dataclass(frozen=True)
class EstimatorSpec:
    """How to estimate per-pixel probabilities (engine.py:88-105).

    ``n_samples`` applies to monte_carlo, ``c`` to semianalytical; ``seed``
    keys the deterministic sample streams.  ``rng`` selects the Monte Carlo
    uniform stream: "splitmix64" (the reference's, bit-exact) or "philox".
    """

    method: str = "closed_form"
    n_samples: int = 2000
    c: int = 10000
    seed: int = 0
    rng: str = "splitmix64"
    precision: str = "fp64"

    def __post_init__(self) -> None:
        if self.method not in ESTIMATOR_METHODS:
            raise ValueError(f"unknown estimator method {self.method!r}")
        if self.n_samples < 1 or self.c < 1:
            raise ValueError("sample counts must be positive")
        if self.rng not in _lib.RNG_CODES:
            raise ValueError(f"unknown rng {self.rng!r}")
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}")


def pixel_index(field: UncertainField, row: int, col: int) -> int:
    """Flat pixel key used for the deterministic per-pixel sample streams (engine.py:482-484)."""
    return row * field.width + col


def _validate(field: UncertainField, estimator: EstimatorSpec, workers: int, channels):
    """engine.py:729-749, in the same order."""
    if isinstance(channels, str):
        channels = (channels,)
    for ch in channels:
        if ch not in CHANNELS:
            raise ValueError(f"unknown channel {ch!r}")
    height, width = field.shape
    if height < 3 or width < 3:
        raise ValueError("field must be at least 3 x 3 to have interior pixels")
    kind = field.model.kind
    method = estimator.method
    if method == "closed_form" and kind == "gaussian":
        raise ValueError("Gaussian fields have no closed form; use monte_carlo")
    if method in ("semianalytical", "combinatorial") and kind != "histogram":
        raise ValueError(f"{method} estimation is defined for histogram fields only")
    if method == "combinatorial" and field.model.bins > COMBINATORIAL_MAX_BINS:
        raise ValueError(
            f"combinatorial estimation refuses more than {COMBINATORIAL_MAX_BINS} bins")
    if workers < 1:
        raise ValueError("workers must be positive")
    return tuple(channels)


def run_rows(dev, estimator: EstimatorSpec, channels, row_begin: int, row_end: int, out: dict,
             counts=None, type_sums=None) -> None:
    """Enqueue the estimator for local rows [row_begin, row_end) into device planes ``out``.

    ``type_sums`` (closed form): a 3-double CUDA tensor the per-type sums of
    these rows are ADDED to, fused into the stencil kernels' epilogue.
    """
    lib = _lib.load()
    s = _lib.stream_ptr()
    pm = out["min"] if "min" in channels else None
    pM = out["max"] if "max" in channels else None
    pS = out["saddle"] if "saddle" in channels else None
    if estimator.method == "closed_form":
        st = dev.ref()
        if estimator.precision == "mixed":
            st = _lib.CpbField.from_buffer_copy(dev.struct)
            st.flags |= _lib.FLAG_MIXED
            st = ctypes.byref(st)
        if type_sums is not None:
            _lib.check(lib.cpb_classify_closed_counts(st, row_begin, row_end, _lib.ptr(pm),
                                                      _lib.ptr(pM), _lib.ptr(pS),
                                                      type_sums.data_ptr(), s))
        else:
            _lib.check(lib.cpb_classify_closed(st, row_begin, row_end, _lib.ptr(pm),
                                               _lib.ptr(pM), _lib.ptr(pS), s))
    elif estimator.method == "monte_carlo":
        seed = int(estimator.seed) & ((1 << 64) - 1)
        _lib.check(lib.cpb_classify_mc(dev.ref(), row_begin, row_end, seed,
                                       int(estimator.n_samples), _lib.RNG_CODES[estimator.rng],
                                       _lib.ptr(pm), _lib.ptr(pM), _lib.ptr(pS), _lib.ptr(counts), s))
    elif estimator.method == "semianalytical":
        seed = int(estimator.seed) & ((1 << 64) - 1)
        _lib.check(lib.cpb_classify_semi(dev.ref(), row_begin, row_end, seed, int(estimator.c),
                                         _lib.ptr(pm), _lib.ptr(pM), _lib.ptr(pS), s))
    else:  # combinatorial (validated: histogram, bins <= COMBINATORIAL_MAX_BINS)
        _lib.check(lib.cpb_classify_combinatorial(dev.ref(), row_begin, row_end, _lib.ptr(pm),
                                                  _lib.ptr(pM), _lib.ptr(pS), s))


def classify_field(
    field: UncertainField,
    estimator: EstimatorSpec | None = None,
    workers: int = 1,
    channels=CHANNELS,
    *,
    output: str = "host",
    counts_out=None,
) -> ProbabilityField:
    """Per-pixel critical-point probabilities over the interior pixels (engine.py:716-787).

    The one-pixel border is marked invalid and unrequested channels stay
    exactly 0.0.  ``output="device"`` keeps the result planes in HBM as CUDA
    tensors (no device-to-host copy); ``counts_out`` (a dict) receives the
    Monte Carlo hit counts as an int64 (3, H, W) device tensor.
    """
    import torch

    estimator = estimator or EstimatorSpec()
    channels = _validate(field, estimator, workers, channels)
    dev = field.device_field()
    H, W = field.shape
    planes = torch.zeros((3, H, W), dtype=torch.float64, device=dev.device)
    out = {"min": planes[0], "max": planes[1], "saddle": planes[2]}
    counts = None
    if counts_out is not None and estimator.method == "monte_carlo":
        counts = torch.zeros((3, H, W), dtype=torch.int64, device=dev.device)
        counts_out["counts"] = counts
    run_rows(dev, estimator, channels, 1, H - 1, out, counts)
    valid = torch.zeros((H, W), dtype=torch.bool, device=dev.device)
    valid[1:-1, 1:-1] = True
    if output == "device":
        return ProbabilityField(planes[0], planes[1], planes[2], valid)
    # one D2H into page-locked memory (torch's caching host allocator: a result
    # array that is dropped returns its buffer for the next call, so repeated
    # calls copy at DMA speed); the channels are views of it (no host copies)
    host_t = torch.empty((3, H, W), dtype=torch.float64, pin_memory=True)
    host_t.copy_(planes, non_blocking=True)
    torch.cuda.current_stream(dev.device).synchronize()
    host = host_t.numpy()
    mask = np.zeros((H, W), dtype=bool)
    mask[1:-1, 1:-1] = True
    return ProbabilityField(host[0], host[1], host[2], mask)
