"""Per-case API of the reference, evaluated as GPU batches.

Mirrors the single-neighbourhood interface of critprob
(/root/reference/pkg/src/critprob):

- distributions ``Support``, ``FiniteDistribution``, ``GaussianSampler``,
  ``uniform`` / ``epanechnikov`` / ``histogram``   distributions.py:38-274, 279-289
- ``NeighborhoodCase``, ``ProbabilityTriple``       engine.py:50-85
- ``local_min_prob``, ``local_max_prob``, ``saddle_prob``, ``closed_form_triple``,
  ``closed_pattern_prob``                           engine.py:127-188
- ``mc_all_patterns``, ``mc_pattern_prob``          engine.py:238-263
- ``semianalytical_prob``                           engine.py:416-441
- ``histogram_min_prob_combinatorial``, ``combinatorial_triple``  engine.py:359-404
- ``case_at``                                       engine.py:466-479
- ``random_case``                                   synth.py:124-151
- ``validate_random_cases``, ``ValidationSummary``  bench.py:215-267

The reference evaluates these one case at a time in Python; here every call
packs its cases into a ``CaseBatch`` (flat device arrays, the
``cpb_case_batch`` of include/critprob_b200.h) and runs one kernel over all
of them: ``closed_form_triples`` / ``mc_all_patterns_batch`` /
``semianalytical_batch`` / ``combinatorial_batch`` take lists of cases (or a
prebuilt ``CaseBatch``) and return an (n, 3) float64 array of (p_min, p_max,
p_saddle).  The scalar functions are batches of one.  There is no CPU path.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

PATTERNS = ("min", "max", "saddle")
MODEL_KINDS = ("uniform", "epanechnikov", "histogram", "gaussian")
COMBINATORIAL_MAX_BINS = 8
_KINDS = ("uniform", "epanechnikov", "histogram")


# ----------------------------------------------------------- distributions
@dataclass(frozen=True)
class Support:
    """Closed support interval (distributions.py:38-52)."""

    lo: float
    hi: float

    @property
    def width(self) -> float:
        return self.hi - self.lo

    def __post_init__(self) -> None:
        if not math.isfinite(self.lo) or not math.isfinite(self.hi):
            raise ValueError("support bounds must be finite")
        if not self.hi > self.lo:
            raise ValueError(f"support must have positive width, got [{self.lo}, {self.hi}]")


class FiniteDistribution:
    """Bounded per-pixel model (distributions.py:105-242); histogram weights are
    stored normalised (w / w.sum()), as the reference constructor does."""

    __slots__ = ("kind", "support", "bin_weights")
    u01_planes = 1

    def __init__(self, kind: str, support: Support, bin_weights=None) -> None:
        if kind not in _KINDS:
            raise ValueError(f"unknown distribution kind {kind!r}")
        if kind == "histogram":
            w = np.asarray(bin_weights, dtype=float)
            if w.ndim != 1 or w.size == 0:
                raise ValueError("histogram needs a 1-D, non-empty weight array")
            if np.any(w < 0.0) or not np.all(np.isfinite(w)):
                raise ValueError("histogram weights must be finite and non-negative")
            total = w.sum()
            if total <= 0.0:
                raise ValueError("histogram weights must not all be zero")
            bin_weights = w / total
        elif bin_weights is not None:
            raise ValueError(f"{kind} takes no bin weights")
        self.kind = kind
        self.support = support
        self.bin_weights = bin_weights

    def __repr__(self) -> str:
        extra = f", bins={self.bin_weights.size}" if self.kind == "histogram" else ""
        return f"FiniteDistribution({self.kind}, [{self.support.lo}, {self.support.hi}]{extra})"

    def negate(self) -> "FiniteDistribution":
        """Distribution of -X (distributions.py:196-200)."""
        w = None if self.bin_weights is None else self.bin_weights[::-1]
        return FiniteDistribution(self.kind, Support(-self.support.hi, -self.support.lo), w)

    def affine(self, alpha: float, beta: float) -> "FiniteDistribution":
        """Distribution of alpha X + beta, alpha > 0 (distributions.py:202-210)."""
        if not alpha > 0.0:
            raise ValueError("affine scale must be positive")
        lo, hi = self.support.lo, self.support.hi
        return FiniteDistribution(self.kind, Support(alpha * lo + beta, alpha * hi + beta),
                                  self.bin_weights)


@dataclass(frozen=True)
class GaussianSampler:
    """Unbounded normal model, Monte Carlo only (distributions.py:245-274)."""

    mean: float
    stddev: float
    u01_planes = 2

    def __post_init__(self) -> None:
        if self.stddev < 0.0 or not math.isfinite(self.stddev):
            raise ValueError("stddev must be finite and non-negative")

    def negate(self) -> "GaussianSampler":
        return GaussianSampler(-self.mean, self.stddev)

    def affine(self, alpha: float, beta: float) -> "GaussianSampler":
        if not alpha > 0.0:
            raise ValueError("affine scale must be positive")
        return GaussianSampler(alpha * self.mean + beta, alpha * self.stddev)


def uniform(lo: float, hi: float) -> FiniteDistribution:
    return FiniteDistribution("uniform", Support(float(lo), float(hi)))


def epanechnikov(mean: float, halfwidth: float) -> FiniteDistribution:
    if not halfwidth > 0.0:
        raise ValueError("halfwidth must be positive")
    return FiniteDistribution("epanechnikov", Support(float(mean - halfwidth), float(mean + halfwidth)))


def histogram(lo: float, hi: float, weights) -> FiniteDistribution:
    return FiniteDistribution("histogram", Support(float(lo), float(hi)), weights)


# ------------------------------------------------------------------ cases
@dataclass(frozen=True)
class NeighborhoodCase:
    """A centre distribution plus its 2 or 4 axis neighbours (engine.py:50-71)."""

    center: object
    neighbors: tuple

    def __post_init__(self) -> None:
        object.__setattr__(self, "neighbors", tuple(self.neighbors))
        if len(self.neighbors) not in (2, 4):
            raise ValueError("a neighborhood has exactly 2 or 4 neighbors")

    def negate(self) -> "NeighborhoodCase":
        return NeighborhoodCase(self.center.negate(), tuple(d.negate() for d in self.neighbors))

    def affine(self, alpha: float, beta: float) -> "NeighborhoodCase":
        return NeighborhoodCase(self.center.affine(alpha, beta),
                                tuple(d.affine(alpha, beta) for d in self.neighbors))


@dataclass(frozen=True)
class ProbabilityTriple:
    p_min: float
    p_max: float
    p_saddle: float

    def __iter__(self):
        return iter((self.p_min, self.p_max, self.p_saddle))

    @property
    def total(self) -> float:
        return self.p_min + self.p_max + self.p_saddle


# ------------------------------------------------------------- the batch
class CaseBatch:
    """n cases of one neighbourhood size as flat device arrays (cpb_case_batch).

    Build it from case objects (``pack``) or, for large batches, straight from
    arrays (``from_arrays``): kind / a / b / bins of shape (n, 1 + k) and the
    histogram weights zero-padded to (n, 1 + k, max_bins).
    """

    def __init__(self, neighbors, kind, a, b, bins, weights):
        import torch

        from .fields import _device

        kind = np.ascontiguousarray(kind, dtype=np.int32)
        if kind.ndim != 2 or kind.shape[1] != neighbors + 1 or neighbors not in (2, 4):
            raise ValueError("a neighborhood has exactly 2 or 4 neighbors")
        n, P = kind.shape
        bins = np.ascontiguousarray(bins, dtype=np.int32).reshape(n, P)
        weights = np.asarray(weights, dtype=np.float64)
        maxb = max(1, int(bins[kind == 2].max()) if np.any(kind == 2) else 1)
        if weights.ndim != 3 or weights.shape[:2] != (n, P) or weights.shape[2] < maxb:
            raise ValueError("weights must be (n, 1 + neighbors, >= max bins)")
        self.n, self.neighbors, self.max_bins = n, neighbors, maxb
        self.kind = kind
        self.bins = bins
        dev = _device()
        flat = np.ascontiguousarray(weights[:, :, :maxb]).reshape(-1)
        woff = (np.arange(n * P, dtype=np.int64) * maxb)
        self._t = {
            "kind": torch.from_numpy(kind.reshape(-1)).to(dev),
            "a": torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to(dev),
            "b": torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64).reshape(-1)).to(dev),
            "bins": torch.from_numpy(bins.reshape(-1)).to(dev),
            "woff": torch.from_numpy(woff).to(dev),
            "weights": torch.from_numpy(flat if flat.size else np.zeros(1)).to(dev),
        }
        self.struct = _lib.CpbCaseBatch(
            n, neighbors, maxb, *[self._t[k].data_ptr() for k in ("kind", "a", "b", "bins", "woff", "weights")])

    @classmethod
    def from_arrays(cls, neighbors, kind, a, b, bins, weights) -> "CaseBatch":
        return cls(neighbors, kind, a, b, bins, weights)

    @classmethod
    def pack(cls, cases) -> "CaseBatch":
        return cls(*pack_arrays(cases))

    def _require_bounded(self) -> None:
        if np.any(self.kind == 3):
            raise TypeError("closed-form evaluation needs bounded distributions; "
                            "Gaussian models support Monte Carlo only")

    def _require_histograms(self) -> None:
        if np.any(self.kind != 2):
            raise ValueError("this estimator is defined for histogram inputs only")

    def _pixels(self, pixels):
        import torch

        if pixels is None:
            return None
        px = np.asarray(pixels, dtype=np.uint64).reshape(-1)
        if px.size != self.n:
            raise ValueError("need one pixel key per case")
        return torch.from_numpy(px.view(np.int64)).to(self._t["kind"].device)

    def _out(self):
        import torch

        return torch.empty((self.n, 3), dtype=torch.float64, device=self._t["kind"].device)

    def _finish(self, out) -> np.ndarray:
        import torch

        torch.cuda.synchronize(out.device)
        return out.cpu().numpy()

    # ---- estimators -------------------------------------------------------
    def closed(self) -> np.ndarray:
        self._require_bounded()
        lib = _lib.load()
        out = self._out()
        _lib.check(lib.cpb_cases_closed(ctypes.byref(self.struct), out.data_ptr(), _lib.stream_ptr()))
        return self._finish(out)

    def monte_carlo(self, n: int, seed: int = 0, pixels=None, counts: bool = False):
        if n < 1:
            raise ValueError("n must be positive")
        import torch

        lib = _lib.load()
        out = self._out()
        px = self._pixels(pixels)
        cnt = torch.empty((self.n, 3), dtype=torch.int64, device=out.device) if counts else None
        _lib.check(lib.cpb_cases_mc(ctypes.byref(self.struct), int(seed) & ((1 << 64) - 1),
                                    _lib.ptr(px), int(n), _lib.ptr(cnt), out.data_ptr(),
                                    _lib.stream_ptr()))
        res = self._finish(out)
        return (res, cnt.cpu().numpy()) if counts else res

    def semianalytical(self, c: int, seed: int = 0, pixels=None) -> np.ndarray:
        if c < 1:
            raise ValueError("c must be positive")
        self._require_histograms()
        lib = _lib.load()
        out = self._out()
        px = self._pixels(pixels)
        _lib.check(lib.cpb_cases_semi(ctypes.byref(self.struct), int(seed) & ((1 << 64) - 1),
                                      _lib.ptr(px), int(c), out.data_ptr(), _lib.stream_ptr()))
        return self._finish(out)

    def combinatorial(self) -> np.ndarray:
        self._require_histograms()
        if self.max_bins > COMBINATORIAL_MAX_BINS:
            raise ValueError(f"combinatorial cost grows as bins**{self.neighbors + 1}; "
                             f"refusing more than {COMBINATORIAL_MAX_BINS} bins")
        lib = _lib.load()
        out = self._out()
        _lib.check(lib.cpb_cases_combinatorial(ctypes.byref(self.struct), out.data_ptr(),
                                               _lib.stream_ptr()))
        return self._finish(out)


def pack_arrays(cases):
    """Case objects -> (neighbors, kind, a, b, bins, weights) host arrays (cpb_case_batch layout)."""
    cases = list(cases)
    if not cases:
        raise ValueError("need at least one case")
    k = len(cases[0].neighbors)
    if any(len(c.neighbors) != k for c in cases):
        raise ValueError("a batch needs one neighbourhood size")
    P = k + 1
    maxb = 1
    for c in cases:
        for d in (c.center, *c.neighbors):
            if getattr(d, "bin_weights", None) is not None:
                maxb = max(maxb, d.bin_weights.size)
    n = len(cases)
    kind = np.zeros((n, P), np.int32)
    a = np.zeros((n, P))
    b = np.zeros((n, P))
    bins = np.ones((n, P), np.int32)
    w = np.zeros((n, P, maxb))
    for i, c in enumerate(cases):
        for p, d in enumerate((c.center, *c.neighbors)):
            # duck-typed, so the reference's own distribution objects pack too
            # (integration.patch_reference)
            if not hasattr(d, "support") and hasattr(d, "stddev"):  # GaussianSampler
                kind[i, p], a[i, p], b[i, p] = 3, d.mean, d.stddev
                continue
            if getattr(d, "kind", None) not in _KINDS or not hasattr(d, "support"):
                raise TypeError(f"unsupported distribution {type(d).__name__}")
            kind[i, p] = _lib.KIND_CODES[d.kind]
            a[i, p], b[i, p] = d.support.lo, d.support.hi
            if d.kind == "histogram":
                bins[i, p] = d.bin_weights.size
                w[i, p, :d.bin_weights.size] = d.bin_weights
    return k, kind, a, b, bins, w


def _cases(cases):
    return cases if isinstance(cases, CaseBatch) else list(cases)


def _count(cases) -> int:
    return cases.n if isinstance(cases, CaseBatch) else len(cases)


def _batches(cases):
    """Group cases by neighbourhood size; returns [(indices, CaseBatch)]."""
    if isinstance(cases, CaseBatch):
        return [(np.arange(cases.n), cases)], cases.n
    cases = list(cases)
    groups = {}
    for i, c in enumerate(cases):
        groups.setdefault(len(c.neighbors), []).append(i)
    return [(np.array(idx), CaseBatch.pack([cases[i] for i in idx])) for idx in groups.values()], len(cases)


def _run(cases, fn, pixels=None) -> np.ndarray:
    groups, n = _batches(cases)
    out = np.empty((n, 3))
    px = None if pixels is None else np.asarray(pixels, dtype=np.uint64).reshape(-1)
    for idx, batch in groups:
        out[idx] = fn(batch, None if px is None else px[idx])
    return out


# ------------------------------------------------------------ batch API
def closed_form_triples(cases) -> np.ndarray:
    """closed_form_triple of every case: (n, 3) float64.

    As in the reference (engine.py:139-142, 177-178) p_max is the minimum
    probability of the NEGATED case, so local_max_prob(c) == local_min_prob(
    c.negate()) holds bit for bit; case objects and their negations go to the
    device as one batch.  (A prebuilt CaseBatch takes p_max from the direct
    product-of-CDFs integral of the same walk instead.)
    """
    cases = _cases(cases)
    if isinstance(cases, CaseBatch):
        return cases.closed()
    n = len(cases)
    both = _run(list(cases) + [c.negate() for c in cases], lambda b, _: b.closed())
    out = both[:n].copy()
    out[:, 1] = both[n:, 0]
    return out


def mc_all_patterns_batch(cases, n: int, seed: int = 0, pixels=None) -> np.ndarray:
    """mc_all_patterns(case_i, n, seed, pixels[i]) (pixel i when pixels is None)."""
    if n < 1:
        raise ValueError("n must be positive")
    cases = _cases(cases)
    if pixels is None:
        pixels = np.arange(_count(cases), dtype=np.uint64)
    return _run(cases, lambda b, px: b.monte_carlo(n, seed, px), pixels)


def semianalytical_batch(cases, c: int, seed: int = 0, pixels=None) -> np.ndarray:
    """semianalytical_prob for min, max, saddle of every case (histogram cases)."""
    if c < 1:
        raise ValueError("c must be positive")
    cases = _cases(cases)
    if pixels is None:
        pixels = np.arange(_count(cases), dtype=np.uint64)
    return _run(cases, lambda b, px: b.semianalytical(c, seed, px), pixels)


def combinatorial_batch(cases) -> np.ndarray:
    """combinatorial_triple of every case (histogram cases, <= 8 bins)."""
    return _run(_cases(cases), lambda b, _: b.combinatorial())


# ------------------------------------------------------ single-case API
def closed_form_triple(case: NeighborhoodCase) -> ProbabilityTriple:
    return ProbabilityTriple(*map(float, closed_form_triples([case])[0]))


def local_min_prob(case: NeighborhoodCase) -> float:
    """Probability that the centre draws strictly below every neighbour (engine.py:127-136)."""
    return closed_form_triple(case).p_min


def local_max_prob(case: NeighborhoodCase) -> float:
    return closed_form_triple(case).p_max


def saddle_prob(case: NeighborhoodCase) -> float:
    return closed_form_triple(case).p_saddle


def closed_pattern_prob(case: NeighborhoodCase, pattern: str) -> float:
    if pattern not in PATTERNS:
        raise ValueError(f"unknown pattern {pattern!r}")
    return dict(zip(PATTERNS, closed_form_triple(case)))[pattern]


def mc_all_patterns(case: NeighborhoodCase, n: int, seed: int = 0, pixel: int = 0) -> ProbabilityTriple:
    """All three pattern fractions from one set of joint draws (engine.py:238-247)."""
    if n < 1:
        raise ValueError("n must be positive")
    return ProbabilityTriple(*map(float, mc_all_patterns_batch([case], n, seed, [pixel])[0]))


def mc_pattern_prob(case: NeighborhoodCase, pattern: str, n: int, seed: int = 0, pixel: int = 0) -> float:
    if pattern not in PATTERNS:
        raise ValueError(f"unknown pattern {pattern!r}")
    if n < 1:
        raise ValueError("n must be positive")
    return dict(zip(PATTERNS, mc_all_patterns(case, n, seed, pixel)))[pattern]


def semianalytical_prob(case: NeighborhoodCase, pattern: str, c: int, seed: int = 0, pixel: int = 0) -> float:
    if pattern not in PATTERNS:
        raise ValueError(f"unknown pattern {pattern!r}")
    if c < 1:
        raise ValueError("c must be positive")
    return float(dict(zip(PATTERNS, semianalytical_batch([case], c, seed, [pixel])[0]))[pattern])


def combinatorial_triple(case: NeighborhoodCase) -> ProbabilityTriple:
    return ProbabilityTriple(*map(float, combinatorial_batch([case])[0]))


def histogram_min_prob_combinatorial(case: NeighborhoodCase) -> float:
    return combinatorial_triple(case).p_min


def case_at(field, row: int, col: int) -> NeighborhoodCase:
    """The 4-neighbourhood at an interior pixel, east, north, west, south (engine.py:466-479)."""
    height, width = field.shape
    if not (1 <= row < height - 1 and 1 <= col < width - 1):
        raise ValueError("neighborhood requires an interior pixel")
    d = field.dist_at
    return NeighborhoodCase(d(row, col), (d(row, col + 1), d(row - 1, col), d(row, col - 1), d(row + 1, col)))


def dist_at(field, row: int, col: int):
    """The pixel's distribution from the stored parameters (UncertainField.dist_at, fields.py:109-121)."""
    p = field.params
    kind = field.model.kind
    if kind == "uniform":
        return uniform(p["lo"][row, col], p["hi"][row, col])
    if kind == "epanechnikov":
        return epanechnikov(p["mean"][row, col], p["halfwidth"][row, col])
    if kind == "histogram":
        return histogram(p["lo"][row, col], p["hi"][row, col], p["weights"][row, col])
    return GaussianSampler(float(p["mean"][row, col]), float(p["stddev"][row, col]))


# ------------------------------------------------------ random cases / fuzz
def random_case(seed: int, model: str = "uniform", neighborhood: int = 4, bins: int = 5) -> NeighborhoodCase:
    """Seeded random neighbourhood whose supports pairwise overlap (synth.py:124-151)."""
    if model not in MODEL_KINDS:
        raise ValueError(f"unknown model kind {model!r}")
    if neighborhood not in (2, 4):
        raise ValueError("neighborhood must be 2 or 4")
    rng = np.random.default_rng(seed)
    count = neighborhood + 1
    centers = rng.uniform(-0.25, 0.25, count)
    halfwidths = rng.uniform(0.4, 0.8, count)
    dists = []
    for c, h in zip(centers, halfwidths):
        if model == "uniform":
            dists.append(uniform(c - h, c + h))
        elif model == "epanechnikov":
            dists.append(epanechnikov(c, h))
        elif model == "histogram":
            weights = rng.uniform(0.05, 1.0, bins)
            dists.append(histogram(c - h, c + h, weights / weights.sum()))
        else:
            dists.append(GaussianSampler(c, 0.5 * h))
    return NeighborhoodCase(dists[0], tuple(dists[1:]))


@dataclass
class ValidationSummary:
    """Fuzz comparison of the closed form against the MC oracle (bench.py:215-232)."""

    model: str
    cases: int
    samples: int
    max_abs_dev: float
    max_se_dev: float
    within_4se: float

    def to_text(self) -> str:
        return (
            f"validate model={self.model}: {self.cases} cases, "
            f"mc n={self.samples}; max |closed-mc| = {self.max_abs_dev:.6f} "
            f"({self.max_se_dev:.2f} standard errors), "
            f"{100.0 * self.within_4se:.1f}% of checks within 4 SE"
        )


def validate_random_cases(cases: int, model: str = "uniform", neighborhood: int = 4,
                          samples: int = 100_000, seed: int = 0, bins: int = 5) -> ValidationSummary:
    """Closed form vs shared-draw MC over seeded random cases (bench.py:235-267),
    as one closed-form batch and one Monte Carlo batch."""
    if cases < 1:
        raise ValueError("cases must be positive")
    batch = CaseBatch.pack([random_case(seed + i, model=model, neighborhood=neighborhood, bins=bins)
                            for i in range(cases)])
    exact = batch.closed()
    est = batch.monte_carlo(samples, seed=seed, pixels=np.arange(cases, dtype=np.uint64))
    se = np.sqrt(np.maximum(exact * (1.0 - exact), 0.0) / samples)
    dev = np.abs(exact - est)
    with np.errstate(divide="ignore", invalid="ignore"):
        dev_se = np.where(se > 0.0, dev / np.where(se > 0.0, se, 1.0), np.where(dev == 0.0, 0.0, np.inf))
    return ValidationSummary(model, cases, samples, float(dev.max()), float(dev_se.max()),
                             float(np.count_nonzero(dev_se <= 4.0)) / dev.size)
