"""CPU oracle for the per-case API -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's single-neighbourhood estimators
(/root/reference/pkg/src/critprob/engine.py:50-459, piecewise.py:65-234,
distributions.py:105-242), used by ``tests/`` to check the batched CUDA
kernels (paper_2407_18015_b200.cases).  Pinned against the reference's own
outputs in tests/golden/cases.npz (tests/test_oracle_golden.py).

A distribution is a dict: {"kind": "uniform"|"epanechnikov"|"histogram",
"lo", "hi", "w" (histogram weights as stored, i.e. already normalised)} or
{"kind": "gaussian", "mean", "std"}; a case is (centre, [neighbours]).
"""

from __future__ import annotations

import math

import numpy as np

from oracle.critprob_oracle import uniforms

KIND_NAMES = ("uniform", "epanechnikov", "histogram", "gaussian")


# --------------------------------------------------------------- packing
def unpack(kind, a, b, bins, weights) -> list:
    """Packed batch arrays (n, P) -> list of cases."""
    cases = []
    for i in range(kind.shape[0]):
        dists = []
        for p in range(kind.shape[1]):
            name = KIND_NAMES[int(kind[i, p])]
            if name == "gaussian":
                dists.append({"kind": name, "mean": float(a[i, p]), "std": float(b[i, p])})
            else:
                d = {"kind": name, "lo": float(a[i, p]), "hi": float(b[i, p])}
                if name == "histogram":
                    d["w"] = np.asarray(weights[i, p, :int(bins[i, p])], dtype=float)
                dists.append(d)
        cases.append((dists[0], dists[1:]))
    return cases


# ------------------------------------------------ piecewise polynomials
class Piecewise:
    """Pieces as coefficient arrays in (x - piece midpoint) (piecewise.py:65-89)."""

    def __init__(self, bp, pieces, below=0.0, above=0.0):
        self.bp = np.asarray(bp, dtype=float)
        self.pieces = [np.atleast_1d(np.asarray(c, dtype=float)) for c in pieces]
        self.below = float(below)
        self.above = float(above)
        self.mid = 0.5 * (self.bp[:-1] + self.bp[1:])

    def antiderivative(self):  # piecewise.py:166-180
        run = 0.0
        out = []
        for i, c in enumerate(self.pieces):
            raw = np.concatenate(([0.0], c / np.arange(1.0, c.size + 1.0)))
            raw[0] = run - np.polynomial.polynomial.polyval(self.bp[i] - self.mid[i], raw)
            out.append(raw)
            run = np.polynomial.polynomial.polyval(self.bp[i + 1] - self.mid[i], raw)
        return Piecewise(self.bp, out, 0.0, run)

    def complement(self):  # survival = 1 - cdf (distributions.py:171-186)
        pieces = []
        for c in self.pieces:
            neg = -c
            neg[0] += 1.0
            pieces.append(neg)
        return Piecewise(self.bp, pieces, 1.0, 1.0 - self.above)

    def local(self, u, v, centre):
        """Coefficients on [u, v] in (x - centre) (piecewise.py:184-197)."""
        m = 0.5 * (u + v)
        if m < self.bp[0]:
            return np.array([self.below])
        if m > self.bp[-1]:
            return np.array([self.above])
        i = int(np.clip(np.searchsorted(self.bp, m, side="right") - 1, 0, len(self.pieces) - 1))
        return _shift(self.pieces[i], centre - self.mid[i])


def _shift(c, off):
    """p(t) with t = s + off, as coefficients in s (piecewise.py:49-62)."""
    out = np.zeros_like(c)
    for k, ak in enumerate(c):
        for j in range(k + 1):
            out[j] += ak * math.comb(k, j) * off ** (k - j)
    return out


def pdf_poly(d) -> Piecewise:  # distributions.py:145-163
    lo, hi = d["lo"], d["hi"]
    if d["kind"] == "uniform":
        return Piecewise([lo, hi], [[1.0 / (hi - lo)]])
    if d["kind"] == "epanechnikov":
        w = 0.5 * (hi - lo)
        return Piecewise([lo, hi], [[0.75 / w, 0.0, -0.75 / w ** 3]])
    h = d["w"].size
    edges = lo + (hi - lo) * np.arange(h + 1) / h
    binw = (hi - lo) / h
    return Piecewise(edges, [[wk / binw] for wk in d["w"]])


def _product_integral(factors, lo, hi) -> float:
    """refine_and_multiply + integrate (piecewise.py:200-234, 123-150), exact per piece."""
    tol = 1e-12 * (hi - lo)
    inner = np.concatenate([f.bp for f in factors])
    inner = np.unique(inner[(inner > lo + tol) & (inner < hi - tol)])
    pts = [lo]
    for p in inner:
        if p - pts[-1] > tol:
            pts.append(float(p))
    pts.append(hi)
    total = 0.0
    for u, v in zip(pts[:-1], pts[1:]):
        c = 0.5 * (u + v)
        coeffs = np.array([1.0])
        for f in factors:
            coeffs = np.convolve(coeffs, f.local(u, v, c))
        anti = np.polynomial.polynomial.polyint(coeffs)
        half = 0.5 * (v - u)
        total += float(np.polynomial.polynomial.polyval(half, anti)
                       - np.polynomial.polynomial.polyval(-half, anti))
    return total


def negate(d):
    if d["kind"] == "gaussian":
        return {"kind": "gaussian", "mean": -d["mean"], "std": d["std"]}
    out = {"kind": d["kind"], "lo": -d["hi"], "hi": -d["lo"]}
    if d["kind"] == "histogram":
        out["w"] = d["w"][::-1].copy()
    return out


def negate_case(case):
    return negate(case[0]), [negate(d) for d in case[1]]


def local_min(case) -> float:  # engine.py:127-136
    c, nb = case
    lo = c["lo"]
    hi = min(d["hi"] for d in (c, *nb))
    if hi <= lo:
        return 0.0
    factors = [pdf_poly(c)] + [pdf_poly(d).antiderivative().complement() for d in nb]
    return _product_integral(factors, lo, hi)


def _half_saddle(case) -> float:  # engine.py:145-163
    c, nb = case
    if len(nb) == 2:
        above, below = [nb[0]], [nb[1]]
    else:
        above, below = [nb[0], nb[2]], [nb[1], nb[3]]
    lo = max(c["lo"], *(d["lo"] for d in below))
    hi = min(c["hi"], *(d["hi"] for d in above))
    if hi <= lo:
        return 0.0
    factors = ([pdf_poly(c)] + [pdf_poly(d).antiderivative().complement() for d in above]
               + [pdf_poly(d).antiderivative() for d in below])
    return _product_integral(factors, lo, hi)


def closed_triple(case) -> tuple:
    """closed_form_triple (engine.py:177-178): min, max (= negated min), saddle."""
    neg = negate_case(case)
    return local_min(case), local_min(neg), _half_saddle(case) + _half_saddle(neg)


# ---------------------------------------------------------- Monte Carlo
def _sample(d, u):
    """FiniteDistribution.sample_u01 / GaussianSampler.sample_u01 (distributions.py:212-274)."""
    if d["kind"] == "gaussian":
        z = np.sqrt(-2.0 * np.log1p(-u[0])) * np.cos(2.0 * np.pi * u[1])
        return d["mean"] + d["std"] * z
    u = u[0]
    lo, hi = d["lo"], d["hi"]
    if d["kind"] == "uniform":
        return (1.0 - u) * lo + u * hi
    if d["kind"] == "epanechnikov":
        m, w = 0.5 * (lo + hi), 0.5 * (hi - lo)
        x = m + w * (2.0 * np.sin(np.arcsin(2.0 * u - 1.0) / 3.0))
        x = np.where(u == 0.0, m - w, x)
        return np.where(u == 1.0, m + w, x)
    w = d["w"]
    h = w.size
    cum = np.concatenate(([0.0], np.cumsum(w)))
    cum[-1] = 1.0
    binw = (hi - lo) / h
    j = np.zeros(u.shape, dtype=np.intp)
    for k in range(1, h):
        j += u >= cum[k]
    cj, wj = cum[j], w[j]
    frac = np.where(wj > 0.0, (u - cj) / np.where(wj > 0.0, wj, 1.0), 0.0)
    e0 = lo + binw * j
    x = (1.0 - frac) * e0 + frac * (e0 + binw)
    return np.where(u == 1.0, lo + binw * h, x)


def _planes(d) -> int:
    return 2 if d["kind"] == "gaussian" else 1


def mc_triple(case, n: int, seed: int, pixel: int) -> tuple:
    """mc_all_patterns (engine.py:238-247) with _case_draws (225-235)."""
    dists = (case[0], *case[1])
    planes = sum(_planes(d) for d in dists)
    u = uniforms(seed, [pixel], planes, n)[0]
    xs, q = [], 0
    for d in dists:
        k = _planes(d)
        xs.append(_sample(d, u[q:q + k]))
        q += k
    c = xs[0]
    if len(xs) == 3:
        a, b = xs[1], xs[2]
        mn = (c < a) & (c < b)
        mx = (c > a) & (c > b)
        sd = ((c < a) & (c > b)) | ((c > a) & (c < b))
    else:
        e, nn, w, s = xs[1:]
        mn = (c < e) & (c < nn) & (c < w) & (c < s)
        mx = (c > e) & (c > nn) & (c > w) & (c > s)
        sd = ((c < e) & (c > nn) & (c < w) & (c > s)) | ((c > e) & (c < nn) & (c > w) & (c < s))
    return float(mn.mean()), float(mx.mean()), float(sd.mean())


# ------------------------------------------------------- semianalytical
def _hist_cdf(d, x):
    """histogram_cdf_values (distributions.py:92-100) with _hist_arrays (engine.py:407-413)."""
    w = d["w"]
    h = w.size
    cum = np.concatenate(([0.0], np.cumsum(w)))
    binw = (d["hi"] - d["lo"]) / h
    j = np.clip(np.floor((x - d["lo"]) / binw).astype(np.intp), 0, h - 1)
    frac = (x - (d["lo"] + binw * j)) / binw
    return np.clip(cum[j] + w[j] * frac, 0.0, 1.0)


def semi_triple(case, c: int, seed: int, pixel: int) -> tuple:
    """semianalytical_prob (engine.py:416-441) for min, max, saddle from the same draws."""
    u = uniforms(seed, [pixel], 1, c)[0]
    x = _sample(case[0], u)
    F = [_hist_cdf(d, x) for d in case[1]]
    mn = 1.0 - F[0]
    for f in F[1:]:
        mn = mn * (1.0 - f)
    mx = F[0].copy()
    for f in F[1:]:
        mx = mx * f
    if len(F) == 2:
        sd = (1.0 - F[0]) * F[1] + F[0] * (1.0 - F[1])
    else:
        e, nn, w, s = F
        sd = (1.0 - e) * nn * (1.0 - w) * s + e * (1.0 - nn) * w * (1.0 - s)
    return float(mn.mean()), float(mx.mean()), float(sd.mean())


# -------------------------------------------------------- combinatorial
def _all_uniform(lo, hi, above, below) -> float:
    """_uniform_kernel_term (engine.py:270-310) via the exact product integral."""
    a = max([lo] + [p[0] for p in below])
    b = min([hi] + [p[1] for p in above])
    if b <= a:
        return 0.0
    factors = [Piecewise([lo, hi], [[1.0 / (hi - lo)]])]
    for p in above:
        factors.append(pdf_poly({"kind": "uniform", "lo": p[0], "hi": p[1]}).antiderivative().complement())
    for p in below:
        factors.append(pdf_poly({"kind": "uniform", "lo": p[0], "hi": p[1]}).antiderivative())
    return _product_integral(factors, a, b)


def comb_triple(case) -> tuple:
    """combinatorial_triple (engine.py:320-404)."""
    import itertools

    dists = (case[0], *case[1])
    grids = []
    for d in dists:
        h = d["w"].size
        grids.append((d["lo"] + (d["hi"] - d["lo"]) * np.arange(h + 1) / h, d["w"]))
    k = len(case[1])
    sad_above, sad_below = ((1,), (2,)) if k == 2 else ((1, 3), (2, 4))
    tot = [0.0, 0.0, 0.0]
    for combo in itertools.product(*(range(w.size) for _, w in grids)):
        wprod = 1.0
        for (_, w), j in zip(grids, combo):
            wprod *= w[j]
        if wprod == 0.0:
            continue
        iv = [(grids[i][0][combo[i]], grids[i][0][combo[i] + 1]) for i in range(len(dists))]
        lo, hi = iv[0]
        nbr = iv[1:]
        tot[0] += wprod * _all_uniform(lo, hi, nbr, [])
        tot[1] += wprod * _all_uniform(lo, hi, [], nbr)
        ab = [iv[i] for i in sad_above]
        be = [iv[i] for i in sad_below]
        tot[2] += wprod * (_all_uniform(lo, hi, ab, be) + _all_uniform(lo, hi, be, ab))
    return tuple(tot)
