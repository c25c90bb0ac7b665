"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``critprob`` read-only from /root/reference/pkg/src, feeds it
small seeded inputs, and stores inputs + outputs under tests/golden/*.npz.
The fixtures travel with the repo; nothing at test time reads
/root/reference.  Reference entry points exercised:

- UncertainField.from_ensemble  (fields.py:125-158)
- UncertainField.from_scalar    (fields.py:160-178)
- classify_field closed form    (engine.py:716-787, 594-629)
- classify_field Monte Carlo    (engine.py:659-666, 632-656)
- classify_field semianalytical (engine.py:669-683)
- classify_field combinatorial  (engine.py:686-702)
- rngstream.unit_block          (rngstream.py:33-48)
- per-case API over seeded random_case / mixed-kind cases (cases.npz):
  closed_form_triple (engine.py:177), mc_all_patterns (238-247),
  semianalytical_prob (416-441), combinatorial_triple (399-404)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from critprob import rngstream  # noqa: E402
from critprob.distributions import GaussianSampler, epanechnikov, histogram, uniform  # noqa: E402
from critprob.engine import (  # noqa: E402
    EstimatorSpec,
    NeighborhoodCase,
    classify_field,
    closed_form_triple,
    combinatorial_triple,
    mc_all_patterns,
    semianalytical_prob,
)
from critprob.fields import EnsembleStack, ModelSpec, UncertainField  # noqa: E402
from critprob.synth import ackley_ensemble, random_case  # noqa: E402


def _ens(seed, shape, members, amp=0.3, base_amp=1.0):
    rng = np.random.default_rng(seed)
    base = rng.uniform(-base_amp, base_amp, shape)
    return (base + rng.uniform(-amp, amp, (members, *shape))).astype(np.float32)


def ensembles() -> dict:
    out = {
        "ackley": ackley_ensemble(13, 11, members=24, noise_amp=0.3, seed=0).values,
        "rand": _ens(11, (9, 10), 24),
        "wide": _ens(5, (8, 12), 7, amp=2.0, base_amp=0.2),
    }
    deg = np.zeros((5, 6, 7), dtype=np.float32)
    deg[:, 2, 2] = 7.0
    deg[:, 3, 4] = -1.5
    deg[1:, 1, 5] = 0.25
    deg[0, 1, 5] = 0.5
    out["degenerate"] = deg
    out["constant"] = np.full((4, 5, 5), 2.5, dtype=np.float32)
    out["single"] = _ens(3, (5, 6), 1)
    big = _ens(21, (7, 9), 40, amp=1e3, base_amp=1e4)
    big[:, 3, 3] = 1e4 + 0.5        # degenerate pixel in a wide-range stack
    out["offset"] = big
    return out


MODELS = [
    ("uniform", 5),
    ("epanechnikov", 5),
    ("gaussian", 5),
    ("histogram", 1),
    ("histogram", 3),
    ("histogram", 5),
    ("histogram", 8),
    ("histogram", 9),
    ("histogram", 16),
]


KIND_CODE = {"uniform": 0, "epanechnikov": 1, "histogram": 2, "gaussian": 3}


def _pack(cases):
    """Flat per-distribution arrays: kind, a, b, bins and zero-padded weights."""
    P = 1 + len(cases[0].neighbors)
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
            if isinstance(d, GaussianSampler):
                kind[i, p], a[i, p], b[i, p] = 3, d.mean, d.stddev
                continue
            kind[i, p] = KIND_CODE[d.kind]
            a[i, p], b[i, p] = d.support.lo, d.support.hi
            if d.kind == "histogram":
                bins[i, p] = d.bin_weights.size
                w[i, p, :d.bin_weights.size] = d.bin_weights
    return {"kind": kind, "a": a, "b": b, "bins": bins, "weights": w}


def case_fixtures() -> dict:
    """Per-case API goldens; groups by neighbourhood size."""
    mixed = NeighborhoodCase(
        epanechnikov(1.0, 0.9),
        (histogram(0.2, 2.2, [0.3, 0.5, 0.2]), uniform(0.5, 2.5), epanechnikov(1.4, 1.0),
         histogram(-0.2, 1.8, [0.25, 0.25, 0.5])))
    kat = NeighborhoodCase(uniform(0.0, 2.0), (uniform(1.0, 3.0), uniform(0.5, 2.5),
                                               uniform(1.5, 3.5), uniform(0.0, 2.0)))
    disjoint = NeighborhoodCase(uniform(0.0, 1.0), tuple(uniform(2.0, 3.0) for _ in range(4)))
    out = {}
    for k in (4, 2):
        cases, spec = [], []
        per = 12 if k == 4 else 6
        for model, bins in (("uniform", 5), ("epanechnikov", 5), ("histogram", 5), ("histogram", 3),
                            ("histogram", 9), ("gaussian", 5)):
            for s in range(per):
                seed = 100 * len(spec) + s
                cases.append(random_case(seed, model=model, neighborhood=k, bins=bins))
                spec.append((seed, KIND_CODE[model], bins))
        if k == 4:
            cases += [mixed, kat, disjoint, disjoint.negate(), mixed.affine(2.5, -1.0),
                      NeighborhoodCase(mixed.center, (mixed.neighbors[0], GaussianSampler(1.0, 0.4),
                                                      mixed.neighbors[2], mixed.neighbors[3]))]
        else:
            cases += [NeighborhoodCase(uniform(0.0, 1.0), (uniform(2.0, 3.0), uniform(-3.0, -2.0))),
                      NeighborhoodCase(mixed.center, mixed.neighbors[:2])]
        pk = _pack(cases)
        n = len(cases)
        closed = np.full((n, 3), np.nan)
        mc = np.zeros((n, 3))
        semi = np.full((n, 3), np.nan)
        comb = np.full((n, 3), np.nan)
        pixels = (np.arange(n, dtype=np.uint64) * np.uint64(7919) + np.uint64(3))
        for i, c in enumerate(cases):
            dists = (c.center, *c.neighbors)
            bounded = not any(isinstance(d, GaussianSampler) for d in dists)
            if bounded:
                closed[i] = tuple(closed_form_triple(c))
            mc[i] = tuple(mc_all_patterns(c, 2001, seed=7, pixel=int(pixels[i])))
            if bounded and all(d.kind == "histogram" for d in dists):
                semi[i] = [semianalytical_prob(c, p, 700, seed=2, pixel=int(pixels[i]))
                           for p in ("min", "max", "saddle")]
                if max(d.bin_weights.size for d in dists) <= 5:
                    comb[i] = tuple(combinatorial_triple(c))
        for key, val in pk.items():
            out[f"k{k}/{key}"] = val
        out[f"k{k}/pixels"] = pixels
        out[f"k{k}/random_spec"] = np.array(spec, dtype=np.int64)  # (seed, kind code, bins) of the first cases
        out[f"k{k}/closed"] = closed
        out[f"k{k}/mc"] = mc
        out[f"k{k}/semi"] = semi
        out[f"k{k}/comb"] = comb
    out["mc/n"] = np.array(2001)
    out["mc/seed"] = np.array(7)
    out["semi/c"] = np.array(700)
    out["semi/seed"] = np.array(2)
    return out


def main() -> None:
    ens = ensembles()
    fit = {}
    closed = {}
    mc = {}
    semi = {}
    comb = {}
    for name, vals in ens.items():
        fit[f"ens/{name}"] = vals
        stack = EnsembleStack(vals)
        for kind, bins in MODELS:
            if vals.shape[0] < 2 and kind in ("epanechnikov", "gaussian"):
                continue
            field = UncertainField.from_ensemble(stack, ModelSpec(kind=kind, bins=bins))
            tag = f"{name}/{kind}/{bins}"
            for pname, arr in field.params.items():
                fit[f"{tag}/{pname}"] = arr
            if min(field.shape) < 3:
                continue
            if kind != "gaussian":
                prob = classify_field(field)
                for ch in ("min", "max", "saddle"):
                    closed[f"{tag}/{ch}"] = prob.channel(ch)
            if name in ("ackley", "rand", "degenerate", "offset") and bins in (1, 5, 9):
                n = 257 if name != "offset" else 64
                est = EstimatorSpec(method="monte_carlo", n_samples=n, seed=9)
                prob = classify_field(field, est)
                for ch in ("min", "max", "saddle"):
                    mc[f"{tag}/{ch}"] = prob.channel(ch)
                mc[f"{tag}/n"] = np.array(n)
            if kind == "histogram" and (bins in (1, 3) or (bins == 5 and name == "degenerate")) \
                    and name in ("ackley", "rand", "degenerate", "offset"):
                prob = classify_field(field, EstimatorSpec(method="combinatorial"))
                for ch in ("min", "max", "saddle"):
                    comb[f"{tag}/{ch}"] = prob.channel(ch)
                comb[f"{tag}/done"] = np.array(1)
            if kind == "histogram" and name in ("ackley", "rand", "degenerate") and bins in (3, 5, 9):
                est = EstimatorSpec(method="semianalytical", c=700, seed=2)
                prob = classify_field(field, est)
                for ch in ("min", "max", "saddle"):
                    semi[f"{tag}/{ch}"] = prob.channel(ch)
                semi[f"{tag}/c"] = np.array(700)

    # closed-form known answers on hand-built 3x3 uniform fields (test_engine.py:147-163)
    lo = np.zeros((3, 3))
    hi = np.ones((3, 3))
    for (r, c), (a, b) in {(1, 1): (0.0, 2.0), (1, 2): (1.0, 3.0), (0, 1): (0.5, 2.5),
                           (1, 0): (1.5, 3.5), (2, 1): (0.0, 2.0)}.items():
        lo[r, c], hi[r, c] = a, b
    field = UncertainField(ModelSpec("uniform"), {"lo": lo, "hi": hi})
    prob = classify_field(field)
    closed["kat3x3/lo"] = lo
    closed["kat3x3/hi"] = hi
    for ch in ("min", "max", "saddle"):
        closed[f"kat3x3/{ch}"] = prob.channel(ch)

    # from_scalar (fields.py:160-178)
    rng = np.random.default_rng(9)
    raster = rng.uniform(0.0, 10.0, (6, 7))
    for eb in (0.5, 0.0):
        f = UncertainField.from_scalar(raster, eb)
        fit[f"scalar/{eb}/lo"] = f.params["lo"]
        fit[f"scalar/{eb}/hi"] = f.params["hi"]
        prob = classify_field(f)
        for ch in ("min", "max", "saddle"):
            closed[f"scalar/{eb}/{ch}"] = prob.channel(ch)
    fit["scalar/raster"] = raster

    # counter RNG (rngstream.py:33-48)
    rng_fx = {}
    px = np.array([0, 1, 17, 2**40 + 3, 2**63 + 5], dtype=np.uint64)
    for seed in (0, 7, -1, 2**64 - 2, 123456789):
        rng_fx[f"{seed}"] = rngstream.unit_block(seed, px, 3, 11)
    rng_fx["pixels"] = px

    # field_io: UCVF bytes, P5 heatmaps, CSV (field_io.py:35-150)
    import tempfile

    from critprob import field_io as fio

    io_fx = {}
    with tempfile.TemporaryDirectory() as tmp:
        stack = EnsembleStack(ens["ackley"])
        fio.save_ensemble(stack, os.path.join(tmp, "e.ucvf"))
        io_fx["ensemble_ucvf"] = np.frombuffer(open(os.path.join(tmp, "e.ucvf"), "rb").read(), np.uint8)
        field = UncertainField.from_ensemble(stack, ModelSpec("uniform"))
        prob = classify_field(field)
        fio.save_probability_field(prob, os.path.join(tmp, "p.ucvf"))
        io_fx["prob_ucvf"] = np.frombuffer(open(os.path.join(tmp, "p.ucvf"), "rb").read(), np.uint8)
        fio.save_probability_field(prob, os.path.join(tmp, "p.csv"), format="csv")
        io_fx["prob_csv"] = np.frombuffer(open(os.path.join(tmp, "p.csv"), "rb").read(), np.uint8)
        for ch in ("min", "max", "saddle"):
            io_fx[f"prob/{ch}"] = prob.channel(ch)
            for g in (1.0, 0.5, 2.2):
                fio.export_heatmap(prob, ch, os.path.join(tmp, "h.pgm"), gamma=g)
                io_fx[f"heat/{ch}/{g}"] = np.frombuffer(open(os.path.join(tmp, "h.pgm"), "rb").read(), np.uint8)
        io_fx["prob/valid"] = prob.valid
    np.savez_compressed(os.path.join(HERE, "io.npz"), **io_fx)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **case_fixtures())
    # synthetic generators used by the acceptance gates (synth.py:54-121)
    from critprob.synth import gaussian_mixture_ensemble

    mix, peaks, outliers = gaussian_mixture_ensemble(32, 32, true_members=6, outlier_members=3, seed=4)
    np.savez_compressed(os.path.join(HERE, "synth.npz"), mixture=mix.values,
                        peaks=np.array(peaks), outlier_peaks=np.array(outliers),
                        ackley=ackley_ensemble(20, 12, members=5, noise_amp=0.3, seed=7).values)

    np.savez_compressed(os.path.join(HERE, "fit.npz"), **fit)
    np.savez_compressed(os.path.join(HERE, "closed.npz"), **closed)
    np.savez_compressed(os.path.join(HERE, "mc.npz"), **mc)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng_fx)
    np.savez_compressed(os.path.join(HERE, "semi.npz"), **semi)
    np.savez_compressed(os.path.join(HERE, "comb.npz"), **comb)
    for f in ("fit", "closed", "mc", "rng", "semi", "comb", "io", "cases", "synth"):
        print(f, os.path.getsize(os.path.join(HERE, f + ".npz")), "bytes")


if __name__ == "__main__":
    main()
