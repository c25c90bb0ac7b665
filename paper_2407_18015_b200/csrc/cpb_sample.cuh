// Inverse-CDF samplers and the histogram CDF lookup shared by the grid
// Monte Carlo / semianalytical kernels (cpb_mc.cu) and the per-case batch
// kernels (cpb_cases.cu).  Every operation is an explicit round-to-nearest
// intrinsic so the draws repeat numpy's float64 arithmetic bit for bit
// (distributions.py:60-100).
#pragma once

#include "cpb_common.cuh"

namespace cpb {

// Per-position sampler state (histogram tables live in shared memory).
struct Sampler {
  double a, b;      // uniform: lo, hi | epanechnikov: mid, half | gaussian: mean, sd | histogram: lo, binw
  const double* wn; // histogram: h renormalised weights (smem)
  const double* cum;// histogram: h+1 prefix sums, cum[h] = 1 (smem)
};

// Root t in [-1, 1] of t^3 - 3t + 2y = 0, i.e. the reference's
// 2 sin(asin(y) / 3) (distributions.py:64-70, y = 2u - 1), without float64
// transcendentals: a single-precision guess (error ~1e-6) and one Halley step
// in float64 (cubic convergence, ~1e-18), so the draw agrees with the
// reference's libm evaluation to an ulp or two -- a strict comparison can only
// flip on a tie within that ulp.  Near |y| = 1 the root is double and the
// Halley step loses its rate, so there the reference formula is evaluated.
CPB_D double epan_root(double y) {
  if (fabs(y) > 0.999) return __dmul_rn(2.0, sin(__ddiv_rn(asin(y), 3.0)));
  const double t = (double)(2.0f * __sinf(asinf((float)y) * (1.0f / 3.0f)));
  const double t2 = t * t;
  const double g = fma(t, t2 - 3.0, 2.0 * y);
  const double gp = 3.0 * (t2 - 1.0);
  return t - (2.0 * g * gp) / fma(2.0 * gp, gp, -g * 6.0 * t);
}

template <int KIND>
CPB_D double draw(const Sampler& s, double u, double u2, int h) {
  if (KIND == CPB_UNIFORM) {  // (1 - u) lo + u hi  (distributions.py:60-61)
    return __dadd_rn(__dmul_rn(__dsub_rn(1.0, u), s.a), __dmul_rn(u, s.b));
  } else if (KIND == CPB_EPANECHNIKOV) {  // distributions.py:64-70
    if (u == 0.0) return __dsub_rn(s.a, s.b);
    if (u == 1.0) return __dadd_rn(s.a, s.b);
    const double root = epan_root(__dsub_rn(__dmul_rn(2.0, u), 1.0));
    return __dadd_rn(s.a, __dmul_rn(s.b, root));
  } else if (KIND == CPB_GAUSSIAN) {  // Box-Muller, engine.py:638-640
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log1p(-u)));
    const double z = __dmul_rn(r, cos(__dmul_rn(6.283185307179586, u2)));
    return __dadd_rn(s.a, __dmul_rn(s.b, z));
  } else {  // histogram_icdf, distributions.py:73-89
    int j = 0;
    for (int k = 1; k < h; ++k) j += (u >= s.cum[k]) ? 1 : 0;
    const double cj = s.cum[j], wj = s.wn[j];
    const double frac = wj > 0.0 ? __ddiv_rn(__dsub_rn(u, cj), wj) : 0.0;
    if (u == 1.0) return __dadd_rn(s.a, __dmul_rn(s.b, (double)h));
    const double e0 = __dadd_rn(s.a, __dmul_rn(s.b, (double)j));
    return __dadd_rn(__dmul_rn(__dsub_rn(1.0, frac), e0), __dmul_rn(frac, __dadd_rn(e0, s.b)));
  }
}

// Histogram CDF at x (histogram_cdf_values, distributions.py:92-100): bin
// floor((x - lo) / binw) clipped to [0, h-1], cum[j] + wn[j] * frac, clipped
// to [0, 1].
CPB_D double hist_cdf_at(const double* wn, const double* cum, double lo, double binw, int h,
                         double x) {
  double t = floor(__ddiv_rn(__dsub_rn(x, lo), binw));
  const int j = (int)fmax(0.0, fmin(t, (double)(h - 1)));
  const double frac = __ddiv_rn(__dsub_rn(x, __dadd_rn(lo, __dmul_rn(binw, (double)j))), binw);
  const double v = __dadd_rn(cum[j], __dmul_rn(wn[j], frac));
  return fmin(fmax(v, 0.0), 1.0);
}

// hist_cdf_at with the two divisions by binw replaced by a multiplication
// with ibinw = 1 / binw (semianalytical estimators, whose tolerance is 1e-13:
// the CDF is continuous, so a bin index off by one where (x - lo) / binw
// rounds across an integer changes the value only by rounding, and the
// quotient itself by an ulp).
// The position in bin units t = (x - lo) / binw is clamped to [0, h] first, so
// the bin is its integer part (capped at h - 1) and the in-bin fraction t - j
// stays in [0, 1]: the value is then in [0, cum[h - 1] + wn[h - 1]] and only
// the top needs the clip (binw is unused: kept for the signature).
CPB_D double hist_cdf_fast(const double* wn, const double* cum, double lo, double binw,
                           double ibinw, int h, double x) {
  (void)binw;
  const double t = fmin(fmax((x - lo) * ibinw, 0.0), (double)h);
  const int j = min((int)t, h - 1);
  const double v = fma(wn[j], t - (double)j, cum[j]);
  return fmin(v, 1.0);
}

}  // namespace cpb
