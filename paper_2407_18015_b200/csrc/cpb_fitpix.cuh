// Per-pixel fit arithmetic shared by the fit kernels (cpb_fit.cu) and the
// fused fit + stencil kernels (cpb_closed.cu): NaN-propagating bounds, the
// exact histogram thresholds and the one-pass multi-model pixel fit.
// Every float64 operation is an explicit round-to-nearest intrinsic in numpy's
// order, so results do not depend on the translation unit's -fmad setting.
//
// Reference: UncertainField.from_ensemble (fields.py:125-158).
#pragma once

#include "cpb_common.cuh"

namespace cpb {
namespace {

CPB_D bool nonfinite(float v) { return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u; }

// NaN-propagating min (PTX min.NaN): a running min over the members is NaN
// iff some member is NaN, so one check after the loop replaces a per-member
// test; +-Inf members show up in the min / max themselves.
CPB_D float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// 1 if x < t else 0, for finite x and a threshold t that is not +0.0 (callers
// map +0 to -0): the sign of fl(x - t) is the sign of x - t (a nonzero
// difference of two floats is at least the smallest subnormal, and no FTZ
// here), and equal operands give +0 -- including x = +-0 against t = -0 --
// so the count update "c += lt_bit(x, t)" is an FADD and a shift-add
// (LEA.HI) per threshold.
CPB_D uint32_t lt_bit(float x, float t) { return __float_as_uint(__fsub_rn(x, t)) >> 31; }

// Smallest float v with floor(fl(fl(v - lo) * scale)) >= k -- the bin index of
// fields.py:147 is monotone in v, so "bin >= k" is "v >= threshold_k" and the
// per-member binning becomes h-1 float compares, bit-exact by construction.
// Order-preserving map of finite floats to uint32 (-0 and +0 adjacent).
CPB_D uint32_t fkey(float f) {
  const uint32_t i = __float_as_uint(f);
  return (i & 0x80000000u) ? ~i : (i | 0x80000000u);
}
CPB_D float fkey_inv(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// The threshold is found on the float order itself: from the FP32 guess
// (normally within an ulp: two evaluations) an exponential search brackets
// the step of the monotone predicate raw(v) >= k inside [vlo, vhi] (the
// pixel's min / max, where raw is 0 and >= h - 1 >= k), then bisection on
// the keys pins it -- exact for any data, e.g. bins whose edge sits within
// 1e-17 of zero, where the step is ~2^40 float ulps away from the guess.
CPB_D __noinline__ float bin_threshold_search(int k, double lo, double scale, float guess, float vlo,
                                              float vhi) {
  const double kk = (double)k;
  auto pred = [&](uint32_t u) {
    return floor(__dmul_rn(__dsub_rn((double)fkey_inv(u), lo), scale)) >= kk;
  };
  const uint32_t kmin = fkey(vlo), kmax = fkey(vhi);
  uint32_t g = fkey(guess);
  g = g < kmin ? kmin : (g > kmax ? kmax : g);
  uint32_t lo_k, hi_k;  // pred(lo_k) false, pred(hi_k) true
  if (pred(g)) {
    hi_k = g;
    uint32_t step = 1;
    for (;;) {
      const uint32_t c = (hi_k - kmin > step) ? hi_k - step : kmin;
      if (!pred(c)) { lo_k = c; break; }
      hi_k = c;
      if (c == kmin) { lo_k = c; break; }  // unreachable: raw(vlo) = 0 < k
      step <<= 1;
    }
  } else {
    lo_k = g;
    uint32_t step = 1;
    for (;;) {
      const uint32_t c = (kmax - lo_k > step) ? lo_k + step : kmax;
      if (pred(c)) { hi_k = c; break; }
      lo_k = c;
      if (c == kmax) { hi_k = c; break; }  // unreachable: raw(vhi) >= h - 1 >= k
      step <<= 1;
    }
  }
  while (hi_k - lo_k > 1) {
    const uint32_t mid = lo_k + (hi_k - lo_k) / 2;
    if (pred(mid)) hi_k = mid; else lo_k = mid;
  }
  return fkey_inv(hi_k);
}

// Fast path: the predicate at the clamped guess and at its neighbour towards
// the step, straight-line; they differ whenever the guess is within an ulp of
// the threshold (the usual case), otherwise the out-of-line search above.
CPB_D float bin_threshold(int k, double lo, double scale, float guess, float vlo, float vhi) {
  const double kk = (double)k;
  auto pred = [&](uint32_t u) {
    return floor(__dmul_rn(__dsub_rn((double)fkey_inv(u), lo), scale)) >= kk;
  };
  const uint32_t kmin = fkey(vlo), kmax = fkey(vhi);
  uint32_t g = fkey(guess);
  g = g < kmin ? kmin : (g > kmax ? kmax : g);
  // pred(kmin) is false and pred(kmax) true, so g - 1 / g + 1 stay in range
  const bool pg = pred(g);
  const uint32_t n = pg ? g - 1u : g + 1u;
  if (pg != pred(n)) return fkey_inv(pg ? g : n);
  return bin_threshold_search(k, lo, scale, guess, vlo, vhi);
}

CPB_D float bin_threshold(int k, double lo, double scale, float vlo, float vhi) {
  return bin_threshold(k, lo, scale, __double2float_rn(__dadd_rn(lo, __ddiv_rn((double)k, scale))),
                       vlo, vhi);
}

// c / M for c in [0, M]: the exact count->weight map of fields.py:151.
__global__ void weight_table_kernel(double* t, int members) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c <= members) t[c] = __ddiv_rn((double)c, (double)members);
}

constexpr int kThreshBinsPix = 8;  // histogram bins counted with per-thread thresholds

struct MultiArgs {
  int64_t npix, wstride;
  int members, bins;
  float* lo[2];       // uniform, histogram bounds (either may be NULL)
  float* hi[2];
  double* mean[2];    // epanechnikov, gaussian moments (either may be NULL)
  double* spread[2];
  void* counts;       // histogram bin counts (bins, npix)
  int wmode;
  uint32_t* range;
};

// One pixel of the multi-model fit: min / max (+ the member sum) in one pass,
// then the histogram binning against exact thresholds and the squared
// deviations in a second pass over the same staged column (member m at
// col[m * stride]); writes every requested plane at p when `write`.
template <int NT>
CPB_D void multi_fit_pixel(const float* col, int stride, const MultiArgs& a, int64_t p, bool write,
                           float& lo_out, float& hi_out) {
  const int M = a.members;
  const bool moments = a.mean[0] || a.mean[1];
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  double sum = 0.0;
  if (moments) {
#pragma unroll 8
    for (int m = 0; m < M; ++m) {
      const float x = col[m * stride];
      lo = fmin_nan(lo, x);
      hi = fmaxf(hi, x);
      sum = __dadd_rn(sum, (double)x);
    }
  } else {
#pragma unroll 8
    for (int m = 0; m < M; ++m) {
      const float x = col[m * stride];
      lo = fmin_nan(lo, x);
      hi = fmaxf(hi, x);
    }
  }
  lo_out = lo;
  hi_out = hi;
  if (write) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (a.lo[i]) {
        a.lo[i][p] = lo;
        a.hi[i][p] = hi;
      }
    }
  }
  // second pass: histogram binning and the squared deviations share each member load
  const bool hist = NT > 0 && a.counts != nullptr;
  constexpr int NB = NT > 0 ? NT : 1;
  uint32_t c[NB + 1];
  float thr[NB];
#pragma unroll
  for (int q = 0; q <= NB; ++q) c[q] = 0u;
  if (hist) {
    const double dlo = (double)lo;
    const double scale = __ddiv_rn((double)a.bins, __dsub_rn((double)hi, dlo));
    const float step = __fsub_rn(hi, lo) * __frcp_rn((float)a.bins);  // a guess: any rounding
#pragma unroll
    for (int q = 1; q < NB; ++q) {
      thr[q] = hi > lo ? bin_threshold(q, dlo, scale, __fmaf_rn((float)q, step, lo), lo, hi) : 0.0f;
      thr[q] = thr[q] == 0.0f ? -0.0f : thr[q];
    }
  }
  const double mean = moments ? __ddiv_rn(sum, (double)M) : 0.0;
  double sq = 0.0;
  if (hist && moments) {
#pragma unroll 4
    for (int m = 0; m < M; ++m) {
      const float x = col[m * stride];
#pragma unroll
      for (int q = 1; q < NB; ++q) c[q] += lt_bit(x, thr[q]);
      const double d = __dsub_rn((double)x, mean);
      sq = __dadd_rn(sq, __dmul_rn(d, d));
    }
  } else if (hist) {
#pragma unroll 4
    for (int m = 0; m < M; ++m) {
      const float x = col[m * stride];
#pragma unroll
      for (int q = 1; q < NB; ++q) c[q] += lt_bit(x, thr[q]);
    }
  } else if (moments) {
#pragma unroll 8
    for (int m = 0; m < M; ++m) {
      const double d = __dsub_rn((double)col[m * stride], mean);
      sq = __dadd_rn(sq, __dmul_rn(d, d));
    }
  }
  if (!write) return;
  if (hist) {
#pragma unroll
    for (int q = 1; q < NB; ++q) c[q] = (uint32_t)M - c[q];
    c[0] = (uint32_t)M;
    const bool flat = !(hi > lo);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint32_t v = flat ? 0u : (b + 1 < NB ? c[b] - c[b + 1] : c[b]);
      if (a.wmode == CPB_WEIGHTS_U8)
        static_cast<uint8_t*>(a.counts)[(int64_t)b * a.wstride + p] = (uint8_t)v;
      else
        static_cast<uint16_t*>(a.counts)[(int64_t)b * a.wstride + p] = (uint16_t)v;
    }
  }
  if (moments) {
    const double sd = __dsqrt_rn(__ddiv_rn(sq, (double)(M - 1)));
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (a.mean[i]) {
        a.mean[i][p] = mean;
        a.spread[i][p] = sd;
      }
    }
  }
}

}  // namespace
}  // namespace cpb
