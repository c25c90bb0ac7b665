// Per-pixel noise-model fit over the member axis, the synthetic ensemble
// generator and the reference-layout materialisation.
//
// Reference: UncertainField.from_ensemble (fields.py:125-158),
// default_epsilon (distributions.py:30-36), from_scalar (fields.py:160-178).
//
// Bit-exactness: every float64 operation below that the reference performs
// in numpy is written with an explicit round-to-nearest intrinsic
// (__dadd_rn, __dmul_rn, ...) so no FMA contraction changes a result, and
// the member reductions run in member order exactly like numpy's axis-0
// reductions (sequential).  min/max and bin counts are exact.
#include <stdlib.h>

#include <algorithm>

#include "cpb_common.cuh"
#include "cpb_tma.cuh"
#include "cpb_fitpix.cuh"

#include <cudaTypedefs.h>

namespace cpb {
namespace {

constexpr int kFitThreads = 256;
constexpr int kRegMembers = 64;  // members kept in registers between passes

struct FitArgs {
  const float* ens;
  int64_t mstride;  // elements between members
  int64_t npix;     // height * width of the slab
  int64_t wstride;  // elements between bin planes of `counts`
  int members;
  int bins;
  float* lo;
  float* hi;
  double* mean;
  double* spread;
  void* counts;     // (bins, npix) uint8 or uint16
  int wmode;
  uint32_t* range;  // [0] ordered min, [1] ordered max, [2] non-finite flag
};

// Histogram bin of value v: clip(floor((v - lo) * (h / (hi - lo))), 0, h-1)
// (fields.py:147-148), evaluated with the same two roundings.
CPB_D int bin_of(float v, double lo, double scale, int h) {
  const double t = floor(__dmul_rn(__dsub_rn((double)v, lo), scale));
  return (int)fmax(0.0, fmin(t, (double)(h - 1)));
}

template <int KIND>
__global__ void __launch_bounds__(kFitThreads) fit_reg_kernel(FitArgs a) {
  extern __shared__ uint32_t s_cnt[];  // (bins, blockDim) per-thread counters (histogram)
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = p < a.npix;
  const int M = a.members;
  float v[kRegMembers];
  float vmin = __int_as_float(0x7f800000), vmax = -__int_as_float(0x7f800000);
  bool bad = false;
  double sum = 0.0;
  if (live) {
    const float* src = a.ens + p;
#pragma unroll
    for (int m = 0; m < kRegMembers; ++m)
      if (m < M) v[m] = __ldcs(src + m * a.mstride);
#pragma unroll
    for (int m = 0; m < kRegMembers; ++m) {
      if (m < M) {
        bad |= nonfinite(v[m]);
        vmin = fminf(vmin, v[m]);
        vmax = fmaxf(vmax, v[m]);
        if (KIND == CPB_EPANECHNIKOV || KIND == CPB_GAUSSIAN) sum = __dadd_rn(sum, (double)v[m]);
      }
    }
    if (KIND == CPB_UNIFORM || KIND == CPB_HISTOGRAM) {
      a.lo[p] = vmin;
      a.hi[p] = vmax;
    }
    if (KIND == CPB_HISTOGRAM) {
      const int h = a.bins;
      for (int b = 0; b < h; ++b) s_cnt[b * blockDim.x + threadIdx.x] = 0u;
      if (vmax > vmin) {  // degenerate pixels are binned at use, once eps is known
        const double lo = (double)vmin, hi = (double)vmax;
        const double scale = __ddiv_rn((double)h, __dsub_rn(hi, lo));
#pragma unroll
        for (int m = 0; m < kRegMembers; ++m)
          if (m < M) s_cnt[bin_of(v[m], lo, scale, h) * blockDim.x + threadIdx.x] += 1u;
      }
      if (a.wmode == CPB_WEIGHTS_U8) {
        uint8_t* c = static_cast<uint8_t*>(a.counts);
        for (int b = 0; b < h; ++b) c[(int64_t)b * a.wstride + p] = (uint8_t)s_cnt[b * blockDim.x + threadIdx.x];
      } else {
        uint16_t* c = static_cast<uint16_t*>(a.counts);
        for (int b = 0; b < h; ++b) c[(int64_t)b * a.wstride + p] = (uint16_t)s_cnt[b * blockDim.x + threadIdx.x];
      }
    }
    if (KIND == CPB_EPANECHNIKOV || KIND == CPB_GAUSSIAN) {
      // numpy: mean = sum / M; var = sum((v - mean)^2) / (M - 1); std = sqrt(var)
      const double mean = __ddiv_rn(sum, (double)M);
      double sq = 0.0;
#pragma unroll
      for (int m = 0; m < kRegMembers; ++m) {
        if (m < M) {
          const double d = __dsub_rn((double)v[m], mean);
          sq = __dadd_rn(sq, __dmul_rn(d, d));
        }
      }
      a.mean[p] = mean;
      a.spread[p] = __dsqrt_rn(__ddiv_rn(sq, (double)(M - 1)));
    }
  }
  merge_range(vmin, vmax, bad, a.range);
}

// Members beyond the register budget: same arithmetic, the second pass
// re-reads the member column (L2-resident right after the first pass).
template <int KIND>
__global__ void __launch_bounds__(kFitThreads) fit_loop_kernel(FitArgs a) {
  extern __shared__ uint32_t s_cnt[];
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = p < a.npix;
  const int M = a.members;
  float vmin = __int_as_float(0x7f800000), vmax = -__int_as_float(0x7f800000);
  bool bad = false;
  if (live) {
    const float* src = a.ens + p;
    double sum = 0.0;
#pragma unroll 8
    for (int m = 0; m < M; ++m) {
      const float x = __ldg(src + (int64_t)m * a.mstride);
      bad |= nonfinite(x);
      vmin = fminf(vmin, x);
      vmax = fmaxf(vmax, x);
      if (KIND == CPB_EPANECHNIKOV || KIND == CPB_GAUSSIAN) sum = __dadd_rn(sum, (double)x);
    }
    if (KIND == CPB_UNIFORM || KIND == CPB_HISTOGRAM) {
      a.lo[p] = vmin;
      a.hi[p] = vmax;
    }
    if (KIND == CPB_HISTOGRAM) {
      const int h = a.bins;
      for (int b = 0; b < h; ++b) s_cnt[b * blockDim.x + threadIdx.x] = 0u;
      if (vmax > vmin) {
        const double lo = (double)vmin, hi = (double)vmax;
        const double scale = __ddiv_rn((double)h, __dsub_rn(hi, lo));
        for (int m = 0; m < M; ++m)
          s_cnt[bin_of(__ldg(src + (int64_t)m * a.mstride), lo, scale, h) * blockDim.x + threadIdx.x] += 1u;
      }
      if (a.wmode == CPB_WEIGHTS_U8) {
        uint8_t* c = static_cast<uint8_t*>(a.counts);
        for (int b = 0; b < h; ++b) c[(int64_t)b * a.wstride + p] = (uint8_t)s_cnt[b * blockDim.x + threadIdx.x];
      } else {
        uint16_t* c = static_cast<uint16_t*>(a.counts);
        for (int b = 0; b < h; ++b) c[(int64_t)b * a.wstride + p] = (uint16_t)s_cnt[b * blockDim.x + threadIdx.x];
      }
    }
    if (KIND == CPB_EPANECHNIKOV || KIND == CPB_GAUSSIAN) {
      const double mean = __ddiv_rn(sum, (double)M);
      double sq = 0.0;
      for (int m = 0; m < M; ++m) {
        const double d = __dsub_rn((double)__ldg(src + (int64_t)m * a.mstride), mean);
        sq = __dadd_rn(sq, __dmul_rn(d, d));
      }
      a.mean[p] = mean;
      a.spread[p] = __dsqrt_rn(__ddiv_rn(sq, (double)(M - 1)));
    }
  }
  merge_range(vmin, vmax, bad, a.range);
}

// ---------------------------------------------------------------------------
// TMA-pipelined fit: the production path.
//
// A persistent CTA of kTmaTile threads owns one pixel per thread of a tile of
// kTmaTile consecutive pixels.  The tile's M member rows form one 2-D box of
// the (members x pixels) tensor view of the ensemble; one TMA instruction
// (cp.async.bulk.tensor.2d, completion on an mbarrier) stages it into shared
// memory through a ring of `stages` buffers, so several tiles per SM are in
// flight while the threads reduce the staged one.  Both passes of the
// two-pass statistics (mean then squared deviations; min/max then bin counts)
// read the staged values, so HBM sees every member value exactly once.
// ---------------------------------------------------------------------------
constexpr int kTmaTile = 128;
constexpr int kThreshBins = 8;  // histogram bins counted with per-thread thresholds

// NT: histogram bin count handled with NT-1 register thresholds (1..kThreshBins),
// or 0 for the shared-memory counters (more bins).
template <int KIND, int NT>
__global__ void __launch_bounds__(kTmaTile) fit_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                           FitArgs a, int stages, int mbox,
                                                           int nbox, int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int M = a.members;
  const int rows = mbox * nbox;  // staged member rows per tile (>= M, OOB rows are zero)
  const int tid = threadIdx.x;
  float* buf = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * rows * kTmaTile * 4);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(full + stages);  // (bins, kTmaTile), bins > kThreshBins
  if (tid == 0) {
    prefetch_tensormap(&map);
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint32_t tile_bytes = (uint32_t)rows * kTmaTile * 4u;
  auto issue = [&](int64_t tile, int s) {  // one thread
    mbar_arrive_expect_tx(&full[s], tile_bytes);
    float* dst = buf + (size_t)s * rows * kTmaTile;
    for (int b = 0; b < nbox; ++b)
      tma_load_2d(dst + (size_t)b * mbox * kTmaTile, &map, (int)(tile * kTmaTile), b * mbox, &full[s], pol);
  };
  if (tid == 0) {
    for (int k = 0; k < stages; ++k) {
      const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
      if (t < ntiles) issue(t, k);
    }
  }
  float vmin = __int_as_float(0x7f800000), vmax = -__int_as_float(0x7f800000);
  bool bad = false;
  int s = 0;           // ring slot of this tile
  uint32_t phase = 0;  // mbarrier phase parity of the slot's current use
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    CPB_ASSERT(s >= 0 && s < stages);
    mbar_wait(&full[s], phase);
    const float* col = buf + (size_t)s * rows * kTmaTile + tid;
    const int64_t p = t * kTmaTile + tid;
    if (p < a.npix) {
      float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
      double sum = 0.0;
#pragma unroll 8
      for (int m = 0; m < M; ++m) {
        const float x = col[m * kTmaTile];
        lo = fmin_nan(lo, x);
        hi = fmaxf(hi, x);
        if (KIND == CPB_EPANECHNIKOV || KIND == CPB_GAUSSIAN) sum = __dadd_rn(sum, (double)x);
      }
      bad |= nonfinite(lo) | nonfinite(hi);
      vmin = fminf(vmin, lo);
      vmax = fmaxf(vmax, hi);
      if (KIND == CPB_UNIFORM || KIND == CPB_HISTOGRAM) {
        a.lo[p] = lo;
        a.hi[p] = hi;
      }
      if (KIND == CPB_HISTOGRAM) {
        const int h = a.bins;
        const double dlo = (double)lo;
        const double scale = __ddiv_rn((double)h, __dsub_rn((double)hi, dlo));
        constexpr int NB = NT > 0 ? NT : 1;
        uint32_t c[NB + 1];
        if (NT > 0) {
          // cumulative counts C_k = #{v >= thr_k}; bin b holds C_b - C_{b+1}
          float thr[NB];
          const float step = __fsub_rn(hi, lo) * __frcp_rn((float)h);  // a guess: any rounding
#pragma unroll
          for (int q = 1; q < NB; ++q)
            thr[q] = hi > lo ? bin_threshold(q, dlo, scale, __fmaf_rn((float)q, step, lo), lo, hi) : 0.0f;
#pragma unroll
          for (int q = 1; q < NB; ++q) thr[q] = thr[q] == 0.0f ? -0.0f : thr[q];  // +0 -> -0
#pragma unroll
          for (int q = 0; q <= NB; ++q) c[q] = 0u;
#pragma unroll 4
          for (int m = 0; m < M; ++m) {
            const float x = col[m * kTmaTile];
#pragma unroll
            for (int q = 1; q < NB; ++q) c[q] += lt_bit(x, thr[q]);  // #{x < thr_q}
          }
#pragma unroll
          for (int q = 1; q < NB; ++q) c[q] = (uint32_t)M - c[q];  // C_q = #{x >= thr_q}
          c[0] = (uint32_t)M;
        } else {
          for (int b = 0; b < h; ++b) cnt[b * kTmaTile + tid] = 0u;
          if (hi > lo)
            for (int m = 0; m < M; ++m) cnt[bin_of(col[m * kTmaTile], dlo, scale, h) * kTmaTile + tid] += 1u;
        }
        const bool flat = !(hi > lo);  // degenerate: counts resolved at use, once eps is known
        if (NT > 0) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const uint32_t v = flat ? 0u : (b + 1 < NB ? c[b] - c[b + 1] : c[b]);
            if (a.wmode == CPB_WEIGHTS_U8)
              static_cast<uint8_t*>(a.counts)[(int64_t)b * a.wstride + p] = (uint8_t)v;
            else
              static_cast<uint16_t*>(a.counts)[(int64_t)b * a.wstride + p] = (uint16_t)v;
          }
        } else {
          for (int b = 0; b < h; ++b) {
            const uint32_t v = flat ? 0u : cnt[b * kTmaTile + tid];
            if (a.wmode == CPB_WEIGHTS_U8)
              static_cast<uint8_t*>(a.counts)[(int64_t)b * a.wstride + p] = (uint8_t)v;
            else
              static_cast<uint16_t*>(a.counts)[(int64_t)b * a.wstride + p] = (uint16_t)v;
          }
        }
      }
      if (KIND == CPB_EPANECHNIKOV || KIND == CPB_GAUSSIAN) {
        const double mean = __ddiv_rn(sum, (double)M);
        double sq = 0.0;
#pragma unroll 8
        for (int m = 0; m < M; ++m) {
          const double d = __dsub_rn((double)col[m * kTmaTile], mean);
          sq = __dadd_rn(sq, __dmul_rn(d, d));
        }
        a.mean[p] = mean;
        a.spread[p] = __dsqrt_rn(__ddiv_rn(sq, (double)(M - 1)));
      }
    }
    __syncthreads();  // every thread is done with stage s
    if (tid == 0) {
      const int64_t tn = t + (int64_t)stages * gridDim.x;
      if (tn < ntiles) issue(tn, s);
    }
    if (++s == stages) {
      s = 0;
      phase ^= 1u;
    }
  }
  merge_range(vmin, vmax, bad, a.range);
}

// d_range words -> {-min, max} as float64 (NaN if a value was non-finite)
__global__ void range_pair_kernel(const uint32_t* range, double* pair) {
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  pair[0] = range[2] ? nan : -(double)ordered_to_float(range[0]);
  pair[1] = range[2] ? nan : (double)ordered_to_float(range[1]);
}

// eps = max(1e-12, 1e-9 * (max - min))  (distributions.py:30-36)
__global__ void pair_eps_kernel(const double* pair, double* eps) {
  const double spread = pair[1] + pair[0];  // max - min, pair[0] = -min
  const double e = 1e-9 * spread;
  *eps = e != e ? e : (e > 1e-12 ? e : 1e-12);
}

// ---------------------------------------------------------------------------
// Several models over ONE read of the ensemble (the reference workflow fits
// one EnsembleStack with every model, fields.py:125-158 per model): each
// TMA-staged tile feeds the shared min / max pass (uniform and histogram
// bounds are the same numbers), the histogram threshold binning and the
// Epanechnikov / Gaussian moment passes, so HBM sees the ensemble once
// instead of once per model.  Same arithmetic as the single-model kernels,
// so every plane is bit-identical to a separate cpb_fit.

template <int NT>
__global__ void __launch_bounds__(kTmaTile) fit_tma_multi_kernel(
    const __grid_constant__ CUtensorMap map, MultiArgs a, int stages, int mbox, int nbox,
    int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int M = a.members;
  const int rows = mbox * nbox;
  const int tid = threadIdx.x;
  float* buf = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * rows * kTmaTile * 4);
  if (tid == 0) {
    prefetch_tensormap(&map);
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint32_t tile_bytes = (uint32_t)rows * kTmaTile * 4u;
  auto issue = [&](int64_t tile, int s) {
    mbar_arrive_expect_tx(&full[s], tile_bytes);
    float* dst = buf + (size_t)s * rows * kTmaTile;
    for (int b = 0; b < nbox; ++b)
      tma_load_2d(dst + (size_t)b * mbox * kTmaTile, &map, (int)(tile * kTmaTile), b * mbox, &full[s], pol);
  };
  if (tid == 0) {
    for (int k = 0; k < stages; ++k) {
      const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
      if (t < ntiles) issue(t, k);
    }
  }
  float vmin = __int_as_float(0x7f800000), vmax = -__int_as_float(0x7f800000);
  bool bad = false;
  int s = 0;           // ring slot of this tile
  uint32_t phase = 0;  // mbarrier phase parity of the slot's current use
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    CPB_ASSERT(s >= 0 && s < stages);
    mbar_wait(&full[s], phase);
    const float* col = buf + (size_t)s * rows * kTmaTile + tid;
    const int64_t p = t * kTmaTile + tid;
    if (p < a.npix) {
      float lo, hi;
      multi_fit_pixel<NT>(col, kTmaTile, a, p, true, lo, hi);
      bad |= nonfinite(lo) | nonfinite(hi);
      vmin = fminf(vmin, lo);
      vmax = fmaxf(vmax, hi);
    }
    __syncthreads();
    if (tid == 0) {
      const int64_t tn = t + (int64_t)stages * gridDim.x;
      if (tn < ntiles) issue(tn, s);
    }
    if (++s == stages) {
      s = 0;
      phase ^= 1u;
    }
  }
  merge_range(vmin, vmax, bad, a.range);
}

// any non-finite value in n floats -> *flag = 1 (float4 loads; exponent all ones)
__global__ void nonfinite_kernel(const float* v, int64_t n, uint32_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  const int64_t n4 = ((reinterpret_cast<uintptr_t>(v) & 15) == 0) ? n / 4 : 0;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  for (int64_t i = t; i < n4; i += stride) {
    const float4 x = __ldcs(v4 + i);
    bad |= ((__float_as_uint(x.x) & 0x7f800000u) == 0x7f800000u) |
           ((__float_as_uint(x.y) & 0x7f800000u) == 0x7f800000u) |
           ((__float_as_uint(x.z) & 0x7f800000u) == 0x7f800000u) |
           ((__float_as_uint(x.w) & 0x7f800000u) == 0x7f800000u);
  }
  for (int64_t i = 4 * n4 + t; i < n; i += stride)
    bad |= (__float_as_uint(v[i]) & 0x7f800000u) == 0x7f800000u;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1u;
}

__global__ void range_init_kernel(uint32_t* range) {
  range[0] = 0xffffffffu;
  range[1] = 0u;
  range[2] = 0u;
}


// fields.py:160-178: lo/hi = v -+ half, half = eb/2 (or eps/2 when eb == 0)
__global__ void from_scalar_kernel(const double* v, int64_t n, double half, double* lo,
                                   double* hi) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double x = v[i];
    lo[i] = __dsub_rn(x, half);
    hi[i] = __dadd_rn(x, half);
  }
}

// Reference-layout float64 params (fields.py:137-158 outputs).
__global__ void materialize_kernel(FieldView f, double* a, double* b, double* w) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= f.npix) return;
  if (f.kind == CPB_EPANECHNIKOV) {
    double m, hw;
    load_epan(f, p, m, hw);
    a[p] = m;
    b[p] = hw;
    return;
  }
  if (f.kind == CPB_GAUSSIAN) {
    a[p] = f.mean[p];
    b[p] = f.spread[p];
    return;
  }
  double lo, hi;
  const bool deg = load_bounds(f, p, lo, hi);
  a[p] = lo;
  b[p] = hi;
  if (f.kind == CPB_HISTOGRAM && w != nullptr) {
    const int h = f.bins;
    const int dbin = deg ? degenerate_bin((double)static_cast<const float*>(f.lo)[p], lo, hi, h) : 0;
    for (int k = 0; k < h; ++k) w[p * h + k] = load_weight(f, p, k, deg, dbin);
  }
}

// bowl(r, c) = 4 (x^2 + y^2) - 3 x^2 y^2, x = c * (2/(W-1)) - 1, y = r * (2/(H-1)) - 1
// value = f32(bowl + amp * (2u - 1)); twin of oracle.synthetic_rows.
__global__ void synth_kernel(float* ens, int64_t mstride, int members, int64_t row0,
                             int64_t nrows, int64_t width, int64_t height, double amp,
                             uint64_t seed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows * width) return;
  const int64_t lr = i / width, c = i - lr * width, r = row0 + lr;
  const double sx = width > 1 ? __ddiv_rn(2.0, (double)(width - 1)) : 0.0;
  const double sy = height > 1 ? __ddiv_rn(2.0, (double)(height - 1)) : 0.0;
  const double x = __dsub_rn(__dmul_rn((double)c, sx), 1.0);
  const double y = __dsub_rn(__dmul_rn((double)r, sy), 1.0);
  const double x2 = __dmul_rn(x, x), y2 = __dmul_rn(y, y);
  const double base = __dsub_rn(__dmul_rn(4.0, __dadd_rn(x2, y2)), __dmul_rn(3.0, __dmul_rn(x2, y2)));
  const uint64_t pk = pixel_key(seed, (uint64_t)(r * width + c));
  for (int m = 0; m < members; ++m) {
    const double u = stream_u01(plane_key(pk, (uint64_t)m), 0);
    const double noise = __dmul_rn(amp, __dsub_rn(__dmul_rn(2.0, u), 1.0));
    ens[(int64_t)m * mstride + i] = __double2float_rn(__dadd_rn(base, noise));
  }
}

}  // namespace

bool encode_tensor_map_2d_f32(CUtensorMap* map, const void* base, uint64_t dim0, uint64_t dim1,
                              uint64_t stride1_bytes, uint32_t box0, uint32_t box1) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !ptr)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  const cuuint64_t dims[2] = {dim0, dim1};
  const cuuint64_t strides[1] = {stride1_bytes};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

inline unsigned grid_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

// cap on persistent fit CTAs per SM (0 = occupancy maximum); a smaller fit
// footprint leaves room for a concurrent stencil (cpb_set_option "fit_ctas_per_sm")
int g_fit_ctas_per_sm = 0;

int launch_fit(const float* ens, int64_t mstride, cpb_field* f, uint32_t* range, bool accumulate,
               cudaStream_t st) {
  FitArgs a;
  a.ens = ens;
  a.mstride = mstride;
  a.npix = f->height * f->width;
  a.wstride = f->plane_stride > 0 ? f->plane_stride : a.npix;
  a.members = f->members;
  a.bins = f->bins;
  a.lo = static_cast<float*>(f->lo);
  a.hi = static_cast<float*>(f->hi);
  a.mean = f->mean;
  a.spread = f->spread;
  a.counts = f->weights;
  a.wmode = f->members <= 255 ? CPB_WEIGHTS_U8 : CPB_WEIGHTS_U16;
  a.range = range;
  f->bounds = CPB_BOUNDS_F32_FITTED;
  f->weights_mode = f->kind == CPB_HISTOGRAM ? a.wmode : CPB_WEIGHTS_F64;
  if (!accumulate) {
    range_init_kernel<<<1, 1, 0, st>>>(range);
    CPB_CHECK_LAUNCH("range init");
  }
  if (a.npix == 0) return CPB_OK;
  if (f->kind == CPB_HISTOGRAM) {
    weight_table_kernel<<<grid_for(f->members + 1, 256), 256, 0, st>>>(f->weight_table, f->members);
    CPB_CHECK_LAUNCH("weight table");
  }
  // production path: TMA-staged tiles (member stride must be a multiple of 16 bytes)
  const int mbox = std::min(f->members, 256);
  const int nbox = (f->members + mbox - 1) / mbox;
  const size_t tile_bytes = (size_t)mbox * nbox * kTmaTile * 4;
  const size_t cnt_bytes =
      (f->kind == CPB_HISTOGRAM && f->bins > kThreshBins) ? (size_t)f->bins * kTmaTile * 4 : 0;
  const bool tma_ok = (mstride % 4 == 0) && ((reinterpret_cast<uintptr_t>(ens) & 15) == 0) &&
                      tile_bytes * 2 + cnt_bytes + 64 <= 200 * 1024;
  if (tma_ok) {
    // ~32 KB of staging per CTA (one 64-member tile): more resident CTAs per SM
    // hide the TMA latency at least as well as a deeper per-CTA ring (histogram
    // 15.6 -> 13.2 ms, uniform unchanged at the HBM limit)
    constexpr size_t kStageBytes = 32 * 1024;
    const int stages = (int)std::min<size_t>(8, std::max<size_t>(1, kStageBytes / tile_bytes));
    const size_t smem = stages * tile_bytes + stages * 8 + cnt_bytes;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // TMA coordinates are int32: split very large slabs into pixel chunks
    const int64_t max_chunk = (int64_t)1 << 30;
    for (int64_t p0 = 0; p0 < a.npix; p0 += max_chunk) {
      FitArgs c = a;
      const int64_t n = std::min(max_chunk, a.npix - p0);
      c.ens = ens + p0;
      c.npix = n;
      c.lo = a.lo ? a.lo + p0 : nullptr;
      c.hi = a.hi ? a.hi + p0 : nullptr;
      c.mean = a.mean ? a.mean + p0 : nullptr;
      c.spread = a.spread ? a.spread + p0 : nullptr;
      c.counts = a.counts ? static_cast<char*>(a.counts) + p0 * (a.wmode == CPB_WEIGHTS_U8 ? 1 : 2) : nullptr;
      CUtensorMap map;
      if (!encode_tensor_map_2d_f32(&map, c.ens, (uint64_t)n, (uint64_t)f->members,
                                    (uint64_t)mstride * 4, kTmaTile, (uint32_t)mbox)) {
        set_error("cuTensorMapEncodeTiled failed");
        return CPB_ECUDA;
      }
      const int64_t ntiles = (n + kTmaTile - 1) / kTmaTile;
#define CPB_FIT_TMA_LAUNCH(KERN)                                                                 \
  do {                                                                                           \
    auto kern = KERN;                                                                            \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);          \
    int per_sm = 1;                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTmaTile, smem);                \
    if (g_fit_ctas_per_sm > 0) per_sm = std::min(per_sm, g_fit_ctas_per_sm);                    \
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * std::max(per_sm, 1));          \
    kern<<<(unsigned)grid, kTmaTile, smem, st>>>(map, c, stages, mbox, nbox, ntiles);            \
  } while (0)
#define CPB_FIT_TMA(K) \
  case K:              \
    CPB_FIT_TMA_LAUNCH((fit_tma_kernel<K, 0>)); \
    break;
      switch (f->kind) {
        CPB_FIT_TMA(CPB_UNIFORM)
        CPB_FIT_TMA(CPB_EPANECHNIKOV)
        CPB_FIT_TMA(CPB_GAUSSIAN)
        case CPB_HISTOGRAM:
          switch (f->bins <= kThreshBins ? f->bins : 0) {
            case 1: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 1>)); break;
            case 2: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 2>)); break;
            case 3: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 3>)); break;
            case 4: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 4>)); break;
            case 5: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 5>)); break;
            case 6: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 6>)); break;
            case 7: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 7>)); break;
            case 8: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 8>)); break;
            default: CPB_FIT_TMA_LAUNCH((fit_tma_kernel<CPB_HISTOGRAM, 0>)); break;
          }
          break;
        default:
          set_error("unknown model kind %d", f->kind);
          return CPB_EINVAL;
      }
#undef CPB_FIT_TMA_LAUNCH
#undef CPB_FIT_TMA
      CPB_CHECK_LAUNCH("fit kernel (TMA)");
    }
    return CPB_OK;
  }
  int threads = kFitThreads;
  size_t smem = 0;
  if (f->kind == CPB_HISTOGRAM) {
    // per-thread bin counters; shrink the block for very many bins
    while ((size_t)f->bins * threads * 4 > 160 * 1024 && threads > 32) threads >>= 1;
    smem = (size_t)f->bins * threads * 4;
    if (smem > 160 * 1024) {
      set_error("histogram fit supports at most %d bins", 160 * 1024 / (32 * 4));
      return CPB_EINVAL;
    }
  }
  const unsigned grid = grid_for(a.npix, threads);
  const bool reg = f->members <= kRegMembers;
#define CPB_FIT_CASE(K)                                                                   \
  case K: {                                                                               \
    auto kern = reg ? fit_reg_kernel<K> : fit_loop_kernel<K>;                             \
    if (smem > 48 * 1024)                                                                 \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<grid, threads, smem, st>>>(a);                                                 \
    break;                                                                                \
  }
  switch (f->kind) {
    CPB_FIT_CASE(CPB_UNIFORM)
    CPB_FIT_CASE(CPB_EPANECHNIKOV)
    CPB_FIT_CASE(CPB_HISTOGRAM)
    CPB_FIT_CASE(CPB_GAUSSIAN)
    default:
      set_error("unknown model kind %d", f->kind);
      return CPB_EINVAL;
  }
#undef CPB_FIT_CASE
  CPB_CHECK_LAUNCH("fit kernel");
  return CPB_OK;
}

int launch_nonfinite(const float* v, int64_t n, uint32_t* flag, cudaStream_t st) {
  if (n <= 0) return CPB_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n / 4 + 255) / 256;
  nonfinite_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8)), 256, 0, st>>>(
      v, n, flag);
  CPB_CHECK_LAUNCH("finiteness check");
  return CPB_OK;
}

int launch_range_to_pair(const uint32_t* range, double* pair, cudaStream_t st) {
  range_pair_kernel<<<1, 1, 0, st>>>(range, pair);
  CPB_CHECK_LAUNCH("range pair kernel");
  return CPB_OK;
}

int launch_pair_to_eps(const double* pair, double* eps, cudaStream_t st) {
  pair_eps_kernel<<<1, 1, 0, st>>>(pair, eps);
  CPB_CHECK_LAUNCH("pair eps kernel");
  return CPB_OK;
}

int launch_from_scalar(const double* v, int64_t n, double half, double* lo, double* hi,
                       cudaStream_t st) {
  if (n == 0) return CPB_OK;
  from_scalar_kernel<<<grid_for(n, 256), 256, 0, st>>>(v, n, half, lo, hi);
  CPB_CHECK_LAUNCH("from_scalar kernel");
  return CPB_OK;
}

int launch_materialize(const cpb_field* f, double* a, double* b, double* w, cudaStream_t st) {
  const FieldView v = make_view(*f);
  if (v.npix == 0) return CPB_OK;
  materialize_kernel<<<grid_for(v.npix, 256), 256, 0, st>>>(v, a, b, w);
  CPB_CHECK_LAUNCH("materialize kernel");
  return CPB_OK;
}

int launch_synth(float* ens, int64_t members, int64_t row0, int64_t nrows, int64_t width,
                 int64_t height, double amp, uint64_t seed, cudaStream_t st) {
  const int64_t n = nrows * width;
  if (n == 0) return CPB_OK;
  synth_kernel<<<grid_for(n, 256), 256, 0, st>>>(ens, n, (int)members, row0, nrows, width, height,
                                                  amp, seed);
  CPB_CHECK_LAUNCH("synth kernel");
  return CPB_OK;
}

}  // namespace cpb

// ---------------------------------------------------------------------------
// Device-side P5 heatmap (field_io.py:138-150): gray = round(255 * clip(p, 0, 1)^gamma)
// (numpy round-half-even), 0 where the pixel is invalid.
// ---------------------------------------------------------------------------
namespace cpb {
namespace {
__global__ void heatmap_kernel(const double* p, const uint8_t* valid, int64_t n, double gamma,
                               uint8_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = fmin(fmax(p[i], 0.0), 1.0);
  double y;
  if (gamma == 1.0) y = x;                 // numpy's power fast paths
  else if (gamma == 0.5) y = __dsqrt_rn(x);
  else if (gamma == 2.0) y = __dmul_rn(x, x);
  else y = pow(x, gamma);
  const double g = rint(__dmul_rn(255.0, y));
  out[i] = (valid && !valid[i]) ? (uint8_t)0 : (uint8_t)g;
}
}  // namespace

int launch_heatmap(const double* p, const uint8_t* valid, int64_t n, double gamma, uint8_t* out,
                   cudaStream_t st) {
  if (n == 0) return CPB_OK;
  heatmap_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, valid, n, gamma, out);
  CPB_CHECK_LAUNCH("heatmap kernel");
  return CPB_OK;
}
}  // namespace cpb

// ---------------------------------------------------------------------------
// Rows whose stencil results depend on eps (for streamed classification with
// a provisional eps): sens[r] = 1 if row r holds a fitted uniform/histogram
// pixel with hi <= lo (widened by eps/2 at use, fields.py:140-143) or an
// Epanechnikov pixel with k * std < eps / 2 (clamped at use, fields.py:156).
// ---------------------------------------------------------------------------
namespace cpb {
namespace {
__global__ void eps_sensitive_rows_kernel(FieldView f, double eps, uint8_t* sens) {
  const int64_t r = blockIdx.x;
  int any = 0;
  for (int64_t c = threadIdx.x; c < f.width; c += blockDim.x) {
    const int64_t i = r * f.width + c;
    if (f.kind == CPB_EPANECHNIKOV) {
      any |= __dmul_rn(f.k, f.spread[i]) < __dmul_rn(0.5, eps);
    } else if (f.kind != CPB_GAUSSIAN && f.bounds == CPB_BOUNDS_F32_FITTED) {
      any |= static_cast<const float*>(f.hi)[i] <= static_cast<const float*>(f.lo)[i];
    }
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) sens[r] = (uint8_t)(any ? 1 : 0);
}
}  // namespace

int launch_eps_sensitive_rows(const cpb_field* fld, double eps, uint8_t* sens, cudaStream_t st) {
  const FieldView f = make_view(*fld);
  if (f.height == 0) return CPB_OK;
  eps_sensitive_rows_kernel<<<(unsigned)f.height, 256, 0, st>>>(f, eps, sens);
  CPB_CHECK_LAUNCH("eps sensitivity kernel");
  return CPB_OK;
}

// Fused fit of several models (see fit_tma_multi_kernel).  Returns 1 (nothing
// launched) when the combination or layout is not covered -- the caller then
// fits the fields one by one.
int launch_fit_multi(const float* ens, int64_t mstride, cpb_field* const* fs, int n,
                     uint32_t* range, bool accumulate, cudaStream_t st) {
  cpb_field* slot[4] = {nullptr, nullptr, nullptr, nullptr};  // uniform, histogram, epan, gaussian
  for (int i = 0; i < n; ++i) {
    const int k = fs[i]->kind;
    const int q = k == CPB_UNIFORM ? 0 : k == CPB_HISTOGRAM ? 1 : k == CPB_EPANECHNIKOV ? 2 : 3;
    if (slot[q]) return 1;
    slot[q] = fs[i];
  }
  const cpb_field* f0 = fs[0];
  if (slot[1] && slot[1]->bins > kThreshBins) return 1;
  const int64_t npix = f0->height * f0->width;
  const int mbox = std::min(f0->members, 256);
  const int nbox = (f0->members + mbox - 1) / mbox;
  const size_t tile_bytes = (size_t)mbox * nbox * kTmaTile * 4;
  if (!((mstride % 4 == 0) && ((reinterpret_cast<uintptr_t>(ens) & 15) == 0) &&
        tile_bytes * 2 + 64 <= 200 * 1024))
    return 1;
  MultiArgs a = {};
  a.npix = npix;
  a.members = f0->members;
  a.wmode = f0->members <= 255 ? CPB_WEIGHTS_U8 : CPB_WEIGHTS_U16;
  a.range = range;
  for (int i = 0; i < 2; ++i) {
    if (slot[i]) {
      a.lo[i] = static_cast<float*>(slot[i]->lo);
      a.hi[i] = static_cast<float*>(slot[i]->hi);
      slot[i]->bounds = CPB_BOUNDS_F32_FITTED;
      slot[i]->weights_mode = CPB_WEIGHTS_F64;
    }
    if (slot[2 + i]) {
      a.mean[i] = slot[2 + i]->mean;
      a.spread[i] = slot[2 + i]->spread;
      slot[2 + i]->bounds = CPB_BOUNDS_F32_FITTED;
      slot[2 + i]->weights_mode = CPB_WEIGHTS_F64;
    }
  }
  int nt = 0;
  if (slot[1]) {
    nt = slot[1]->bins;
    a.bins = nt;
    a.counts = slot[1]->weights;
    a.wstride = slot[1]->plane_stride > 0 ? slot[1]->plane_stride : npix;
    slot[1]->weights_mode = a.wmode;
  }
  if (!accumulate) {
    range_init_kernel<<<1, 1, 0, st>>>(range);
    CPB_CHECK_LAUNCH("range init");
  }
  if (npix == 0) return CPB_OK;
  if (slot[1]) {
    weight_table_kernel<<<grid_for(a.members + 1, 256), 256, 0, st>>>(slot[1]->weight_table, a.members);
    CPB_CHECK_LAUNCH("weight table");
  }
  // one 32 KB stage per CTA (6-7 CTAs / SM): with the issue-bound fused passes,
  // more resident CTAs hide the TMA latency better than a deeper ring per CTA
  // (19.7 vs 23.4 ms at config 5)
  const int stages = 1;
  const size_t smem = stages * tile_bytes + stages * 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t max_chunk = (int64_t)1 << 30;
  for (int64_t p0 = 0; p0 < npix; p0 += max_chunk) {
    MultiArgs c = a;
    const int64_t cn = std::min(max_chunk, npix - p0);
    c.npix = cn;
    for (int i = 0; i < 2; ++i) {
      if (c.lo[i]) { c.lo[i] += p0; c.hi[i] += p0; }
      if (c.mean[i]) { c.mean[i] += p0; c.spread[i] += p0; }
    }
    if (c.counts) c.counts = static_cast<char*>(c.counts) + p0 * (a.wmode == CPB_WEIGHTS_U8 ? 1 : 2);
    CUtensorMap map;
    if (!encode_tensor_map_2d_f32(&map, ens + p0, (uint64_t)cn, (uint64_t)a.members,
                                  (uint64_t)mstride * 4, kTmaTile, (uint32_t)mbox)) {
      set_error("cuTensorMapEncodeTiled failed");
      return CPB_ECUDA;
    }
    const int64_t ntiles = (cn + kTmaTile - 1) / kTmaTile;
#define CPB_MULTI(NTV)                                                                         \
  case NTV: {                                                                                  \
    auto kern = fit_tma_multi_kernel<NTV>;                                                     \
    const int threads = kTmaTile;                                                              \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    int per_sm = 1;                                                                            \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);               \
    if (g_fit_ctas_per_sm > 0) per_sm = std::min(per_sm, g_fit_ctas_per_sm);                  \
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * std::max(per_sm, 1));        \
    kern<<<(unsigned)grid, threads, smem, st>>>(map, c, stages, mbox, nbox, ntiles);           \
  } break;
    switch (nt) {
      CPB_MULTI(0) CPB_MULTI(1) CPB_MULTI(2) CPB_MULTI(3) CPB_MULTI(4)
      CPB_MULTI(5) CPB_MULTI(6) CPB_MULTI(7) CPB_MULTI(8)
      default: return 1;
    }
#undef CPB_MULTI
    CPB_CHECK_LAUNCH("fused multi-model fit kernel");
  }
  return CPB_OK;
}

}  // namespace cpb
