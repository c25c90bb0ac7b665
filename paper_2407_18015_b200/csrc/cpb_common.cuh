// Shared device helpers for the critprob B200 kernels.
//
// Reference citations are /root/reference/pkg/src/critprob/<file>:<line>.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/critprob_b200.h"

#define CPB_HD __host__ __device__ __forceinline__
#define CPB_D __device__ __forceinline__

namespace cpb {

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

// Bounds-check build (CPB_NVCC_EXTRA=-DCPB_BOUNDS_CHECK=1, tools/build_variant.sh):
// every CPB_ASSERT on a shared-memory / ring index traps with its location, so
// the GPU test suite run against that build doubles as an out-of-bounds check
// (compute-sanitizer is not available on this pool).  Compiled out otherwise.
#if defined(CPB_BOUNDS_CHECK) && CPB_BOUNDS_CHECK
#define CPB_ASSERT(cond)                                                                 \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("CPB_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define CPB_ASSERT(cond) \
  do {                   \
  } while (0)
#endif

#define CPB_CHECK_LAUNCH(what)                                              \
  do {                                                                      \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) return ::cpb::cuda_status(_e, what);             \
  } while (0)

// ---------------------------------------------------------------------------
// Gauss-Legendre tables: the exact bits of numpy.polynomial.legendre.leggauss(n)
// (piecewise.py:29-31); 3 nodes for uniform/histogram, 8 for epanechnikov
// (engine.py:600-601).
// ---------------------------------------------------------------------------
// Device code reads the nodes / weights from constant memory, so a DFMA takes
// them as a c[bank][offset] operand instead of materialising each 64-bit
// immediate with two UMOVs per use inside the piece loops.
__constant__ double c_gl3[6] = {-0x1.8c97ef43f7248p-1, 0.0, 0x1.8c97ef43f7248p-1,
                                0x1.1c71c71c71c73p-1, 0x1.c71c71c71c71cp-1, 0x1.1c71c71c71c73p-1};
__constant__ double c_gl8[16] = {
    -0x1.ebab1cb0acc66p-1, -0x1.97e4ab249f41ep-1, -0x1.0d129583284b4p-1, -0x1.77ac94f3c7344p-3,
    0x1.77ac94f3c7344p-3,  0x1.0d129583284b4p-1,  0x1.97e4ab249f41ep-1,  0x1.ebab1cb0acc66p-1,
    0x1.9ea1d04ca03aep-4,  0x1.c76fb531d2b94p-3,  0x1.413c50a25560ep-2,  0x1.736360b19933dp-2,
    0x1.736360b19933dp-2,  0x1.413c50a25560ep-2,  0x1.c76fb531d2b94p-3,  0x1.9ea1d04ca03aep-4};

struct GL3 {
  static constexpr int n = 3;
  CPB_HD static double x(int i) {
#ifdef __CUDA_ARCH__
    return c_gl3[i];
#else
    return i == 0 ? -0x1.8c97ef43f7248p-1 : (i == 1 ? 0.0 : 0x1.8c97ef43f7248p-1);
#endif
  }
  CPB_HD static double w(int i) {
#ifdef __CUDA_ARCH__
    return c_gl3[3 + i];
#else
    return i == 1 ? 0x1.c71c71c71c71cp-1 : 0x1.1c71c71c71c73p-1;
#endif
  }
};

// numpy leggauss(n) bits by node count, as (positive node, weight) pairs from
// the outermost node in, plus the centre weight for odd counts; constant
// memory like c_gl3 / c_gl8.  Offsets: n = 2 at 0, 3 at 2, 5 at 5, 6 at 10,
// 8 at 16.
__constant__ double c_glsym[24] = {
    0x1.279a74590331cp-1, 0x1.0000000000000p+0,                                     // 2
    0x1.8c97ef43f7248p-1, 0x1.1c71c71c71c73p-1, 0x1.c71c71c71c71cp-1,               // 3
    0x1.cff6ce0533a69p-1, 0x1.13b23fd99b705p-1, 0x1.e539ec36e0393p-3,               // 5
    0x1.ea1da25ae4158p-2, 0x1.23456789abcddp-1,
    0x1.dd6ca4e80a01dp-1, 0x1.528a09655c95ep-1, 0x1.e8b12d03675c5p-3,               // 6
    0x1.5edf601e2dbf5p-3, 0x1.716b7b5794c1ep-2, 0x1.df24d499545e8p-2,
    0x1.ebab1cb0acc66p-1, 0x1.97e4ab249f41ep-1, 0x1.0d129583284b4p-1,               // 8
    0x1.77ac94f3c7344p-3, 0x1.9ea1d04ca03aep-4, 0x1.c76fb531d2b94p-3,
    0x1.413c50a25560ep-2, 0x1.736360b19933dp-2};

// Symmetric Gauss-Legendre rule with NN nodes (device code only): x(i), w(i)
// for the node pairs +-x(i), w0() the centre weight (odd NN).  Used by the
// degree-adaptive Epanechnikov stencil: a piece whose integrand has degree
// 2 + 3k (k neighbours inside their support) is integrated exactly by
// NN = 2, 3, 5, 6, 8 nodes for k = 0..4.
template <int NN>
struct GLSym {
  static constexpr int pairs = NN / 2;
  static constexpr int off = NN == 2 ? 0 : NN == 3 ? 2 : NN == 5 ? 5 : NN == 6 ? 10 : 16;
  static_assert(NN == 2 || NN == 3 || NN == 5 || NN == 6 || NN == 8, "no table");
  CPB_D static double x(int i) { return c_glsym[off + i]; }
  CPB_D static double w(int i) { return c_glsym[off + pairs + i]; }
  CPB_D static double w0() { return NN % 2 ? c_glsym[off + 2 * pairs] : 0.0; }
};

struct GL8 {
  static constexpr int n = 8;
  CPB_HD static double x(int i) {
#ifdef __CUDA_ARCH__
    return c_gl8[i];
#else
    switch (i) {
      case 0: return -0x1.ebab1cb0acc66p-1;
      case 1: return -0x1.97e4ab249f41ep-1;
      case 2: return -0x1.0d129583284b4p-1;
      case 3: return -0x1.77ac94f3c7344p-3;
      case 4: return 0x1.77ac94f3c7344p-3;
      case 5: return 0x1.0d129583284b4p-1;
      case 6: return 0x1.97e4ab249f41ep-1;
      default: return 0x1.ebab1cb0acc66p-1;
    }
#endif
  }
  CPB_HD static double w(int i) {
#ifdef __CUDA_ARCH__
    return c_gl8[8 + i];
#else
    switch (i) {
      case 0: case 7: return 0x1.9ea1d04ca03aep-4;
      case 1: case 6: return 0x1.c76fb531d2b94p-3;
      case 2: case 5: return 0x1.413c50a25560ep-2;
      default: return 0x1.736360b19933dp-2;
    }
#endif
  }
};


// ---------------------------------------------------------------------------
// keyed splitmix64 stream (rngstream.py:18-48)
// ---------------------------------------------------------------------------
constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSaltPixel = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kSaltPlane = 0x94D049BB133111EBull;

CPB_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// base = mix(seed + phi); pixel key = mix(base ^ px * S1); plane key = mix(pk ^ plane * S2)
CPB_HD uint64_t pixel_key(uint64_t seed, uint64_t px) {
  const uint64_t base = mix64(seed + kPhi);
  return mix64(base ^ (px * kSaltPixel));
}
CPB_HD uint64_t plane_key(uint64_t pk, uint64_t plane) { return mix64(pk ^ (plane * kSaltPlane)); }

// u = (mix(key + (i+1) * phi) >> 11) * 2^-53, exactly (a 53-bit integer is exact in f64)
CPB_D double stream_u01(uint64_t key, uint64_t i) {
  const uint64_t z = mix64(key + (i + 1ull) * kPhi);
  return __dmul_rn((double)(z >> 11), 0x1p-53);
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. 2011), used only for CPB_RNG_PHILOX
// ---------------------------------------------------------------------------
CPB_D uint4 philox4x32_10(uint4 ctr, uint2 key) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += W0;
    key.y += W1;
  }
  return ctr;
}
CPB_D double u53_from(uint32_t a, uint32_t b) {
  return __dmul_rn((double)(((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6)), 0x1p-53);
}

// ---------------------------------------------------------------------------
// order-preserving float <-> uint32 (for atomic min/max of the global range)
// ---------------------------------------------------------------------------
CPB_HD uint32_t float_to_ordered(float f) {
  uint32_t b;
#ifdef __CUDA_ARCH__
  b = __float_as_uint(f);
#else
  memcpy(&b, &f, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
CPB_HD float ordered_to_float(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(b);
#else
  memcpy(&f, &b, 4);
#endif
  return f;
}

// ---------------------------------------------------------------------------
// numpy's pairwise summation of a contiguous run (what w.sum(axis=1) does
// for the histogram renormalisation, engine.py:538 / 651): sequential below
// 8 terms, 8 interleaved accumulators up to 128, recursive halving above.
// ---------------------------------------------------------------------------
template <typename Get>
CPB_D double pairwise_sum_block(const Get& get, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, get(off + i));
    return r;
  }
  double r0 = get(off + 0), r1 = get(off + 1), r2 = get(off + 2), r3 = get(off + 3);
  double r4 = get(off + 4), r5 = get(off + 5), r6 = get(off + 6), r7 = get(off + 7);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, get(off + i + 0));
    r1 = __dadd_rn(r1, get(off + i + 1));
    r2 = __dadd_rn(r2, get(off + i + 2));
    r3 = __dadd_rn(r3, get(off + i + 3));
    r4 = __dadd_rn(r4, get(off + i + 4));
    r5 = __dadd_rn(r5, get(off + i + 5));
    r6 = __dadd_rn(r6, get(off + i + 6));
    r7 = __dadd_rn(r7, get(off + i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, get(off + i));
  return res;
}

template <typename Get>
__device__ double pairwise_sum_rec(const Get& get, int off, int n) {
  if (n <= 128) return pairwise_sum_block(get, off, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum_rec(get, off, n2), pairwise_sum_rec(get, off + n2, n - n2));
}

template <typename Get>
CPB_D double pairwise_sum(const Get& get, int n) {
  return n <= 128 ? pairwise_sum_block(get, 0, n) : pairwise_sum_rec(get, 0, n);
}

// ---------------------------------------------------------------------------
// The semianalytical mean's summation (engine.py:439 / 683 average the c
// per-draw pattern terms): lane l of a warp adds terms l, l + 32, ... in
// order, then a fixed xor-shuffle tree adds the 32 lane sums.  The grid
// kernel (semi_kernel) and the per-case kernel (cases_semi_kernel) both sum
// through this ONE function, so a grid vertex and the same neighbourhood as
// a case give bit-identical results, as the reference's two numpy paths do
// (test_engine.py:574-582); the association differs from numpy's pairwise
// sum by ~1e-16 relative.  Valid in every lane.
// ---------------------------------------------------------------------------
// the conditional pattern terms of one draw (_conditional_pattern,
// engine.py:444-459) from the neighbour CDFs F[1..4] (E, N, W, S) at the draw
CPB_D void semi_terms4(const double F[5], double t[3]) {
  const double e = F[1], nn = F[2], w = F[3], s = F[4];
  t[0] = __dmul_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, e), __dsub_rn(1.0, nn)), __dsub_rn(1.0, w)),
                   __dsub_rn(1.0, s));
  t[1] = __dmul_rn(__dmul_rn(__dmul_rn(e, nn), w), s);
  const double t1 = __dmul_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, e), nn), __dsub_rn(1.0, w)), s);
  const double t2 = __dmul_rn(__dmul_rn(__dmul_rn(e, __dsub_rn(1.0, nn)), w), __dsub_rn(1.0, s));
  t[2] = __dadd_rn(t1, t2);
}

// the same for a two-neighbour (1-D) case, F[1..2]
CPB_D void semi_terms2(const double F[3], double t[3]) {
  t[0] = __dmul_rn(__dsub_rn(1.0, F[1]), __dsub_rn(1.0, F[2]));
  t[1] = __dmul_rn(F[1], F[2]);
  t[2] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, F[1]), F[2]), __dmul_rn(F[1], __dsub_rn(1.0, F[2])));
}

template <typename Term>
CPB_D void warp_strided_sum3(const Term& term, int64_t n, int lane, double r[3]) {
  r[0] = r[1] = r[2] = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    double t[3];
    term(i, t);
#pragma unroll
    for (int q = 0; q < 3; ++q) r[q] = __dadd_rn(r[q], t[q]);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
#pragma unroll
    for (int q = 0; q < 3; ++q) r[q] = __dadd_rn(r[q], __shfl_xor_sync(0xffffffffu, r[q], d));
  }
}

// ---------------------------------------------------------------------------
// parameter access for one pixel of a cpb_field
// ---------------------------------------------------------------------------
// Block-level merge of the per-thread range into the global words.
CPB_D void merge_range(float vmin, float vmax, bool bad, uint32_t* range) {
  uint32_t omin = float_to_ordered(vmin), omax = float_to_ordered(vmax);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    omin = min(omin, __shfl_xor_sync(0xffffffffu, omin, s));
    omax = max(omax, __shfl_xor_sync(0xffffffffu, omax, s));
  }
  const unsigned anybad = __any_sync(0xffffffffu, bad);
  __shared__ uint32_t s_min[32], s_max[32], s_bad[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { s_min[warp] = omin; s_max[warp] = omax; s_bad[warp] = anybad; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    omin = lane < nw ? s_min[lane] : 0xffffffffu;
    omax = lane < nw ? s_max[lane] : 0u;
    uint32_t b = lane < nw ? s_bad[lane] : 0u;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      omin = min(omin, __shfl_xor_sync(0xffffffffu, omin, s));
      omax = max(omax, __shfl_xor_sync(0xffffffffu, omax, s));
      b |= __shfl_xor_sync(0xffffffffu, b, s);
    }
    if (lane == 0) {
      atomicMin(range + 0, omin);
      atomicMax(range + 1, omax);
      if (b) atomicOr(range + 2, 1u);
    }
  }
}

struct FieldView {
  int kind, bins, members, bounds, wmode;
  int mixed;        // CPB_FLAG_MIXED: single-precision GL evaluation in the closed form
  int64_t height, width, row0, gwidth;
  int64_t npix;     // height * width
  int64_t wstride;  // elements between histogram bin planes
  double eps, k;
  const double* eps_dev;
  const void* lo;
  const void* hi;
  const double* mean;
  const double* spread;
  const void* weights;
  const double* wtab;
};

inline FieldView make_view(const cpb_field& f) {
  FieldView v;
  v.kind = f.kind; v.bins = f.bins; v.members = f.members; v.bounds = f.bounds;
  v.wmode = f.weights_mode; v.height = f.height; v.width = f.width; v.row0 = f.row0;
  v.gwidth = f.global_width; v.npix = f.height * f.width;
  v.wstride = f.plane_stride > 0 ? f.plane_stride : v.npix;
  v.eps = f.eps; v.k = f.k;
  v.eps_dev = f.eps_device;
  v.lo = f.lo; v.hi = f.hi; v.mean = f.mean; v.spread = f.spread; v.weights = f.weights;
  v.wtab = f.weight_table;
  v.mixed = (f.flags & CPB_FLAG_MIXED) ? 1 : 0;
  return v;
}

CPB_D double field_eps(const FieldView& v) { return v.eps_dev ? __ldg(v.eps_dev) : v.eps; }

// Support bounds of a uniform/histogram pixel, widened like fields.py:140-143
// when the stored (fitted, f32) range is degenerate.  Returns true if widened.
CPB_D bool load_bounds(const FieldView& v, int64_t idx, double& lo, double& hi) {
  if (v.bounds == CPB_BOUNDS_F64) {
    lo = __ldg(static_cast<const double*>(v.lo) + idx);
    hi = __ldg(static_cast<const double*>(v.hi) + idx);
    return false;
  }
  lo = (double)__ldg(static_cast<const float*>(v.lo) + idx);
  hi = (double)__ldg(static_cast<const float*>(v.hi) + idx);
  if (hi <= lo) {
    const double c = lo, h = __dmul_rn(0.5, field_eps(v));
    lo = __dsub_rn(c, h);
    hi = __dadd_rn(c, h);
    return true;
  }
  return false;
}

// Epanechnikov mean / half-width: max(k * std, 0.5 * eps) (fields.py:156).
CPB_D void load_epan(const FieldView& v, int64_t idx, double& m, double& hw) {
  m = __ldg(v.mean + idx);
  const double s = __ldg(v.spread + idx);
  const double a = __dmul_rn(v.k, s), b = __dmul_rn(0.5, field_eps(v));
  hw = a > b ? a : (b > a ? b : a);  // np.maximum (no NaN inputs here)
}

// Bin that a degenerate fitted histogram pixel puts all its members in:
// clip(floor((c - lo') * (h / (hi' - lo'))), 0, h-1) with the widened bounds
// (fields.py:140-148; every member equals the centre c).
CPB_D int degenerate_bin(double c, double lo, double hi, int h) {
  const double scale = __ddiv_rn((double)h, __dsub_rn(hi, lo));
  double t = floor(__dmul_rn(__dsub_rn(c, lo), scale));
  int b = (int)fmax(0.0, fmin(t, (double)(h - 1)));
  return b;
}

// Weight w_b of bin b at pixel idx (before renormalisation): count/M from the
// exact table, the degenerate one-hot, or the stored float64 weight.
CPB_D double load_weight(const FieldView& v, int64_t idx, int b, bool degenerate, int dbin) {
  if (v.wmode == CPB_WEIGHTS_F64)
    return __ldg(static_cast<const double*>(v.weights) + (int64_t)b * v.wstride + idx);
  if (degenerate) return b == dbin ? 1.0 : 0.0;  // M/M == 1.0 exactly
  unsigned c;
  if (v.wmode == CPB_WEIGHTS_U8)
    c = __ldg(static_cast<const uint8_t*>(v.weights) + (int64_t)b * v.wstride + idx);
  else
    c = __ldg(static_cast<const uint16_t*>(v.weights) + (int64_t)b * v.wstride + idx);
  return __ldg(v.wtab + c);
}

}  // namespace cpb
