// Monte Carlo pattern estimator and the keyed uniform stream.
//
// Reference: _mc_chunk (engine.py:659-666), _position_samples
// (engine.py:632-656), the inverse CDFs (distributions.py:60-89),
// _pattern_stats (engine.py:195-222) and rngstream.unit_block
// (rngstream.py:33-48).
//
// One warp per vertex: the 32 lanes split the n joint draws, each lane keeps
// integer hit counts, and a warp reduction gives exact totals (integer sums
// are order-free, so results do not depend on the launch shape).  With the
// splitmix64 stream each draw is the reference's (seed, pixel, plane, i)
// uniform and the inverse CDFs repeat numpy's float64 operations with
// explicit round-to-nearest intrinsics, so uniform and histogram counts are
// bit-identical to the reference; Epanechnikov draws (the cubic's root by a
// float guess + one float64 Halley step, cpb_sample.cuh) and Gaussian draws
// (log1p/cos) can differ from glibc's by an ulp or two, which flips a strict
// comparison only on a tie within that distance (never observed).
#include "cpb_common.cuh"
#include "cpb_sample.cuh"

namespace cpb {
namespace {

constexpr int kMcWarps = 4;  // warps (vertices in flight) per block

struct McArgs {
  int64_t row_begin, nvert, cols;  // interior columns per row = width - 2
  uint64_t seed;
  int64_t n;
  double* pmin;
  double* pmax;
  double* psad;
  int64_t* counts;  // optional: 3 planes (min, max, saddle)
};

template <int KIND, int RNG>
__global__ void __launch_bounds__(kMcWarps * 32) mc_kernel(FieldView f, McArgs a) {
  extern __shared__ double s_tab[];  // per warp: 5 x (h wn + h+1 cum)
  // two-stage sampling for the costly inverse CDFs (see below): a 64-entry
  // ring per warp of candidate draws (C value, sample index, type, u_N)
  constexpr bool kSplit = KIND == CPB_EPANECHNIKOV || KIND == CPB_HISTOGRAM;
  constexpr int kQ = kSplit ? kMcWarps * 64 : 1;
  __shared__ double q_x[kQ], q_u[kQ];
  __shared__ int64_t q_i[kQ];
  __shared__ unsigned char q_t[kQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = f.bins;
  const int tab = 2 * h + 1;
  double* my_tab = s_tab + (size_t)warp * 5 * tab;
  const int64_t warps_total = (int64_t)gridDim.x * kMcWarps;
  for (int64_t v = (int64_t)blockIdx.x * kMcWarps + warp; v < a.nvert; v += warps_total) {
    const int64_t r = a.row_begin + v / a.cols, c = 1 + v % a.cols;
    const int64_t idx = r * f.width + c;
    const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
    Sampler s[5];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      if (KIND == CPB_UNIFORM) {
        load_bounds(f, at[p], s[p].a, s[p].b);
      } else if (KIND == CPB_EPANECHNIKOV) {
        double m, hw;
        load_epan(f, at[p], m, hw);
        const double lo = __dsub_rn(m, hw), hi = __dadd_rn(m, hw);  // engine.py:645-649
        s[p].a = __dmul_rn(0.5, __dadd_rn(lo, hi));
        s[p].b = __dmul_rn(0.5, __dsub_rn(hi, lo));
      } else if (KIND == CPB_GAUSSIAN) {
        s[p].a = __ldg(f.mean + at[p]);
        s[p].b = __ldg(f.spread + at[p]);
      } else {
        double lo, hi;
        const bool deg = load_bounds(f, at[p], lo, hi);
        s[p].a = lo;
        s[p].b = __ddiv_rn(__dsub_rn(hi, lo), (double)h);  // binw, engine.py:655
        s[p].wn = my_tab + p * tab;
        s[p].cum = my_tab + p * tab + h;
        if (lane == p) {  // one lane per position builds its tables (engine.py:650-654)
          const int dbin =
              deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at[p]), lo, hi, h) : 0;
          const double total =
              pairwise_sum([&](int b) { return load_weight(f, at[p], b, deg, dbin); }, h);
          double* wn = my_tab + p * tab;
          double* cum = wn + h;
          double run = 0.0;
          cum[0] = 0.0;
          for (int b = 0; b < h; ++b) {
            wn[b] = __ddiv_rn(load_weight(f, at[p], b, deg, dbin), total);
            run = __dadd_rn(run, wn[b]);
            cum[b + 1] = run;
          }
          cum[h] = 1.0;
        }
      }
    }
    if (KIND == CPB_HISTOGRAM) __syncwarp();
    uint64_t key[10];
    const uint64_t px = (uint64_t)((f.row0 + r) * f.gwidth + c);
    constexpr int per = KIND == CPB_GAUSSIAN ? 2 : 1;
    if (RNG == CPB_RNG_SPLITMIX) {
      const uint64_t pk = pixel_key(a.seed, px);
#pragma unroll
      for (int q = 0; q < 5 * per; ++q) key[q] = plane_key(pk, (uint64_t)q);
    }
    uint32_t cmin = 0, cmax = 0, csad = 0;
    if (kSplit) {
      // Two stages: every pattern needs C against E and W on the same side
      // (min: both less, max: both greater, saddle: either), so a joint
      // draw first samples C, E, W; only the candidates (~half on most
      // vertices) are queued, warp-compacted, and draw N and S 32 at a time.
      // Same samples, same strict comparisons: the counts are unchanged.
      double* qx = q_x + warp * 64;
      double* qu = q_u + warp * 64;
      int64_t* qi = q_i + warp * 64;
      unsigned char* qt = q_t + warp * 64;
      int qh = 0, qn = 0;  // warp-uniform ring head and length
      const uint2 k2 = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
      auto philox_u = [&](int64_t i, int q, double& lo_u, double& hi_u) {
        const uint4 o = philox4x32_10(
            make_uint4((uint32_t)i, (uint32_t)((uint64_t)i >> 32) ^ ((uint32_t)q << 24),
                       (uint32_t)px, (uint32_t)(px >> 32)), k2);
        lo_u = u53_from(o.x, o.y);
        hi_u = u53_from(o.z, o.w);
      };
      auto stage2 = [&](int cnt) {
        if (lane < cnt) {
          const int e = (qh + lane) & 63;
          const int64_t i = qi[e];
          const double x0 = qx[e];
          double u2, u4, unused;
          if (RNG == CPB_RNG_SPLITMIX) {
            u2 = stream_u01(key[2], (uint64_t)i);
            u4 = stream_u01(key[4], (uint64_t)i);
          } else {
            u2 = qu[e];
            philox_u(i, 2, u4, unused);
          }
          const double x2 = draw<KIND>(s[2], u2, 0.0, h), x4 = draw<KIND>(s[4], u4, 0.0, h);
          const bool lns = x0 < x2 && x0 < x4, gns = x0 > x2 && x0 > x4;
          if (qt[e] == 1) {
            cmin += lns;
            csad += gns;
          } else {
            cmax += gns;
            csad += lns;
          }
        }
        qh = (qh + cnt) & 63;
        qn -= cnt;
      };
      for (int64_t base = 0; base < a.n; base += 32) {
        const int64_t i = base + lane;
        int ty = 0;
        double x0 = 0.0, u2 = 0.0;
        if (i < a.n) {
          double u0, u1, u3;
          if (RNG == CPB_RNG_SPLITMIX) {
            u0 = stream_u01(key[0], (uint64_t)i);
            u1 = stream_u01(key[1], (uint64_t)i);
            u3 = stream_u01(key[3], (uint64_t)i);
          } else {
            philox_u(i, 0, u0, u1);
            philox_u(i, 1, u2, u3);
          }
          x0 = draw<KIND>(s[0], u0, 0.0, h);
          const double x1 = draw<KIND>(s[1], u1, 0.0, h), x3 = draw<KIND>(s[3], u3, 0.0, h);
          ty = (x0 < x1 && x0 < x3) ? 1 : ((x0 > x1 && x0 > x3) ? 2 : 0);
        }
        const unsigned m = __ballot_sync(0xffffffffu, ty != 0);
        CPB_ASSERT(qn + __popc(m) <= 64);
        if (ty) {
          const int e = (qh + qn + __popc(m & ((1u << lane) - 1u))) & 63;
          qx[e] = x0;
          qi[e] = i;
          qt[e] = (unsigned char)ty;
          if (RNG != CPB_RNG_SPLITMIX) qu[e] = u2;
        }
        qn += __popc(m);
        __syncwarp();
        if (qn >= 32) {
          stage2(32);
          __syncwarp();
        }
      }
      if (qn > 0) stage2(qn);
      __syncwarp();
    }
    for (int64_t i = kSplit ? a.n : lane; i < a.n; i += 32) {
      double u[10];
      if (RNG == CPB_RNG_SPLITMIX) {
#pragma unroll
        for (int q = 0; q < 5 * per; ++q) u[q] = stream_u01(key[q], (uint64_t)i);
      } else {
        const uint2 k2 = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
#pragma unroll
        for (int q = 0; q < (5 * per + 1) / 2; ++q) {
          const uint4 o = philox4x32_10(
              make_uint4((uint32_t)i, (uint32_t)((uint64_t)i >> 32) ^ ((uint32_t)q << 24),
                         (uint32_t)px, (uint32_t)(px >> 32)), k2);
          u[2 * q] = u53_from(o.x, o.y);
          if (2 * q + 1 < 5 * per) u[2 * q + 1] = u53_from(o.z, o.w);
        }
      }
      double x[5];
#pragma unroll
      for (int p = 0; p < 5; ++p)
        x[p] = draw<KIND>(s[p], u[p * per], per == 2 ? u[p * per + 1] : 0.0, h);
      // strict comparisons, ties count against every pattern (engine.py:213-221)
      const bool lE = x[0] < x[1], lN = x[0] < x[2], lW = x[0] < x[3], lS = x[0] < x[4];
      const bool gE = x[0] > x[1], gN = x[0] > x[2], gW = x[0] > x[3], gS = x[0] > x[4];
      cmin += (lE & lN & lW & lS);
      cmax += (gE & gN & gW & gS);
      csad += ((lE & gN & lW & gS) | (gE & lN & gW & lS));
    }
    cmin = __reduce_add_sync(0xffffffffu, cmin);
    cmax = __reduce_add_sync(0xffffffffu, cmax);
    csad = __reduce_add_sync(0xffffffffu, csad);
    if (lane == 0) {
      const double n = (double)a.n;  // np.mean of booleans: float64 count / n
      if (a.pmin) a.pmin[idx] = __ddiv_rn((double)cmin, n);
      if (a.pmax) a.pmax[idx] = __ddiv_rn((double)cmax, n);
      if (a.psad) a.psad[idx] = __ddiv_rn((double)csad, n);
      if (a.counts) {
        const int64_t plane = f.npix;
        a.counts[idx] = cmin;
        a.counts[plane + idx] = cmax;
        a.counts[2 * plane + idx] = csad;
      }
    }
    if (KIND == CPB_HISTOGRAM) __syncwarp();
  }
}

// Semianalytical estimator (histogram fields only): engine.py:416-459 and the
// grid chunk engine.py:669-683.  c centre draws from the keyed stream (plane 0)
// through the histogram inverse CDF (cum[-1] forced to 1, engine.py:654),
// each neighbour contributes its exact CDF at the draw (histogram_cdf_values,
// distributions.py:92-100, with the plain prefix sums), and the conditional
// pattern probabilities (_conditional_pattern, engine.py:444-459) are averaged.
// One warp per vertex; the draws are summed by warp_strided_sum3, the same
// function the per-case kernel uses (bit-identical grid and per-case results).
__global__ void __launch_bounds__(kMcWarps * 32) semi_kernel(FieldView f, McArgs a) {
  extern __shared__ double s_tab[];  // per warp: 5 x (h wn + h+1 cum) + 1 x (h+1) centre cum
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = f.bins;
  const int tab = 2 * h + 1;
  double* my_tab = s_tab + (size_t)warp * (5 * tab + h + 1);
  double* ccum = my_tab + 5 * tab;  // centre prefix sums with cum[h] = 1 (sampling)
  const int64_t warps_total = (int64_t)gridDim.x * kMcWarps;
  for (int64_t v = (int64_t)blockIdx.x * kMcWarps + warp; v < a.nvert; v += warps_total) {
    const int64_t r = a.row_begin + v / a.cols, c = 1 + v % a.cols;
    const int64_t idx = r * f.width + c;
    const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
    double lo[5], binw[5], ibinw[5];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      double l, hh;
      const bool deg = load_bounds(f, at[p], l, hh);
      lo[p] = l;
      binw[p] = __ddiv_rn(__dsub_rn(hh, l), (double)h);
      ibinw[p] = 1.0 / binw[p];
      if (lane == p) {
        const int dbin = deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at[p]), l, hh, h) : 0;
        const double total = pairwise_sum([&](int b) { return load_weight(f, at[p], b, deg, dbin); }, h);
        double* wn = my_tab + p * tab;
        double* cum = wn + h;
        CPB_ASSERT(p * tab + 2 * h + 1 <= 5 * tab + h + 1);
        double run = 0.0;
        cum[0] = 0.0;
        for (int b = 0; b < h; ++b) {
          wn[b] = __ddiv_rn(load_weight(f, at[p], b, deg, dbin), total);
          run = __dadd_rn(run, wn[b]);
          cum[b + 1] = run;
        }
        if (p == 0) {
          for (int b = 0; b <= h; ++b) ccum[b] = cum[b];
          ccum[h] = 1.0;
        }
      }
    }
    __syncwarp();
    Sampler sc;
    sc.a = lo[0];
    sc.b = binw[0];
    sc.wn = my_tab;
    sc.cum = ccum;
    const uint64_t px = (uint64_t)((f.row0 + r) * f.gwidth + c);
    const uint64_t key = plane_key(pixel_key(a.seed, px), 0);
    auto term = [&](int64_t i, double t[3]) {
      const double x = draw<CPB_HISTOGRAM>(sc, stream_u01(key, (uint64_t)i), 0.0, h);
      double F[5];
#pragma unroll
      for (int p = 1; p < 5; ++p)
        F[p] = hist_cdf_fast(my_tab + p * tab, my_tab + p * tab + h, lo[p], binw[p], ibinw[p], h, x);
      semi_terms4(F, t);
    };
    double sum[3];
    warp_strided_sum3(term, a.n, lane, sum);
    if (lane == 0) {
      const double n = (double)a.n;
      if (a.pmin) a.pmin[idx] = __ddiv_rn(sum[0], n);
      if (a.pmax) a.pmax[idx] = __ddiv_rn(sum[1], n);
      if (a.psad) a.psad[idx] = __ddiv_rn(sum[2], n);
    }
    __syncwarp();
  }
}

__global__ void unit_block_kernel(uint64_t seed, const uint64_t* px, int64_t npix, int planes,
                                  int64_t start, int64_t n, double* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = npix * planes * n;
  if (t >= total) return;
  const int64_t i = t % n, q = (t / n) % planes, p = t / (n * planes);
  const uint64_t key = plane_key(pixel_key(seed, px[p]), (uint64_t)q);
  out[t] = stream_u01(key, (uint64_t)(start + i));
}

}  // namespace

int launch_mc(const cpb_field* fld, int64_t row_begin, int64_t row_end, uint64_t seed, int64_t n,
              int rng, double* pmin, double* pmax, double* psad, int64_t* counts, cudaStream_t st) {
  const FieldView f = make_view(*fld);
  const int64_t rows = row_end - row_begin;
  if (rows <= 0 || f.width < 3) return CPB_OK;
  if (n < 1) {
    set_error("sample counts must be positive");
    return CPB_EINVAL;
  }
  // per-vertex hit counts are uint32 (summed across the warp by __reduce_add_sync)
  if (n > 0xffffffffll) {
    set_error("n_samples too large (at most 2^32 - 1 per vertex)");
    return CPB_EINVAL;
  }
  McArgs a;
  a.row_begin = row_begin;
  a.cols = f.width - 2;
  a.nvert = rows * a.cols;
  a.seed = seed;
  a.n = n;
  a.pmin = pmin;
  a.pmax = pmax;
  a.psad = psad;
  a.counts = counts;
  const size_t smem = f.kind == CPB_HISTOGRAM ? (size_t)kMcWarps * 5 * (2 * f.bins + 1) * sizeof(double) : 0;
  if (smem > 200 * 1024) {
    set_error("too many histogram bins for the Monte Carlo sampler tables");
    return CPB_EINVAL;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (a.nvert + kMcWarps - 1) / kMcWarps;
  const unsigned grid = (unsigned)(want < (int64_t)sms * 64 ? want : (int64_t)sms * 64);
#define CPB_MC_LAUNCH(K, R)                                                                  \
  do {                                                                                       \
    auto kern = mc_kernel<K, R>;                                                             \
    if (smem > 48 * 1024)                                                                    \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    kern<<<grid, kMcWarps * 32, smem, st>>>(f, a);                                           \
  } while (0)
#define CPB_MC_KIND(K)                                                                       \
  case K:                                                                                    \
    if (rng == CPB_RNG_PHILOX) CPB_MC_LAUNCH(K, CPB_RNG_PHILOX);                             \
    else CPB_MC_LAUNCH(K, CPB_RNG_SPLITMIX);                                                 \
    break;
  switch (f.kind) {
    CPB_MC_KIND(CPB_UNIFORM)
    CPB_MC_KIND(CPB_EPANECHNIKOV)
    CPB_MC_KIND(CPB_HISTOGRAM)
    CPB_MC_KIND(CPB_GAUSSIAN)
    default:
      set_error("unknown model kind %d", f.kind);
      return CPB_EINVAL;
  }
#undef CPB_MC_KIND
#undef CPB_MC_LAUNCH
  CPB_CHECK_LAUNCH("monte carlo kernel");
  return CPB_OK;
}

int launch_semi(const cpb_field* fld, int64_t row_begin, int64_t row_end, uint64_t seed, int64_t c,
                double* pmin, double* pmax, double* psad, cudaStream_t st) {
  const FieldView f = make_view(*fld);
  const int64_t rows = row_end - row_begin;
  if (rows <= 0 || f.width < 3) return CPB_OK;
  if (f.kind != CPB_HISTOGRAM) {
    set_error("semianalytical estimation is defined for histogram fields only");
    return CPB_EINVAL;
  }
  if (c < 1) {
    set_error("sample counts must be positive");
    return CPB_EINVAL;
  }
  McArgs a;
  a.row_begin = row_begin;
  a.cols = f.width - 2;
  a.nvert = rows * a.cols;
  a.seed = seed;
  a.n = c;
  a.pmin = pmin;
  a.pmax = pmax;
  a.psad = psad;
  a.counts = nullptr;
  const size_t smem = (size_t)kMcWarps * (5 * (2 * f.bins + 1) + f.bins + 1) * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("too many histogram bins for the semianalytical tables");
    return CPB_EINVAL;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (a.nvert + kMcWarps - 1) / kMcWarps;
  const unsigned grid = (unsigned)(want < (int64_t)sms * 64 ? want : (int64_t)sms * 64);
  if (smem > 48 * 1024) cudaFuncSetAttribute(semi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  semi_kernel<<<grid, kMcWarps * 32, smem, st>>>(f, a);
  CPB_CHECK_LAUNCH("semianalytical kernel");
  return CPB_OK;
}

int launch_unit_block(uint64_t seed, const uint64_t* px, int64_t npix, int planes, int64_t start,
                      int64_t n, double* out, cudaStream_t st) {
  const int64_t total = npix * planes * n;
  if (total == 0) return CPB_OK;
  unit_block_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(seed, px, npix, planes, start, n, out);
  CPB_CHECK_LAUNCH("unit_block kernel");
  return CPB_OK;
}

}  // namespace cpb
