// Batched per-case estimators: many independent neighbourhoods per launch.
//
// Reference: the single-case API of engine.py -- NeighborhoodCase (50-71),
// local_min_prob / local_max_prob / saddle_prob / closed_form_triple
// (127-178), mc_all_patterns (238-247, draws from _case_draws 225-235),
// semianalytical_prob (416-459) and the combinatorial terms (270-404) -- which
// the reference evaluates one case at a time in Python (validate_random_cases,
// bench.py:235-267; acceptance #2, test_acceptance.py:75-97: 1500 cases x
// 1e6 joint draws).  Here a batch is n_cases x (1 + k) distributions
// (k = 2 or 4 neighbours) of arbitrary, possibly mixed kinds, laid out as
// flat device arrays (cpb_case_batch).
//
// Closed form.  The reference multiplies piecewise polynomials on the union
// of all breakpoints and integrates each piece exactly (refine_and_multiply,
// piecewise.py:200-234).  One thread per case walks the same union here as a
// k+1-way merge of the distributions' sorted breakpoints (support ends, or
// histogram bin edges lo + (hi - lo) j / h as in pdf_poly,
// distributions.py:156-162), keeping per distribution the index of its next
// breakpoint and, for histograms, the running CDF at the current bin start;
// on a piece every factor is then one polynomial and Gauss-Legendre
// quadrature with 3 nodes (degree <= 4: uniform / histogram) or 8 nodes
// (degree <= 14: any Epanechnikov factor) integrates it exactly.  All four
// integrals (min, max, saddle halves) share the walk over the centre support:
// outside an integral's range one factor is an exact 0 (a neighbour below its
// support has CDF 0, above it survival 0), so no range bookkeeping is needed.
//
// Monte Carlo.  The draws are the reference's: plane q of case i is keyed by
// (seed, pixel_i, q) with planes assigned in position order (a Gaussian
// takes two), each transformed by the same inverse CDF as the grid path
// (cpb_sample.cuh); counts are integers, so the split of the n draws over
// blocks and the atomic accumulation are exact and the probabilities are
// bit-identical to mc_all_patterns for uniform / histogram kinds.
#include <stdlib.h>

#include "cpb_common.cuh"
#include "cpb_sample.cuh"

namespace cpb {

int workspace_alloc(void** p, size_t bytes, cudaStream_t st);
void workspace_free(void* p, cudaStream_t st);

namespace {

constexpr int kMaxPos = 5;
constexpr int kCaseThreads = 128;     // closed form: one case per thread
constexpr int kMcThreads = 256;       // Monte Carlo: one (case, sample chunk) per block
constexpr int kMcPerThread = 32;      // draws per thread per block
constexpr int kCombThreads = 256;     // combinatorial / semianalytical: one case per block
constexpr int kCombMaxBins = 8;       // COMBINATORIAL_MAX_BINS, engine.py:44

struct Batch {
  int64_t n;
  int k;   // neighbours
  int maxb;
  const int32_t* kind;
  const double* a;
  const double* b;
  const int32_t* bins;
  const int64_t* woff;
  const double* w;
};

Batch make_batch(const cpb_case_batch& c) {
  return Batch{c.n_cases, c.neighbors, c.max_bins, c.kind, c.a, c.b, c.bins, c.woff, c.weights};
}

// ------------------------------------------------------------ closed form
// Walk state of one distribution.
struct Walk {
  int kind, h, nb, j;   // nb breakpoints; j = index of the next one not yet passed
  double lo, hi, span;  // support; span = hi - lo
  double m, ih;         // epanechnikov: mid, 1/halfwidth | uniform: -, 1/(hi - lo)
  double binw, cum;     // histogram: bin width, CDF at the current bin start
  const double* w;      // histogram: bin weights
};

CPB_D double breakpoint(const Walk& d, int j) {
  if (d.kind != CPB_HISTOGRAM) return j == 0 ? d.lo : d.hi;
  // edges = lo + (hi - lo) * arange(h + 1) / h  (distributions.py:158)
  return __dadd_rn(d.lo, __ddiv_rn(__dmul_rn(d.span, (double)j), (double)d.h));
}

CPB_D void pass_through(Walk& d, double x) {
  while (d.j < d.nb && breakpoint(d, d.j) <= x) {
    if (d.kind == CPB_HISTOGRAM && d.j >= 1) d.cum = __dadd_rn(d.cum, d.w[d.j - 1]);
    ++d.j;
  }
}

// CDF of a neighbour at x inside the current piece.
CPB_D double walk_cdf(const Walk& d, double x) {
  if (d.j == 0) return 0.0;
  if (d.j >= d.nb) return 1.0;
  if (d.kind == CPB_UNIFORM) return (x - d.lo) * d.ih;
  if (d.kind == CPB_EPANECHNIKOV) {
    const double u = fmin(fmax((x - d.m) * d.ih, -1.0), 1.0);
    return fma(u, fma(-0.25, u * u, 0.75), 0.5);
  }
  const int bin = d.j - 1;
  return d.cum + d.w[bin] * ((x - breakpoint(d, bin)) / d.binw);
}

// Density of the centre at x inside the current piece.
CPB_D double walk_pdf(const Walk& d, double x) {
  if (d.kind == CPB_UNIFORM) return d.ih;
  if (d.kind == CPB_EPANECHNIKOV) {
    const double u = (x - d.m) * d.ih;
    return 0.75 * d.ih * (1.0 - u * u);
  }
  return d.w[d.j - 1] / d.binw;
}

CPB_D void init_walk(const Batch& B, int64_t di, Walk& d) {
  d.kind = B.kind[di];
  d.lo = B.a[di];
  d.hi = B.b[di];
  d.span = d.hi - d.lo;
  d.j = 0;
  d.cum = 0.0;
  d.w = nullptr;
  d.h = 1;
  d.nb = 2;
  d.m = 0.5 * (d.lo + d.hi);
  d.ih = d.kind == CPB_EPANECHNIKOV ? 1.0 / (0.5 * d.span) : 1.0 / d.span;
  d.binw = d.span;
  if (d.kind == CPB_HISTOGRAM) {
    d.h = B.bins[di];
    d.nb = d.h + 1;
    d.w = B.w + B.woff[di];
    d.binw = d.span / (double)d.h;
  }
}

// g[0..3] = min, max, saddle t1, saddle t2 integrands (without the centre pdf).
CPB_D void case_integrands(const double* F, int k, double g[4]) {
  if (k == 2) {
    const double sa = 1.0 - F[1], sb = 1.0 - F[2];
    g[0] = sa * sb;
    g[1] = F[1] * F[2];
    g[2] = sa * F[2];  // below the first neighbour, above the second (engine.py:149-152)
    g[3] = F[1] * sb;  // its mirror (the negated case)
    return;
  }
  const double sE = 1.0 - F[1], sN = 1.0 - F[2], sW = 1.0 - F[3], sS = 1.0 - F[4];
  g[0] = (sE * sN) * (sW * sS);
  g[1] = (F[1] * F[2]) * (F[3] * F[4]);
  g[2] = (sE * sW) * (F[2] * F[4]);  // below E, W and above N, S (engine.py:152-153)
  g[3] = (sN * sS) * (F[1] * F[3]);
}

// Integrand values at x: g[r] = pdf_C(x) * factors_r(x) when WITH_PDF, else
// the factors only (a piecewise-constant centre density is applied per piece).
template <bool WITH_PDF>
CPB_D void node_values(Walk* d, int P, double x, double g[4]) {
  double F[kMaxPos];
  for (int p = 1; p < P; ++p) F[p] = walk_cdf(d[p], x);
  case_integrands(F, P - 1, g);
  if (WITH_PDF) {
    const double pdf = walk_pdf(d[0], x);
#pragma unroll
    for (int r = 0; r < 4; ++r) g[r] *= pdf;
  }
}

// GL sums over symmetric node pairs: s = w_0 g(mid) [odd n] + sum_j w_j (g(mid - t_j)
// + g(mid + t_j)).  For a constant integrand this is exactly 2 g (the pair
// weights of leggauss(3) and leggauss(8) add to exactly 2 in this order), so
// certain / impossible patterns come out as exactly 1 and 0, as the
// reference's exact polynomial integration gives them (test_engine.py:114-143).
template <class GL>
CPB_D void walk_integrals(Walk* d, int P, double acc[4]) {
  for (int r = 0; r < 4; ++r) acc[r] = 0.0;
  const double hiC = d[0].hi;
  double x0 = d[0].lo;
  for (int p = 0; p < P; ++p) pass_through(d[p], x0);
  const bool pdf_const = d[0].kind != CPB_EPANECHNIKOV;
  int guard = 0;
  while (x0 < hiC && guard++ < 1 << 20) {
    double x1 = hiC;
    for (int p = 0; p < P; ++p)
      if (d[p].j < d[p].nb) x1 = fmin(x1, breakpoint(d[p], d[p].j));
    if (x1 > x0) {
      const double half = 0.5 * (x1 - x0), mid = 0.5 * (x1 + x0);
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      if (GL::n % 2 == 1) {  // centre node
        double g[4];
        if (pdf_const) node_values<false>(d, P, mid, g);
        else node_values<true>(d, P, mid, g);
#pragma unroll
        for (int r = 0; r < 4; ++r) s[r] = GL::w(GL::n / 2) * g[r];
      }
#pragma unroll
      for (int j = 0; j < GL::n / 2; ++j) {
        const double t = half * GL::x(GL::n - 1 - j);  // positive node
        double gm[4], gp[4];
        if (pdf_const) {
          node_values<false>(d, P, mid - t, gm);
          node_values<false>(d, P, mid + t, gp);
        } else {
          node_values<true>(d, P, mid - t, gm);
          node_values<true>(d, P, mid + t, gp);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) s[r] = fma(GL::w(GL::n - 1 - j), gm[r] + gp[r], s[r]);
      }
      const double scale = pdf_const ? half * walk_pdf(d[0], mid) : half;
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fma(scale, s[r], acc[r]);
    } else {
      x1 = x0;
    }
    x0 = x1;
    for (int p = 0; p < P; ++p) pass_through(d[p], x0);
  }
}

__global__ void __launch_bounds__(kCaseThreads) cases_closed_kernel(Batch B, double* out) {
  const int64_t c = (int64_t)blockIdx.x * kCaseThreads + threadIdx.x;
  if (c >= B.n) return;
  const int P = B.k + 1;
  Walk d[kMaxPos];
  bool epan = false, bounded = true;
  for (int p = 0; p < P; ++p) {
    init_walk(B, c * P + p, d[p]);
    epan |= d[p].kind == CPB_EPANECHNIKOV;
    bounded &= d[p].kind != CPB_GAUSSIAN;
  }
  double acc[4];
  if (!bounded) {
    acc[0] = acc[1] = acc[2] = acc[3] = __longlong_as_double(0x7ff8000000000000ll);
  } else if (epan) {
    walk_integrals<GL8>(d, P, acc);
  } else {
    walk_integrals<GL3>(d, P, acc);
  }
  out[3 * c + 0] = acc[0];
  out[3 * c + 1] = acc[1];
  out[3 * c + 2] = acc[2] + acc[3];
}

// ------------------------------------------------------------ Monte Carlo
struct PosTab {
  int kind, h, plane;
  Sampler s;
};

// Loads the samplers of case c into shared memory (thread p handles position
// p): histogram weights as stored (FiniteDistribution keeps w / w.sum()) and
// the prefix sums with cum[h] forced to 1 (sample_u01, distributions.py:223-226).
CPB_D void load_samplers(const Batch& B, int64_t c, PosTab* pt, double* tab, int tabw,
                         bool force_last) {
  const int P = B.k + 1;
  const int p = threadIdx.x;
  if (p < P) {
    const int64_t di = c * P + p;
    PosTab t;
    t.kind = B.kind[di];
    t.h = t.kind == CPB_HISTOGRAM ? B.bins[di] : 1;
    const double lo = B.a[di], hi = B.b[di];
    if (t.kind == CPB_EPANECHNIKOV) {
      t.s.a = __dmul_rn(0.5, __dadd_rn(lo, hi));
      t.s.b = __dmul_rn(0.5, __dsub_rn(hi, lo));
    } else if (t.kind == CPB_HISTOGRAM) {
      t.s.a = lo;
      t.s.b = __ddiv_rn(__dsub_rn(hi, lo), (double)t.h);
    } else {
      t.s.a = lo;
      t.s.b = hi;
    }
    t.s.wn = tab + p * tabw;
    t.s.cum = tab + p * tabw + t.h;
    if (t.kind == CPB_HISTOGRAM) {
      CPB_ASSERT(t.h >= 1 && 2 * t.h + 1 <= tabw);
      const double* w = B.w + B.woff[di];
      double* wn = tab + p * tabw;
      double* cum = wn + t.h;
      double run = 0.0;
      cum[0] = 0.0;
      for (int q = 0; q < t.h; ++q) {
        wn[q] = w[q];
        run = __dadd_rn(run, w[q]);
        cum[q + 1] = run;
      }
      if (force_last) cum[t.h] = 1.0;
    }
    pt[p] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // plane offsets in position order (_case_draws, engine.py:225-235)
    int q = 0;
    for (int i = 0; i < P; ++i) {
      pt[i].plane = q;
      q += pt[i].kind == CPB_GAUSSIAN ? 2 : 1;
    }
  }
  __syncthreads();
}

CPB_D double draw_any(const PosTab& t, double u, double u2) {
  switch (t.kind) {
    case CPB_UNIFORM: return draw<CPB_UNIFORM>(t.s, u, u2, 1);
    case CPB_EPANECHNIKOV: return draw<CPB_EPANECHNIKOV>(t.s, u, u2, 1);
    case CPB_GAUSSIAN: return draw<CPB_GAUSSIAN>(t.s, u, u2, 1);
    default: return draw<CPB_HISTOGRAM>(t.s, u, u2, t.h);
  }
}

template <int KIND>
CPB_D double draw_k(const PosTab& t, double u, double u2) {
  if (KIND < 0) return draw_any(t, u, u2);
  return draw<KIND < 0 ? 0 : KIND>(t.s, u, u2, KIND == CPB_HISTOGRAM ? t.h : 1);
}

// The sample loop for P positions (compile time) whose kinds are all KIND
// (or mixed, KIND = -1): everything per position lives in registers.
template <int P, int KIND>
CPB_D void mc_loop(const PosTab (&t)[P], const uint64_t (&key)[2 * P], int64_t base, int64_t n,
                   uint32_t& cmin, uint32_t& cmax, uint32_t& csad) {
#pragma unroll 2
  for (int r = 0; r < kMcPerThread; ++r) {
    const int64_t i = base + (int64_t)r * kMcThreads + threadIdx.x;
    if (i >= n) break;
    double x[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const double u = stream_u01(key[2 * p], (uint64_t)i);
      const bool gauss = KIND == CPB_GAUSSIAN || (KIND < 0 && t[p].kind == CPB_GAUSSIAN);
      const double u2 = gauss ? stream_u01(key[2 * p + 1], (uint64_t)i) : 0.0;
      x[p] = draw_k<KIND>(t[p], u, u2);
    }
    // strict comparisons, ties count against every pattern (_pattern_stats, engine.py:195-222)
    if (P == 3) {
      const bool la = x[0] < x[1], lb = x[0] < x[2 % P], ga = x[0] > x[1], gb = x[0] > x[2 % P];
      cmin += la & lb;
      cmax += ga & gb;
      csad += (la & gb) | (ga & lb);
    } else {
      const bool lE = x[0] < x[1], lN = x[0] < x[2 % P], lW = x[0] < x[3 % P], lS = x[0] < x[4 % P];
      const bool gE = x[0] > x[1], gN = x[0] > x[2 % P], gW = x[0] > x[3 % P], gS = x[0] > x[4 % P];
      cmin += lE & lN & lW & lS;
      cmax += gE & gN & gW & gS;
      csad += (lE & gN & lW & gS) | (gE & lN & gW & lS);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kMcThreads) cases_mc_kernel(Batch B, uint64_t seed,
                                                              const uint64_t* pixels, int64_t n,
                                                              int64_t chunks,
                                                              unsigned long long* counts) {
  constexpr int P = K + 1;
  extern __shared__ double s_tab[];
  __shared__ PosTab pt[kMaxPos];
  __shared__ uint32_t red[3][kMcThreads / 32];
  const int64_t c = (int64_t)blockIdx.x / chunks;
  const int64_t chunk = (int64_t)blockIdx.x % chunks;
  const int tabw = 2 * B.maxb + 1;
  load_samplers(B, c, pt, s_tab, tabw, true);
  const uint64_t px = pixels ? pixels[c] : (uint64_t)c;
  const uint64_t pk = pixel_key(seed, px);
  PosTab t[P];
  uint64_t key[2 * P];
  bool same = true;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    t[p] = pt[p];
    key[2 * p] = plane_key(pk, (uint64_t)t[p].plane);
    key[2 * p + 1] = plane_key(pk, (uint64_t)t[p].plane + 1);
    same &= t[p].kind == t[0].kind;
  }
  uint32_t cmin = 0, cmax = 0, csad = 0;
  const int64_t base = chunk * (int64_t)kMcThreads * kMcPerThread;
  switch (same ? t[0].kind : -1) {
    case CPB_UNIFORM: mc_loop<P, CPB_UNIFORM>(t, key, base, n, cmin, cmax, csad); break;
    case CPB_EPANECHNIKOV: mc_loop<P, CPB_EPANECHNIKOV>(t, key, base, n, cmin, cmax, csad); break;
    case CPB_HISTOGRAM: mc_loop<P, CPB_HISTOGRAM>(t, key, base, n, cmin, cmax, csad); break;
    case CPB_GAUSSIAN: mc_loop<P, CPB_GAUSSIAN>(t, key, base, n, cmin, cmax, csad); break;
    default: mc_loop<P, -1>(t, key, base, n, cmin, cmax, csad); break;
  }
  cmin = __reduce_add_sync(0xffffffffu, cmin);
  cmax = __reduce_add_sync(0xffffffffu, cmax);
  csad = __reduce_add_sync(0xffffffffu, csad);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][warp] = cmin;
    red[1][warp] = cmax;
    red[2][warp] = csad;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    unsigned long long sum = 0;
    for (int q = 0; q < kMcThreads / 32; ++q) sum += red[threadIdx.x][q];
    if (sum) atomicAdd(counts + 3 * c + threadIdx.x, sum);
  }
}

__global__ void cases_finish_kernel(const unsigned long long* counts, int64_t ncases, int64_t n,
                                    double* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * ncases) return;
  out[t] = __ddiv_rn((double)counts[t], (double)n);  // np.mean of booleans
}

// -------------------------------------------------------- semianalytical
// histogram cases only: c centre draws (plane 0), each neighbour's exact CDF
// at the draw from the plain prefix sums (_hist_arrays, engine.py:407-413),
// the conditional patterns of _conditional_pattern (engine.py:444-459)
// averaged.  One warp per case: the draws are summed by warp_strided_sum3,
// the function the grid kernel (semi_kernel) uses, so a grid vertex and the
// same neighbourhood as a case agree bitwise (test_engine.py:574-582).
constexpr int kSemiThreads = 32;
__global__ void __launch_bounds__(kSemiThreads) cases_semi_kernel(Batch B, uint64_t seed,
                                                                  const uint64_t* pixels, int64_t cnt,
                                                                  double* out) {
  extern __shared__ double s_tab[];
  __shared__ PosTab pt[kMaxPos];
  const int64_t c = blockIdx.x;
  const int lane = threadIdx.x;
  const int P = B.k + 1;
  const int tabw = 2 * B.maxb + 1;
  double* ccum = s_tab + kMaxPos * tabw;  // centre prefix sums with cum[h] = 1
  load_samplers(B, c, pt, s_tab, tabw, false);
  if (threadIdx.x == 0) {
    for (int q = 0; q <= pt[0].h; ++q) ccum[q] = pt[0].s.cum[q];
    ccum[pt[0].h] = 1.0;
  }
  __syncthreads();
  bool hist = true;
  for (int p = 0; p < P; ++p) hist &= pt[p].kind == CPB_HISTOGRAM;
  Sampler sc = pt[0].s;
  sc.cum = ccum;
  const uint64_t px = pixels ? pixels[c] : (uint64_t)c;
  const uint64_t key = plane_key(pixel_key(seed, px), 0);
  double ib[kMaxPos];
  for (int p = 0; p < P; ++p) ib[p] = 1.0 / pt[p].s.b;
  auto term = [&](int64_t i, double t[3]) {
    const double x = draw<CPB_HISTOGRAM>(sc, stream_u01(key, (uint64_t)i), 0.0, pt[0].h);
    double F[kMaxPos];
    for (int p = 1; p < P; ++p)
      F[p] = hist_cdf_fast(pt[p].s.wn, pt[p].s.cum, pt[p].s.a, pt[p].s.b, ib[p], pt[p].h, x);
    if (P == 3)
      semi_terms2(F, t);
    else
      semi_terms4(F, t);
  };
  double sum[3] = {0.0, 0.0, 0.0};
  if (hist) warp_strided_sum3(term, cnt, lane, sum);
  if (lane < 3) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    out[3 * c + lane] = hist ? __ddiv_rn(sum[lane], (double)cnt) : nan;
  }
}

// --------------------------------------------------------- combinatorial
// Eq. 5 for histogram cases (engine.py:320-404): the sum over every
// combination of one bin per position of (product of the bin masses) x (the
// all-uniform probability with each position uniform on its bin, edges of
// _histogram_grid, engine.py:313-317).  One block per case; threads take
// combinations (itertools.product order, centre slowest), each all-uniform
// term comes from the same breakpoint walk, and a fixed block tree adds the
// partial sums (deterministic; re-associates the reference's running sum).
__global__ void __launch_bounds__(kCombThreads) cases_comb_kernel(Batch B, double* out) {
  __shared__ double red[3][kCombThreads];
  const int64_t c = blockIdx.x;
  const int P = B.k + 1;
  int h[kMaxPos];
  const double* wts[kMaxPos];
  double lo[kMaxPos], span[kMaxPos];
  bool hist = true;
  int64_t ncomb = 1;
  for (int p = 0; p < P; ++p) {
    const int64_t di = c * P + p;
    hist &= B.kind[di] == CPB_HISTOGRAM;
    h[p] = hist ? B.bins[di] : 1;
    wts[p] = hist ? B.w + B.woff[di] : nullptr;
    lo[p] = B.a[di];
    span[p] = B.b[di] - B.a[di];
    ncomb *= h[p];
  }
  double smin = 0.0, smax = 0.0, ssad = 0.0;
  for (int64_t q = threadIdx.x; hist && q < ncomb; q += kCombThreads) {
    int64_t rest = q;
    int ib[kMaxPos];
    for (int p = P - 1; p >= 0; --p) {
      ib[p] = (int)(rest % h[p]);
      rest /= h[p];
    }
    double wprod = 1.0;
    for (int p = 0; p < P; ++p) wprod *= wts[p][ib[p]];
    if (wprod == 0.0) continue;
    Walk d[kMaxPos];
    for (int p = 0; p < P; ++p) {
      const double e0 = lo[p] + (span[p] * (double)ib[p]) / (double)h[p];
      const double e1 = lo[p] + (span[p] * (double)(ib[p] + 1)) / (double)h[p];
      d[p].kind = CPB_UNIFORM;
      d[p].h = 1;
      d[p].nb = 2;
      d[p].j = 0;
      d[p].lo = e0;
      d[p].hi = e1;
      d[p].span = e1 - e0;
      d[p].ih = 1.0 / d[p].span;
      d[p].m = 0.5 * (e0 + e1);
      d[p].binw = d[p].span;
      d[p].cum = 0.0;
      d[p].w = nullptr;
    }
    double acc[4];
    walk_integrals<GL3>(d, P, acc);
    smin = fma(wprod, acc[0], smin);
    smax = fma(wprod, acc[1], smax);
    ssad = fma(wprod, acc[2] + acc[3], ssad);
  }
  red[0][threadIdx.x] = smin;
  red[1][threadIdx.x] = smax;
  red[2][threadIdx.x] = ssad;
  __syncthreads();
  for (int s = kCombThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int r = 0; r < 3; ++r) red[r][threadIdx.x] += red[r][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 3) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    out[3 * c + threadIdx.x] = hist ? red[threadIdx.x][0] : nan;
  }
}

int check_batch(const cpb_case_batch* b, double* out) {
  if (!b || !out) {
    set_error("case batch and output must not be NULL");
    return CPB_EINVAL;
  }
  if (b->neighbors != 2 && b->neighbors != 4) {
    set_error("a neighborhood has exactly 2 or 4 neighbors");
    return CPB_EINVAL;
  }
  if (b->n_cases < 0 || b->max_bins < 1 || b->max_bins > 4096) {
    set_error("n_cases must be >= 0 and max_bins in [1, 4096]");
    return CPB_EINVAL;
  }
  if (b->n_cases > 0 && (!b->kind || !b->a || !b->b || !b->bins || !b->woff || !b->weights)) {
    set_error("case batch arrays must not be NULL");
    return CPB_EINVAL;
  }
  return CPB_OK;
}

}  // namespace

int launch_cases_closed(const cpb_case_batch* b, double* out, cudaStream_t st) {
  if (int s = check_batch(b, out)) return s;
  if (b->n_cases == 0) return CPB_OK;
  const Batch B = make_batch(*b);
  cases_closed_kernel<<<(unsigned)((B.n + kCaseThreads - 1) / kCaseThreads), kCaseThreads, 0, st>>>(B, out);
  CPB_CHECK_LAUNCH("per-case closed-form kernel");
  return CPB_OK;
}

int launch_cases_mc(const cpb_case_batch* b, uint64_t seed, const uint64_t* pixels, int64_t n,
                    unsigned long long* counts, double* out, cudaStream_t st) {
  if (int s = check_batch(b, out)) return s;
  if (n < 1) {
    set_error("n must be positive");
    return CPB_EINVAL;
  }
  if (b->n_cases == 0) return CPB_OK;
  const Batch B = make_batch(*b);
  const int64_t per_block = (int64_t)kMcThreads * kMcPerThread;
  const int64_t chunks = (n + per_block - 1) / per_block;
  if (chunks * B.n > 0x7fffffffll) {
    set_error("n_cases * n too large for one launch");
    return CPB_EINVAL;
  }
  const size_t smem = (size_t)kMaxPos * (2 * B.maxb + 1) * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("too many histogram bins (%d) for the per-case sampler tables", B.maxb);
    return CPB_EINVAL;
  }
  // caller-provided counts, or stream-ordered scratch from the library pool
  struct Scratch {
    unsigned long long* p = nullptr;
    cudaStream_t st;
    ~Scratch() { workspace_free(p, st); }
  } scratch{nullptr, st};
  unsigned long long* cnt = counts;
  if (!cnt) {
    if (int s = workspace_alloc((void**)&scratch.p, (size_t)B.n * 3 * sizeof(unsigned long long), st)) return s;
    cnt = scratch.p;
  }
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)B.n * 3 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_status(e, "memset counts");
  auto kern = B.k == 2 ? cases_mc_kernel<2> : cases_mc_kernel<4>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)(chunks * B.n), kMcThreads, smem, st>>>(B, seed, pixels, n, chunks, cnt);
  CPB_CHECK_LAUNCH("per-case Monte Carlo kernel");
  cases_finish_kernel<<<(unsigned)((3 * B.n + 255) / 256), 256, 0, st>>>(cnt, B.n, n, out);
  CPB_CHECK_LAUNCH("per-case Monte Carlo finish");
  return CPB_OK;
}

int launch_cases_semi(const cpb_case_batch* b, uint64_t seed, const uint64_t* pixels, int64_t c,
                      double* out, cudaStream_t st) {
  if (int s = check_batch(b, out)) return s;
  if (c < 1) {
    set_error("c must be positive");
    return CPB_EINVAL;
  }
  if (b->n_cases == 0) return CPB_OK;
  const Batch B = make_batch(*b);
  const size_t smem = ((size_t)kMaxPos * (2 * B.maxb + 1) + B.maxb + 1) * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("too many histogram bins (%d) for the per-case semianalytical tables", B.maxb);
    return CPB_EINVAL;
  }
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(cases_semi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cases_semi_kernel<<<(unsigned)B.n, kSemiThreads, smem, st>>>(B, seed, pixels, c, out);
  CPB_CHECK_LAUNCH("per-case semianalytical kernel");
  return CPB_OK;
}

int launch_cases_combinatorial(const cpb_case_batch* b, double* out, cudaStream_t st) {
  if (int s = check_batch(b, out)) return s;
  if (b->max_bins > kCombMaxBins) {
    set_error("combinatorial cost grows as bins**%d; refusing more than %d bins",
              b->neighbors + 1, kCombMaxBins);
    return CPB_EINVAL;
  }
  if (b->n_cases == 0) return CPB_OK;
  const Batch B = make_batch(*b);
  cases_comb_kernel<<<(unsigned)B.n, kCombThreads, 0, st>>>(B, out);
  CPB_CHECK_LAUNCH("per-case combinatorial kernel");
  return CPB_OK;
}

}  // namespace cpb
