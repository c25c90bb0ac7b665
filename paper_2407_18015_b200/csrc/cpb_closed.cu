// Closed-form min / max / saddle probabilities: the four-neighbour stencil.
//
// Reference: engine.py:580-629 (_product_integral, _closed_chunk), the node
// evaluators engine.py:508-561 and breakpoints engine.py:564-577, driven by
// classify_field engine.py:716-787.
//
// Per vertex the reference integrates pdf_C * prod(F or 1-F) over four ranges
// with Gauss-Legendre quadrature on the partition given by all support (or
// bin) edges clipped to the range.  Every range endpoint is itself an edge
// and every range lies inside the centre support, so the partition of
// [lo_C, hi_C] by all edges, restricted to a range, IS the reference's
// partition of that range.  The kernel therefore sorts / merges the edges
// once, evaluates the four neighbour CDFs once per node, and feeds all four
// integrals (min, max, saddle t1, saddle t2) from the shared node values,
// adding a piece's contribution to the integrals whose range contains it.
//
// Arithmetic is float64 throughout (closed-form parity bar: 1e-12 absolute,
// the reference's own grid-vs-case tolerance, test_engine.py:548-559).
#include "cpb_common.cuh"

namespace cpb {
namespace {

constexpr int kClosedThreads = 128;
enum { C_ = 0, E_ = 1, N_ = 2, W_ = 3, S_ = 4 };

CPB_D double dmin(double a, double b) { return a < b ? a : b; }
CPB_D double dmax(double a, double b) { return a > b ? a : b; }
CPB_D double clamp01(double x) { return dmin(dmax(x, 0.0), 1.0); }
CPB_D void cswap(double& a, double& b) {
  const double lo = dmin(a, b), hi = dmax(a, b);
  a = lo;
  b = hi;
}

// Batcher merge of four sorted (lo, hi) pairs: 15 compare-exchanges.
CPB_D void merge_pairs8(double* k) {
  cswap(k[0], k[2]); cswap(k[1], k[3]); cswap(k[1], k[2]);
  cswap(k[4], k[6]); cswap(k[5], k[7]); cswap(k[5], k[6]);
  cswap(k[0], k[4]); cswap(k[1], k[5]); cswap(k[2], k[6]); cswap(k[3], k[7]);
  cswap(k[2], k[4]); cswap(k[3], k[5]);
  cswap(k[1], k[2]); cswap(k[3], k[4]); cswap(k[5], k[6]);
}

// Ranges of the four integrals (engine.py:603-628):
//   min : [lo_C, min(all hi)]                         factors S_E S_N S_W S_S
//   max : [max(all lo), hi_C]                         factors F_E F_N F_W F_S
//   t1  : [max(lo_C, lo_N, lo_S), min(hi_C, hi_E, hi_W)]  S_E S_W F_N F_S
//   t2  : [max(lo_C, lo_E, lo_W), min(hi_C, hi_N, hi_S)]  S_N S_S F_E F_W
struct Ranges {
  double lo[4], hi[4];
};
CPB_D Ranges make_ranges(const double* lo, const double* hi) {
  Ranges r;
  r.lo[0] = lo[C_];
  r.hi[0] = dmin(dmin(dmin(hi[C_], hi[E_]), dmin(hi[N_], hi[W_])), hi[S_]);
  r.lo[1] = dmax(dmax(dmax(lo[C_], lo[E_]), dmax(lo[N_], lo[W_])), lo[S_]);
  r.hi[1] = hi[C_];
  r.lo[2] = dmax(dmax(lo[C_], lo[N_]), lo[S_]);
  r.hi[2] = dmin(dmin(hi[C_], hi[E_]), hi[W_]);
  r.lo[3] = dmax(dmax(lo[C_], lo[E_]), lo[W_]);
  r.hi[3] = dmin(dmin(hi[C_], hi[N_]), hi[S_]);
  return r;
}

// The four integrands from the neighbour CDF values at one node.
CPB_D void integrands(const double* F, double g[4]) {
  const double sE = 1.0 - F[E_], sN = 1.0 - F[N_], sW = 1.0 - F[W_], sS = 1.0 - F[S_];
  const double sesw = sE * sW, snss = sN * sS;
  const double fefw = F[E_] * F[W_], fnfs = F[N_] * F[S_];
  g[0] = sesw * snss;
  g[1] = fefw * fnfs;
  g[2] = sesw * fnfs;
  g[3] = snss * fefw;
}

CPB_D void store(double* pmin, double* pmax, double* psad, int64_t idx, const double acc[4]) {
  if (pmin) pmin[idx] = acc[0];
  if (pmax) pmax[idx] = acc[1];
  if (psad) psad[idx] = acc[2] + acc[3];
}

struct Window {
  int64_t row_begin;
  int ntiles;  // column tiles per row
};

CPB_D bool vertex(const FieldView& f, const Window& w, int64_t& idx) {
  const int64_t t = blockIdx.x;
  const int64_t r = w.row_begin + t / w.ntiles;
  const int64_t c = 1 + (t % w.ntiles) * blockDim.x + threadIdx.x;
  if (c >= f.width - 1) return false;
  idx = r * f.width + c;
  return true;
}

// Per-piece state of the neighbour CDFs.  A piece [a, b] of the shared
// partition lies wholly below, inside or above each neighbour's support (the
// support ends are partition points), so on that piece the clipped CDF
// argument of engine.py:518 / 530 is  fma(x - ref, beta, alpha)  with
// (beta, alpha) = (scale, 0) inside and (0, below | above) outside: one DADD
// and one FMA per node and neighbour instead of a clip.  The node x itself is
// rounded exactly like the reference's  mids + halves * xi  (no contraction),
// so even supports that are tiny next to their offset (degenerate pixels
// widened by eps) see the same arguments as the reference.
CPB_D void piece_state(double mid, double lo, double hi, double scale, double below, double above,
                       double& alpha, double& beta) {
  const bool inside = mid > lo && mid < hi;
  alpha = inside ? 0.0 : (mid >= hi ? above : below);
  beta = inside ? scale : 0.0;
}

CPB_D double node_x(double mid, double half, double xi) { return __dadd_rn(mid, __dmul_rn(half, xi)); }

// ----------------------------------------------------------------- uniform
// pdf_C = 1/(hi_C - lo_C); F_P(x) = clip((x - lo_P)/(hi_P - lo_P), 0, 1)
// (engine.py:510-520), 3-node Gauss-Legendre per piece (integrand degree 4).
__global__ void __launch_bounds__(kClosedThreads) closed_uniform_kernel(
    FieldView f, Window w, double* pmin, double* pmax, double* psad) {
  int64_t idx;
  if (!vertex(f, w, idx)) return;
  const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
  double lo[5], hi[5], inv[5];
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    load_bounds(f, at[p], lo[p], hi[p]);
    inv[p] = 1.0 / (hi[p] - lo[p]);
  }
  const Ranges rg = make_ranges(lo, hi);
  double k[8];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    k[2 * p - 2] = dmin(dmax(lo[p], lo[C_]), hi[C_]);
    k[2 * p - 1] = dmin(dmax(hi[p], lo[C_]), hi[C_]);
  }
  merge_pairs8(k);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double a = lo[C_];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double b = i < 8 ? k[i] : hi[C_];
    if (b > a) {
      const double half = 0.5 * (b - a), mid = 0.5 * (b + a);
      double al[5], be[5];
#pragma unroll
      for (int p = 1; p < 5; ++p) piece_state(mid, lo[p], hi[p], inv[p], 0.0, 1.0, al[p], be[p]);
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < GL3::n; ++j) {
        const double x = node_x(mid, half, GL3::x(j));
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p) F[p] = fma(x - lo[p], be[p], al[p]);
        integrands(F, g);
#pragma unroll
        for (int r = 0; r < 4; ++r) s[r] = fma(GL3::w(j), g[r], s[r]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (a >= rg.lo[r] && b <= rg.hi[r]) acc[r] = fma(s[r], half, acc[r]);
    }
    a = dmax(a, b);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] *= inv[C_];
  store(pmin, pmax, psad, idx, acc);
}

// ------------------------------------------------------------ epanechnikov
// pdf_C = 0.75/hw_C (1 - u^2), u unclipped; F_P = 0.5 + 0.75u - 0.25u^3 with
// u clipped to [-1, 1] (engine.py:521-533); 8-node Gauss-Legendre (degree 14).
// Outside a neighbour's support the affine form pins u to -1 or +1, where the
// cubic gives exactly 0 or 1, so no clip is evaluated per node.
CPB_D double epan_cdf(double u) { return fma(u, fma(-0.25, u * u, 0.75), 0.5); }

__global__ void __launch_bounds__(kClosedThreads) closed_epan_kernel(
    FieldView f, Window w, double* pmin, double* pmax, double* psad) {
  int64_t idx;
  if (!vertex(f, w, idx)) return;
  const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
  double m[5], ih[5], lo[5], hi[5];
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    double hw;
    load_epan(f, at[p], m[p], hw);
    ih[p] = 1.0 / hw;
    lo[p] = m[p] - hw;  // _support_bounds, engine.py:502-505
    hi[p] = m[p] + hw;
  }
  const double pdf0 = 0.75 * ih[C_];
  const Ranges rg = make_ranges(lo, hi);
  double k[8];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    k[2 * p - 2] = dmin(dmax(lo[p], lo[C_]), hi[C_]);
    k[2 * p - 1] = dmin(dmax(hi[p], lo[C_]), hi[C_]);
  }
  merge_pairs8(k);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double a = lo[C_];
#pragma unroll 1
  for (int i = 0; i < 9; ++i) {
    double b = hi[C_];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == i) b = k[q];
    if (b > a) {
      const double half = 0.5 * (b - a), mid = 0.5 * (b + a);
      double al[5], be[5];
#pragma unroll
      for (int p = 1; p < 5; ++p) piece_state(mid, lo[p], hi[p], ih[p], -1.0, 1.0, al[p], be[p]);
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < GL8::n; ++j) {
        const double x = node_x(mid, half, GL8::x(j));
        const double uc = (x - m[C_]) * ih[C_];
        const double wp = GL8::w(j) * (pdf0 * fma(-uc, uc, 1.0));
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p) F[p] = epan_cdf(fma(x - m[p], be[p], al[p]));
        integrands(F, g);
#pragma unroll
        for (int r = 0; r < 4; ++r) s[r] = fma(wp, g[r], s[r]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (a >= rg.lo[r] && b <= rg.hi[r]) acc[r] = fma(s[r], half, acc[r]);
    }
    a = dmax(a, b);
  }
  store(pmin, pmax, psad, idx, acc);
}

// --------------------------------------------------------------- histogram
// Renormalised weights wn = w / sum(w), cum = [0, cumsum(wn)], binw = (hi-lo)/h;
// pdf_C = wn[j]/binw, F_P = clip(cum[j] + wn[j] (x - (lo + binw j))/binw, 0, 1)
// (engine.py:534-559, distributions.py:92-100); edges lo + (hi-lo) k/h
// (engine.py:565-571).  Instead of sorting 5(h+1) edges the kernel sweeps
// the five sorted edge lists in merge order, carrying each neighbour's
// current bin (and its running prefix sum) from piece to piece.
struct HistPos {
  double lo, hi, width, binw, ibinw, itotal;
  bool deg;
  int dbin;
  int64_t at;
};

struct Sweep {  // neighbour state inside the current piece: F(x) = c + s (x - e)
  int j;        // current bin; -1 below the support, h above it
  double next;  // next edge strictly ahead (+inf when none)
  double cum;   // prefix sum of wn over bins < j (sequential, like np.cumsum)
  double wj;    // wn[j]
  double c, s, e;
};

CPB_D double edge_at(const HistPos& P, int k, int h) {
  // kinks of engine.py:570-571; the last edge is the support end itself so
  // range endpoints coincide exactly with partition points
  return k >= h ? P.hi : P.lo + P.width * ((double)k / (double)h);
}

CPB_D double wn_at(const FieldView& f, const HistPos& P, int b) {
  return load_weight(f, P.at, b, P.deg, P.dbin) * P.itotal;
}

CPB_D void enter_bin(const FieldView& f, const HistPos& P, Sweep& st, int h) {
  // advance from bin st.j to st.j + 1
  if (st.j >= 0 && st.j < h) st.cum += st.wj;
  st.j += 1;
  if (st.j >= h) {
    st.c = 1.0; st.s = 0.0; st.e = 0.0;
    st.next = __longlong_as_double(0x7ff0000000000000ll);
    return;
  }
  st.wj = wn_at(f, P, st.j);
  st.c = st.cum;
  st.s = st.wj * P.ibinw;
  st.e = P.lo + P.binw * (double)st.j;
  st.next = edge_at(P, st.j + 1, h);
}

// Fallback for very many bins (> kHistSmemMaxBins): per-thread state, weights
// read from global memory.
__global__ void __launch_bounds__(kClosedThreads) closed_hist_global_kernel(
    FieldView f, Window w, double* pmin, double* pmax, double* psad) {
  int64_t idx;
  if (!vertex(f, w, idx)) return;
  const int h = f.bins;
  const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
  HistPos P[5];
  double lo[5], hi[5];
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    HistPos& q = P[p];
    q.at = at[p];
    q.deg = load_bounds(f, at[p], q.lo, q.hi);
    q.dbin = 0;
    if (q.deg) q.dbin = degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at[p]), q.lo, q.hi, h);
    q.width = q.hi - q.lo;
    q.binw = q.width / (double)h;
    q.ibinw = 1.0 / q.binw;
    const double total = pairwise_sum([&](int b) { return load_weight(f, q.at, b, q.deg, q.dbin); }, h);
    q.itotal = 1.0 / total;
    lo[p] = q.lo;
    hi[p] = q.hi;
  }
  const Ranges rg = make_ranges(lo, hi);
  const double x0 = lo[C_], xend = hi[C_];
  // neighbour states at the start of the sweep
  Sweep st[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    st[p].j = -1; st[p].cum = 0.0; st[p].wj = 0.0; st[p].c = 0.0; st[p].s = 0.0; st[p].e = 0.0;
    st[p].next = P[p].lo;
    while (st[p].next <= x0) enter_bin(f, P[p], st[p], h);
  }
  // centre: bin jc, pdf = wn[jc]/binw
  int jc = 0;
  double pdf = wn_at(f, P[C_], 0) * P[C_].ibinw;
  double nextc = edge_at(P[C_], 1, h);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double x = x0;
  while (x < xend) {
    const double xn = dmin(dmin(nextc, dmin(st[E_].next, st[N_].next)), dmin(st[W_].next, st[S_].next));
    if (xn > x) {
      const double half = 0.5 * (xn - x), mid = 0.5 * (xn + x);
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < GL3::n; ++j) {
        const double xx = mid + half * GL3::x(j);
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p) F[p] = st[p].c + st[p].s * (xx - st[p].e);
        integrands(F, g);
#pragma unroll
        for (int r = 0; r < 4; ++r) s[r] += GL3::w(j) * g[r];
      }
      const double scale = pdf * half;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (x >= rg.lo[r] && xn <= rg.hi[r]) acc[r] += s[r] * scale;
    }
    if (nextc == xn) {
      ++jc;
      if (jc >= h) {
        nextc = __longlong_as_double(0x7ff0000000000000ll);
      } else {
        pdf = wn_at(f, P[C_], jc) * P[C_].ibinw;
        nextc = edge_at(P[C_], jc + 1, h);
      }
    }
#pragma unroll
    for (int p = 1; p < 5; ++p)
      if (st[p].next == xn) enter_bin(f, P[p], st[p], h);
    x = dmax(x, xn);
  }
  store(pmin, pmax, psad, idx, acc);
}

// Shared-memory histogram stencil (the production path for bins <= 64).
// A block of TW threads computes TW consecutive vertices of one row.  First the
// block stages the 3 x (TW + 2) pixels the stencil touches: support bounds,
// bin widths and the renormalised weights wn = w / sum(w) (numpy pairwise
// order for the sum), all in float64 shared memory; then every thread sweeps
// its five edge lists reading only shared memory.
constexpr int kHistSmemMaxBins = 64;

struct HistTile {
  int sw;            // staged row width = TW + 2
  double* lo;        // [3 * sw]
  double* hi;
  double* width;     // hi - lo
  double* binw;
  double* ibinw;
  double* wn;        // [bins][3 * sw]
  double* kh;        // k / h for k = 0..h
};

struct NState {      // one neighbour inside the current piece: F(x) = c + s (x - e)
  int j;
  double next, cum, wj, c, s, e;
};

CPB_D void nb_enter(const HistTile& T, int i, int h, double hi, NState& st) {
  if (st.j >= 0) st.cum += st.wj;  // np.cumsum order
  st.j += 1;
  if (st.j >= h) {
    st.c = 1.0; st.s = 0.0; st.e = 0.0; st.wj = 0.0;
    st.next = __longlong_as_double(0x7ff0000000000000ll);
    return;
  }
  const int n = 3 * T.sw;
  st.wj = T.wn[st.j * n + i];
  st.c = st.cum;
  st.s = st.wj * T.ibinw[i];
  st.e = T.lo[i] + T.binw[i] * (double)st.j;
  st.next = st.j + 1 >= h ? hi : T.lo[i] + T.width[i] * T.kh[st.j + 1];
}

__global__ void closed_hist_smem_kernel(FieldView f, Window w, double* pmin, double* pmax,
                                        double* psad) {
  extern __shared__ double sm[];
  const int TW = blockDim.x, sw = TW + 2, n = 3 * sw, h = f.bins;
  HistTile T;
  T.sw = sw;
  T.lo = sm;
  T.hi = sm + n;
  T.width = sm + 2 * n;
  T.binw = sm + 3 * n;
  T.ibinw = sm + 4 * n;
  T.wn = sm + 5 * n;
  T.kh = T.wn + (size_t)h * n;
  const int64_t tile = blockIdx.x % w.ntiles;
  const int64_t r = w.row_begin + blockIdx.x / w.ntiles;
  const int64_t c0 = tile * TW;  // staged columns [c0, c0 + sw)
  for (int k = threadIdx.x; k <= h; k += TW) T.kh[k] = (double)k / (double)h;
  for (int i = threadIdx.x; i < n; i += TW) {
    const int64_t rr = r - 1 + i / sw, cc = c0 + i % sw;
    if (cc >= f.width) continue;
    const int64_t at = rr * f.width + cc;
    double lo, hi;
    const bool deg = load_bounds(f, at, lo, hi);
    const int dbin = deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at), lo, hi, h) : 0;
    for (int b = 0; b < h; ++b) T.wn[b * n + i] = load_weight(f, at, b, deg, dbin);
    const double total = pairwise_sum([&](int b) { return T.wn[b * n + i]; }, h);
    const double it = 1.0 / total;
    for (int b = 0; b < h; ++b) T.wn[b * n + i] *= it;
    T.lo[i] = lo;
    T.hi[i] = hi;
    T.width[i] = hi - lo;
    T.binw[i] = (hi - lo) / (double)h;
    T.ibinw[i] = 1.0 / T.binw[i];
  }
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t c = c0 + 1 + t;
  if (c >= f.width - 1) return;
  const int64_t idx = r * f.width + c;
  const int li[5] = {sw + t + 1, sw + t + 2, t + 1, sw + t, 2 * sw + t + 1};  // C E N W S
  double lo[5], hi[5];
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    lo[p] = T.lo[li[p]];
    hi[p] = T.hi[li[p]];
  }
  const Ranges rg = make_ranges(lo, hi);
  const double x0 = lo[C_], xend = hi[C_];
  NState st[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    st[p].j = -1; st[p].cum = 0.0; st[p].wj = 0.0; st[p].c = 0.0; st[p].s = 0.0; st[p].e = 0.0;
    st[p].next = lo[p];
    while (st[p].next <= x0) nb_enter(T, li[p], h, hi[p], st[p]);
  }
  const int ic = li[C_];
  int jc = 0;
  double pdf = T.wn[ic] * T.ibinw[ic];
  double nextc = h > 1 ? T.lo[ic] + T.width[ic] * T.kh[1] : xend;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double x = x0;
  while (x < xend) {
    const double xn = dmin(dmin(nextc, dmin(st[E_].next, st[N_].next)), dmin(st[W_].next, st[S_].next));
    if (xn > x) {
      const double half = 0.5 * (xn - x), mid = 0.5 * (xn + x);
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < GL3::n; ++j) {
        const double xx = node_x(mid, half, GL3::x(j));
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p) F[p] = fma(xx - st[p].e, st[p].s, st[p].c);
        integrands(F, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fma(GL3::w(j), g[q], s[q]);
      }
      const double scale = pdf * half;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (x >= rg.lo[q] && xn <= rg.hi[q]) acc[q] = fma(s[q], scale, acc[q]);
    }
    if (nextc == xn) {
      ++jc;
      if (jc >= h) {
        nextc = __longlong_as_double(0x7ff0000000000000ll);
      } else {
        pdf = T.wn[jc * n + ic] * T.ibinw[ic];
        nextc = jc + 1 >= h ? xend : T.lo[ic] + T.width[ic] * T.kh[jc + 1];
      }
    }
#pragma unroll
    for (int p = 1; p < 5; ++p)
      if (st[p].next == xn) nb_enter(T, li[p], h, hi[p], st[p]);
    x = dmax(x, xn);
  }
  store(pmin, pmax, psad, idx, acc);
}

}  // namespace

int launch_closed(const cpb_field* fld, int64_t row_begin, int64_t row_end, double* pmin,
                  double* pmax, double* psad, cudaStream_t st) {
  const FieldView f = make_view(*fld);
  const int64_t rows = row_end - row_begin;
  if (rows <= 0 || f.width < 3) return CPB_OK;
  Window w;
  w.row_begin = row_begin;
  w.ntiles = (int)((f.width - 2 + kClosedThreads - 1) / kClosedThreads);
  const int64_t blocks = rows * w.ntiles;
  if (blocks > 0x7fffffffll) {
    set_error("grid too large for one launch (%lld blocks)", (long long)blocks);
    return CPB_EINVAL;
  }
  switch (f.kind) {
    case CPB_UNIFORM:
      closed_uniform_kernel<<<(unsigned)blocks, kClosedThreads, 0, st>>>(f, w, pmin, pmax, psad);
      break;
    case CPB_EPANECHNIKOV:
      closed_epan_kernel<<<(unsigned)blocks, kClosedThreads, 0, st>>>(f, w, pmin, pmax, psad);
      break;
    case CPB_HISTOGRAM: {
      if (f.bins > kHistSmemMaxBins) {
        closed_hist_global_kernel<<<(unsigned)blocks, kClosedThreads, 0, st>>>(f, w, pmin, pmax, psad);
        break;
      }
      // tile width so the staged float64 weights fit comfortably in shared memory
      int tw = 128;
      while (tw > 32 && (size_t)(5 + f.bins) * 3 * (tw + 2) * 8 > 64 * 1024) tw >>= 1;
      Window wh = w;
      wh.ntiles = (int)((f.width - 2 + tw - 1) / tw);
      const int64_t hb = rows * wh.ntiles;
      const size_t smem = ((size_t)(5 + f.bins) * 3 * (tw + 2) + f.bins + 1) * 8;
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(closed_hist_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      closed_hist_smem_kernel<<<(unsigned)hb, tw, smem, st>>>(f, wh, pmin, pmax, psad);
      break;
    }
    default:
      set_error("Gaussian fields have no closed form; use monte_carlo");
      return CPB_EINVAL;
  }
  CPB_CHECK_LAUNCH("closed-form kernel");
  return CPB_OK;
}

}  // namespace cpb
