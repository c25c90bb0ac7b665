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
#include <stdlib.h>

#include <algorithm>

#include "cpb_common.cuh"
#include "cpb_tma.cuh"
#include "cpb_fitpix.cuh"

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

// integrands with the two saddle terms summed: g[2] = t1 + t2
CPB_D void integrands3(const double* F, double g[3]) {
  const double sE = 1.0 - F[E_], sN = 1.0 - F[N_], sW = 1.0 - F[W_], sS = 1.0 - F[S_];
  const double sesw = sE * sW, snss = sN * sS;
  const double fefw = F[E_] * F[W_], fnfs = F[N_] * F[S_];
  g[0] = sesw * snss;
  g[1] = fefw * fnfs;
  g[2] = fma(sesw, fnfs, snss * fefw);
}

// GL3 sums of the four integrands on one piece from the neighbour CDFs at
// the piece midpoint (Fm) and their slopes times the node offset (d): with
// F = Fm +- d at the nodes mid +- tau, each pair product X*Y is Pe +- Po
// (Pe = x0 y0 + dx dy, Po = x0 dy + y0 dx), so an integrand P*Q summed over
// the two symmetric nodes is 2 (Pe Qe + Po Qo) and the midpoint value is
// x0 y0 * ... : 58 FP64 operations instead of 69 for three separate nodes.
// s[q] = w1 g_q(mid) + w0 (g_q(mid - tau) + g_q(mid + tau)).
CPB_D void gl3_sym_sums(const double* Fm, const double* d, double s[4]) {
  struct Pair { double p0, pe, po; };
  auto pair = [](double x0, double dx, double y0, double dy) {
    Pair r;
    r.p0 = x0 * y0;
    r.pe = fma(dx, dy, r.p0);
    r.po = fma(x0, dy, y0 * dx);
    return r;
  };
  const double sE = 1.0 - Fm[E_], sN = 1.0 - Fm[N_], sW = 1.0 - Fm[W_], sS = 1.0 - Fm[S_];
  // survival slopes are -d
  const Pair sesw = pair(sE, -d[E_], sW, -d[W_]), snss = pair(sN, -d[N_], sS, -d[S_]);
  const Pair fefw = pair(Fm[E_], d[E_], Fm[W_], d[W_]), fnfs = pair(Fm[N_], d[N_], Fm[S_], d[S_]);
  const double w1 = GL3::w(1), w0x2 = 2.0 * GL3::w(0);
  auto term = [&](const Pair& P, const Pair& Q) {
    const double gs = fma(P.po, Q.po, P.pe * Q.pe);
    return fma(w0x2, gs, w1 * (P.p0 * Q.p0));
  };
  s[0] = term(sesw, snss);
  s[1] = term(fefw, fnfs);
  s[2] = term(sesw, fnfs);
  s[3] = term(snss, fefw);
}

// gl3_sym_sums with the saddle integrals summed inside: s[2] = t1 + t2 (the
// stencils only ever report the saddle sum), 37 FP64 operations.
CPB_D void gl3_sym_sums3(const double* Fm, const double* d, double s[3]) {
  struct Pair { double p0, pe, po; };
  auto pair = [](double x0, double dx, double y0, double dy) {
    Pair r;
    r.p0 = x0 * y0;
    r.pe = fma(dx, dy, r.p0);
    r.po = fma(x0, dy, y0 * dx);
    return r;
  };
  const double sE = 1.0 - Fm[E_], sN = 1.0 - Fm[N_], sW = 1.0 - Fm[W_], sS = 1.0 - Fm[S_];
  const Pair sesw = pair(sE, -d[E_], sW, -d[W_]), snss = pair(sN, -d[N_], sS, -d[S_]);
  const Pair fefw = pair(Fm[E_], d[E_], Fm[W_], d[W_]), fnfs = pair(Fm[N_], d[N_], Fm[S_], d[S_]);
  const double w1 = GL3::w(1), w0x2 = 2.0 * GL3::w(0);
  auto term = [&](const Pair& P, const Pair& Q) {
    const double gs = fma(P.po, Q.po, P.pe * Q.pe);
    return fma(w0x2, gs, w1 * (P.p0 * Q.p0));
  };
  s[0] = term(sesw, snss);
  s[1] = term(fefw, fnfs);
  const double gs = fma(sesw.po, fnfs.po, fma(sesw.pe, fnfs.pe, fma(snss.po, fefw.po, snss.pe * fefw.pe)));
  const double g0 = fma(sesw.p0, fnfs.p0, snss.p0 * fefw.p0);
  s[2] = fma(w0x2, gs, w1 * g0);
}

// gl3_sym_sums3 before the Gauss-Legendre weights: s = w0x2 gs + w1 g0, the
// caller accumulates gs and g0 separately and weights the totals once.
CPB_D void gl3_sym_parts3(const double* Fm, const double* d, double gs[3], double g0[3]) {
  struct Pair { double p0, pe, po; };
  auto pair = [](double x0, double dx, double y0, double dy) {
    Pair r;
    r.p0 = x0 * y0;
    r.pe = fma(dx, dy, r.p0);
    r.po = fma(x0, dy, y0 * dx);
    return r;
  };
  const double sE = 1.0 - Fm[E_], sN = 1.0 - Fm[N_], sW = 1.0 - Fm[W_], sS = 1.0 - Fm[S_];
  const Pair sesw = pair(sE, -d[E_], sW, -d[W_]), snss = pair(sN, -d[N_], sS, -d[S_]);
  const Pair fefw = pair(Fm[E_], d[E_], Fm[W_], d[W_]), fnfs = pair(Fm[N_], d[N_], Fm[S_], d[S_]);
  gs[0] = fma(sesw.po, snss.po, sesw.pe * snss.pe);
  g0[0] = sesw.p0 * snss.p0;
  gs[1] = fma(fefw.po, fnfs.po, fefw.pe * fnfs.pe);
  g0[1] = fefw.p0 * fnfs.p0;
  gs[2] = fma(sesw.po, fnfs.po, fma(sesw.pe, fnfs.pe, fma(snss.po, fefw.po, snss.pe * fefw.pe)));
  g0[2] = fma(sesw.p0, fnfs.p0, snss.p0 * fefw.p0);
}

// gl3_sym_sums in single precision (the mixed-precision closed form: the
// partition, node offsets and accumulation stay float64, the per-piece GL3
// evaluation runs on the FP32 pipes).
CPB_D void gl3_sym_sums_f(const float* Fm, const float* d, float s[4]) {
  struct Pair { float p0, pe, po; };
  auto pair = [](float x0, float dx, float y0, float dy) {
    Pair r;
    r.p0 = x0 * y0;
    r.pe = fmaf(dx, dy, r.p0);
    r.po = fmaf(x0, dy, y0 * dx);
    return r;
  };
  const float sE = 1.0f - Fm[E_], sN = 1.0f - Fm[N_], sW = 1.0f - Fm[W_], sS = 1.0f - Fm[S_];
  const Pair sesw = pair(sE, -d[E_], sW, -d[W_]), snss = pair(sN, -d[N_], sS, -d[S_]);
  const Pair fefw = pair(Fm[E_], d[E_], Fm[W_], d[W_]), fnfs = pair(Fm[N_], d[N_], Fm[S_], d[S_]);
  const float w1 = (float)GL3::w(1), w0x2 = (float)(2.0 * GL3::w(0));
  auto term = [&](const Pair& P, const Pair& Q) {
    const float gs = fmaf(P.po, Q.po, P.pe * Q.pe);
    return fmaf(w0x2, gs, w1 * (P.p0 * Q.p0));
  };
  s[0] = term(sesw, snss);
  s[1] = term(fefw, fnfs);
  s[2] = term(sesw, fnfs);
  s[3] = term(snss, fefw);
}

CPB_D void store(double* pmin, double* pmax, double* psad, int64_t idx, const double acc[4]) {
  if (pmin) pmin[idx] = acc[0];
  if (pmax) pmax[idx] = acc[1];
  if (psad) psad[idx] = acc[2] + acc[3];
}

// Expected per-type counts (sum of each channel over the launch's vertices,
// SURVEY.md §8 e): every WARP reduces its lanes' (p_min, p_max, p_saddle) with
// a fixed shuffle tree and writes one partial triple (no block barrier, so
// warps still retire independently); counts_reduce_kernel and
// counts_finish_kernel add the partials with a fixed tree.  Deterministic for
// a given launch shape.  Every lane of a warp must call it (dead lanes pass 0).
CPB_D void warp_partial_sums(double v0, double v1, double v2, double* partial) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, d);
    v1 += __shfl_xor_sync(0xffffffffu, v1, d);
    v2 += __shfl_xor_sync(0xffffffffu, v2, d);
  }
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int wpb = (blockDim.x * blockDim.y + 31) / 32;
  if ((tid & 31) == 0) {
    const int64_t w = ((int64_t)blockIdx.x + (int64_t)blockIdx.y * gridDim.x) * wpb + (tid >> 5);
    partial[3 * w] = v0;
    partial[3 * w + 1] = v1;
    partial[3 * w + 2] = v2;
  }
}

constexpr int kCountChunks = 1024;

// stage 1: chunk c of the warp partials -> chunk[c] (fixed tree per block)
__global__ void counts_reduce_kernel(const double* partial, int64_t n, double* chunk) {
  __shared__ double red[256][3];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t b = b0 + threadIdx.x; b < b1; b += 256) {
    a0 += partial[3 * b];
    a1 += partial[3 * b + 1];
    a2 += partial[3 * b + 2];
  }
  red[threadIdx.x][0] = a0;
  red[threadIdx.x][1] = a1;
  red[threadIdx.x][2] = a2;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int c = 0; c < 3; ++c) red[threadIdx.x][c] += red[threadIdx.x + w][c];
    __syncthreads();
  }
  if (threadIdx.x < 3) chunk[3 * blockIdx.x + threadIdx.x] = red[0][threadIdx.x];
}

// stage 2: the chunks -> counts[0..2] (added)
__global__ void counts_finish_kernel(const double* chunk, int64_t n, double* counts) {
  __shared__ double red[256][3];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t b = threadIdx.x; b < n; b += 256) {
    a0 += chunk[3 * b];
    a1 += chunk[3 * b + 1];
    a2 += chunk[3 * b + 2];
  }
  red[threadIdx.x][0] = a0;
  red[threadIdx.x][1] = a1;
  red[threadIdx.x][2] = a2;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int c = 0; c < 3; ++c) red[threadIdx.x][c] += red[threadIdx.x + w][c];
    __syncthreads();
  }
  if (threadIdx.x < 3) counts[threadIdx.x] += red[0][threadIdx.x];
}

__global__ void rows_partial_kernel(const double* pmin, const double* pmax, const double* psad,
                                    int64_t row_begin, int64_t cols, int64_t width, int64_t nvert,
                                    double* partial) {
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvert;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = (row_begin + v / cols) * width + 1 + v % cols;
    if (pmin) v0 += pmin[idx];
    if (pmax) v1 += pmax[idx];
    if (psad) v2 += psad[idx];
  }
  warp_partial_sums(v0, v1, v2, partial);
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
// argument of engine.py:518 / 530 is affine in x:  fma(x - ref, beta, alpha)
// with (beta, alpha) = (scale, 0) inside and (0, below | above) outside --
// no clip per node.  The same below/above flags give each piece's membership
// in the four integration ranges (range_masks).
//
// Two evaluation modes per vertex:
//  - exact: every node x is rounded like the reference's  mids + halves * xi
//    (no contraction) before the subtraction, so supports that are tiny next
//    to their offset (eps-widened degenerate pixels) see the reference's
//    arguments bit for bit;
//  - fast (|x| / support width <= kFastRatio at all five positions): the
//    CDF is evaluated at the piece midpoint and moved to the symmetric nodes
//    mid +- tau along its slope, which skips the per-node x rounding; the
//    difference to the reference is <= ulp(x) / width * kFastRatio-bounded,
//    i.e. < 3e-14 in every probability (tolerance 1e-12).
constexpr double kFastRatio = 256.0;

CPB_D void piece_flags(double mid, double lo, double hi, bool& below, bool& above) {
  above = mid >= hi;
  below = mid <= lo;
}

// Which of the four integrals a piece belongs to.  The ranges of
// engine.py:603-628 start at max(lo) / end at min(hi) of some positions, and
// a position's lo / hi are its first / last partition edge, so a piece is in
// the min range iff no neighbour is above it, in the max range iff none is
// below, t1 iff N, S are not below and E, W not above, t2 vice versa.  But
// outside exactly those pieces one factor of the integrand is an exact zero
// (a neighbour below its support has F = 0, above it S = 1 - 1 = 0, and the
// piece states reproduce those values exactly), so the contribution is 0
// either way: every piece can feed all four integrals unmasked.  The masks
// are therefore all-true; evaluating them (previous revision) cost ~13 % of
// the histogram stencil.
CPB_D void range_masks(bool, bool, bool, bool, bool, bool, bool, bool, bool m[4]) {
  m[0] = m[1] = m[2] = m[3] = true;
}

CPB_D double node_x(double mid, double half, double xi) { return __dadd_rn(mid, __dmul_rn(half, xi)); }

CPB_D double piece_end(const double* k, double hiC, int i) {
  double b = hiC;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q == i) b = k[q];
  return b;
}

// ----------------------------------------------------------------- uniform
// Batcher merge of four sorted (key, tag) pairs: one compare per exchange,
// the tag (2 (p - 1) + {0: lo, 1: hi}) travels with its key.
CPB_D void tcswap(double& a, double& b, int& ta, int& tb) {
  const bool sw = b < a;
  const double x = sw ? b : a, y = sw ? a : b;
  const int u = sw ? tb : ta, v = sw ? ta : tb;
  a = x; b = y; ta = u; tb = v;
}
CPB_D void merge_pairs8_tagged(double* k, int* t) {
  tcswap(k[0], k[2], t[0], t[2]); tcswap(k[1], k[3], t[1], t[3]); tcswap(k[1], k[2], t[1], t[2]);
  tcswap(k[4], k[6], t[4], t[6]); tcswap(k[5], k[7], t[5], t[7]); tcswap(k[5], k[6], t[5], t[6]);
  tcswap(k[0], k[4], t[0], t[4]); tcswap(k[1], k[5], t[1], t[5]); tcswap(k[2], k[6], t[2], t[6]);
  tcswap(k[3], k[7], t[3], t[7]);
  tcswap(k[2], k[4], t[2], t[4]); tcswap(k[3], k[5], t[3], t[5]);
  tcswap(k[1], k[2], t[1], t[2]); tcswap(k[3], k[4], t[3], t[4]); tcswap(k[5], k[6], t[5], t[6]);
}

// uniform_pieces with the piece states tracked from the merge tags: every
// partition point is some neighbour's (clamped) support end, so crossing it
// moves that neighbour below -> inside -> above.  A 2-bit crossing count per
// neighbour replaces the per-piece midpoint comparisons (8 FP64-pipe compares
// per piece), and the 9 pieces are unrolled so the keys are static registers.
// Ties are harmless: coincident points bound zero-width pieces, which add
// exactly 0, and a count of 2 means "above" whatever the tie order.
template <bool FAST>
CPB_D void uniform_pieces_tagged(const double* lo, const double* hi, const double* inv,
                                 const double* k, const int* t, double acc[4]) {
  double a = lo[C_];
  unsigned cnt = 0;  // 2 bits per neighbour p at bit 2 (p - 1)
  double accs[3] = {0.0, 0.0, 0.0};  // FAST: node-pair sums (acc: midpoint sums)
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double b = i < 8 ? k[i] : hi[C_];
    // every piece is evaluated (a zero-width one adds s * 0 = exactly 0): no
    // per-piece branch, so the nine unrolled pieces schedule as one block
    // (fused uniform kernel 15.5 -> 15.0 ms)
    {
      const double half = 0.5 * (b - a), mid = 0.5 * (b + a);
      double al[5], be[5];
#pragma unroll
      for (int p = 1; p < 5; ++p) {
        const unsigned c = (cnt >> (2 * (p - 1))) & 3u;
        const bool in = c == 1u;
        be[p] = in ? inv[p] : 0.0;
        al[p] = in ? (FAST ? (mid - lo[p]) * inv[p] : 0.0) : (c == 2u ? 1.0 : 0.0);
      }
      double s[4];
      if (FAST) {
        const double tau = half * GL3::x(2);
        double d[5];
#pragma unroll
        for (int p = 1; p < 5; ++p) d[p] = tau * be[p];
        double gs[3];
        gl3_sym_parts3(al, d, gs, s);
#pragma unroll
        for (int r = 0; r < 3; ++r) accs[r] = fma(gs[r], half, accs[r]);
      } else {
        double F[5], g[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) s[r] = 0.0;
#pragma unroll
        for (int j = 0; j < GL3::n; ++j) {
          const double x = node_x(mid, half, GL3::x(j));
#pragma unroll
          for (int p = 1; p < 5; ++p) F[p] = fma(x - lo[p], be[p], al[p]);
          integrands(F, g);
#pragma unroll
          for (int r = 0; r < 4; ++r) s[r] = fma(GL3::w(j), g[r], s[r]);
        }
        s[2] += s[3];
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) acc[r] = fma(s[r], half, acc[r]);  // acc[3] stays 0
      a = b;
    }
    if (i < 8) cnt += 1u << (2 * (t[i] >> 1));
  }
  if (FAST) {  // the Gauss-Legendre weights, once per vertex
    const double w1 = GL3::w(1), w0x2 = 2.0 * GL3::w(0);
#pragma unroll
    for (int r = 0; r < 3; ++r) acc[r] = fma(w0x2, accs[r], w1 * acc[r]);
  }
}

// The four integrals of one all-uniform neighbourhood from its supports and
// the merged, tagged partition points k / t.
CPB_D void uniform_integrals_merged(const double* lo, const double* hi, const double* k,
                                    const int* t, double acc[4]) {
  double inv[5];
  bool fast = true;
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    inv[p] = 1.0 / (hi[p] - lo[p]);
    fast &= (fabs(lo[p]) + fabs(hi[p])) * inv[p] <= kFastRatio;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] = 0.0;
  if (fast) uniform_pieces_tagged<true>(lo, hi, inv, k, t, acc);
  else uniform_pieces_tagged<false>(lo, hi, inv, k, t, acc);
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] *= inv[C_];
}

// The four integrals (min, max, saddle t1, t2) of one all-uniform
// neighbourhood given its five supports [lo_P, hi_P] (P = C, E, N, W, S).
CPB_D void uniform_integrals(const double* lo, const double* hi, double acc[4]) {
  double k[8];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    k[2 * p - 2] = dmin(dmax(lo[p], lo[C_]), hi[C_]);
    k[2 * p - 1] = dmin(dmax(hi[p], lo[C_]), hi[C_]);
  }
  int t[8] = {0, 1, 2, 3, 4, 5, 6, 7};
  merge_pairs8_tagged(k, t);
  uniform_integrals_merged(lo, hi, k, t, acc);
}

CPB_D void tcswapf(float& a, float& b, int& ta, int& tb);

// Fitted float supports (not eps-widened): the clamped partition points are
// floats themselves, so clamping and the tagged merge run exactly on the FP32
// / integer pipes (FMNMX, FSETP + SEL) instead of FP64 compares.
CPB_D void uniform_integrals_f32keys(const float* rl, const float* rh, const double* lo,
                                     const double* hi, double acc[4]) {
  float kf[8];
  int t[8];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    kf[2 * p - 2] = fminf(fmaxf(rl[p], rl[C_]), rh[C_]);
    kf[2 * p - 1] = fminf(fmaxf(rh[p], rl[C_]), rh[C_]);
    t[2 * p - 2] = 2 * p - 2;
    t[2 * p - 1] = 2 * p - 1;
  }
  tcswapf(kf[0], kf[2], t[0], t[2]); tcswapf(kf[1], kf[3], t[1], t[3]); tcswapf(kf[1], kf[2], t[1], t[2]);
  tcswapf(kf[4], kf[6], t[4], t[6]); tcswapf(kf[5], kf[7], t[5], t[7]); tcswapf(kf[5], kf[6], t[5], t[6]);
  tcswapf(kf[0], kf[4], t[0], t[4]); tcswapf(kf[1], kf[5], t[1], t[5]); tcswapf(kf[2], kf[6], t[2], t[6]);
  tcswapf(kf[3], kf[7], t[3], t[7]);
  tcswapf(kf[2], kf[4], t[2], t[4]); tcswapf(kf[3], kf[5], t[3], t[5]);
  tcswapf(kf[1], kf[2], t[1], t[2]); tcswapf(kf[3], kf[4], t[3], t[4]); tcswapf(kf[5], kf[6], t[5], t[6]);
  double k[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) k[q] = (double)kf[q];
  uniform_integrals_merged(lo, hi, k, t, acc);
}

// The four integrals of the uniform vertex idx from the field's planes: with
// fitted float planes and no degenerate pixel the merge runs on float keys,
// otherwise load_bounds widens degenerate pixels by eps / 2 (fields.py:140-143).
CPB_D void uniform_vertex(const FieldView& f, int64_t idx, double acc[4]) {
  {
    const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
    double lo[5], hi[5];
    if (f.bounds == CPB_BOUNDS_F32_FITTED) {
      // all ten loads in flight before any use, then the eps widening of
      // degenerate pixels (load_bounds)
      float rl[5], rh[5];
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        rl[p] = __ldg(static_cast<const float*>(f.lo) + at[p]);
        rh[p] = __ldg(static_cast<const float*>(f.hi) + at[p]);
      }
      bool deg = false;
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        lo[p] = (double)rl[p];
        hi[p] = (double)rh[p];
        deg |= !(hi[p] > lo[p]);
      }
      if (deg) {
        const double he = __dmul_rn(0.5, field_eps(f));
#pragma unroll
        for (int p = 0; p < 5; ++p) {
          if (!(hi[p] > lo[p])) {
            const double c = lo[p];
            lo[p] = __dsub_rn(c, he);
            hi[p] = __dadd_rn(c, he);
          }
        }
        uniform_integrals(lo, hi, acc);
      } else {
        uniform_integrals_f32keys(rl, rh, lo, hi, acc);
      }
    } else {
#pragma unroll
      for (int p = 0; p < 5; ++p) load_bounds(f, at[p], lo[p], hi[p]);
      uniform_integrals(lo, hi, acc);
    }
  }
}

__global__ void __launch_bounds__(kClosedThreads) closed_uniform_kernel(
    FieldView f, Window w, double* pmin, double* pmax, double* psad, double* partial) {
  int64_t idx = 0;
  const bool live = vertex(f, w, idx);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (live) {
    uniform_vertex(f, idx, acc);
    store(pmin, pmax, psad, idx, acc);
  }
  if (partial) warp_partial_sums(acc[0], acc[1], acc[2] + acc[3], partial);
}

// ------------------------------------------------ uniform, mixed precision
// CPB_FLAG_MIXED: the five supports are re-centred on lo_C in float64 and the
// rest -- merge, piece states, GL3 sums -- runs in single precision on the
// FP32 pipes, with a compensated (Kahan) sum over the pieces.  Absolute error
// bound 1e-6 (north_star); measured ~1e-7 (tests/test_gpu_parity.py).
CPB_D void tcswapf(float& a, float& b, int& ta, int& tb) {
  const bool sw = b < a;
  const float x = sw ? b : a, y = sw ? a : b;
  const int u = sw ? tb : ta, v = sw ? ta : tb;
  a = x; b = y; ta = u; tb = v;
}

CPB_D void kahan_add(float& sum, float& c, float v) {
  const float y = v - c;
  const float t = sum + y;
  c = (t - sum) - y;
  sum = t;
}

CPB_D void uniform_integrals_f(const double* lo, const double* hi, double out[3]) {
  const double ref = lo[C_];
  float l[5], h[5], inv[5];
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    l[p] = (float)(lo[p] - ref);
    h[p] = (float)(hi[p] - ref);
    inv[p] = 1.0f / (h[p] - l[p]);
  }
  float k[8];
  int t[8];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    k[2 * p - 2] = fminf(fmaxf(l[p], l[C_]), h[C_]);
    k[2 * p - 1] = fminf(fmaxf(h[p], l[C_]), h[C_]);
    t[2 * p - 2] = 2 * p - 2;
    t[2 * p - 1] = 2 * p - 1;
  }
  tcswapf(k[0], k[2], t[0], t[2]); tcswapf(k[1], k[3], t[1], t[3]); tcswapf(k[1], k[2], t[1], t[2]);
  tcswapf(k[4], k[6], t[4], t[6]); tcswapf(k[5], k[7], t[5], t[7]); tcswapf(k[5], k[6], t[5], t[6]);
  tcswapf(k[0], k[4], t[0], t[4]); tcswapf(k[1], k[5], t[1], t[5]); tcswapf(k[2], k[6], t[2], t[6]);
  tcswapf(k[3], k[7], t[3], t[7]);
  tcswapf(k[2], k[4], t[2], t[4]); tcswapf(k[3], k[5], t[3], t[5]);
  tcswapf(k[1], k[2], t[1], t[2]); tcswapf(k[3], k[4], t[3], t[4]); tcswapf(k[5], k[6], t[5], t[6]);
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f}, cmp[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  float a = l[C_];
  unsigned cnt = 0;
  const float tau_x = (float)GL3::x(2);
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const float b = i < 8 ? k[i] : h[C_];
    if (b > a) {
      const float half = 0.5f * (b - a), mid = 0.5f * (b + a), tau = half * tau_x;
      float Fm[5], d[5];
#pragma unroll
      for (int p = 1; p < 5; ++p) {
        const unsigned c = (cnt >> (2 * (p - 1))) & 3u;
        const bool in = c == 1u;
        Fm[p] = in ? (mid - l[p]) * inv[p] : (c == 2u ? 1.0f : 0.0f);
        d[p] = in ? tau * inv[p] : 0.0f;
      }
      float sp[4];
      gl3_sym_sums_f(Fm, d, sp);
#pragma unroll
      for (int r = 0; r < 4; ++r) kahan_add(acc[r], cmp[r], sp[r] * half);
      a = b;
    }
    if (i < 8) cnt += 1u << (2 * (t[i] >> 1));
  }
  out[0] = (double)(acc[0] * inv[C_]);
  out[1] = (double)(acc[1] * inv[C_]);
  out[2] = (double)((acc[2] + acc[3]) * inv[C_]);
}

__global__ void __launch_bounds__(kClosedThreads) closed_uniform_f32_kernel(
    FieldView f, Window w, double* pmin, double* pmax, double* psad, double* partial) {
  int64_t idx = 0;
  const bool live = vertex(f, w, idx);
  double res[3] = {0.0, 0.0, 0.0};
  if (live) {
    const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
    double lo[5], hi[5];
    bool fast = true;
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      load_bounds(f, at[p], lo[p], hi[p]);
      fast &= fabs(lo[p]) + fabs(hi[p]) <= kFastRatio * (hi[p] - lo[p]);
    }
    if (fast) {
      uniform_integrals_f(lo, hi, res);
    } else {  // tiny supports far from 0 (eps-widened pixels): the fp64 exact mode
      double acc[4];
      uniform_integrals(lo, hi, acc);
      res[0] = acc[0];
      res[1] = acc[1];
      res[2] = acc[2] + acc[3];
    }
    if (pmin) pmin[idx] = res[0];
    if (pmax) pmax[idx] = res[1];
    if (psad) psad[idx] = res[2];
  }
  if (partial) warp_partial_sums(res[0], res[1], res[2], partial);
}

// ------------------------------------------- fused fit + uniform stencil
// One pass over the ensemble for a UNIFORM field: the fit (fields.py:137-143)
// and the closed-form stencil (engine.py:594-629) in the same CTA, so the
// fitted lo / hi reach the stencil through a shared-memory row ring instead of
// HBM, and the FP64 stencil of one row overlaps the TMA stream of the next.
//
// Work item = (column band, segment of vertex rows).  A CTA of kFuseCols
// threads owns the kFuseCols columns [c0, c0 + kFuseCols), c0 a multiple of
// kFuseCols, and walks its segment's rows top to bottom (one halo row above
// and below): per row, ONE 2-D TMA box (kFuseCols pixels x M members,
// UTMALDG) of exactly the band's own 512 bytes per member row -- 128-byte
// aligned, so DRAM moves no byte the band does not use -- lands in a single
// shared stage; each thread reduces its column's members (FMNMX3.NAN /
// FMNMX3) into a 4-row ring of (lo, hi), one barrier, the next row's TMA is
// issued, and vertex row r - 1 is stencilled from ring rows r - 2, r - 1, r.
// Items come from an atomic work counter (persistent CTAs, dynamic balance).
// The band's two edge columns need a neighbouring band's fit: the CTA that
// completes the second of the two bands around a band boundary (a counter per
// segment and boundary, fenced) then computes that boundary's two columns of
// the segment from the fitted planes, still hot in L2 (every item also writes
// its two halo rows, so the segment's own items wrote every pixel those
// vertices read).  2 of 128 vertices, against the 8
// extra halo pixels per member row (12.5 % more DRAM sectors) an overlapping
// box would read.  An edge vertex touching a degenerate pixel is flagged for
// closed_fuse_edges_kernel (it needs the final eps).
//
// The fitted planes are also written (they are the field's params and the
// input of the finish pass).  A band-row whose stencil touches a degenerate
// pixel (lo == hi: the eps widening needs the GLOBAL range, unknown until the
// whole ensemble is read) is not computed here: it is queued in `pending`
// (and flagged) and computed by closed_fuse_pending_kernel once eps is final.
#ifndef CPB_FUSE_SEG
#define CPB_FUSE_SEG 128
#endif
#ifndef CPB_FUSE_MINB
#define CPB_FUSE_MINB 4
#endif
#ifndef CPB_FUSE_EVICT_FIRST  // evict_normal: the halo rows / columns another item re-reads hit L2
#define CPB_FUSE_EVICT_FIRST 0
#endif
constexpr int kFuseCols = 128, kFuseBox = kFuseCols, kFuseRing = kFuseCols + 2;
constexpr int kFuseSeg = CPB_FUSE_SEG;
constexpr int kFuseMaxMembers = 256;
constexpr int kFuseFinishBlocks = 592;

struct FuseArgs {
  int64_t height, width;       // local field (the ensemble holds every row)
  int64_t row_begin, row_end;  // vertex rows to stencil
  int members;
  int nbands, nsegs;
  int64_t nitems;
  float* lo;
  float* hi;
  uint32_t* range;
  double* pmin;
  double* pmax;
  double* psad;
  double* partial;  // (nitems * kFuseCols / 32) warp triples, or null
  int* pending;     // [0] count, then band-rows (row * nbands + band)
  unsigned char* pflag;  // [(row - row_begin) * nbands + band] = 1: pending band-row (zero at launch)
  int* bdone;            // [segment][band boundary 0..nbands] adjacent bands done (zero at launch)
  unsigned char* eflag;  // [edge vertex] = 1: left to the finish pass (degenerate pixel; zero at launch)
  double* edge_partial;  // (nsegs * (nbands + 1) * kFuseCols / 32) warp triples: in-kernel edge vertices
  int* work;        // work counter, zero at launch
  MultiArgs mf;     // NT >= 0: the planes of every fitted model (multi_fit_pixel)
};

CPB_D void fuse_fit_column(const float* col, int M, float& lo, float& hi) {
  lo = __int_as_float(0x7f800000);
  hi = -__int_as_float(0x7f800000);
  int m = 0;
  for (; m + 2 <= M; m += 2) {
    const float x0 = col[m * kFuseBox], x1 = col[(m + 1) * kFuseBox];
    float r3;
    asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r3) : "f"(lo), "f"(x0), "f"(x1));
    lo = r3;
    hi = fmaxf(hi, fmaxf(x0, x1));
  }
  if (m < M) {
    const float x = col[m * kFuseBox];
    float r2;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r2) : "f"(lo), "f"(x));
    lo = r2;
    hi = fmaxf(hi, x);
  }
}

// Edge vertex e of the range: row (e / per_row), boundary b = (e % per_row) / 2,
// column b kFuseCols - 1 + (e & 1) -- the two columns on either side of band
// boundary b (the fused kernel computes columns 1 .. kFuseCols - 2 of a band).
CPB_D int64_t fuse_edge_col(int64_t k) { return (k >> 1) * kFuseCols - 1 + (k & 1); }

// The two edge columns b kFuseCols - 1, b kFuseCols of row segment [v0, v1)
// at band boundary b (both bands around it are done): fitted float planes, no
// eps -- a vertex touching a degenerate pixel is flagged for the finish pass;
// pending band-rows are skipped (the pending pass redoes them whole).  Fixed
// thread mapping, one partial triple per warp per (segment, boundary).
CPB_D void fuse_boundary_edges(const FuseArgs& a, int64_t seg, int64_t b, int64_t v0, int64_t v1) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t per_row = 2 * (int64_t)(a.nbands + 1);
  const int64_t n = 2 * (v1 - v0);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t e = t; e < n; e += kFuseCols) {
    const int64_t lr = (v0 - a.row_begin) + (e >> 1), k = 2 * b + (e & 1), c = fuse_edge_col(k);
    if (c < 1 || c > a.width - 2 || __ldcg(a.pflag + lr * a.nbands + c / kFuseCols)) continue;
    const int64_t idx = (a.row_begin + lr) * a.width + c;
    const int64_t at[5] = {idx, idx + 1, idx - a.width, idx - 1, idx + a.width};
    float rl[5], rh[5];
    bool deg = false;
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      rl[p] = __ldcg(a.lo + at[p]);  // L2: written by other CTAs of this launch
      rh[p] = __ldcg(a.hi + at[p]);
      deg |= !(rh[p] > rl[p]);
    }
    if (deg) {
      a.eflag[lr * per_row + k] = 1;
      continue;
    }
    double lo5[5], hi5[5], acc[4];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      lo5[p] = (double)rl[p];
      hi5[p] = (double)rh[p];
    }
    uniform_integrals_f32keys(rl, rh, lo5, hi5, acc);
    store(a.pmin, a.pmax, a.psad, idx, acc);
    s0 += acc[0];
    s1 += acc[1];
    s2 += acc[2] + acc[3];
  }
  if (a.edge_partial) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, d);
      s1 += __shfl_xor_sync(0xffffffffu, s1, d);
      s2 += __shfl_xor_sync(0xffffffffu, s2, d);
    }
    if (lane == 0) {
      double* q = a.edge_partial + 3 * ((seg * (a.nbands + 1) + b) * (kFuseCols / 32) + warp);
      q[0] = s0;
      q[1] = s1;
      q[2] = s2;
    }
  }
}

// NT < 0: the uniform field alone (min / max per column); NT >= 0: every model
// of a.mf in the same pass (multi_fit_pixel<NT>: NT histogram bins, 0 = none),
// the uniform one stencilled.
template <int NT>
__global__ void __launch_bounds__(kFuseCols, CPB_FUSE_MINB) closed_fuse_uniform_kernel(
    const __grid_constant__ CUtensorMap map, FuseArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int M = a.members, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float* stage = reinterpret_cast<float*>(smem);                            // [M][kFuseBox]
  float2* ring = reinterpret_cast<float2*>(stage + (size_t)M * kFuseBox);  // [4][kFuseRing]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + 4 * kFuseRing);
  __shared__ int64_t s_item;
  __shared__ int s_last2[2];
  if (t == 0) {
    prefetch_tensormap(&map);
    mbar_init(full, 1);
    fence_mbar_init();
  }
#if CPB_FUSE_EVICT_FIRST
  const uint64_t pol = policy_evict_first();
#else
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#endif
  const uint32_t box_bytes = (uint32_t)M * kFuseBox * 4u;
  uint32_t phase = 0;
  float vmin = __int_as_float(0x7f800000), vmax = -__int_as_float(0x7f800000);
  bool bad = false;
  for (;;) {
    __syncthreads();  // the previous item is done with the stage and the ring
    if (t == 0) s_item = atomicAdd(a.work, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= a.nitems) break;
    const int band = (int)(item % a.nbands);
    const int64_t seg = item / a.nbands;
    const int64_t c0 = (int64_t)band * kFuseCols;
    const int64_t v0 = a.row_begin + seg * kFuseSeg;
    const int64_t v1 = min(v0 + (int64_t)kFuseSeg, a.row_end);
    const int64_t f0 = v0 - 1;  // fitted rows [f0, v1]
    const int nfit = (int)(v1 - v0) + 2;
    const int64_t c = c0 + t;
    const bool col_ok = c < a.width;
    if (t == 0) {
      mbar_arrive_expect_tx(full, box_bytes);
      tma_load_2d(stage, &map, (int)(f0 * a.width + c0), 0, full, pol);
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    unsigned degmask = 0;  // bit j % 4: ring row j holds a degenerate pixel
    for (int j = 0; j < nfit; ++j) {
      const int64_t r = f0 + j;
      mbar_wait(full, phase);
      phase ^= 1u;
      // every fitted row is written to the planes, the segment's halo rows
      // included (the neighbouring segment writes the same values): the edge
      // vertices and the finish passes read them there
      const bool live = col_ok && r < a.height;
      float lo, hi;
      if constexpr (NT < 0)
        fuse_fit_column(stage + t, M, lo, hi);
      else
        multi_fit_pixel<NT>(stage + t, kFuseBox, a.mf, r * a.width + c, live, lo, hi);
      float2* rrow = ring + (j & 3) * kFuseRing;
      CPB_ASSERT(1 + t < kFuseRing);
      rrow[1 + t] = make_float2(lo, hi);
      if (live) {
        bad |= ((__float_as_uint(lo) & 0x7f800000u) == 0x7f800000u) |
               ((__float_as_uint(hi) & 0x7f800000u) == 0x7f800000u);
        vmin = fminf(vmin, lo);
        vmax = fmaxf(vmax, hi);
        if (NT < 0) {
          a.lo[r * a.width + c] = lo;
          a.hi[r * a.width + c] = hi;
        }
      }
      const int rowdeg = __syncthreads_or(live && !(hi > lo));
      if (t == 0 && j + 1 < nfit) {  // every thread is done with the stage
        mbar_arrive_expect_tx(full, box_bytes);
        tma_load_2d(stage, &map, (int)((r + 1) * a.width + c0), 0, full, pol);
      }
      degmask = (degmask & ~(1u << (j & 3))) | ((rowdeg ? 1u : 0u) << (j & 3));
      if (j < 2) continue;
      // stencil vertex row r - 1 from ring rows j - 2 (N), j - 1 (C, E, W), j (S)
      const int64_t vr = r - 1;
      const unsigned need = (1u << (j & 3)) | (1u << ((j - 1) & 3)) | (1u << ((j - 2) & 3));
      if (degmask & need) {
        if (t == 0) {
          const int q = atomicAdd(a.pending, 1);
          a.pending[1 + q] = (int)(vr * a.nbands + band);
          a.pflag[(vr - a.row_begin) * a.nbands + band] = 1;
        }
        continue;
      }
      // the band's edge columns t = 0, kFuseCols - 1 need the neighbouring
      // bands' fits: closed_fuse_edges_kernel computes them
      if (t >= 1 && t <= kFuseCols - 2 && c <= a.width - 2) {
        const float2* rn = ring + ((j - 2) & 3) * kFuseRing + 1 + t;
        const float2* rc = ring + ((j - 1) & 3) * kFuseRing + 1 + t;
        const float2* rs = ring + (j & 3) * kFuseRing + 1 + t;
        const float2 pc = rc[0], pe = rc[1], pw = rc[-1], pn = rn[0], ps = rs[0];
        const float rl[5] = {pc.x, pe.x, pn.x, pw.x, ps.x};
        const float rh[5] = {pc.y, pe.y, pn.y, pw.y, ps.y};
        double lo5[5], hi5[5], acc[4];
#pragma unroll
        for (int p = 0; p < 5; ++p) {
          lo5[p] = (double)rl[p];
          hi5[p] = (double)rh[p];
        }
        uniform_integrals_f32keys(rl, rh, lo5, hi5, acc);
        const int64_t idx = vr * a.width + c;
        store(a.pmin, a.pmax, a.psad, idx, acc);
        s0 += acc[0];
        s1 += acc[1];
        s2 += acc[2] + acc[3];
      }
    }
    if (a.partial) {  // this item's warp partials (fixed tree: deterministic)
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, d);
        s1 += __shfl_xor_sync(0xffffffffu, s1, d);
        s2 += __shfl_xor_sync(0xffffffffu, s2, d);
      }
      if (lane == 0) {
        double* q = a.partial + 3 * (item * (kFuseCols / 32) + warp);
        q[0] = s0;
        q[1] = s1;
        q[2] = s2;
      }
    }
    // the second band done around a boundary computes that boundary's edge
    // columns of the segment (boundaries 0 and nbands have one band)
    __threadfence();  // this item's planes and flags before its counts
    __syncthreads();
    if (t < 2) {
      const int b = band + t;
      const int need = (b == 0 || b == a.nbands) ? 1 : 2;
      s_last2[t] = atomicAdd(a.bdone + seg * (a.nbands + 1) + b, 1) == need - 1;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (s_last2[q]) {
        __threadfence();  // the other band's planes and flags
        fuse_boundary_edges(a, seg, band + q, v0, v1);
      }
    }
  }
  merge_range(vmin, vmax, bad, a.range);
}

// The band-rows the fused kernel left for the final eps: the ordinary uniform
// vertex code (load_bounds widens degenerate pixels by eps / 2) over the fitted
// planes.  Block b takes pending entries b, b + grid, ... (fixed order).
// pending[0] == -1 (the fallback when the ensemble cannot be TMA-streamed):
// every band-row of [row_begin, row_end).
__global__ void __launch_bounds__(kFuseCols) closed_fuse_pending_kernel(
    FieldView f, const int* pending, int nbands, int64_t row_begin, int64_t row_end, double* pmin,
    double* pmax, double* psad, double* partial) {
  const int t = threadIdx.x;
  const bool all = pending[0] < 0;
  const int64_t count = all ? (row_end - row_begin) * nbands : pending[0];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t e = blockIdx.x; e < count; e += gridDim.x) {
    const int64_t code = all ? row_begin * nbands + e : pending[1 + e];
    const int64_t vr = code / nbands;
    const int64_t c = (int64_t)(code % nbands) * kFuseCols + t;
    if (c < 1 || c > f.width - 2) continue;
    const int64_t idx = vr * f.width + c;
    const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
    double lo[5], hi[5], acc[4];
#pragma unroll
    for (int p = 0; p < 5; ++p) load_bounds(f, at[p], lo[p], hi[p]);
    uniform_integrals(lo, hi, acc);
    store(pmin, pmax, psad, idx, acc);
    s0 += acc[0];
    s1 += acc[1];
    s2 += acc[2] + acc[3];
  }
  if (partial) warp_partial_sums(s0, s1, s2, partial);
}

// The edge vertices the fused kernel flagged (a degenerate pixel among the
// five: they need the final eps), in a fixed order: the uniform vertex code of
// closed_uniform_kernel over the fitted planes (load_bounds widens degenerate
// pixels by eps / 2).  One edge vertex per thread, one partial triple per warp.
// pending[0] == -1 (no fused pass ran): every edge vertex of the range.
__global__ void __launch_bounds__(kFuseCols) closed_fuse_edges_kernel(
    FieldView f, const int* pending, const unsigned char* pflag, const unsigned char* eflag,
    int nbands, int64_t row_begin, int64_t row_end, double* pmin, double* pmax, double* psad,
    double* partial) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  const int64_t per_row = 2 * (int64_t)(nbands + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pending[0] >= 0 && e < (row_end - row_begin) * per_row && eflag[e]) {
    const int64_t lr = e / per_row, c = fuse_edge_col(e % per_row);
    if (!pflag[lr * nbands + c / kFuseCols]) {
      const int64_t idx = (row_begin + lr) * f.width + c;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      uniform_vertex(f, idx, acc);
      store(pmin, pmax, psad, idx, acc);
      s0 = acc[0];
      s1 = acc[1];
      s2 = acc[2] + acc[3];
    }
  }
  if (partial) warp_partial_sums(s0, s1, s2, partial);
}

// --------------------------------------------------------- combinatorial
// Eq. 5 cross-check for histogram fields (engine.py:320-404, grid chunk
// engine.py:686-702): the sum over every combination of one bin per position
// of (product of the bin masses) x (the all-uniform probability with each
// position uniform on its bin).  One warp per vertex; lanes take combinations
// (C index slowest, itertools.product order) and the all-uniform terms come
// from uniform_integrals; a fixed warp tree adds the lane partials.
// Weights are renormalised like dist.histogram (w / w.sum(), a 1-D numpy
// pairwise sum) and the bin edges are lo + (hi - lo) * k / h
// (_histogram_grid, engine.py:313-317).
constexpr int kCombWarps = 4;
constexpr int COMB_MAX_BINS = 8;  // COMBINATORIAL_MAX_BINS, engine.py:44

__global__ void __launch_bounds__(kCombWarps * 32) combinatorial_kernel(
    FieldView f, int64_t row_begin, int64_t nvert, int64_t cols, double* pmin, double* pmax,
    double* psad) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v = (int64_t)blockIdx.x * kCombWarps + warp;
  if (v >= nvert) return;
  const int h = f.bins;
  const int64_t r = row_begin + v / cols, c = 1 + v % cols;
  const int64_t idx = r * f.width + c;
  const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
  double wn[5][COMB_MAX_BINS], edge[5][COMB_MAX_BINS + 1];
#pragma unroll
  for (int p = 0; p < 5; ++p) {
    double lo, hi;
    const bool deg = load_bounds(f, at[p], lo, hi);
    const int dbin = deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at[p]), lo, hi, h) : 0;
    double w[COMB_MAX_BINS];
#pragma unroll
    for (int b = 0; b < COMB_MAX_BINS; ++b) w[b] = b < h ? load_weight(f, at[p], b, deg, dbin) : 0.0;
    double total = 0.0;  // numpy pairwise sum, h <= 8: sequential below 8 terms
    if (h < 8) {
#pragma unroll
      for (int b = 0; b < COMB_MAX_BINS; ++b)
        if (b < h) total = __dadd_rn(total, w[b]);
    } else {
      total = __dadd_rn(__dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3])),
                        __dadd_rn(__dadd_rn(w[4], w[5]), __dadd_rn(w[6], w[7])));
    }
#pragma unroll
    for (int b = 0; b < COMB_MAX_BINS; ++b) wn[p][b] = b < h ? __ddiv_rn(w[b], total) : 0.0;
    const double width = __dsub_rn(hi, lo);
#pragma unroll
    for (int b = 0; b <= COMB_MAX_BINS; ++b)
      edge[p][b] = b <= h ? __dadd_rn(lo, __ddiv_rn(__dmul_rn(width, (double)b), (double)h)) : 0.0;
  }
  int64_t ncomb = 1;
  for (int p = 0; p < 5; ++p) ncomb *= h;
  double s_min = 0.0, s_max = 0.0, s_sad = 0.0;
  for (int64_t q = lane; q < ncomb; q += 32) {
    int64_t rest = q;
    int ib[5];
#pragma unroll
    for (int p = 4; p >= 0; --p) {
      ib[p] = (int)(rest % h);
      rest /= h;
    }
    double wprod = 1.0, lo[5], hi[5];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      double wb = 0.0, a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < COMB_MAX_BINS; ++k) {
        if (k == ib[p]) {
          wb = wn[p][k];
          a = edge[p][k];
          b = edge[p][k + 1];
        }
      }
      wprod = __dmul_rn(wprod, wb);
      lo[p] = a;
      hi[p] = b;
    }
    if (wprod == 0.0) continue;
    double t[4];
    uniform_integrals(lo, hi, t);
    s_min = fma(wprod, t[0], s_min);
    s_max = fma(wprod, t[1], s_max);
    s_sad = fma(wprod, t[2] + t[3], s_sad);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    s_min += __shfl_xor_sync(0xffffffffu, s_min, d);
    s_max += __shfl_xor_sync(0xffffffffu, s_max, d);
    s_sad += __shfl_xor_sync(0xffffffffu, s_sad, d);
  }
  if (lane == 0) {
    if (pmin) pmin[idx] = s_min;
    if (pmax) pmax[idx] = s_max;
    if (psad) psad[idx] = s_sad;
  }
}

// ------------------------------------------------------------ epanechnikov
// pdf_C = 0.75/hw_C (1 - u^2), u unclipped; F_P = 0.5 + 0.75u - 0.25u^3 with
// u clipped to [-1, 1] (engine.py:521-533); 8-node Gauss-Legendre (degree 14).
// Outside a neighbour's support the affine form pins u to -1 or +1, where the
// cubic gives exactly 0 or 1.
CPB_D double epan_cdf(double u) { return fma(u, fma(-0.25, u * u, 0.75), 0.5); }

// Exact-mode Epanechnikov piece (a vertex outside the fast-mode ratio, see
// kFastRatio): 8 nodes, every node x rounded like the reference's
// mids + halves * xi before the subtraction.  The neighbour states (2 bits
// each, from the merge tags: 0 below, 1 inside, 2 above) replace midpoint
// comparisons.
CPB_D void epan_piece_exact(double a, double b, const double* m, const double* ih, unsigned state,
                            double s[4]) {
  const double pdf0 = 0.75 * ih[C_];
  const double half = 0.5 * (b - a), mid = 0.5 * (b + a);
  double al[5], be[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    const unsigned c = (state >> (2 * (p - 1))) & 3u;
    const bool in = c == 1u;
    be[p] = in ? ih[p] : 0.0;
    al[p] = in ? 0.0 : (c == 2u ? 1.0 : -1.0);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) s[r] = 0.0;  // s[2] = t1 + t2, s[3] stays 0
#pragma unroll
  for (int j = 0; j < GL8::n; ++j) {
    const double x = node_x(mid, half, GL8::x(j));
    const double uc = (x - m[C_]) * ih[C_];
    const double wp = GL8::w(j) * (pdf0 * fma(-uc, uc, 1.0));
    double F[5], g[3];
#pragma unroll
    for (int p = 1; p < 5; ++p) F[p] = epan_cdf(fma(x - m[p], be[p], al[p]));
    integrands3(F, g);
#pragma unroll
    for (int r = 0; r < 3; ++r) s[r] = fma(wp, g[r], s[r]);
  }
}

// Fast-mode Epanechnikov piece with nn symmetric Gauss-Legendre nodes
// (nn = 3, 5, 6 or 8, warp-uniform; the nodes and weights are read from
// c_glsym).  On a piece where k of the four neighbour CDFs are non-constant
// (the others are pinned to an exact 0 or 1 by their state) the integrands
// have degree 2 + 3k, so nn = 3, 5, 6, 8 nodes integrate them exactly for
// k <= 1, 2, 3, 4 (the reference always uses 8, engine.py:600-601; the
// difference is rounding).  One loop over the node pairs for every nn keeps
// the kernel small (four unrolled variants thrashed the instruction cache).
CPB_D void epan_piece_n(double a, double b, const double* m, const double* ih, unsigned state,
                        int nn, double s[4]) {
  const double pdf0 = 0.75 * ih[C_];
  const double half = 0.5 * (b - a), mid = 0.5 * (b + a);
  double al[5], be[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    const unsigned c = (state >> (2 * (p - 1))) & 3u;
    const bool in = c == 1u;
    be[p] = in ? ih[p] : 0.0;
    al[p] = in ? (mid - m[p]) * ih[p] : (c == 2u ? 1.0 : -1.0);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) s[r] = 0.0;  // s[2] = t1 + t2, s[3] stays 0
  const double uc0 = (mid - m[C_]) * ih[C_];
  auto node = [&](double t, double wpj) {
    const double uc = fma(t, ih[C_], uc0);
    const double wp = wpj * fma(-uc, uc, 1.0);
    double F[5], g[3];
#pragma unroll
    for (int p = 1; p < 5; ++p) F[p] = epan_cdf(fma(t, be[p], al[p]));
    integrands3(F, g);
#pragma unroll
    for (int r = 0; r < 3; ++r) s[r] = fma(wp, g[r], s[r]);
  };
  const int pairs = nn >> 1;
  const int off = nn == 3 ? 2 : (nn == 5 ? 5 : (nn == 6 ? 10 : 16));
#pragma unroll 1
  for (int j = 0; j < pairs; ++j) {
    const double tau = half * c_glsym[off + j];
    const double wpj = c_glsym[off + pairs + j] * pdf0;
    node(-tau, wpj);
    node(tau, wpj);
  }
  if (nn & 1) node(0.0, c_glsym[off + 2 * pairs] * pdf0);
}

// Piece-parallel Epanechnikov stencil.  With one vertex per lane, a warp
// iterates over the UNION of its lanes' pieces (9 on smooth fields) although a
// vertex has ~5 non-empty pieces, so ~45 % of the 8-node piece evaluations are
// idle lanes.  Here each lane first builds its vertex's non-empty pieces; the
// warp compacts all of them into one list (warp prefix sum) and then evaluates
// it 32 pieces per round, each lane reading its piece's vertex constants from
// shared memory.  The list is sorted by piece degree class (counting sort with
// one packed warp scan) so each round runs ONE node count on all lanes -- the
// largest its pieces need (epan_piece_n): ~5.4 instead of 8 node evaluations
// per piece on smooth fields.  A warp owns 32 consecutive vertices of one row
// (row-aligned segments), so the rounds a vertex's pieces fall in, and hence
// its rounding, do not depend on how the rows are split into launches, slabs
// or chunks.  Per-piece results land in shared memory and every vertex sums
// its own pieces in a fixed order (class, then piece), so the result is
// deterministic.
constexpr int kPPWarps = 4;

// closed_pp_kernel's per-warp layout: ROWS rows of vertex constants
// (Epanechnikov m, ih, plus the MX float copies), the piece ends, and per slot
// the (owner lane, neighbour states, degree class) word in the r2 slot.  Slot
// e is read and written only by lane e % 32, so its results overwrite its own
// (a, b, owner) words, and the vertex's fast-mode flag is the sign of its
// centre ih row.  Epanechnikov fp64: 9.25 KB per warp, six 4-warp blocks per
// SM (24 warps).
template <int ROWS>
struct PPSmem {
  double vd[ROWS][32];
  double pa[9 * 32], pb[9 * 32];  // piece ends, then results min / max
  double r2[9 * 32];              // owner | state << 8 | class << 16, then result saddle (t1 + t2)
};

// Mixed-precision Epanechnikov piece (CPB_FLAG_MIXED): positions re-centred on
// the centre mean in float64 by the owner lane, the 8-node evaluation in FP32.
CPB_D float epan_cdf_f(float u) { return fmaf(u, fmaf(-0.25f, u * u, 0.75f), 0.5f); }

CPB_D void integrands_f(const float* F, float g[4]) {
  const float sE = 1.0f - F[E_], sN = 1.0f - F[N_], sW = 1.0f - F[W_], sS = 1.0f - F[S_];
  const float sesw = sE * sW, snss = sN * sS;
  const float fefw = F[E_] * F[W_], fnfs = F[N_] * F[S_];
  g[0] = sesw * snss;
  g[1] = fefw * fnfs;
  g[2] = sesw * fnfs;
  g[3] = snss * fefw;
}

CPB_D void epan_piece_f(float a, float b, const float* m, const float* ih, unsigned state,
                        float s[4]) {
  const float pdf0 = 0.75f * ih[C_];
  const float half = 0.5f * (b - a), mid = 0.5f * (b + a);
  float al[5], be[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    const unsigned c = (state >> (2 * (p - 1))) & 3u;
    const bool in = c == 1u;
    be[p] = in ? ih[p] : 0.0f;
    al[p] = in ? (mid - m[p]) * ih[p] : (c == 2u ? 1.0f : -1.0f);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) s[r] = 0.0f;
  const float uc0 = (mid - m[C_]) * ih[C_];
#pragma unroll
  for (int j = 0; j < GL8::n / 2; ++j) {
    const float tau = half * (float)GL8::x(7 - j);
    const float wj = (float)GL8::w(j);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const float t = side ? tau : -tau;
      const float uc = fmaf(t, ih[C_], uc0);
      const float wp = wj * (pdf0 * fmaf(-uc, uc, 1.0f));
      float F[5], g[4];
#pragma unroll
      for (int p = 1; p < 5; ++p) F[p] = epan_cdf_f(fmaf(t, be[p], al[p]));
      integrands_f(F, g);
#pragma unroll
      for (int r = 0; r < 4; ++r) s[r] = fmaf(wp, g[r], s[r]);
    }
  }
}

// Vertex constants m[5], ih[5] (+ MX: their float copies re-centred on m_C).
template <bool MX>
__global__ void __launch_bounds__(kPPWarps * 32, 6) closed_pp_kernel(
    FieldView f, int64_t row_begin, int64_t row_end, int64_t cols, int64_t segs, double* pmin,
    double* pmax, double* psad, double* partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int ROWS = MX ? 15 : 10;
  constexpr int FR = 5;  // centre ih row: sign = !fast
  PPSmem<ROWS>& S = reinterpret_cast<PPSmem<ROWS>*>(smem_raw)[warp];
  const int64_t g = (int64_t)blockIdx.x * kPPWarps + warp;  // row segment
  const int64_t r = row_begin + g / segs, c = 1 + (g % segs) * 32 + lane;
  const bool live = r < row_end && c <= cols;
  int64_t idx = 0;
  int n = 0;
  double pts[10];
  int tg[8];
  double mref = 0.0;  // MX: the centre mean, origin of the float coordinates
  bool vfast = false;
  if (live) {
    idx = r * f.width + c;
    const int64_t at[5] = {idx, idx + 1, idx - f.width, idx - 1, idx + f.width};
    double lo[5], hi[5];
    bool fast = true;
    {
      double m[5], ih[5], sd[5];
      // all ten loads (and eps) in flight before any use: the division's
      // slow-path call below would otherwise serialise them per position
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        m[p] = __ldg(f.mean + at[p]);
        sd[p] = __ldg(f.spread + at[p]);
      }
      const double heps = __dmul_rn(0.5, field_eps(f));
      mref = m[0];
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        const double ks = __dmul_rn(f.k, sd[p]);
        const double hw = ks > heps ? ks : (heps > ks ? heps : ks);  // load_epan (fields.py:156)
        ih[p] = 1.0 / hw;
        lo[p] = m[p] - hw;  // _support_bounds, engine.py:502-505
        hi[p] = m[p] + hw;
        fast &= (fabs(m[p]) + hw) * ih[p] <= kFastRatio;
      }
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        S.vd[p][lane] = m[p];
        S.vd[5 + p][lane] = ih[p];
      }
      if (MX) {  // float copies re-centred on the centre mean (fp64 subtraction), rows 10..
        float* vf = reinterpret_cast<float*>(&S.vd[10][0]);
#pragma unroll
        for (int p = 0; p < 5; ++p) {
          vf[p * 32 + lane] = (float)(m[p] - m[C_]);
          vf[(5 + p) * 32 + lane] = (float)ih[p];
        }
      }
    }
    if (!fast) S.vd[FR][lane] = -S.vd[FR][lane];
    vfast = fast;
    double k[8];
#pragma unroll
    for (int p = 1; p < 5; ++p) {
      k[2 * p - 2] = dmin(dmax(lo[p], lo[C_]), hi[C_]);
      k[2 * p - 1] = dmin(dmax(hi[p], lo[C_]), hi[C_]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) tg[q] = q;
    merge_pairs8_tagged(k, tg);
    pts[0] = lo[C_];
#pragma unroll
    for (int q = 0; q < 8; ++q) pts[q + 1] = k[q];
    pts[9] = hi[C_];
#pragma unroll
    for (int i = 0; i < 9; ++i) n += pts[i + 1] > pts[i] ? 1 : 0;
  }
  // Class of a piece from k, the number of neighbours inside their support on
  // it (+1 per lo crossed, -1 per hi crossed): 0 = 8 nodes (k = 4, and every
  // piece of an exact-mode or mixed-precision vertex), 1 = 6 (k = 3), 2 = 5
  // (k = 2), 3 = 3 nodes (k <= 1).  Counts of classes 0..2 are packed 9-bit
  // fields of one word (a warp holds <= 288 pieces); class 3 is the rest.
  auto piece_class = [&](int kin) -> int {
    if (MX || !vfast) return 0;
    return kin >= 4 ? 0 : 4 - max(kin, 1);
  };
  unsigned mine = 0;  // my pieces of classes 0..2
  if (live) {
    int kin = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (pts[i + 1] > pts[i]) {
        const int cl = piece_class(kin);
        mine += cl < 3 ? 1u << (9 * cl) : 0u;
      }
      if (i < 8) kin += (tg[i] & 1) ? -1 : 1;
    }
  }
  // warp scans of the packed class counts and of the piece counts
  unsigned incl = mine;
  int incn = n;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, d);
    const int yn = __shfl_up_sync(0xffffffffu, incn, d);
    if (lane >= d) {
      incl += y;
      incn += yn;
    }
  }
  const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
  const int total = __shfl_sync(0xffffffffu, incn, 31);
  const int t0 = (int)(tot & 511u), t1 = (int)((tot >> 9) & 511u), t2 = (int)((tot >> 18) & 511u);
  // first positions of my pieces: classes 0..2 packed (class bases added), class 3
  const unsigned ex = incl - mine;
  const unsigned start = ex + ((unsigned)t0 << 9) + ((unsigned)(t0 + t1) << 18);
  const int ex3 = (incn - n) - (int)(ex & 511u) - (int)((ex >> 9) & 511u) - (int)((ex >> 18) & 511u);
  const int start3 = t0 + t1 + t2 + ex3;
  if (live) {
    unsigned pos = start;
    int pos3 = start3;
    unsigned cnt = 0;
    int kin = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (pts[i + 1] > pts[i]) {
        const int cl = piece_class(kin);
        int q;
        if (cl < 3) {
          q = (int)((pos >> (9 * cl)) & 511u);
          pos += 1u << (9 * cl);
        } else {
          q = pos3++;
        }
        CPB_ASSERT(q < 9 * 32);
        if (MX && vfast) {  // float position in the first word of the slot
          reinterpret_cast<float*>(&S.pa[q])[0] = (float)(pts[i] - mref);
          reinterpret_cast<float*>(&S.pb[q])[0] = (float)(pts[i + 1] - mref);
        } else {
          S.pa[q] = pts[i];
          S.pb[q] = pts[i + 1];
        }
        reinterpret_cast<unsigned*>(&S.r2[q])[0] = (unsigned)lane | (cnt << 8) | ((unsigned)cl << 16);
      }
      if (i < 8) {
        cnt += 1u << (2 * (tg[i] >> 1));
        kin += (tg[i] & 1) ? -1 : 1;
      }
    }
  }
  __syncwarp();
  for (int e0 = 0; e0 < total; e0 += 32) {
    const int e = e0 + lane;
    const bool act = e < total;
    const unsigned os = act ? reinterpret_cast<const unsigned*>(&S.r2[e])[0] : 0u;
    const int cl = act ? (int)((os >> 16) & 7u) : 7;
    // the round runs the node count its most demanding piece needs (the list is
    // sorted by class, so rounds are uniform except at class boundaries)
    const int rc = __reduce_min_sync(0xffffffffu, cl);
    if (!act) continue;
    const int o = (int)(os & 0xffu);
    CPB_ASSERT(e < 9 * 32 && o < 32);
    const unsigned st = (os >> 8) & 0xffu;
    const bool vf_ = S.vd[FR][o] > 0.0;
    const double a = S.pa[e], b = S.pb[e];
    if (MX && vf_) {
      const float* vf = reinterpret_cast<const float*>(&S.vd[10][0]);
      float mf[5], ihf[5], sf[4];
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        mf[p] = vf[p * 32 + o];
        ihf[p] = vf[(5 + p) * 32 + o];
      }
      const float fa = reinterpret_cast<const float*>(&S.pa[e])[0];
      const float fb = reinterpret_cast<const float*>(&S.pb[e])[0];
      epan_piece_f(fa, fb, mf, ihf, st, sf);
      const double hf = 0.5 * (double)(fb - fa);
      S.pa[e] = (double)sf[0] * hf;
      S.pb[e] = (double)sf[1] * hf;
      S.r2[e] = (double)(sf[2] + sf[3]) * hf;
      continue;
    }
    double m[5], ih[5], s[4];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      m[p] = S.vd[p][o];
      ih[p] = p == 0 ? fabs(S.vd[5][o]) : S.vd[5 + p][o];
    }
    if (!vf_) epan_piece_exact(a, b, m, ih, st, s);
    else epan_piece_n(a, b, m, ih, st, rc == 0 ? 8 : (rc == 1 ? 6 : (rc == 2 ? 5 : 3)), s);
    const double half = 0.5 * (b - a);
    S.pa[e] = s[0] * half;
    S.pb[e] = s[1] * half;
    S.r2[e] = s[2] * half + s[3] * half;
  }
  __syncwarp();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (live) {
    // my pieces of class q are contiguous from their first position; sum class by class
    const int n3 = n - (int)(mine & 511u) - (int)((mine >> 9) & 511u) - (int)((mine >> 18) & 511u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int b0 = q < 3 ? (int)((start >> (9 * q)) & 511u) : start3;
      const int nq = q < 3 ? (int)((mine >> (9 * q)) & 511u) : n3;
      for (int e = b0; e < b0 + nq; ++e) {
        acc[0] += S.pa[e];
        acc[1] += S.pb[e];
        acc[2] += S.r2[e];
      }
    }
    store(pmin, pmax, psad, idx, acc);
  }
  if (partial) warp_partial_sums(acc[0], acc[1], acc[2] + acc[3], partial);
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
// block stages the 3 x (TW + 2) pixels the stencil touches -- support bounds
// and the renormalised weights wn = w / sum(w) (numpy pairwise order for the
// sum) -- in float64 shared memory; then every thread sweeps its five sorted
// edge lists in merge order (the partition of engine.py:580-582 without a
// sort), carrying each neighbour's current bin and running prefix sum
// (np.cumsum order) from piece to piece.  The per-edge advance is written as
// selects, not branches, so lanes advancing different neighbours never
// diverge.
constexpr int kHistSmemMaxBins = 64;
constexpr int kHistThreads = 128;

struct Nb {          // one neighbour: constants + state inside the current piece
  double lo, width, binw;
  int i;             // staged pixel index
  int j;             // current bin; -1 below the support, h above it
  double next;       // next edge strictly ahead (+inf when none)
  double c, s, e;    // F(x) = c + s (x - e); c = prefix sum of wn below bin j
};

template <int MINB>
__global__ void __launch_bounds__(kHistThreads, MINB) closed_hist_smem_kernel(
    FieldView f, Window w, double* pmin, double* pmax, double* psad) {
  extern __shared__ double sm[];
  const int TW = blockDim.x, sw = TW + 2, n = 3 * sw, h = f.bins;
  // layout: lo[n] hi[n] ibinw[n] wn[h][n] kh[h+1]
  const int o_hi = n, o_ib = 2 * n, o_wn = 3 * n, o_kh = (3 + h) * n;
  const int64_t tile = blockIdx.x % w.ntiles;
  const int64_t r = w.row_begin + blockIdx.x / w.ntiles;
  const int64_t c0 = tile * TW;  // staged columns [c0, c0 + sw)
  for (int k = threadIdx.x; k <= h; k += TW) sm[o_kh + k] = (double)k / (double)h;
  const double invM = 1.0 / (double)f.members;
  for (int i = threadIdx.x; i < n; i += TW) {
    const int64_t rr = r - 1 + i / sw, cc = c0 + i % sw;
    if (cc >= f.width) continue;
    const int64_t at = rr * f.width + cc;
    double lo, hi;
    const bool deg = load_bounds(f, at, lo, hi);
    const int dbin = deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at), lo, hi, h) : 0;
    for (int b = 0; b < h; ++b) {
      double wb;
      if (f.wmode == CPB_WEIGHTS_F64) {
        wb = __ldg(static_cast<const double*>(f.weights) + (int64_t)b * f.wstride + at);
      } else if (deg) {
        wb = b == dbin ? 1.0 : 0.0;
      } else {
        const unsigned cnt = f.wmode == CPB_WEIGHTS_U8
            ? (unsigned)__ldg(static_cast<const uint8_t*>(f.weights) + (int64_t)b * f.wstride + at)
            : (unsigned)__ldg(static_cast<const uint16_t*>(f.weights) + (int64_t)b * f.wstride + at);
        wb = (double)cnt * invM;  // count / M to within an ulp (closed-form tolerance)
      }
      sm[o_wn + b * n + i] = wb;
    }
    const double total = pairwise_sum([&](int b) { return sm[o_wn + b * n + i]; }, h);
    const double it = 1.0 / total;
    for (int b = 0; b < h; ++b) sm[o_wn + b * n + i] *= it;
    sm[i] = lo;
    sm[o_hi + i] = hi;
    sm[o_ib + i] = 1.0 / ((hi - lo) / (double)h);
  }
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t c = c0 + 1 + t;
  if (c >= f.width - 1) return;
  const int64_t idx = r * f.width + c;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double dh = (double)h;
  const int ic = sw + t + 1;
  const double x0 = sm[ic], xend = sm[o_hi + ic];
  bool fast = true;  // see kFastRatio: all five |x| / bin width within bounds
  {
    const int li[5] = {sw + t + 1, sw + t + 2, t + 1, sw + t, 2 * sw + t + 1};
#pragma unroll
    for (int p = 0; p < 5; ++p)
      fast &= (fabs(sm[li[p]]) + fabs(sm[o_hi + li[p]])) * sm[o_ib + li[p]] <= kFastRatio;
  }
  Nb nb[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    const int li = p == E_ ? sw + t + 2 : (p == N_ ? t + 1 : (p == W_ ? sw + t : 2 * sw + t + 1));
    Nb& q = nb[p];
    q.i = li;
    q.lo = sm[li];
    q.width = sm[o_hi + li] - q.lo;
    q.binw = q.width / dh;
    q.j = -1; q.c = 0.0; q.s = 0.0; q.e = 0.0;
    q.next = q.lo;
  }
  // one merge step of neighbour q, applied when `adv` (selects, no branches)
  auto step = [&](Nb& q, bool adv) {
    const int j1 = q.j + 1;
    const bool in = j1 < h;
    const double w1 = sm[o_wn + (in ? j1 : h - 1) * n + q.i];
    const double w0 = (q.j >= 0 && q.j < h) ? sm[o_wn + q.j * n + q.i] : 0.0;
    const double kh = sm[o_kh + (j1 + 1 < h ? j1 + 1 : h)];
    const double nxt = j1 + 1 < h ? fma(q.width, kh, q.lo) : (j1 + 1 == h ? sm[o_hi + q.i] : inf);
    const double c1 = q.c + w0;                          // np.cumsum order
    const double e1 = fma(q.binw, (double)j1, q.lo);     // lo + binw * j (distributions.py:97)
    q.j = adv ? j1 : q.j;
    q.c = adv ? (in ? c1 : 1.0) : q.c;
    q.s = adv ? (in ? w1 * sm[o_ib + q.i] : 0.0) : q.s;
    q.e = adv ? (in ? e1 : 0.0) : q.e;
    q.next = adv ? (in ? nxt : inf) : q.next;
  };
#pragma unroll
  for (int p = 1; p < 5; ++p)
    while (nb[p].next <= x0) step(nb[p], true);
  const double cwidth = xend - x0, cibinw = sm[o_ib + ic];
  int jc = 0;
  double pdf = sm[o_wn + ic] * cibinw;
  double nextc = h > 1 ? fma(cwidth, sm[o_kh + 1], x0) : xend;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double x = x0;
  while (x < xend) {
    const double xn =
        dmin(dmin(nextc, dmin(nb[E_].next, nb[N_].next)), dmin(nb[W_].next, nb[S_].next));
    // the piece [x, xn]; coincident edges give a zero-width piece worth exactly 0
    const double half = 0.5 * (xn - x), mid = 0.5 * (xn + x);
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (fast) {
      double Fm[5], F[5], g[4];
      const double tau = half * GL3::x(2);
#pragma unroll
      for (int p = 1; p < 5; ++p) Fm[p] = fma(mid - nb[p].e, nb[p].s, nb[p].c);
      integrands(Fm, g);
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] = GL3::w(1) * g[q];
#pragma unroll
      for (int side = 0; side < 2; ++side) {
#pragma unroll
        for (int p = 1; p < 5; ++p) F[p] = fma(side ? tau : -tau, nb[p].s, Fm[p]);
        integrands(F, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fma(GL3::w(0), g[q], s[q]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < GL3::n; ++j) {
        const double xx = node_x(mid, half, GL3::x(j));
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p) F[p] = fma(xx - nb[p].e, nb[p].s, nb[p].c);
        integrands(F, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fma(GL3::w(j), g[q], s[q]);
      }
    }
    bool m[4];
    range_masks(nb[E_].j < 0, nb[N_].j < 0, nb[W_].j < 0, nb[S_].j < 0, nb[E_].j >= h,
                nb[N_].j >= h, nb[W_].j >= h, nb[S_].j >= h, m);
    const double scale = pdf * half;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double add = fma(s[q], scale, acc[q]);
      acc[q] = m[q] ? add : acc[q];
    }
    {  // centre list
      const bool adv = nextc == xn;
      const int j1 = jc + 1;
      const double pdf1 = sm[o_wn + (j1 < h ? j1 : h - 1) * n + ic] * cibinw;
      const double kh = sm[o_kh + (j1 + 1 < h ? j1 + 1 : h)];
      const double nx1 = j1 + 1 < h ? fma(cwidth, kh, x0) : (j1 + 1 == h ? xend : inf);
      jc = adv ? j1 : jc;
      pdf = adv ? pdf1 : pdf;
      nextc = adv ? nx1 : nextc;
    }
#pragma unroll
    for (int p = 1; p < 5; ++p) step(nb[p], nb[p].next == xn);
    x = dmax(x, xn);
  }
  store(pmin, pmax, psad, idx, acc);
}

// Table-driven histogram stencil (the production path for bins <= kTabMaxBins).
// A block computes a TH x TW tile of vertices.  It stages the (TH + 2) x
// (TW + 2) pixels around the tile as per-pixel STATE TABLES: for every
// position k in the merged sweep (k = 0 below the support, k = b + 1 inside
// bin b, k = h + 1 above) the CDF on that stretch is
// F(x) = CUM[k] + SL[k] (x - EV[k]) and the next edge ahead is NX[k].  CUM is
// the sequential prefix sum of wn = w / sum(w) (np.cumsum and numpy pairwise
// sum orders, engine.py:538-540), SL = wn / binw, EV = lo + binw b
// (distributions.py:97) and NX the kinks of engine.py:570-571 (the last one is
// the support end itself).  The sweep over the five sorted edge lists then
// only increments integer positions and re-reads four table entries (one
// address, constant offsets), with no floating-point bookkeeping and no
// divergent branches.
constexpr int kTabTW = 32, kTabTH = 8, kTabMaxBins = 16;
constexpr int kTabSW = kTabTW + 2, kTabP = kTabSW * (kTabTH + 2);

// numpy pairwise summation of exactly N <= 8 terms (sequential below 8, one
// 8-accumulator tree at 8)
template <int N>
CPB_D double pairwise_small(const double* w) {
  if (N < 8) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) r = __dadd_rn(r, w[i]);
    return r;
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(w[0], w[1 % N]), __dadd_rn(w[2 % N], w[3 % N])),
                   __dadd_rn(__dadd_rn(w[4 % N], w[5 % N]), __dadd_rn(w[6 % N], w[7 % N])));
}

// numpy pairwise summation of w[0..n) for n <= 16 (register array, unrolled)
CPB_D double pairwise16(const double* w, int n) {
  if (n < 8) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < n) r = __dadd_rn(r, w[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = w[j];
  if (n == 16) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], w[8 + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
  for (int i = 8; i < 16; ++i)
    if (n < 16 && i < n) res = __dadd_rn(res, w[i]);
  return res;
}

// The merged sweep of one vertex over its five state-table lists (see
// closed_hist_tab_kernel).  FAST (all five pixels fast-mode): midpoint CDFs
// B + (SL/2) s2 and symmetric node pairs; the lists then never need EV, so an
// advance reads (B, SL/2) and NX only.
template <bool FAST>
CPB_D void hist_sweep(const double* T, int h, const int* ip, const bool* pf, double acc[4]) {
  constexpr int P = kTabP;
  double accs[3] = {0.0, 0.0, 0.0};  // FAST: node-pair sums (acc holds the midpoint ones)
  constexpr int K4 = 4 * P;
  const double x0 = T[2 * P + 2 * ip[0] + 1];                     // lo_C (NX of state 0)
  // each list is a pointer to its current state's table column; advancing
  // is one predicated add of the state stride
  const double* tp[5];
  double cc_[5], ss[5], ee[5], nx[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    // first state whose next edge lies beyond lo_C: the first three edges
    // tested with independent loads (one shared-memory latency for all four
    // lists), the rare rest by walking
    const double* t = T + 2 * ip[p];
    const int k = (t[2 * P + 1] <= x0) + (t[K4 + 2 * P + 1] <= x0) + (t[2 * K4 + 2 * P + 1] <= x0);
    t += k * K4;
    if (k == 3)
      while (t[2 * P + 1] <= x0) t += K4;
    CPB_ASSERT(t >= T && t < T + (size_t)(h + 2) * K4);
    tp[p] = t;
    const double2 a = *reinterpret_cast<const double2*>(t);
    cc_[p] = a.x;
    ss[p] = a.y;
    if (FAST) {
      ee[p] = 0.0;
      nx[p] = t[2 * P + 1];
    } else {
      const double2 b = *reinterpret_cast<const double2*>(t + 2 * P);
      ee[p] = b.x;
      nx[p] = b.y;
    }
  }
  const double* tcp = T + K4 + 2 * ip[0];
  double pdf = tcp[1], nextc = tcp[2 * P + 1];
  double x = x0;
  // x reaches hi_C exactly when the centre list leaves its last bin (its
  // next edge bounds every xn), so the loop test is a pointer compare
  const double* const tend = T + (size_t)(h + 1) * K4 + 2 * ip[0];
  while (tcp != tend) {
    const double xn = dmin(dmin(nextc, dmin(nx[E_], nx[N_])), dmin(nx[W_], nx[S_]));
    // the piece [x, xn]; coincident edges give a zero-width piece worth exactly 0
    // (ss = SL / 2, pdf = SL_C / 2: the halves of half and mid are folded in)
    const double s2 = xn + x, hd = xn - x;
    double s[4];
    const double scale = pdf * hd;
    if (FAST) {
      double Fm[5], d[5];
      const double tau = hd * GL3::x(2);
#pragma unroll
      for (int p = 1; p < 5; ++p) {
        Fm[p] = fma(ss[p], s2, cc_[p]);
        d[p] = tau * ss[p];
      }
      double gs[3];
      gl3_sym_parts3(Fm, d, gs, s);
#pragma unroll
      for (int q = 0; q < 3; ++q) accs[q] = fma(gs[q], scale, accs[q]);
    } else {
      const double half = 0.5 * hd, mid = 0.5 * s2;
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] = 0.0;
#pragma unroll
      for (int j = 0; j < GL3::n; ++j) {
        const double xx = node_x(mid, half, GL3::x(j));
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p)
          F[p] = pf[p] ? fma(2.0 * ss[p], xx, cc_[p]) : fma(xx - ee[p], 2.0 * ss[p], cc_[p]);
        integrands(F, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fma(GL3::w(j), g[q], s[q]);
      }
      s[2] += s[3];
    }
    // No range masks: outside an integral's range some factor is an exact 0
    // (a neighbour below its support has F = 0, above it S = 1 - 1 = 0), so
    // the piece adds exactly 0 -- the range limits of engine.py:603-628 are
    // implied by the clipped CDFs.
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[q] = fma(s[q], scale, acc[q]);  // acc[3] stays 0
    // advance every list whose next edge is xn; only those lanes re-read
    // their state (predicated loads: shared-memory wavefronts, not the FP64
    // pipe, were the busiest unit with all five lists re-read every piece)
    if (nextc == xn) {
      tcp += K4;
      CPB_ASSERT(tcp < T + (size_t)(h + 2) * K4);
      pdf = tcp[1];
      nextc = tcp[2 * P + 1];
    }
#pragma unroll
    for (int p = 1; p < 5; ++p) {
      if (nx[p] == xn) {
        tp[p] += K4;
        CPB_ASSERT(tp[p] < T + (size_t)(h + 2) * K4);
        const double2 a = *reinterpret_cast<const double2*>(tp[p]);
        cc_[p] = a.x;
        ss[p] = a.y;
        if (FAST) {
          nx[p] = tp[p][2 * P + 1];
        } else {
          const double2 b = *reinterpret_cast<const double2*>(tp[p] + 2 * P);
          ee[p] = b.x;
          nx[p] = b.y;
        }
      }
    }
    x = xn;  // every next edge lies beyond x, so the partition only moves forward
  }
  if (FAST) {  // the Gauss-Legendre weights, once per vertex
    const double w1 = GL3::w(1), w0x2 = 2.0 * GL3::w(0);
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[q] = fma(w0x2, accs[q], w1 * acc[q]);
  }
}

// HB: bin count when <= 8 (compile-time: exact-size staging loops), else 16
// (runtime bins 9..16).
// Register cap: 2 blocks of 256 threads per SM (shared memory allows no more);
// at <= 6 bins 96 registers measured 0.6 % faster than the 112 the compiler
// picks under __launch_bounds__(256, 2) (88: spills; 104: 4 % slower).
template <int HB>
__global__ void __maxnreg__(HB <= 6 ? 96 : 128) closed_hist_tab_kernel(
    FieldView f, int64_t row_begin, int64_t row_end, int ctiles, double* pmin, double* pmax,
    double* psad, double* partial) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = kTabP, SW = kTabSW;
  const int h = HB <= 8 ? HB : f.bins;
  // [(h + 2) states][2 pairs][P pixels] of double2: (CUM, SL) then (EV, NX), so
  // a list advance is two 16-byte loads (conflict-free: 8 lanes x 16 B)
  // The EV slot of the below-support state (never read as EV: its SL is 0)
  // holds the fast-mode flag, 0 when (|lo| + |hi|) / binw <= kFastRatio.
  // The first pair holds (B, SL / 2): on a fast-mode pixel B = CUM - SL EV,
  // so on a piece with midpoint sum s2 = a + b the CDF at the midpoint is one
  // FMA, B + (SL / 2) s2 (|SL EV| <= kFastRatio there bounds the cancellation
  // to ~1e-14); on the other pixels B = CUM (exact-mode evaluation).
  double* T = sm;
  const int64_t r0 = row_begin + (int64_t)(blockIdx.x / ctiles) * kTabTH;
  const int64_t c0 = (int64_t)(blockIdx.x % ctiles) * kTabTW;  // staged cols [c0, c0 + SW)
  const int tid = threadIdx.y * kTabTW + threadIdx.x;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double dh = (double)h, invM = 1.0 / (double)f.members;
  // per-pixel state tables from (lo, hi, raw weights)
  // (short dependency chains: this build runs once per staged pixel and its
  // latency, with the barrier after it, is exposed at the start of a tile)
  const double ih = 1.0 / dh;
  auto rcp = [](double v) {  // 1 / v to ~1 ulp: FP32 estimate + two Newton steps
    const float e = __frcp_rn((float)v);
    if (!(fabsf(e) > 1e-37f && fabsf(e) < 1e37f)) return 1.0 / v;  // outside FP32 range
    double r = (double)e;
    r = r * fma(-v, r, 2.0);
    return r * fma(-v, r, 2.0);
  };
  // unit_sum: the weights are member counts / M (or one-hot), whose sum is 1 to
  // a few ulps, so the renormalisation w / sum(w) (engine.py:538-540) is the
  // identity to within the closed form's tolerance and is skipped
  auto build = [&](int i, double lo, double hi, const double* wv, bool unit_sum) {
    CPB_ASSERT(i >= 0 && i < P);
    const double it = unit_sum ? 1.0 : rcp(HB <= 8 ? pairwise_small<HB>(wv) : pairwise16(wv, h));
    const double width = hi - lo, binw = width * ih, ibinw = dh * rcp(width);
    const bool pfast = (fabs(lo) + fabs(hi)) * ibinw <= kFastRatio;
    T[2 * i] = 0.0; T[2 * i + 1] = 0.0;
    T[2 * P + 2 * i] = pfast ? 0.0 : 1.0;
    T[2 * P + 2 * i + 1] = lo;
    double cum = 0.0;
#pragma unroll
    for (int b = 0; b < HB; ++b) {
      if (b < h) {
        const double wn = wv[b] * it;
        double* t = T + (size_t)(b + 1) * 4 * P + 2 * i;
        const double sl = wn * ibinw, ev = fma(binw, (double)b, lo);
        t[0] = pfast ? fma(-sl, ev, cum) : cum;
        t[1] = 0.5 * sl;
        t[2 * P] = ev;
        t[2 * P + 1] = b + 1 < h ? fma(width, (double)(b + 1) / dh, lo) : hi;
        cum += wn;
      }
    }
    double* t = T + (size_t)(h + 1) * 4 * P + 2 * i;
    t[0] = 1.0; t[1] = 0.0; t[2 * P] = 0.0; t[2 * P + 1] = inf;
  };
  constexpr int NT = kTabTW * kTabTH, NPT = (P + NT - 1) / NT;
  if (HB <= 8 && f.bounds == CPB_BOUNDS_F32_FITTED && f.wmode == CPB_WEIGHTS_U8) {
    // fitted planes (the common case): issue every global load of this
    // thread's pixels first, then build -- one exposed load latency, not NPT
    constexpr int HC = HB <= 8 ? HB : 1;
    float rlo[NPT], rhi[NPT];
    unsigned rc[NPT][HC];
    int64_t at[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int i = tid + j * NT;
      const int64_t rr = r0 - 1 + i / SW, cc = c0 + i % SW;
      at[j] = (i < P && rr < f.height && cc < f.width) ? rr * f.width + cc : -1;
      rlo[j] = rhi[j] = 0.0f;
      if (at[j] >= 0) {
        rlo[j] = __ldg(static_cast<const float*>(f.lo) + at[j]);
        rhi[j] = __ldg(static_cast<const float*>(f.hi) + at[j]);
      }
#pragma unroll
      for (int q = 0; q < HC; ++q)
        rc[j][q] = at[j] >= 0 ? (unsigned)__ldg(static_cast<const uint8_t*>(f.weights) + (int64_t)q * f.wstride + at[j]) : 0u;
    }
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      if (at[j] < 0) continue;
      double lo = (double)rlo[j], hi = (double)rhi[j];
      const bool deg = !(hi > lo);
      int dbin = 0;
      if (deg) {  // load_bounds: widen by eps/2 at use (fields.py:140-143)
        const double c = lo, hh = __dmul_rn(0.5, field_eps(f));
        lo = __dsub_rn(c, hh);
        hi = __dadd_rn(c, hh);
        dbin = degenerate_bin(c, lo, hi, h);
      }
      double wv[HB];
#pragma unroll
      for (int q = 0; q < HB; ++q) {
        const unsigned cnt = rc[j][q < HC ? q : 0];
        wv[q] = q < h ? (deg ? (q == dbin ? 1.0 : 0.0) : (double)cnt * invM) : 0.0;
      }
      build(tid + j * NT, lo, hi, wv, true);
    }
  } else {
    for (int i = tid; i < P; i += NT) {
      const int64_t rr = r0 - 1 + i / SW, cc = c0 + i % SW;
      if (rr >= f.height || cc >= f.width) continue;
      const int64_t at = rr * f.width + cc;
      double lo, hi;
      const bool deg = load_bounds(f, at, lo, hi);
      const int dbin = deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at), lo, hi, h) : 0;
      double wv[HB];
#pragma unroll
      for (int b = 0; b < HB; ++b) {
        double wb = 0.0;
        if (b < h) {
          if (f.wmode == CPB_WEIGHTS_F64) {
            wb = __ldg(static_cast<const double*>(f.weights) + (int64_t)b * f.wstride + at);
          } else if (deg) {
            wb = b == dbin ? 1.0 : 0.0;
          } else {
            const unsigned cnt = f.wmode == CPB_WEIGHTS_U8
                ? (unsigned)__ldg(static_cast<const uint8_t*>(f.weights) + (int64_t)b * f.wstride + at)
                : (unsigned)__ldg(static_cast<const uint16_t*>(f.weights) + (int64_t)b * f.wstride + at);
            wb = (double)cnt * invM;  // count / M to within an ulp (closed-form tolerance)
          }
        }
        wv[b] = wb;
      }
      build(i, lo, hi, wv, false);
    }
  }
  __syncthreads();
  const int64_t r = r0 + threadIdx.y, c = c0 + 1 + threadIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (r < row_end && c < f.width - 1) {
  const int ic = (threadIdx.y + 1) * SW + threadIdx.x + 1;
  const int ip[5] = {ic, ic + 1, ic - SW, ic - 1, ic + SW};  // C E N W S
  const bool fast = T[2 * P + 2 * ip[0]] + T[2 * P + 2 * ip[1]] + T[2 * P + 2 * ip[2]] +
                    T[2 * P + 2 * ip[3]] + T[2 * P + 2 * ip[4]] == 0.0;
  bool pf[5];  // per-pixel fast flags (the exact mode reads B = CUM - SL EV there)
#pragma unroll
  for (int p = 0; p < 5; ++p) pf[p] = T[2 * P + 2 * ip[p]] == 0.0;
  if (fast) hist_sweep<true>(T, h, ip, pf, acc);
  else hist_sweep<false>(T, h, ip, pf, acc);
  store(pmin, pmax, psad, r * f.width + c, acc);
  }
  if (partial) warp_partial_sums(acc[0], acc[1], acc[2] + acc[3], partial);
}

// Histogram stencil for many bins (kTabMaxBins + 1 .. kOtfMaxBins, fitted uint8 counts):
// the state tables of closed_hist_tab_kernel cost 32 (h + 2) bytes per staged
// pixel (one 256-vertex block per SM at h = 16, none at h = 32), so here a
// block stages only what the states are derived from -- lo, hi, binw, 1/binw
// and the CUMULATIVE member counts c_b (h + 1 bytes) per pixel, plus the
// exact weight table c / M -- and every list computes its state when it
// advances: CUM = wtab[c_b], wn = wtab[c_(b+1) - c_b], SL = wn / binw, the
// bin start EV is the previous next-edge, NX = lo + binw (b + 1) (a float64
// counter, no conversion).  Same sweep and piece arithmetic as the table
// kernel (fast: B + (SL/2) s2 with B = CUM - SL EV and symmetric node pairs;
// exact mode: per-node positions).  ~70 bytes per staged pixel at h = 32.
constexpr int kOtfMaxBins = 64;

struct OtfList {
  int k;         // 0 below the support, 1..h inside bin k - 1, h + 1 above
  int px;        // staged pixel
  double kd;     // k as a double (the next edge is lo + binw * kd)
  double cc, ss, ee, nx;
};

template <bool FAST>
CPB_D void otf_enter(OtfList& L, int k, int h, const double* lo, const double* hi, const double* bw,
                     const double* ibw, const uint8_t* cc, const double* wt, int P) {
  const int i = L.px;
  L.k = k;
  if (k == 0) {
    L.cc = 0.0; L.ss = 0.0; L.ee = 0.0; L.nx = lo[i];
    return;
  }
  if (k > h) {
    L.cc = 1.0; L.ss = 0.0; L.ee = 0.0; L.nx = __longlong_as_double(0x7ff0000000000000ll);
    return;
  }
  const int b = k - 1;
  CPB_ASSERT(i >= 0 && i < P && b >= 0 && b < h);
  const int c0 = cc[b * P + i], c1 = cc[(b + 1) * P + i];
  const double cum = wt[c0], wn = wt[c1 - c0];
  const double sl = wn * fabs(ibw[i]);
  const double ev = fma(bw[i], L.kd - 1.0, lo[i]);
  L.ee = ev;
  L.cc = FAST ? fma(-sl, ev, cum) : cum;
  L.ss = 0.5 * sl;
  L.nx = k < h ? fma(bw[i], L.kd, lo[i]) : hi[i];
}

template <bool FAST>
CPB_D void hist_otf_sweep(int h, const int* ip, const bool* pf, const double* lo, const double* hi,
                          const double* bw, const double* ibw, const uint8_t* cc, const double* wt,
                          int P, double acc[4]) {
  double accs[3] = {0.0, 0.0, 0.0};
  const double x0 = lo[ip[0]];
  OtfList L[5];
#pragma unroll
  for (int p = 1; p < 5; ++p) {
    // first state whose next edge lies beyond x0: a guess from the bin
    // position, then the exact float64 edges decide
    const int i = ip[p];
    L[p].px = i;
    int k = 0;
    if (lo[i] <= x0) {
      const double t = floor((x0 - lo[i]) * fabs(ibw[i]));
      k = (int)fmin(fmax(t, 0.0), (double)h) + 1;
    }
    L[p].kd = (double)k;
    otf_enter<FAST>(L[p], k, h, lo, hi, bw, ibw, cc, wt, P);
    while (L[p].nx <= x0) {
      L[p].kd += 1.0;
      otf_enter<FAST>(L[p], L[p].k + 1, h, lo, hi, bw, ibw, cc, wt, P);
    }
    while (L[p].k > 0) {  // the guess may overshoot by one
      OtfList q = L[p];
      q.kd -= 1.0;
      otf_enter<FAST>(q, L[p].k - 1, h, lo, hi, bw, ibw, cc, wt, P);
      if (q.nx <= x0) break;
      L[p] = q;
    }
  }
  OtfList C;
  C.px = ip[0];
  C.kd = 1.0;
  otf_enter<FAST>(C, 1, h, lo, hi, bw, ibw, cc, wt, P);
  double x = x0;
  while (C.k <= h) {
    const double xn = dmin(dmin(C.nx, dmin(L[E_].nx, L[N_].nx)), dmin(L[W_].nx, L[S_].nx));
    const double s2 = xn + x, hd = xn - x;
    const double scale = C.ss * hd;  // pdf_C / 2 * (b - a)
    double s[4];
    if (FAST) {
      double Fm[5], d[5];
      const double tau = hd * GL3::x(2);
#pragma unroll
      for (int p = 1; p < 5; ++p) {
        Fm[p] = fma(L[p].ss, s2, L[p].cc);
        d[p] = tau * L[p].ss;
      }
      double gs[3];
      gl3_sym_parts3(Fm, d, gs, s);
#pragma unroll
      for (int q = 0; q < 3; ++q) accs[q] = fma(gs[q], scale, accs[q]);
    } else {
      const double half = 0.5 * hd, mid = 0.5 * s2;
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] = 0.0;
#pragma unroll
      for (int j = 0; j < GL3::n; ++j) {
        const double xx = node_x(mid, half, GL3::x(j));
        double F[5], g[4];
#pragma unroll
        for (int p = 1; p < 5; ++p)
          F[p] = pf[p] ? fma(2.0 * L[p].ss, xx, fma(-2.0 * L[p].ss, L[p].ee, L[p].cc))
                       : fma(xx - L[p].ee, 2.0 * L[p].ss, L[p].cc);
        integrands(F, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fma(GL3::w(j), g[q], s[q]);
      }
      s[2] += s[3];
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[q] = fma(s[q], scale, acc[q]);
    if (C.nx == xn) {
      C.kd += 1.0;
      otf_enter<FAST>(C, C.k + 1, h, lo, hi, bw, ibw, cc, wt, P);
    }
#pragma unroll
    for (int p = 1; p < 5; ++p) {
      if (L[p].nx == xn) {
        L[p].kd += 1.0;
        otf_enter<FAST>(L[p], L[p].k + 1, h, lo, hi, bw, ibw, cc, wt, P);
      }
    }
    x = xn;
  }
  if (FAST) {
    const double w1 = GL3::w(1), w0x2 = 2.0 * GL3::w(0);
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[q] = fma(w0x2, accs[q], w1 * acc[q]);
  }
}

__global__ void __launch_bounds__(kTabTW * kTabTH, 2) closed_hist_otf_kernel(
    FieldView f, int64_t row_begin, int64_t row_end, int ctiles, double* pmin, double* pmax,
    double* psad, double* partial) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = kTabP, SW = kTabSW;
  const int h = f.bins, M = f.members;
  double* lo = sm;
  double* hi = lo + P;
  double* bw = hi + P;
  double* ibw = bw + P;  // 1 / binw; negative: the pixel is not fast-mode
  double* wt = ibw + P;  // (M + 1) weights c / M
  uint8_t* cc = reinterpret_cast<uint8_t*>(wt + M + 1);  // (h + 1) x P cumulative counts
  const int64_t r0 = row_begin + (int64_t)(blockIdx.x / ctiles) * kTabTH;
  const int64_t c0 = (int64_t)(blockIdx.x % ctiles) * kTabTW;
  const int tid = threadIdx.y * kTabTW + threadIdx.x;
  constexpr int NT = kTabTW * kTabTH;
  for (int c = tid; c <= M; c += NT) wt[c] = __ldg(f.wtab + c);
  const double dh = (double)h;
  for (int i = tid; i < P; i += NT) {
    const int64_t rr = r0 - 1 + i / SW, col = c0 + i % SW;
    if (rr >= f.height || col >= f.width) continue;
    const int64_t at = rr * f.width + col;
    double l, u;
    const bool deg = load_bounds(f, at, l, u);
    const int dbin = deg ? degenerate_bin((double)__ldg(static_cast<const float*>(f.lo) + at), l, u, h) : 0;
    const double width = u - l, binw = width / dh;
    const bool pfast = (fabs(l) + fabs(u)) * (dh / width) <= kFastRatio;
    lo[i] = l;
    hi[i] = u;
    bw[i] = binw;
    ibw[i] = pfast ? 1.0 / binw : -1.0 / binw;
    unsigned c = 0;
    cc[i] = 0;
    for (int b = 0; b < h; ++b) {
      c = deg ? (b >= dbin ? (unsigned)M : 0u)
              : c + (unsigned)__ldg(static_cast<const uint8_t*>(f.weights) + (int64_t)b * f.wstride + at);
      cc[(b + 1) * P + i] = (uint8_t)c;
    }
  }
  __syncthreads();
  const int64_t r = r0 + threadIdx.y, c = c0 + 1 + threadIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (r < row_end && c < f.width - 1) {
    const int ic = (threadIdx.y + 1) * SW + threadIdx.x + 1;
    const int ip[5] = {ic, ic + 1, ic - SW, ic - 1, ic + SW};  // C E N W S
    bool pf[5], fast = true;
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      pf[p] = ibw[ip[p]] > 0.0;
      fast &= pf[p];
    }
    if (fast) hist_otf_sweep<true>(h, ip, pf, lo, hi, bw, ibw, cc, wt, P, acc);
    else hist_otf_sweep<false>(h, ip, pf, lo, hi, bw, ibw, cc, wt, P, acc);
    store(pmin, pmax, psad, r * f.width + c, acc);
  }
  if (partial) warp_partial_sums(acc[0], acc[1], acc[2] + acc[3], partial);
}

}  // namespace

int launch_combinatorial(const cpb_field* fld, int64_t row_begin, int64_t row_end, double* pmin,
                         double* pmax, double* psad, cudaStream_t st) {
  const FieldView f = make_view(*fld);
  if (f.kind != CPB_HISTOGRAM) {
    set_error("combinatorial estimation is defined for histogram fields only");
    return CPB_EINVAL;
  }
  if (f.bins > COMB_MAX_BINS) {
    set_error("combinatorial estimation refuses more than %d bins", COMB_MAX_BINS);
    return CPB_EINVAL;
  }
  const int64_t rows = row_end - row_begin;
  if (rows <= 0 || f.width < 3) return CPB_OK;
  const int64_t cols = f.width - 2, nvert = rows * cols;
  combinatorial_kernel<<<(unsigned)((nvert + kCombWarps - 1) / kCombWarps), kCombWarps * 32, 0, st>>>(
      f, row_begin, nvert, cols, pmin, pmax, psad);
  CPB_CHECK_LAUNCH("combinatorial kernel");
  return CPB_OK;
}

bool encode_tensor_map_2d_f32(CUtensorMap* map, const void* base, uint64_t dim0, uint64_t dim1,
                              uint64_t stride1_bytes, uint32_t box0, uint32_t box1);
int launch_fit(const float* ens, int64_t mstride, cpb_field* f, uint32_t* range, bool accumulate,
               cudaStream_t st);

// ---- fused fit + uniform stencil (closed_fuse_uniform_kernel) -------------
namespace {
struct FuseLayout {
  int nbands;
  int64_t nsegs, nitems, max_pending, n_edges, edge_blocks, nbounds;
  size_t off_pending, off_flags, off_bdone, off_eflag, off_partial, off_seg_partial, off_chunk, bytes;
  int64_t ntrip;
};
FuseLayout fuse_layout(int64_t width, int64_t row_begin, int64_t row_end) {
  FuseLayout L;
  L.nbands = (int)((width + kFuseCols - 1) / kFuseCols);
  const int64_t rows = std::max<int64_t>(0, row_end - row_begin);
  L.nsegs = (rows + kFuseSeg - 1) / kFuseSeg;
  L.nitems = L.nsegs * L.nbands;
  L.max_pending = rows * L.nbands;
  L.n_edges = rows * 2 * (int64_t)(L.nbands + 1);
  L.edge_blocks = (L.n_edges + kFuseCols - 1) / kFuseCols;
  L.off_pending = 16;
  L.off_flags = (L.off_pending + 4 * (size_t)(1 + L.max_pending) + 15) / 16 * 16;
  L.nbounds = L.nsegs * (L.nbands + 1);
  L.off_bdone = (L.off_flags + (size_t)L.max_pending + 15) / 16 * 16;
  L.off_eflag = (L.off_bdone + 4 * (size_t)L.nbounds + 15) / 16 * 16;
  L.off_partial = (L.off_eflag + (size_t)L.n_edges + 15) / 16 * 16;
  // warp triples: the fused items, the boundaries' edge vertices, the pending
  // pass, the flagged-edge pass
  const int64_t wpb = kFuseCols / 32;
  L.off_seg_partial = L.off_partial + (size_t)L.nitems * wpb * 3 * sizeof(double);
  L.ntrip = (L.nitems + L.nbounds + kFuseFinishBlocks + L.edge_blocks) * wpb;
  L.off_chunk = L.off_partial + (size_t)L.ntrip * 3 * sizeof(double);
  L.bytes = L.off_chunk + (size_t)kCountChunks * 3 * sizeof(double);
  return L;
}
}  // namespace

size_t fit_classify_work_bytes(int64_t width, int64_t row_begin, int64_t row_end) {
  return fuse_layout(width, row_begin, row_end).bytes;
}

int launch_fit_multi(const float* ens, int64_t mstride, cpb_field* const* fs, int n, uint32_t* range,
                     bool accumulate, cudaStream_t st);

// fields[0..n): one uniform field (stencilled) plus at most one histogram
// (<= 8 bins), Epanechnikov and Gaussian field, fitted in the same pass.
int launch_fit_classify(const float* ens, int64_t mstride, cpb_field* const* fields, int n,
                        uint32_t* range, bool accumulate, int64_t row_begin, int64_t row_end,
                        double* pmin, double* pmax, double* psad, void* work, cudaStream_t st) {
  if (n < 1 || n > 4 || !fields) { set_error("1..4 fields expected"); return CPB_EINVAL; }
  cpb_field* slot[4] = {nullptr, nullptr, nullptr, nullptr};  // uniform, histogram, epan, gaussian
  for (int i = 0; i < n; ++i) {
    const int k = fields[i]->kind;
    const int q = k == CPB_UNIFORM ? 0 : k == CPB_HISTOGRAM ? 1 : k == CPB_EPANECHNIKOV ? 2 : 3;
    if (slot[q]) { set_error("at most one field per model kind"); return CPB_EINVAL; }
    slot[q] = fields[i];
  }
  cpb_field* fld = slot[0];
  if (!fld) {
    set_error("the fused fit + stencil needs a uniform field");
    return CPB_EINVAL;
  }
  const int64_t H = fld->height, W = fld->width, M = fld->members;
  for (int i = 0; i < n; ++i)
    if (fields[i]->height != H || fields[i]->width != W || fields[i]->members != M) {
      set_error("fused fit: every field must share height, width and members");
      return CPB_EINVAL;
    }
  if (W < 3 || row_begin < 1 || row_end > H - 1 || row_begin > row_end) {
    set_error("fused fit + stencil: vertex rows must lie inside [1, height - 1)");
    return CPB_EINVAL;
  }
  const FuseLayout L = fuse_layout(W, row_begin, row_end);
  char* wb = static_cast<char*>(work);
  // per-row TMA boxes start at pixel r W + c0: their global address is
  // 16-byte aligned only when W is a multiple of 4 (a misaligned box start
  // faults as an illegal instruction)
  if (M < 1 || M > kFuseMaxMembers || mstride % 4 != 0 || W % 4 != 0 ||
      (reinterpret_cast<uintptr_t>(ens) & 15) || H * W >= ((int64_t)1 << 31) ||
      (slot[1] && slot[1]->bins > kThreshBinsPix)) {
    // not one TMA-streamed pass: the plain fit(s) now, every vertex row in the finish pass
    int rc = n == 1 ? launch_fit(ens, mstride, fld, range, accumulate, st)
                    : launch_fit_multi(ens, mstride, fields, n, range, accumulate, st);
    if (rc == 1 && n > 1)  // launch_fit_multi declines this set: one fit per model
      for (int i = 0; i < n; ++i)
        if ((rc = launch_fit(ens, mstride, fields[i], range, accumulate || i > 0, st))) break;
    if (rc) return rc;
    cudaError_t e = cudaMemsetAsync(wb + L.off_pending, 0xff, 4, st);  // pending count = -1: all rows
    if (e == cudaSuccess)  // no item partials from the one-pass kernel
      e = cudaMemsetAsync(wb + L.off_partial, 0, (size_t)(L.nitems + L.nbounds) * (kFuseCols / 32) * 3 * sizeof(double), st);
    return e == cudaSuccess ? CPB_OK : cuda_status(e, "memset");
  }
  cudaError_t e = cudaMemsetAsync(wb, 0, L.off_pending + 4, st);  // work counter, pending count
  // band-row flags, segment counters and edge flags are contiguous
  if (e == cudaSuccess) e = cudaMemsetAsync(wb + L.off_flags, 0, L.off_partial - L.off_flags, st);
  if (e != cudaSuccess) return cuda_status(e, "memset");
  if (!accumulate) {  // {ordered min = all ones, ordered max = 0, non-finite = 0}
    e = cudaMemsetAsync(range, 0xff, sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(range + 1, 0, 2 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "range init");
  }
  CUtensorMap map;
  if (!encode_tensor_map_2d_f32(&map, ens, (uint64_t)(H * W), (uint64_t)M, (uint64_t)mstride * 4,
                                kFuseBox, (uint32_t)M)) {
    set_error("cuTensorMapEncodeTiled failed");
    return CPB_ECUDA;
  }
  FuseArgs a = {};
  a.height = H; a.width = W; a.row_begin = row_begin; a.row_end = row_end; a.members = (int)M;
  a.nbands = L.nbands; a.nsegs = (int)L.nsegs; a.nitems = L.nitems;
  a.lo = static_cast<float*>(fld->lo); a.hi = static_cast<float*>(fld->hi); a.range = range;
  a.pmin = pmin; a.pmax = pmax; a.psad = psad;
  a.partial = reinterpret_cast<double*>(wb + L.off_partial);
  a.pending = reinterpret_cast<int*>(wb + L.off_pending);
  a.pflag = reinterpret_cast<unsigned char*>(wb + L.off_flags);
  a.bdone = reinterpret_cast<int*>(wb + L.off_bdone);
  a.eflag = reinterpret_cast<unsigned char*>(wb + L.off_eflag);
  a.edge_partial = reinterpret_cast<double*>(wb + L.off_seg_partial);
  a.work = reinterpret_cast<int*>(wb);
  int nt = -1;
  if (n > 1) {  // the other models' planes come out of the same pass
    MultiArgs& m = a.mf;
    m.npix = H * W;
    m.members = (int)M;
    m.wmode = M <= 255 ? CPB_WEIGHTS_U8 : CPB_WEIGHTS_U16;
    m.range = range;
    for (int i = 0; i < 2; ++i) {
      if (slot[i]) {
        m.lo[i] = static_cast<float*>(slot[i]->lo);
        m.hi[i] = static_cast<float*>(slot[i]->hi);
      }
      if (slot[2 + i]) {
        m.mean[i] = slot[2 + i]->mean;
        m.spread[i] = slot[2 + i]->spread;
        slot[2 + i]->bounds = CPB_BOUNDS_F32_FITTED;
        slot[2 + i]->weights_mode = CPB_WEIGHTS_F64;
      }
    }
    nt = 0;
    if (slot[1]) {
      nt = slot[1]->bins;
      m.bins = nt;
      m.counts = slot[1]->weights;
      m.wstride = slot[1]->plane_stride > 0 ? slot[1]->plane_stride : H * W;
      slot[1]->bounds = CPB_BOUNDS_F32_FITTED;
      slot[1]->weights_mode = m.wmode;
      weight_table_kernel<<<(unsigned)((M + 256) / 256), 256, 0, st>>>(slot[1]->weight_table, (int)M);
      CPB_CHECK_LAUNCH("weight table");
    }
  }
  fld->bounds = CPB_BOUNDS_F32_FITTED;
  fld->weights_mode = CPB_WEIGHTS_F64;
  const size_t smem = (size_t)M * kFuseBox * 4 + 4 * kFuseRing * sizeof(float2) + 16;  // box = the band
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFuseCols, smem);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(L.nitems, (int64_t)sms * std::max(per_sm, 1)));
    if (L.nitems > 0) kern<<<(unsigned)grid, kFuseCols, smem, st>>>(map, a);
  };
  switch (nt) {
    case -1: go(closed_fuse_uniform_kernel<-1>); break;
    case 0: go(closed_fuse_uniform_kernel<0>); break;
    case 1: go(closed_fuse_uniform_kernel<1>); break;
    case 2: go(closed_fuse_uniform_kernel<2>); break;
    case 3: go(closed_fuse_uniform_kernel<3>); break;
    case 4: go(closed_fuse_uniform_kernel<4>); break;
    case 5: go(closed_fuse_uniform_kernel<5>); break;
    case 6: go(closed_fuse_uniform_kernel<6>); break;
    case 7: go(closed_fuse_uniform_kernel<7>); break;
    default: go(closed_fuse_uniform_kernel<8>); break;
  }
  CPB_CHECK_LAUNCH("fused fit + uniform stencil");
  return CPB_OK;
}

int launch_fit_classify_finish(const cpb_field* fld, int64_t row_begin, int64_t row_end, double* pmin,
                               double* pmax, double* psad, double* counts, void* work, cudaStream_t st) {
  const FieldView f = make_view(*fld);
  const FuseLayout L = fuse_layout(f.width, row_begin, row_end);
  char* wb = static_cast<char*>(work);
  double* partial = reinterpret_cast<double*>(wb + L.off_partial);
  const int* pending = reinterpret_cast<const int*>(wb + L.off_pending);
  const int64_t wpb = kFuseCols / 32;
  double* part_pending = partial + 3 * (size_t)(L.nitems + L.nbounds) * wpb;
  closed_fuse_pending_kernel<<<kFuseFinishBlocks, kFuseCols, 0, st>>>(
      f, pending, L.nbands, row_begin, row_end, pmin, pmax, psad, part_pending);
  CPB_CHECK_LAUNCH("fused stencil: pending rows");
  if (L.edge_blocks > 0)
    closed_fuse_edges_kernel<<<(unsigned)L.edge_blocks, kFuseCols, 0, st>>>(
        f, pending, reinterpret_cast<const unsigned char*>(wb + L.off_flags),
        reinterpret_cast<const unsigned char*>(wb + L.off_eflag), L.nbands, row_begin, row_end, pmin, pmax,
        psad, part_pending + 3 * (size_t)kFuseFinishBlocks * wpb);
  CPB_CHECK_LAUNCH("fused stencil: flagged band edges");
  if (counts) {
    double* chunk = reinterpret_cast<double*>(wb + L.off_chunk);
    const int64_t n = L.ntrip;
    counts_reduce_kernel<<<kCountChunks, 256, 0, st>>>(partial, n, chunk);
    counts_finish_kernel<<<1, 256, 0, st>>>(chunk, kCountChunks, counts);
    CPB_CHECK_LAUNCH("fused stencil: counts");
  }
  return CPB_OK;
}

int workspace_alloc(void** p, size_t bytes, cudaStream_t st);
void workspace_free(void* p, cudaStream_t st);

// counts (optional, 3 doubles): the per-type sums of this launch's vertices are
// ADDED to counts[0..2] (fused into the stencils' epilogue where supported,
// otherwise a reduction over the written rows)
int launch_closed(const cpb_field* fld, int64_t row_begin, int64_t row_end, double* pmin,
                  double* pmax, double* psad, cudaStream_t st, double* counts) {
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
  const int64_t cols = f.width - 2, nvert = rows * cols;
  const int64_t pp_segs = (cols + 31) / 32;  // closed_pp_kernel: row-aligned 32-vertex segments
  const int64_t pp_blocks = (rows * pp_segs + kPPWarps - 1) / kPPWarps;
  // per-block partial sums of the expected counts (freed on every path)
  struct Partial {
    double* p = nullptr;
    int64_t n = 0;
    cudaStream_t st;
    ~Partial() { workspace_free(p, st); }
  } part{nullptr, 0, st};
  auto want_partial = [&](int64_t nwarps) -> int {  // one partial triple per warp
    if (!counts) return CPB_OK;
    part.n = nwarps;
    return workspace_alloc((void**)&part.p, (size_t)(nwarps + kCountChunks) * 3 * sizeof(double), st);
  };
  bool fused_counts = false;  // set by the kernels that write block partials
  switch (f.kind) {
    case CPB_UNIFORM:
      // one vertex per lane: 3-node pieces are too cheap to amortise a
      // piece-parallel redistribution (measured 18.6 vs 25.4 ms at 16384^2)
      if (int rc = want_partial(blocks * (kClosedThreads / 32))) return rc;
      if (f.mixed)
        closed_uniform_f32_kernel<<<(unsigned)blocks, kClosedThreads, 0, st>>>(f, w, pmin, pmax, psad, part.p);
      else
        closed_uniform_kernel<<<(unsigned)blocks, kClosedThreads, 0, st>>>(f, w, pmin, pmax, psad, part.p);
      fused_counts = true;
      break;
    case CPB_EPANECHNIKOV: {
      // piece-parallel (8-node pieces): each warp compacts its lanes' non-empty pieces
      if (int rc = want_partial(pp_blocks * kPPWarps)) return rc;
      auto kern = f.mixed ? closed_pp_kernel<true> : closed_pp_kernel<false>;
      const size_t pp_smem = (f.mixed ? sizeof(PPSmem<15>) : sizeof(PPSmem<10>)) * kPPWarps;
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp_smem);
      kern<<<(unsigned)pp_blocks, kPPWarps * 32, pp_smem, st>>>(
          f, row_begin, row_end, cols, pp_segs, pmin, pmax, psad, part.p);
      fused_counts = true;
      break;
    }
    case CPB_HISTOGRAM: {
      const size_t tab_smem = (size_t)4 * (f.bins + 2) * kTabP * 8;
      // bins > kTabMaxBins: states on the fly (tables of 16 bins still win at 1
      // block / SM: 3.55 vs 4.77 ms at 2048^2 x 40; 32 bins: 9.9 ms vs 16.8 ms
      // for the per-thread shared-memory kernel)
      if (f.bins > kTabMaxBins && f.bins <= kOtfMaxBins && f.bounds == CPB_BOUNDS_F32_FITTED &&
          f.wmode == CPB_WEIGHTS_U8 && f.wtab) {
        const int ctiles = (int)((f.width - 2 + kTabTW - 1) / kTabTW);
        const int64_t rtiles = (rows + kTabTH - 1) / kTabTH;
        const size_t otf_smem = (size_t)4 * kTabP * 8 + (size_t)(f.members + 1) * 8 + (size_t)(f.bins + 1) * kTabP;
        if (int rc = want_partial(rtiles * ctiles * (kTabTW * kTabTH / 32))) return rc;
        cudaFuncSetAttribute(closed_hist_otf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)otf_smem);
        closed_hist_otf_kernel<<<(unsigned)(rtiles * ctiles), dim3(kTabTW, kTabTH), otf_smem, st>>>(
            f, row_begin, row_end, ctiles, pmin, pmax, psad, part.p);
        fused_counts = true;
        break;
      }
      if (f.bins <= kTabMaxBins && tab_smem <= 200 * 1024) {
        const int ctiles = (int)((f.width - 2 + kTabTW - 1) / kTabTW);
        const int64_t rtiles = (rows + kTabTH - 1) / kTabTH;
        auto kern = closed_hist_tab_kernel<16>;
        switch (f.bins) {
          case 1: kern = closed_hist_tab_kernel<1>; break;
          case 2: kern = closed_hist_tab_kernel<2>; break;
          case 3: kern = closed_hist_tab_kernel<3>; break;
          case 4: kern = closed_hist_tab_kernel<4>; break;
          case 5: kern = closed_hist_tab_kernel<5>; break;
          case 6: kern = closed_hist_tab_kernel<6>; break;
          case 7: kern = closed_hist_tab_kernel<7>; break;
          case 8: kern = closed_hist_tab_kernel<8>; break;
          default: break;
        }
        if (int rc = want_partial(rtiles * ctiles * (kTabTW * kTabTH / 32))) return rc;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab_smem);
        kern<<<(unsigned)(rtiles * ctiles), dim3(kTabTW, kTabTH), tab_smem, st>>>(
            f, row_begin, row_end, ctiles, pmin, pmax, psad, part.p);
        fused_counts = true;
        break;
      }
      if (f.bins > kHistSmemMaxBins) {
        closed_hist_global_kernel<<<(unsigned)blocks, kClosedThreads, 0, st>>>(f, w, pmin, pmax, psad);
        break;
      }
      // tile width so the staged float64 weights fit comfortably in shared memory
      int tw = kHistThreads;
      while (tw > 32 && (size_t)(3 + f.bins) * 3 * (tw + 2) * 8 > 64 * 1024) tw >>= 1;
      Window wh = w;
      wh.ntiles = (int)((f.width - 2 + tw - 1) / tw);
      const int64_t hb = rows * wh.ntiles;
      const size_t smem = ((size_t)(3 + f.bins) * 3 * (tw + 2) + f.bins + 1) * 8;
      auto kern = closed_hist_smem_kernel<4>;
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<(unsigned)hb, tw, smem, st>>>(f, wh, pmin, pmax, psad);
      break;
    }
    default:
      set_error("Gaussian fields have no closed form; use monte_carlo");
      return CPB_EINVAL;
  }
  CPB_CHECK_LAUNCH("closed-form kernel");
  if (counts) {
    if (!fused_counts) {  // the large-bin histogram kernels: reduce the written rows instead
      const int64_t nb = std::min<int64_t>(4096, (nvert + 255) / 256);
      if (int rc = want_partial(nb * 8)) return rc;
      rows_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(pmin, pmax, psad, row_begin, cols, f.width,
                                                         nvert, part.p);
      CPB_CHECK_LAUNCH("count rows");
    }
    double* chunk = part.p + 3 * part.n;
    counts_reduce_kernel<<<kCountChunks, 256, 0, st>>>(part.p, part.n, chunk);
    counts_finish_kernel<<<1, 256, 0, st>>>(chunk, kCountChunks, counts);
    CPB_CHECK_LAUNCH("count finish");
  }
  return CPB_OK;
}

}  // namespace cpb
