/*
 * critprob_b200.h -- C ABI of the B200-native critical-point probability path.
 *
 * Drop-in boundary for the grid hot path of the reference package
 * `critprob` (arXiv 2407.18015).  The reference has no FFI: its boundary is
 * the Python API, and each entry point below replaces one step of it
 * (citations are /root/reference/pkg/src/critprob/<file>:<line>):
 *
 *   cpb_fit              UncertainField.from_ensemble      fields.py:125-158
 *   cpb_fit_multi        from_ensemble of several models over one stack (one HBM pass)
 *   cpb_from_scalar      UncertainField.from_scalar        fields.py:160-178
 *   cpb_epsilon          default_epsilon                   distributions.py:30-36
 *   cpb_classify_closed  classify_field, closed form       engine.py:716-787 (+ _closed_chunk 594-629)
 *   cpb_classify_mc      classify_field, monte_carlo       engine.py:716-787 (+ _mc_chunk 659-666)
 *   cpb_materialize      UncertainField.params             fields.py:86-103 (reference f64 layout)
 *   cpb_unit_block       rngstream.unit_block              rngstream.py:33-48
 *   cpb_run_host         from_ensemble + classify_field with host buffers (one call, H2D/D2H inside)
 *   cpb_cases_*          the per-case API (NeighborhoodCase, engine.py:50-459) over a batch of cases
 *
 * Conventions
 *   - Plain pointers and sizes; no framework types.  "d_" pointers are CUDA
 *     device memory, "h_" pointers host memory.  `stream` is a cudaStream_t
 *     (NULL = legacy default stream).  Calls only enqueue work unless noted.
 *   - Every function returns a cpb_status; cpb_last_error() describes the
 *     last failure on the calling thread.
 *   - The library never frees caller memory.  A cpb_field only carries
 *     pointers to caller-owned device planes (see cpb_field_plane_bytes).
 *   - Grids are row-major (H, W); ensembles are member-major (M, H, W)
 *     float32, exactly the reference's EnsembleStack layout (fields.py:42-56).
 *   - Results are identical for any launch configuration or row-slab split
 *     (the reference's worker-count invariance, engine.py:724-727).
 */
#ifndef CRITPROB_B200_H
#define CRITPROB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPB_ABI_VERSION 1

typedef enum {
  CPB_OK = 0,
  CPB_EINVAL = 1,      /* invalid argument (reference: ValueError) */
  CPB_ECUDA = 2,       /* CUDA runtime error */
  CPB_ENOMEM = 4,      /* device or pinned-host allocation failed */
  CPB_ENONFINITE = 5   /* ensemble holds NaN/Inf (reference: ValueError, fields.py:54-55) */
} cpb_status;

/* Model kinds (fields.py:21, MODEL_KINDS order). */
enum { CPB_UNIFORM = 0, CPB_EPANECHNIKOV = 1, CPB_HISTOGRAM = 2, CPB_GAUSSIAN = 3 };

/* Channel bits (fields.py:22, CHANNELS). */
enum { CPB_CH_MIN = 1, CPB_CH_MAX = 2, CPB_CH_SADDLE = 4, CPB_CH_ALL = 7 };

/* Monte Carlo uniform streams. */
enum {
  CPB_RNG_SPLITMIX = 0, /* the reference keyed splitmix64 stream: bit-exact (rngstream.py) */
  CPB_RNG_PHILOX = 1    /* Philox4x32-10 keyed by (seed, pixel, plane): statistical parity only */
};

/* cpb_field.flags */
enum {
  CPB_FLAG_MIXED = 1 /* closed form: float64 partition / node offsets / accumulation, single-
                        precision Gauss-Legendre evaluation (north_star bound 1e-6 absolute;
                        measured in tests/test_gpu_parity.py) */
};

/* Storage of the support bounds / histogram weights inside a cpb_field. */
enum {
  CPB_BOUNDS_F32_FITTED = 0, /* lo/hi = raw member min/max (exact in f32); lo==hi pixels are
                                widened by eps/2 at use, as fields.py:140-143 does at fit time */
  CPB_BOUNDS_F64 = 1         /* lo/hi given in float64 and used as-is (user-built fields) */
};
enum {
  CPB_WEIGHTS_U8 = 0,  /* member counts per bin (members <= 255); weight = count / members */
  CPB_WEIGHTS_U16 = 1, /* member counts per bin (members <= 65535) */
  CPB_WEIGHTS_F64 = 2  /* float64 weights as given (user-built fields) */
};

/*
 * Compact device-resident fitted field (a row slab of the global grid).
 * Planes are row-major (height, width); histogram weights are bin planes
 * (bins, height, width) so every per-bin read is coalesced.
 *
 *   uniform / histogram : lo, hi  (float if bounds == F32_FITTED else double)
 *   epanechnikov        : mean, spread (spread = std(ddof=1) when fitted; the
 *                         half-width used is max(k * spread, eps / 2), i.e.
 *                         fields.py:156.  User-built fields pass k = 1, eps = 0
 *                         and spread = half-width.)
 *   gaussian            : mean, spread (= stddev)
 *   histogram           : weights (CPB_WEIGHTS_*), weight_table = d_ptr to
 *                         (members + 1) doubles c / members (filled by cpb_fit)
 */
typedef struct cpb_field {
  int32_t kind;
  int32_t bins;
  int32_t members;
  int32_t bounds;        /* CPB_BOUNDS_* */
  int32_t weights_mode;  /* CPB_WEIGHTS_* */
  int32_t flags;        /* CPB_FLAG_* */
  int64_t height;        /* local rows (a slab includes its halo rows) */
  int64_t width;
  int64_t row0;          /* global row index of local row 0 (Monte Carlo pixel keys) */
  int64_t global_width;  /* pixel key = global_row * global_width + col (engine.py:752-754) */
  int64_t plane_stride;  /* elements between histogram bin planes; 0 = height * width.  Lets a
                            slab view (offset base pointers, fewer rows) address the bin planes
                            of a taller allocation, e.g. a row slab with halo rows */
  const double* eps_device; /* optional device pointer: when set, kernels read eps from it
                            instead of `eps` (no host round trip between fit and classify;
                            filled by cpb_pair_to_eps) */
  double eps;            /* from the GLOBAL ensemble range (distributions.py:30-36) */
  double k;              /* epanechnikov k (fields.py:31) */
  void* lo;
  void* hi;
  double* mean;
  double* spread;
  void* weights;
  double* weight_table;
} cpb_field;

/* ABI version and last error (thread-local). */
int cpb_abi_version(void);
const char* cpb_last_error(void);

/* Process-wide tunables (results never depend on them):
 *   "fit_ctas_per_sm"  cap on the persistent fit CTAs per SM (0 = occupancy
 *                      maximum); a smaller fit footprint lets a stencil running
 *                      on another stream share the SMs. */
int cpb_set_option(const char* name, int64_t value);

/* Bytes of device memory each plane of a fitted field needs
 * (lo, hi, mean, spread, weights, weight_table, range scratch), written into
 * out[7].  Mirrors the layout cpb_fit writes. */
int cpb_field_plane_bytes(int32_t kind, int32_t bins, int32_t members, int64_t height,
                          int64_t width, size_t out[7]);

/* eps = max(1e-12, 1e-9 * (gmax - gmin))  -- distributions.py:30-36. */
double cpb_epsilon(double gmin, double gmax);

/*
 * Fit one model per pixel over the member axis (fields.py:133-158).
 * d_ens: member-major float32, element (m, r, c) at d_ens[m * member_stride + r * width + c]
 *        for local rows r in [0, f->height).
 * Writes the compact planes of `f` and, into d_range[0..2], the float32 min
 * and max over all values read plus a non-finite flag (d_range is 3 x
 * uint32 device words; decode with cpb_read_range; accumulate != 0 merges into
 * the words instead of resetting them first, for chunked fits).  `f` must have kind, bins,
 * members, height, width and the plane pointers set; `f->bounds` and
 * `f->weights_mode` are set by this call.  Bit-exact with the reference:
 * min/max and counts exactly, mean/std by the same sequential two-pass order.
 */
int cpb_fit(const float* d_ens, int64_t member_stride, cpb_field* f, uint32_t* d_range,
            int32_t accumulate, void* stream);

/* Device-side eps, no host synchronisation: cpb_range_to_pair turns the
 * d_range words of cpb_fit into d_pair = {-min, max} (float64; NaN when a
 * value was non-finite), ready for a MAX all-reduce across row slabs;
 * cpb_pair_to_eps writes eps = max(1e-12, 1e-9 * (max - min)) to d_eps
 * (distributions.py:30-36), for cpb_field.eps_device. */
int cpb_range_to_pair(const uint32_t* d_range, double* d_pair, void* stream);
int cpb_pair_to_eps(const double* d_pair, double* d_eps, void* stream);

/* Fit several models of ONE ensemble in a single pass over it (the reference
 * workflow: one EnsembleStack, from_ensemble per model).  All fields share
 * height, width and members; each gets exactly the planes cpb_fit would write
 * (bit-identical), and d_range receives the shared data range.  At most one
 * field per kind is fused (histograms with <= 8 bins); other sets are fitted
 * one after another. */
int cpb_fit_multi(const float* d_ens, int64_t member_stride, cpb_field* const* fields,
                  int32_t n_fields, uint32_t* d_range, int32_t accumulate, void* stream);

/* Synchronous finiteness check of n device floats (EnsembleStack's
 * isfinite validation, fields.py:54-55, run in HBM instead of on the host):
 * CPB_ENONFINITE if any value is NaN or +-Inf. */
int cpb_check_finite(const float* d_values, int64_t n, void* stream);

/*
 * Fused fit + closed-form stencil of a UNIFORM field, one pass over the
 * ensemble (fields.py:137-143 + engine.py:594-629; the reference workflow
 * classify_field(from_ensemble(stack, ModelSpec("uniform")))).  The fitted
 * lo / hi reach the stencil through shared memory, not HBM, so the ensemble
 * stream and the FP64 stencil overlap inside each SM.
 *   cpb_fit_classify      fits rows [row_begin - 1, row_end] of `f` (writes those
 *                         rows of its planes and d_range, as cpb_fit does; the full
 *                         field for row_begin = 1, row_end = height - 1) and writes
 *                         p_min / p_max / p_saddle for
 *                         vertex rows [row_begin, row_end) (1 <= row_begin, row_end
 *                         <= height - 1), except vertex rows whose stencil holds a
 *                         degenerate pixel (lo == hi: their eps widening needs the
 *                         GLOBAL range), which are queued in d_work;
 *   cpb_fit_classify_finish   once f's eps is final (f->eps, or f->eps_device, e.g.
 *                         after the cross-slab MAX all-reduce) computes the queued
 *                         rows and ADDS the expected per-type counts of all
 *                         [row_begin, row_end) vertices to d_counts (optional).
 * d_work: cpb_fit_classify_work_bytes() bytes of device scratch, the same
 * (width, row_begin, row_end) for both calls.  The one-pass kernel needs
 * members <= 256, a 16-byte aligned ensemble with member_stride % 4 == 0 and
 * < 2^31 pixels; other stacks are fitted by cpb_fit and stencilled in the
 * finish pass.  Results equal cpb_fit + cpb_classify_closed bit for bit.
 */
int cpb_fit_classify_work_bytes(int64_t width, int64_t row_begin, int64_t row_end, size_t* bytes);
int cpb_fit_classify(const float* d_ens, int64_t member_stride, cpb_field* f, uint32_t* d_range,
                     int32_t accumulate, int64_t row_begin, int64_t row_end, double* d_pmin,
                     double* d_pmax, double* d_psaddle, void* d_work, void* stream);
/* cpb_fit_classify for several models of one stack (the reference workflow of
 * fitting one EnsembleStack with every model): fields[] holds exactly one
 * uniform field -- the one stencilled -- plus at most one histogram (<= 8 bins
 * for the one-pass kernel), Epanechnikov and Gaussian field, all fitted in the
 * same pass over the ensemble with the planes cpb_fit_multi writes.  Finish
 * with cpb_fit_classify_finish on the uniform field. */
int cpb_fit_multi_classify(const float* d_ens, int64_t member_stride, cpb_field* const* fields,
                           int32_t n_fields, uint32_t* d_range, int32_t accumulate, int64_t row_begin,
                           int64_t row_end, double* d_pmin, double* d_pmax, double* d_psaddle,
                           void* d_work, void* stream);
int cpb_fit_classify_finish(const cpb_field* f, int64_t row_begin, int64_t row_end, double* d_pmin,
                            double* d_pmax, double* d_psaddle, double* d_counts, void* d_work,
                            void* stream);

/* Synchronously read back a d_range written by cpb_fit; returns
 * CPB_ENONFINITE if any value was NaN/Inf. */
int cpb_read_range(const uint32_t* d_range, double* gmin, double* gmax, void* stream);

/* Uniform field from a float64 raster with a +-error_bound/2 band
 * (fields.py:160-178).  d_lo/d_hi are float64 planes; eps is the raster's
 * epsilon, used when error_bound == 0. */
int cpb_from_scalar(const double* d_values, int64_t height, int64_t width, double error_bound,
                    double eps, double* d_lo, double* d_hi, void* stream);

/*
 * Closed-form min/max/saddle probabilities (engine.py:594-629) for local rows
 * [row_begin, row_end) and columns [1, width-1); rows row_begin-1 and row_end
 * must exist in `f`.  Output planes are (f->height, f->width) float64; a NULL
 * pointer skips that channel.  Entries outside the computed window are not
 * touched (callers zero them: ProbabilityField.empty, fields.py:209-212).
 * Gauss-Legendre quadrature on the breakpoint partition in float64.
 */
int cpb_classify_closed(const cpb_field* f, int64_t row_begin, int64_t row_end, double* d_pmin,
                        double* d_pmax, double* d_psaddle, void* stream);

/* cpb_classify_closed plus the expected per-type counts of the launch's
 * vertices (sum of p_min, p_max, p_saddle over rows [row_begin, row_end)),
 * ADDED to d_counts[0..2] (3 device doubles): fused into the stencil kernels'
 * epilogue (per-block partials, summed in block order: deterministic). */
int cpb_classify_closed_counts(const cpb_field* f, int64_t row_begin, int64_t row_end,
                               double* d_pmin, double* d_pmax, double* d_psaddle, double* d_counts,
                               void* stream);

/*
 * Monte Carlo pattern fractions (engine.py:195-222, 632-666): n_samples joint
 * inverse-CDF draws per vertex, strict comparisons, p = count / n.  With
 * CPB_RNG_SPLITMIX the draws are the reference's keyed stream, so counts
 * are identical to the reference's.  d_counts (optional, int64 x 3 planes
 * min/max/saddle, same shape as the outputs) receives the raw hit counts.
 */
int cpb_classify_mc(const cpb_field* f, int64_t row_begin, int64_t row_end, uint64_t seed,
                    int64_t n_samples, int32_t rng, double* d_pmin, double* d_pmax,
                    double* d_psaddle, int64_t* d_counts, void* stream);

/*
 * Semianalytical estimator, histogram fields only (engine.py:416-459, grid
 * chunk engine.py:669-683): c centre draws from the keyed stream (plane 0,
 * the same draws as the reference), exact neighbour CDFs at each draw, the
 * conditional pattern probabilities averaged.  Per-draw arithmetic repeats
 * numpy's; the mean re-associates numpy's pairwise sum (~1e-16 relative).
 */
int cpb_classify_semi(const cpb_field* f, int64_t row_begin, int64_t row_end, uint64_t seed,
                      int64_t c, double* d_pmin, double* d_pmax, double* d_psaddle,
                      void* stream);

/*
 * Combinatorial (Eq. 5) cross-check, histogram fields with bins <= 8
 * (engine.py:320-404, grid chunk engine.py:686-702): sum over all bins^5
 * bin combinations of the bin-mass product times the all-uniform
 * probabilities.  Agrees with the closed form to ~1e-12 (the reference's own
 * acceptance bar is 1e-9, test_acceptance.py:100-108).
 */
int cpb_classify_combinatorial(const cpb_field* f, int64_t row_begin, int64_t row_end,
                               double* d_pmin, double* d_pmax, double* d_psaddle, void* stream);

/*
 * Reference-layout float64 parameters (fields.py:86-103, what from_ensemble
 * returns): uniform/histogram -> d_a = lo, d_b = hi (widened),
 * d_weights = (H, W, bins) weights; epanechnikov -> d_a = mean,
 * d_b = halfwidth; gaussian -> d_a = mean, d_b = stddev.
 */
int cpb_materialize(const cpb_field* f, double* d_a, double* d_b, double* d_weights,
                    void* stream);

/* Uniform [0, 1) draws of the keyed splitmix64 stream, shape (npix, planes, n),
 * samples [start, start + n) -- rngstream.py:33-48. */
int cpb_unit_block(uint64_t seed, const uint64_t* d_pixels, int64_t npix, int32_t planes,
                   int64_t start, int64_t n, double* d_out, void* stream);

/* Synthetic member-major ensemble rows [row0, row0 + nrows) of a height x width
 * grid: value = f32(bowl(r, c) + noise_amp * (2u - 1)), u = keyed stream
 * (seed, r * width + c, plane m, sample 0).  The host twin is
 * oracle.critprob_oracle.synthetic_rows (bit-identical). */
int cpb_synth_ensemble(float* d_ens, int64_t members, int64_t row0, int64_t nrows, int64_t width,
                       int64_t height, double noise_amp, uint64_t seed, void* stream);

/*
 * One-call host path: host ensemble in, host probabilities out.  Streams the
 * ensemble through the device in row chunks (H2D overlapped with the fit),
 * fits, classifies all interior rows and copies the three float64 planes and
 * the validity mask back.  h_ens should be pinned (cpb_host_alloc) for full
 * PCIe bandwidth.  method: 0 = closed form, 1 = Monte Carlo.
 * Synchronous; returns CPB_ENONFINITE on NaN/Inf input.
 */
int cpb_run_host(const float* h_ens, int64_t members, int64_t height, int64_t width,
                 int32_t kind, int32_t bins, double k, int32_t method, uint64_t seed,
                 int64_t n_samples, uint32_t channels, double* h_pmin, double* h_pmax,
                 double* h_psaddle, uint8_t* h_valid);

/*
 * Several models over ONE upload of the ensemble (the reference workflow
 * `stack = EnsembleStack(v); for model: classify_field(from_ensemble(stack,
 * model))`): every row chunk crossing PCIe is fitted for all n_models models
 * while resident, and the vertex rows a chunk completes are stencilled and
 * copied back while later chunks are still crossing PCIe (the eps of the rows
 * seen so far is kept on the device; rows whose result depends on eps are
 * redone with the final eps, so the output equals the whole-stack result).
 * Model i is (kinds[i], bins[i], ks[i]); h_out[3*i + c] receives channel c
 * (min, max, saddle) of model i (NULL skips).  Device scratch comes from a
 * library-owned stream-ordered pool that keeps its memory between calls
 * (see cpb_release_workspace).
 */
int cpb_run_host_models(const float* h_ens, int64_t members, int64_t height, int64_t width,
                        int32_t n_models, const int32_t* kinds, const int32_t* bins,
                        const double* ks, int32_t method, uint64_t seed, int64_t n_samples,
                        uint32_t channels, double* const* h_out, uint8_t* h_valid);

/* P5 heatmap bytes of one probability plane (export_heatmap, field_io.py:138-150):
 * d_out[i] = round_half_even(255 * clip(d_p[i], 0, 1)^gamma), 0 where d_valid[i]
 * is 0 (d_valid may be NULL). */
int cpb_heatmap(const double* d_p, const uint8_t* d_valid, int64_t n, double gamma,
                uint8_t* d_out, void* stream);

/*
 * Batched per-case API.  A batch is n_cases neighbourhoods (NeighborhoodCase,
 * engine.py:50-71), each a centre plus `neighbors` (2 or 4) distributions in
 * the reference's order (east, north, west, south | first, second), stored
 * position-major per case: distribution d = case * (1 + neighbors) + position.
 * Kinds may be mixed inside a case.  All arrays are device memory.
 *   uniform / epanechnikov / histogram : a = support lo, b = support hi
 *                                        (epanechnikov(mean, hw) has support mean -+ hw)
 *   gaussian (GaussianSampler)          : a = mean, b = stddev (Monte Carlo only)
 *   histogram                           : bins[d] bins, weights[woff[d] + j], already
 *                                         normalised (FiniteDistribution stores w / w.sum())
 * Outputs are n_cases x 3 float64 (p_min, p_max, p_saddle) per case.
 */
typedef struct cpb_case_batch {
  int64_t n_cases;
  int32_t neighbors;       /* 2 or 4 */
  int32_t max_bins;        /* largest histogram bin count in the batch (1 if none) */
  const int32_t* kind;     /* CPB_UNIFORM | CPB_EPANECHNIKOV | CPB_HISTOGRAM | CPB_GAUSSIAN */
  const double* a;
  const double* b;
  const int32_t* bins;
  const int64_t* woff;
  const double* weights;
} cpb_case_batch;

/* closed_form_triple (engine.py:177-178) of every case: exact piecewise
 * integration on the breakpoint union.  Cases holding a Gaussian yield NaN
 * (the reference raises TypeError; check kinds before calling). */
int cpb_cases_closed(const cpb_case_batch* batch, double* d_out, void* stream);

/* mc_all_patterns(case_i, n, seed, pixel_i) (engine.py:238-247) of every case:
 * pixel_i = d_pixels[i] (NULL: i).  Bit-identical to the reference for
 * uniform / histogram kinds.  d_counts (n_cases x 3 uint64, optional) receives
 * the pattern counts. */
int cpb_cases_mc(const cpb_case_batch* batch, uint64_t seed, const uint64_t* d_pixels, int64_t n,
                 uint64_t* d_counts, double* d_out, void* stream);

/* semianalytical_prob(case_i, pattern, c, seed, pixel_i) for all three patterns
 * (engine.py:416-441); histogram-only cases (others yield NaN). */
int cpb_cases_semi(const cpb_case_batch* batch, uint64_t seed, const uint64_t* d_pixels, int64_t c,
                   double* d_out, void* stream);

/* combinatorial_triple (engine.py:399-404, Eq. 5); histogram-only cases with
 * at most 8 bins (CPB_EINVAL above, as the reference's ValueError). */
int cpb_cases_combinatorial(const cpb_case_batch* batch, double* d_out, void* stream);

/* Pinned host memory for cpb_run_host buffers. */
int cpb_host_alloc(void** ptr, size_t bytes);
int cpb_host_free(void* ptr);

/* Return the current device's cached workspace (the pool cpb_run_host* draw
 * their device scratch from) to the driver.  Reports the bytes released. */
int cpb_release_workspace(size_t* released_bytes);

#ifdef __cplusplus
}
#endif

#endif /* CRITPROB_B200_H */
