// C ABI entry points (include/critprob_b200.h): argument validation, error
// reporting and the one-call host pipeline.  Kernels live in cpb_fit.cu,
// cpb_closed.cu and cpb_mc.cu.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <chrono>
#include <vector>

#include "cpb_common.cuh"

#include <nvtx3/nvToolsExt.h>

// NVTX range around every compute entry point (header-only NVTX 3: a no-op
// unless a tool such as Nsight Systems / Compute is attached), so a trace of
// the reference-facing calls lines up with the kernels they launch.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define CPB_NVTX_RANGE(name) NvtxRange cpb_nvtx_range_(name)

namespace cpb {

int launch_fit(const float* ens, int64_t mstride, cpb_field* f, uint32_t* range, bool accumulate,
               cudaStream_t st);
int launch_from_scalar(const double* v, int64_t n, double half, double* lo, double* hi,
                       cudaStream_t st);
int launch_range_to_pair(const uint32_t* range, double* pair, cudaStream_t st);
int launch_nonfinite(const float* v, int64_t n, uint32_t* flag, cudaStream_t st);
size_t fit_classify_work_bytes(int64_t width, int64_t row_begin, int64_t row_end);
int launch_fit_classify(const float* ens, int64_t mstride, cpb_field* const* fields, int n,
                        uint32_t* range, bool accumulate, int64_t row_begin, int64_t row_end,
                        double* pmin, double* pmax, double* psad, void* work, cudaStream_t st);
int launch_fit_classify_finish(const cpb_field* f, int64_t row_begin, int64_t row_end, double* pmin,
                               double* pmax, double* psad, double* counts, void* work, cudaStream_t st);
int launch_pair_to_eps(const double* pair, double* eps, cudaStream_t st);
int launch_materialize(const cpb_field* f, double* a, double* b, double* w, cudaStream_t st);
int launch_synth(float* ens, int64_t members, int64_t row0, int64_t nrows, int64_t width,
                 int64_t height, double amp, uint64_t seed, cudaStream_t st);
int launch_closed(const cpb_field* f, int64_t row_begin, int64_t row_end, double* pmin,
                  double* pmax, double* psad, cudaStream_t st, double* counts);
int launch_mc(const cpb_field* f, int64_t row_begin, int64_t row_end, uint64_t seed, int64_t n,
              int rng, double* pmin, double* pmax, double* psad, int64_t* counts, cudaStream_t st);
int launch_unit_block(uint64_t seed, const uint64_t* px, int64_t npix, int planes, int64_t start,
                      int64_t n, double* out, cudaStream_t st);
int launch_semi(const cpb_field* f, int64_t row_begin, int64_t row_end, uint64_t seed, int64_t c,
                double* pmin, double* pmax, double* psad, cudaStream_t st);
int launch_combinatorial(const cpb_field* f, int64_t row_begin, int64_t row_end, double* pmin,
                         double* pmax, double* psad, cudaStream_t st);
int launch_heatmap(const double* p, const uint8_t* valid, int64_t n, double gamma, uint8_t* out,
                   cudaStream_t st);
int launch_eps_sensitive_rows(const cpb_field* f, double eps, uint8_t* sens, cudaStream_t st);
int launch_fit_multi(const float* ens, int64_t mstride, cpb_field* const* fs, int n, uint32_t* range,
                     bool accumulate, cudaStream_t st);
int launch_cases_closed(const cpb_case_batch* b, double* out, cudaStream_t st);
int launch_cases_mc(const cpb_case_batch* b, uint64_t seed, const uint64_t* pixels, int64_t n,
                    unsigned long long* counts, double* out, cudaStream_t st);
int launch_cases_semi(const cpb_case_batch* b, uint64_t seed, const uint64_t* pixels, int64_t c,
                      double* out, cudaStream_t st);
int launch_cases_combinatorial(const cpb_case_batch* b, double* out, cudaStream_t st);

extern int g_fit_ctas_per_sm;
int workspace_alloc(void** p, size_t bytes, cudaStream_t st);
void workspace_free(void* p, cudaStream_t st);

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return e == cudaErrorMemoryAllocation ? CPB_ENOMEM : CPB_ECUDA;
}

static int check_field(const cpb_field* f, bool need_eps) {
  if (!f) { set_error("field is NULL"); return CPB_EINVAL; }
  if (f->kind < CPB_UNIFORM || f->kind > CPB_GAUSSIAN) {
    set_error("unknown model kind %d", f->kind);
    return CPB_EINVAL;
  }
  if (f->height < 0 || f->width < 0) { set_error("negative field extent"); return CPB_EINVAL; }
  if (f->kind == CPB_HISTOGRAM && f->bins < 1) { set_error("bins must be at least 1"); return CPB_EINVAL; }
  if (need_eps && !(f->eps >= 0.0)) { set_error("field eps is not set"); return CPB_EINVAL; }
  return CPB_OK;
}

}  // namespace cpb

using namespace cpb;

extern "C" {

int cpb_abi_version(void) { return CPB_ABI_VERSION; }

int cpb_set_option(const char* name, int64_t value) {
  if (!name) { set_error("NULL option name"); return CPB_EINVAL; }
  if (strcmp(name, "fit_ctas_per_sm") == 0) {
    if (value < 0 || value > 32) { set_error("fit_ctas_per_sm must be in [0, 32]"); return CPB_EINVAL; }
    g_fit_ctas_per_sm = (int)value;
    return CPB_OK;
  }
  set_error("unknown option %s", name);
  return CPB_EINVAL;
}

const char* cpb_last_error(void) { return g_err; }

double cpb_epsilon(double gmin, double gmax) {
  // distributions.py:30-36
  const double spread = gmax - gmin;
  const double e = 1e-9 * spread;
  return e > 1e-12 ? e : 1e-12;
}

int cpb_field_plane_bytes(int32_t kind, int32_t bins, int32_t members, int64_t height,
                          int64_t width, size_t out[7]) {
  if (!out || height < 0 || width < 0 || members < 1) {
    set_error("invalid field extent");
    return CPB_EINVAL;
  }
  const size_t n = (size_t)height * (size_t)width;
  for (int i = 0; i < 7; ++i) out[i] = 0;
  if (kind == CPB_UNIFORM || kind == CPB_HISTOGRAM) {
    out[0] = out[1] = n * sizeof(float);
  } else if (kind == CPB_EPANECHNIKOV || kind == CPB_GAUSSIAN) {
    out[2] = out[3] = n * sizeof(double);
  } else {
    set_error("unknown model kind %d", kind);
    return CPB_EINVAL;
  }
  if (kind == CPB_HISTOGRAM) {
    if (bins < 1) { set_error("bins must be at least 1"); return CPB_EINVAL; }
    if (members > 65535) { set_error("histogram fit supports at most 65535 members"); return CPB_EINVAL; }
    out[4] = n * (size_t)bins * (members <= 255 ? 1 : 2);
    out[5] = (size_t)(members + 1) * sizeof(double);
  }
  out[6] = 3 * sizeof(uint32_t);
  return CPB_OK;
}

int cpb_fit(const float* d_ens, int64_t member_stride, cpb_field* f, uint32_t* d_range,
            int32_t accumulate, void* stream) {
  CPB_NVTX_RANGE("cpb_fit");
  int s = check_field(f, false);
  if (s) return s;
  if (f->members < 1) { set_error("ensemble needs at least one member"); return CPB_EINVAL; }
  if (f->members < 2 && (f->kind == CPB_EPANECHNIKOV || f->kind == CPB_GAUSSIAN)) {
    set_error("%s fit needs at least two members",
              f->kind == CPB_EPANECHNIKOV ? "epanechnikov" : "gaussian");
    return CPB_EINVAL;
  }
  if (f->kind == CPB_HISTOGRAM && f->members > 65535) {
    set_error("histogram fit supports at most 65535 members");
    return CPB_EINVAL;
  }
  if (member_stride < f->height * f->width) { set_error("member_stride smaller than a member plane"); return CPB_EINVAL; }
  if (!d_ens || !d_range) { set_error("NULL ensemble or range pointer"); return CPB_EINVAL; }
  return launch_fit(d_ens, member_stride, f, d_range, accumulate != 0, (cudaStream_t)stream);
}

int cpb_fit_multi(const float* d_ens, int64_t member_stride, cpb_field* const* fields,
                  int32_t n_fields, uint32_t* d_range, int32_t accumulate, void* stream) {
  CPB_NVTX_RANGE("cpb_fit_multi");
  if (!fields || n_fields < 1 || n_fields > 16) { set_error("1..16 fields expected"); return CPB_EINVAL; }
  for (int i = 0; i < n_fields; ++i) {
    cpb_field* f = fields[i];
    if (!f) { set_error("NULL field"); return CPB_EINVAL; }
    if (f->height != fields[0]->height || f->width != fields[0]->width ||
        f->members != fields[0]->members) {
      set_error("fields of one fused fit must share height, width and members");
      return CPB_EINVAL;
    }
  }
  // validation (and, when the fused kernel does not cover the set, the fits
  // themselves) through the single-model entry point
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < n_fields; ++i) {
    int s = check_field(fields[i], false);
    if (s) return s;
    cpb_field* f = fields[i];
    if (f->members < 1) { set_error("ensemble needs at least one member"); return CPB_EINVAL; }
    if (f->members < 2 && (f->kind == CPB_EPANECHNIKOV || f->kind == CPB_GAUSSIAN)) {
      set_error("%s fit needs at least two members", f->kind == CPB_EPANECHNIKOV ? "epanechnikov" : "gaussian");
      return CPB_EINVAL;
    }
    if (f->kind == CPB_HISTOGRAM && f->members > 65535) {
      set_error("histogram fit supports at most 65535 members");
      return CPB_EINVAL;
    }
  }
  if (member_stride < fields[0]->height * fields[0]->width) { set_error("member_stride smaller than a member plane"); return CPB_EINVAL; }
  if (!d_ens || !d_range) { set_error("NULL ensemble or range pointer"); return CPB_EINVAL; }
  const int rc = n_fields > 1 ? launch_fit_multi(d_ens, member_stride, fields, n_fields, d_range, accumulate != 0, st) : 1;
  if (rc != 1) return rc;
  for (int i = 0; i < n_fields; ++i) {
    int s = launch_fit(d_ens, member_stride, fields[i], d_range, accumulate != 0 || i > 0, st);
    if (s) return s;
  }
  return CPB_OK;
}

int cpb_read_range(const uint32_t* d_range, double* gmin, double* gmax, void* stream) {
  uint32_t h[3];
  cudaError_t e = cudaMemcpyAsync(h, d_range, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "read range");
  if (h[2]) { set_error("ensemble values must be finite"); return CPB_ENONFINITE; }
  if (gmin) *gmin = (double)ordered_to_float(h[0]);
  if (gmax) *gmax = (double)ordered_to_float(h[1]);
  return CPB_OK;
}

int cpb_fit_classify_work_bytes(int64_t width, int64_t row_begin, int64_t row_end, size_t* bytes) {
  if (!bytes || width < 3 || row_begin > row_end) { set_error("invalid arguments"); return CPB_EINVAL; }
  *bytes = fit_classify_work_bytes(width, row_begin, row_end);
  return CPB_OK;
}

int cpb_fit_classify(const float* d_ens, int64_t member_stride, cpb_field* f, uint32_t* d_range,
                     int32_t accumulate, int64_t row_begin, int64_t row_end, double* d_pmin,
                     double* d_pmax, double* d_psaddle, void* d_work, void* stream) {
  CPB_NVTX_RANGE("cpb_fit_classify");
  if (!d_ens || !f || !d_range || !d_work || !f->lo || !f->hi) { set_error("null argument"); return CPB_EINVAL; }
  return launch_fit_classify(d_ens, member_stride, &f, 1, d_range, accumulate != 0, row_begin, row_end,
                             d_pmin, d_pmax, d_psaddle, d_work, (cudaStream_t)stream);
}

int cpb_fit_multi_classify(const float* d_ens, int64_t member_stride, cpb_field* const* fields,
                           int32_t n_fields, uint32_t* d_range, int32_t accumulate, int64_t row_begin,
                           int64_t row_end, double* d_pmin, double* d_pmax, double* d_psaddle,
                           void* d_work, void* stream) {
  CPB_NVTX_RANGE("cpb_fit_multi_classify");
  if (!d_ens || !fields || !d_range || !d_work) { set_error("null argument"); return CPB_EINVAL; }
  for (int i = 0; i < n_fields; ++i)
    if (!fields[i]) { set_error("null field"); return CPB_EINVAL; }
  return launch_fit_classify(d_ens, member_stride, fields, n_fields, d_range, accumulate != 0, row_begin,
                             row_end, d_pmin, d_pmax, d_psaddle, d_work, (cudaStream_t)stream);
}

int cpb_fit_classify_finish(const cpb_field* f, int64_t row_begin, int64_t row_end, double* d_pmin,
                            double* d_pmax, double* d_psaddle, double* d_counts, void* d_work,
                            void* stream) {
  CPB_NVTX_RANGE("cpb_fit_classify_finish");
  if (int rc = check_field(f, true)) return rc;
  if (!d_work) { set_error("null workspace"); return CPB_EINVAL; }
  return launch_fit_classify_finish(f, row_begin, row_end, d_pmin, d_pmax, d_psaddle, d_counts, d_work,
                                    (cudaStream_t)stream);
}

int cpb_check_finite(const float* d_values, int64_t n, void* stream) {
  CPB_NVTX_RANGE("cpb_check_finite");
  if (n < 0 || (n > 0 && !d_values)) { set_error("invalid values"); return CPB_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* flag = nullptr;
  if (int rc = workspace_alloc((void**)&flag, sizeof(uint32_t), st)) return rc;
  uint32_t h = 0;
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(uint32_t), st);
  int rc = e == cudaSuccess ? launch_nonfinite(d_values, n, flag, st) : cuda_status(e, "memset");
  if (rc == CPB_OK) {
    e = cudaMemcpyAsync(&h, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_status(e, "finiteness flag");
  }
  workspace_free(flag, st);
  if (rc == CPB_OK && h) { set_error("ensemble values must be finite"); return CPB_ENONFINITE; }
  return rc;
}

int cpb_range_to_pair(const uint32_t* d_range, double* d_pair, void* stream) {
  if (!d_range || !d_pair) { set_error("NULL range or pair pointer"); return CPB_EINVAL; }
  return launch_range_to_pair(d_range, d_pair, (cudaStream_t)stream);
}

int cpb_pair_to_eps(const double* d_pair, double* d_eps, void* stream) {
  if (!d_pair || !d_eps) { set_error("NULL pair or eps pointer"); return CPB_EINVAL; }
  return launch_pair_to_eps(d_pair, d_eps, (cudaStream_t)stream);
}

int cpb_from_scalar(const double* d_values, int64_t height, int64_t width, double error_bound,
                    double eps, double* d_lo, double* d_hi, void* stream) {
  CPB_NVTX_RANGE("cpb_from_scalar");
  if (!(error_bound >= 0.0)) { set_error("error bound must be nonnegative"); return CPB_EINVAL; }
  double half = 0.5 * error_bound;
  if (half <= 0.0) half = 0.5 * eps;  // fields.py:174-176
  return launch_from_scalar(d_values, height * width, half, d_lo, d_hi, (cudaStream_t)stream);
}

int cpb_classify_closed(const cpb_field* f, int64_t row_begin, int64_t row_end, double* d_pmin,
                        double* d_pmax, double* d_psaddle, void* stream) {
  CPB_NVTX_RANGE("cpb_classify_closed");
  int s = check_field(f, true);
  if (s) return s;
  if (f->kind == CPB_GAUSSIAN) {
    set_error("Gaussian fields have no closed form; use monte_carlo");
    return CPB_EINVAL;
  }
  if (row_begin < 1 || row_end > f->height - 1 || f->width < 3) {
    if (row_end > row_begin) {
      set_error("rows [%lld, %lld) need a one-row halo inside the field",
                (long long)row_begin, (long long)row_end);
      return CPB_EINVAL;
    }
  }
  return launch_closed(f, row_begin, row_end, d_pmin, d_pmax, d_psaddle, (cudaStream_t)stream, nullptr);
}

int cpb_classify_closed_counts(const cpb_field* f, int64_t row_begin, int64_t row_end,
                               double* d_pmin, double* d_pmax, double* d_psaddle, double* d_counts,
                               void* stream) {
  CPB_NVTX_RANGE("cpb_classify_closed_counts");
  if (!d_counts) { set_error("d_counts must not be NULL"); return CPB_EINVAL; }
  int s = check_field(f, true);
  if (s) return s;
  if (f->kind == CPB_GAUSSIAN) {
    set_error("Gaussian fields have no closed form; use monte_carlo");
    return CPB_EINVAL;
  }
  if (row_begin < 1 || row_end > f->height - 1 || f->width < 3) {
    if (row_end > row_begin) {
      set_error("rows [%lld, %lld) need a one-row halo inside the field",
                (long long)row_begin, (long long)row_end);
      return CPB_EINVAL;
    }
  }
  return launch_closed(f, row_begin, row_end, d_pmin, d_pmax, d_psaddle, (cudaStream_t)stream, d_counts);
}

int cpb_classify_mc(const cpb_field* f, int64_t row_begin, int64_t row_end, uint64_t seed,
                    int64_t n_samples, int32_t rng, double* d_pmin, double* d_pmax,
                    double* d_psaddle, int64_t* d_counts, void* stream) {
  CPB_NVTX_RANGE("cpb_classify_mc");
  int s = check_field(f, true);
  if (s) return s;
  if (rng != CPB_RNG_SPLITMIX && rng != CPB_RNG_PHILOX) { set_error("unknown rng %d", rng); return CPB_EINVAL; }
  if (row_begin < 1 || row_end > f->height - 1 || f->width < 3) {
    if (row_end > row_begin) {
      set_error("rows [%lld, %lld) need a one-row halo inside the field",
                (long long)row_begin, (long long)row_end);
      return CPB_EINVAL;
    }
  }
  return launch_mc(f, row_begin, row_end, seed, n_samples, rng, d_pmin, d_pmax, d_psaddle,
                   d_counts, (cudaStream_t)stream);
}

int cpb_classify_semi(const cpb_field* f, int64_t row_begin, int64_t row_end, uint64_t seed,
                      int64_t c, double* d_pmin, double* d_pmax, double* d_psaddle,
                      void* stream) {
  CPB_NVTX_RANGE("cpb_classify_semi");
  int s = check_field(f, true);
  if (s) return s;
  if (row_begin < 1 || row_end > f->height - 1 || f->width < 3) {
    if (row_end > row_begin) {
      set_error("rows [%lld, %lld) need a one-row halo inside the field",
                (long long)row_begin, (long long)row_end);
      return CPB_EINVAL;
    }
  }
  return launch_semi(f, row_begin, row_end, seed, c, d_pmin, d_pmax, d_psaddle,
                     (cudaStream_t)stream);
}

int cpb_classify_combinatorial(const cpb_field* f, int64_t row_begin, int64_t row_end,
                               double* d_pmin, double* d_pmax, double* d_psaddle, void* stream) {
  CPB_NVTX_RANGE("cpb_classify_combinatorial");
  int s = check_field(f, true);
  if (s) return s;
  if (row_begin < 1 || row_end > f->height - 1 || f->width < 3) {
    if (row_end > row_begin) {
      set_error("rows [%lld, %lld) need a one-row halo inside the field",
                (long long)row_begin, (long long)row_end);
      return CPB_EINVAL;
    }
  }
  return launch_combinatorial(f, row_begin, row_end, d_pmin, d_pmax, d_psaddle,
                              (cudaStream_t)stream);
}

int cpb_materialize(const cpb_field* f, double* d_a, double* d_b, double* d_weights,
                    void* stream) {
  CPB_NVTX_RANGE("cpb_materialize");
  int s = check_field(f, true);
  if (s) return s;
  return launch_materialize(f, d_a, d_b, d_weights, (cudaStream_t)stream);
}

int cpb_unit_block(uint64_t seed, const uint64_t* d_pixels, int64_t npix, int32_t planes,
                   int64_t start, int64_t n, double* d_out, void* stream) {
  CPB_NVTX_RANGE("cpb_unit_block");
  if (npix < 0 || planes < 0 || n < 0 || start < 0) { set_error("negative extent"); return CPB_EINVAL; }
  return launch_unit_block(seed, d_pixels, npix, planes, start, n, d_out, (cudaStream_t)stream);
}

int cpb_synth_ensemble(float* d_ens, int64_t members, int64_t row0, int64_t nrows, int64_t width,
                       int64_t height, double noise_amp, uint64_t seed, void* stream) {
  CPB_NVTX_RANGE("cpb_synth_ensemble");
  if (members < 1 || nrows < 0 || width < 1 || height < 1 || row0 < 0 || row0 + nrows > height) {
    set_error("invalid synthetic ensemble extent");
    return CPB_EINVAL;
  }
  return launch_synth(d_ens, members, row0, nrows, width, height, noise_amp, seed,
                      (cudaStream_t)stream);
}

int cpb_heatmap(const double* d_p, const uint8_t* d_valid, int64_t n, double gamma,
                uint8_t* d_out, void* stream) {
  CPB_NVTX_RANGE("cpb_heatmap");
  if (!(gamma > 0.0)) { set_error("gamma must be positive"); return CPB_EINVAL; }
  if (n < 0 || (n > 0 && (!d_p || !d_out))) { set_error("invalid heatmap buffers"); return CPB_EINVAL; }
  return launch_heatmap(d_p, d_valid, n, gamma, d_out, (cudaStream_t)stream);
}

int cpb_host_alloc(void** ptr, size_t bytes) {
  cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) return cuda_status(e, "cudaHostAlloc");
  return CPB_OK;
}

int cpb_host_free(void* ptr) {
  cudaError_t e = cudaFreeHost(ptr);
  if (e != cudaSuccess) return cuda_status(e, "cudaFreeHost");
  return CPB_OK;
}

// ---------------------------------------------------------------------------
// One-call host pipeline.
// ---------------------------------------------------------------------------
namespace {

// Library-owned stream-ordered pool per device.  Its release threshold is
// unbounded, so a host call's multi-GB scratch stays mapped for the next call:
// with the default pool every call re-maps (and at the final synchronize
// unmaps) tens of GB, which costs 0.1-3 s of host time per call.
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

int workspace_pool(cudaMemPool_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) { set_error("device ordinal out of range"); return CPB_EINVAL; }
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    e = cudaMemPoolCreate(&g_pool[dev], &props);
    if (e != cudaSuccess) { g_pool[dev] = nullptr; return cuda_status(e, "cudaMemPoolCreate"); }
    uint64_t keep = ~0ull;
    e = cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemPoolSetAttribute");
  }
  *out = g_pool[dev];
  return CPB_OK;
}

}  // namespace
}  // extern "C"

namespace cpb {
int workspace_alloc(void** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool;
  if (int rc = workspace_pool(&pool)) return rc;
  cudaError_t e = cudaMallocFromPoolAsync(p, bytes, pool, st);
  if (e != cudaSuccess) { *p = nullptr; return cuda_status(e, "cudaMallocFromPoolAsync"); }
  return CPB_OK;
}

void workspace_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}
}  // namespace cpb

extern "C" {

namespace {

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  int alloc(size_t bytes, cudaStream_t s) {
    st = s;
    if (bytes == 0) return CPB_OK;
    cudaMemPool_t pool;
    if (int rc = workspace_pool(&pool)) return rc;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, s);
    if (e != cudaSuccess) { p = nullptr; return cuda_status(e, "cudaMallocAsync"); }
    return CPB_OK;
  }
};

struct Streams {
  cudaStream_t s[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Streams() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (s[i]) { cudaStreamSynchronize(s[i]); cudaStreamDestroy(s[i]); }
    }
  }
};

}  // namespace

int cpb_run_host_models(const float* h_ens, int64_t members, int64_t height, int64_t width,
                        int32_t n_models, const int32_t* kinds, const int32_t* bins,
                        const double* ks, int32_t method, uint64_t seed, int64_t n_samples,
                        uint32_t channels, double* const* h_out, uint8_t* h_valid) {
  CPB_NVTX_RANGE("cpb_run_host_models");
  if (!h_ens || members < 1 || height < 1 || width < 1) {
    set_error("ensemble needs at least one member and one pixel");
    return CPB_EINVAL;
  }
  if (height < 3 || width < 3) { set_error("field must be at least 3 x 3 to have interior pixels"); return CPB_EINVAL; }
  if (method != 0 && method != 1) { set_error("method must be 0 (closed form) or 1 (monte carlo)"); return CPB_EINVAL; }
  if (n_models < 1 || n_models > 16 || !kinds || !bins || !ks) { set_error("1..16 models expected"); return CPB_EINVAL; }
  for (int i = 0; i < n_models; ++i) {
    if (method == 0 && kinds[i] == CPB_GAUSSIAN) { set_error("Gaussian fields have no closed form; use monte_carlo"); return CPB_EINVAL; }
    if (members < 2 && (kinds[i] == CPB_EPANECHNIKOV || kinds[i] == CPB_GAUSSIAN)) {
      set_error("%s fit needs at least two members", kinds[i] == CPB_EPANECHNIKOV ? "epanechnikov" : "gaussian");
      return CPB_EINVAL;
    }
  }
  const int nm = n_models;
  const auto t_start = std::chrono::steady_clock::now();
  auto host_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  };
  size_t pb[16][7];
  int s;
  for (int i = 0; i < nm; ++i)
    if ((s = cpb_field_plane_bytes(kinds[i], bins[i], (int32_t)members, height, width, pb[i]))) return s;
  // streams: ss.s[0..1] chunk ring (H2D + fits), sx[0] stencils, sx[1] D2H
  Streams ss, sx;
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&ss.s[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ss.ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sx.s[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sx.ev[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_status(e, "stream setup");
  cudaStream_t s0 = ss.s[0], scls = sx.s[0], scopy = sx.s[1];
  size_t max_pitch = 0;
  {
    int dev = 0, mp = 0;
    e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mp, cudaDevAttrMaxPitch, dev);
    if (e != cudaSuccess) return cuda_status(e, "device attribute");
    max_pitch = (size_t)(unsigned)mp;
    if (const char* v = getenv("CPB_HOST_MAX_PITCH")) max_pitch = (size_t)atoll(v);  // tests
  }
  const size_t plane = (size_t)height * width;
  const size_t row_bytes = (size_t)members * width * sizeof(float);
  static const size_t chunk_bytes = [] {  // CPB_HOST_CHUNK_BYTES overrides, for tests
    const char* v = getenv("CPB_HOST_CHUNK_BYTES");
    return v ? (size_t)atoll(v) : (size_t)(256u << 20);
  }();
  int64_t chunk = (int64_t)std::max<size_t>(2, chunk_bytes / row_bytes);
  if (chunk > height) chunk = height;
  const int64_t nchunks = (height + chunk - 1) / chunk;
  // per-model compact planes, the device eps of every chunk, outputs
  DevBuf planes[16][7], epsbuf[16], pair[16], out[16], sens[16];
  cpb_field fm[16];
  for (int i = 0; i < nm; ++i) {
    for (int q = 0; q < 7; ++q)
      if ((s = planes[i][q].alloc(pb[i][q], s0))) return s;
    if ((s = epsbuf[i].alloc((size_t)nchunks * sizeof(double), s0)) ||
        (s = pair[i].alloc(2 * sizeof(double), s0)) || (s = sens[i].alloc((size_t)height, s0)) ||
        (s = out[i].alloc(3 * plane * sizeof(double), s0)))
      return s;
    // the stencils write every interior vertex; only the border columns of the
    // copied rows need zeros (two strided columns per plane, not 3 x H x W)
    for (int c = 0; c < 3 && e == cudaSuccess; ++c) {
      double* base = (double*)out[i].p + c * plane;
      e = cudaMemset2DAsync(base, width * sizeof(double), 0, sizeof(double), (size_t)height, s0);
      if (e == cudaSuccess)
        e = cudaMemset2DAsync(base + width - 1, width * sizeof(double), 0, sizeof(double),
                              (size_t)height, s0);
    }
    if (e != cudaSuccess) return cuda_status(e, "memset");
    cpb_field& f = fm[i];
    f = cpb_field{};
    f.kind = kinds[i]; f.bins = bins[i]; f.members = (int32_t)members;
    f.height = height; f.width = width; f.row0 = 0; f.global_width = width;
    f.k = ks[i]; f.eps = 0.0;
    f.lo = planes[i][0].p; f.hi = planes[i][1].p; f.mean = (double*)planes[i][2].p;
    f.spread = (double*)planes[i][3].p; f.weights = planes[i][4].p;
    f.weight_table = (double*)planes[i][5].p;
  }
  DevBuf ebuf[2];
  for (int i = 0; i < 2; ++i)
    if ((s = ebuf[i].alloc((size_t)chunk * row_bytes, s0))) return s;
  e = cudaEventRecord(ss.ev[0], s0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ss.s[1], ss.ev[0], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(scls, ss.ev[0], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(scopy, ss.ev[0], 0);
  if (e != cudaSuccess) return cuda_status(e, "event");
  struct Launch { int64_t r0, r1, chunk; };
  std::vector<Launch> launches;
  // per-chunk events (the ring events are reused, so the stencil stream waits on its own copy)
  std::vector<cudaEvent_t> fitted((size_t)nchunks, nullptr), classified((size_t)nchunks, nullptr);
  struct EvVec {
    std::vector<cudaEvent_t>* a; std::vector<cudaEvent_t>* b; cudaStream_t st[4];
    ~EvVec() {  // destroyed before the buffers: drain every stream first (also on
                // an error return, when work may still be queued on any of them)
      for (cudaStream_t x : st)
        if (x) cudaStreamSynchronize(x);
      for (auto* v : {a, b})
        for (auto ev : *v) if (ev) cudaEventDestroy(ev);
    }
  } evguard{&fitted, &classified, {ss.s[0], ss.s[1], scls, scopy}};
  for (int64_t j = 0; j < nchunks; ++j) {
    e = cudaEventCreateWithFlags(&fitted[j], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&classified[j], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e, "event create");
  }
  auto classify_rows = [&](int i, int64_t r0, int64_t r1, const double* eps_dev, double eps_host,
                           cudaStream_t st) -> int {
    cpb_field f = fm[i];
    f.eps_device = eps_dev;
    f.eps = eps_host;
    double* pmin = (double*)out[i].p;
    double* om = (channels & CPB_CH_MIN) ? pmin : nullptr;
    double* oM = (channels & CPB_CH_MAX) ? pmin + plane : nullptr;
    double* oS = (channels & CPB_CH_SADDLE) ? pmin + 2 * plane : nullptr;
    if (method == 0) return cpb_classify_closed(&f, r0, r1, om, oM, oS, st);
    return cpb_classify_mc(&f, r0, r1, seed, n_samples, CPB_RNG_SPLITMIX, om, oM, oS, nullptr, st);
  };
  // unrequested channels are never computed: their host planes are zeroed on
  // the host instead (the reference leaves them exactly 0.0, test_engine.py:616-623)
  auto copy_rows = [&](int i, int64_t r0, int64_t r1) -> int {
    const double* base = (const double*)out[i].p;
    for (int c = 0; c < 3; ++c) {
      double* dst = h_out ? h_out[3 * i + c] : nullptr;
      if (!dst || r1 <= r0 || !(channels & (1u << c))) continue;
      const size_t off = (size_t)r0 * width, n = (size_t)(r1 - r0) * width;
      cudaError_t ce = cudaMemcpyAsync(dst + off, base + c * plane + off, n * sizeof(double),
                                       cudaMemcpyDeviceToHost, scopy);
      if (ce != cudaSuccess) return cuda_status(ce, "D2H probabilities");
    }
    return CPB_OK;
  };
  // CPB_HOST_TRACE=1: per-chunk timeline on stderr (H2D done, fits done, stencil done)
  static const bool trace = getenv("CPB_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, st);
    tev.push_back(ev);
  };
  tmark(s0);
  const double t_setup = host_ms();
  int64_t next_row = 1;  // first vertex row not yet classified
  for (int64_t j = 0; j < nchunks; ++j) {
    const int64_t r0 = j * chunk, nr = std::min(chunk, height - r0);
    const int b = (int)(j & 1);
    cudaStream_t st = ss.s[b];
    // one 2-D copy: M member rows of nr*W floats, source pitch = member plane;
    // a member plane wider than the driver's maximum pitch (grids of >= 2^29
    // pixels) goes as one plain copy per member instead
    if (plane * sizeof(float) <= max_pitch) {
      e = cudaMemcpy2DAsync(ebuf[b].p, (size_t)nr * width * sizeof(float), h_ens + r0 * width,
                            plane * sizeof(float), (size_t)nr * width * sizeof(float), (size_t)members,
                            cudaMemcpyHostToDevice, st);
    } else {
      for (int64_t m = 0; m < members && e == cudaSuccess; ++m)
        e = cudaMemcpyAsync((float*)ebuf[b].p + m * nr * width, h_ens + m * plane + r0 * width,
                            (size_t)nr * width * sizeof(float), cudaMemcpyHostToDevice, st);
    }
    if (e != cudaSuccess) return cuda_status(e, "H2D ensemble chunk");
    tmark(st);
    if (j > 0) {  // range accumulation is serialised across the ring by chunk order
      e = cudaStreamWaitEvent(st, ss.ev[b ^ 1], 0);
      if (e != cudaSuccess) return cuda_status(e, "event wait");
    }
    const size_t off = (size_t)r0 * width;
    // one pass over the chunk for all models (cpb_fit_multi); the shared data
    // range accumulates in model 0's range words
    cpb_field fcs[16];
    cpb_field* fptr[16];
    uint32_t* rng0 = (uint32_t*)planes[0][6].p;
    for (int i = 0; i < nm; ++i) {
      cpb_field& fc = fcs[i];
      fc = fm[i];
      fc.height = nr;
      fc.lo = pb[i][0] ? (char*)planes[i][0].p + off * sizeof(float) : nullptr;
      fc.hi = pb[i][1] ? (char*)planes[i][1].p + off * sizeof(float) : nullptr;
      fc.mean = pb[i][2] ? (double*)planes[i][2].p + off : nullptr;
      fc.spread = pb[i][3] ? (double*)planes[i][3].p + off : nullptr;
      // bin planes are (bins, H, W): the chunk view offsets the base pointer and
      // keeps the full-grid plane stride
      fc.weights = pb[i][4] ? (char*)planes[i][4].p + off * (members <= 255 ? 1 : 2) : nullptr;
      fc.plane_stride = (int64_t)plane;
      fptr[i] = &fc;
    }
    if ((s = cpb_fit_multi((const float*)ebuf[b].p, (int64_t)nr * width, fptr, nm, rng0, j > 0, st)))
      return s;
    for (int i = 0; i < nm; ++i) {
      fm[i].bounds = fcs[i].bounds;
      fm[i].weights_mode = fcs[i].weights_mode;
      // provisional eps of the rows fitted so far (exact once the last chunk is in)
      if ((s = cpb_range_to_pair(rng0, (double*)pair[i].p, st)) ||
          (s = cpb_pair_to_eps((const double*)pair[i].p, (double*)epsbuf[i].p + j, st)))
        return s;
    }
    if ((e = cudaEventRecord(ss.ev[b], st)) != cudaSuccess || (e = cudaEventRecord(fitted[j], st)) != cudaSuccess)
      return cuda_status(e, "event record");
    tmark(st);
    // stencil the vertex rows whose three rows are now fitted, copy them back
    const int64_t hi_row = (j + 1 == nchunks) ? height - 1 : std::min(r0 + nr - 1, height - 1);
    if (hi_row > next_row) {
      e = cudaStreamWaitEvent(scls, fitted[j], 0);
      if (e != cudaSuccess) return cuda_status(e, "event wait");
      for (int i = 0; i < nm; ++i)
        if ((s = classify_rows(i, next_row, hi_row, (const double*)epsbuf[i].p + j, 0.0, scls))) return s;
      launches.push_back({next_row, hi_row, j});
      tmark(scls);
      if ((e = cudaEventRecord(classified[j], scls)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(scopy, classified[j], 0)) != cudaSuccess)
        return cuda_status(e, "event");
      for (int i = 0; i < nm; ++i)
        if ((s = copy_rows(i, next_row, hi_row))) return s;
      next_row = hi_row;
    }
  }
  const double t_enqueued = host_ms();
  // host work while the device pipeline runs: the border rows of the outputs
  // (never copied back; zero like the reference's invalid border) and the mask
  for (int i = 0; i < nm; ++i)
    for (int c = 0; c < 3; ++c)
      if (double* dst = h_out ? h_out[3 * i + c] : nullptr) {
        if (!(channels & (1u << c))) {
          memset(dst, 0, plane * sizeof(double));
          continue;
        }
        memset(dst, 0, (size_t)width * sizeof(double));
        memset(dst + (size_t)(height - 1) * width, 0, (size_t)width * sizeof(double));
      }
  if (h_valid) {
    for (int64_t r = 0; r < height; ++r) {
      uint8_t* row = h_valid + r * width;
      const uint8_t inner = (r > 0 && r < height - 1) ? 1 : 0;
      memset(row, inner, (size_t)width);
      row[0] = 0;
      row[width - 1] = 0;
    }
  }
  // exactness: rows stencilled with a provisional eps are redone where some
  // pixel's result depends on eps (degenerate / clamped pixels; normally none)
  e = cudaStreamSynchronize(ss.s[0]);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ss.s[1]);
  if (e != cudaSuccess) return cuda_status(e, "synchronize");
  std::vector<double> eps_host((size_t)nchunks);
  std::vector<uint8_t> sens_host((size_t)height);
  for (int i = 0; i < nm; ++i) {
    e = cudaMemcpy(eps_host.data(), epsbuf[i].p, (size_t)nchunks * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_status(e, "D2H eps");
    const double eps_final = eps_host[(size_t)nchunks - 1];
    if (eps_final != eps_final) { set_error("ensemble values must be finite"); return CPB_ENONFINITE; }
    fm[i].eps = eps_final;
    bool stale = false;
    for (const Launch& L : launches) stale |= eps_host[(size_t)L.chunk] != eps_final;
    if (!stale) continue;
    if ((s = launch_eps_sensitive_rows(&fm[i], eps_final, (uint8_t*)sens[i].p, scls))) return s;
    e = cudaMemcpyAsync(sens_host.data(), sens[i].p, (size_t)height, cudaMemcpyDeviceToHost, scls);
    if (e == cudaSuccess) e = cudaStreamSynchronize(scls);
    if (e != cudaSuccess) return cuda_status(e, "D2H sensitivity");
    for (const Launch& L : launches) {
      if (eps_host[(size_t)L.chunk] == eps_final) continue;
      for (int64_t v = L.r0; v < L.r1;) {
        if (!(sens_host[v - 1] | sens_host[v] | sens_host[v + 1])) { ++v; continue; }
        int64_t w = v + 1;
        while (w < L.r1 && (sens_host[w - 1] | sens_host[w] | sens_host[w + 1])) ++w;
        if ((s = classify_rows(i, v, w, nullptr, eps_final, scls))) return s;
        cudaEvent_t done;
        if ((e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming)) != cudaSuccess)
          return cuda_status(e, "event");
        e = cudaEventRecord(done, scls);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(scopy, done, 0);
        cudaEventDestroy(done);
        if (e != cudaSuccess) return cuda_status(e, "event");
        if ((s = copy_rows(i, v, w))) return s;
        v = w;
      }
    }
  }
  e = cudaStreamSynchronize(scls);
  if (e == cudaSuccess) e = cudaStreamSynchronize(scopy);
  if (e != cudaSuccess) return cuda_status(e, "synchronize");
  if (trace) {
    fprintf(stderr, "cpb_trace_host setup=%.1f enqueued=%.1f done=%.1f ms\n", t_setup, t_enqueued, host_ms());
    for (size_t q = 1; q < tev.size(); ++q) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[q]);
      fprintf(stderr, "%s%.2f", q == 1 ? "cpb_trace_ms " : " ", ms);
    }
    fprintf(stderr, "\n");
    for (auto ev : tev) cudaEventDestroy(ev);
  }
  return CPB_OK;
}

int cpb_cases_closed(const cpb_case_batch* batch, double* d_out, void* stream) {
  CPB_NVTX_RANGE("cpb_cases_closed");
  return launch_cases_closed(batch, d_out, (cudaStream_t)stream);
}

int cpb_cases_mc(const cpb_case_batch* batch, uint64_t seed, const uint64_t* d_pixels, int64_t n,
                 uint64_t* d_counts, double* d_out, void* stream) {
  CPB_NVTX_RANGE("cpb_cases_mc");
  return launch_cases_mc(batch, seed, d_pixels, n, (unsigned long long*)d_counts, d_out,
                         (cudaStream_t)stream);
}

int cpb_cases_semi(const cpb_case_batch* batch, uint64_t seed, const uint64_t* d_pixels, int64_t c,
                   double* d_out, void* stream) {
  CPB_NVTX_RANGE("cpb_cases_semi");
  return launch_cases_semi(batch, seed, d_pixels, c, d_out, (cudaStream_t)stream);
}

int cpb_cases_combinatorial(const cpb_case_batch* batch, double* d_out, void* stream) {
  CPB_NVTX_RANGE("cpb_cases_combinatorial");
  return launch_cases_combinatorial(batch, d_out, (cudaStream_t)stream);
}

int cpb_release_workspace(size_t* released_bytes) {
  cudaMemPool_t pool;
  if (int rc = workspace_pool(&pool)) return rc;
  uint64_t before = 0, after = 0;
  cudaError_t e = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &before);
  if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
  if (e == cudaSuccess) e = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &after);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemPoolTrimTo");
  if (released_bytes) *released_bytes = (size_t)(before - after);
  return CPB_OK;
}

int cpb_run_host(const float* h_ens, int64_t members, int64_t height, int64_t width,
                 int32_t kind, int32_t bins, double k, int32_t method, uint64_t seed,
                 int64_t n_samples, uint32_t channels, double* h_pmin, double* h_pmax,
                 double* h_psaddle, uint8_t* h_valid) {
  CPB_NVTX_RANGE("cpb_run_host");
  double* outs[3] = {h_pmin, h_pmax, h_psaddle};
  return cpb_run_host_models(h_ens, members, height, width, 1, &kind, &bins, &k, method, seed,
                             n_samples, channels, outs, h_valid);
}

}  // extern "C"
