// Instruction throughput of the FP64-pipe operations the closed-form stencils
// issue besides DFMA (compares, conversions), against the FP32 / integer ones
// that could replace them.  One JSON line: giga-ops/s and ops per SM per clock
// (at the attribute clock) for each kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_rates tools/pipe_rates.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048, kIlp = 8;

#define KERNEL_BEGIN(name, T)                                      \
  __global__ void name(T* out, T a, T b, int64_t tb) {             \
    T x[kIlp];                                                      \
    unsigned acc[kIlp];                                             \
    _Pragma("unroll") for (int i = 0; i < kIlp; ++i) {              \
      x[i] = (T)(threadIdx.x * 1e-3 + i);                           \
      acc[i] = 0;                                                   \
    }                                                               \
    for (int it = 0; it < kIters; ++it) {                           \
      _Pragma("unroll") for (int i = 0; i < kIlp; ++i) {
#define KERNEL_END(T)                                               \
      }                                                             \
    }                                                               \
    T s = 0;                                                        \
    unsigned u = 0;                                                 \
    _Pragma("unroll") for (int i = 0; i < kIlp; ++i) {              \
      s += x[i];                                                    \
      u += acc[i];                                                  \
    }                                                               \
    if (s == (T)1.2345 || u == 77777u) out[0] = s + (T)u;           \
  }

// reference: DFMA
KERNEL_BEGIN(k_dfma, double) x[i] = fma(x[i], a, b); KERNEL_END(double)
KERNEL_BEGIN(k_dadd, double) x[i] = x[i] + b; KERNEL_END(double)
KERNEL_BEGIN(k_dmul, double) x[i] = x[i] * a; KERNEL_END(double)
// DSETP: compare against a value that changes through integer ops only
KERNEL_BEGIN(k_dsetp, double)
  const double t = __longlong_as_double(tb + (int64_t)(it * kIlp + i));
  acc[i] += (x[i] < t) ? 1u : 0u;
KERNEL_END(double)
// same structure with FSETP (FP32 compare) -- isolates the DSETP cost
KERNEL_BEGIN(k_fsetp, float)
  const float t = __int_as_float((int)tb + (it * kIlp + i));
  acc[i] += (x[i] < t) ? 1u : 0u;
KERNEL_END(float)
// 64-bit integer compare (ISETP + ISETP.EX)
KERNEL_BEGIN(k_isetp64, double)
  const int64_t t = tb + (int64_t)(it * kIlp + i);
  acc[i] += (__double_as_longlong(x[i]) < t) ? 1u : 0u;
KERNEL_END(double)
// double -> float conversion (F2F.F32.F64) feeding an FP32 add
KERNEL_BEGIN(k_d2f, double)
  const double t = __longlong_as_double(tb + (int64_t)(it * kIlp + i));
  acc[i] += __float_as_uint((float)t);
KERNEL_END(double)
// float -> double conversion (F2F.F64.F32) feeding an integer add
KERNEL_BEGIN(k_f2d, double)
  const float t = __int_as_float((int)tb + (it * kIlp + i));
  acc[i] += (unsigned)__double2hiint((double)t);
KERNEL_END(double)
// fmin on doubles (DSETP.MIN + two SELs)
KERNEL_BEGIN(k_dmin, double)
  x[i] = fmin(x[i], __longlong_as_double(tb + (int64_t)(it * kIlp + i)));
KERNEL_END(double)
// FP32 min (FMNMX)
KERNEL_BEGIN(k_fmin, float)
  x[i] = fminf(x[i], __int_as_float((int)tb + (it * kIlp + i)));
KERNEL_END(float)

template <typename K, typename T>
static double rate(K kern, int blocks, int threads, T* d, T a, T b, int64_t tb) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(d, a, b, tb);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, a, b, tb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return (double)blocks * threads * kIters * kIlp / (best * 1e-3);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount, threads = 256, blocks = sms * 8;
  void* d;
  cudaMalloc(&d, 64);
  double* dd = (double*)d;
  float* df = (float*)d;
  const int64_t tbd = __builtin_bit_cast(int64_t, 0.5);
  const int64_t tbf = (int64_t)__builtin_bit_cast(int32_t, 0.5f);
  struct R { const char* n; double r; } rs[] = {
      {"dfma", rate(k_dfma, blocks, threads, dd, 0.999999, 1e-7, 0)},
      {"dadd", rate(k_dadd, blocks, threads, dd, 0.999999, 1e-7, 0)},
      {"dmul", rate(k_dmul, blocks, threads, dd, 0.999999, 1e-7, 0)},
      {"dsetp", rate(k_dsetp, blocks, threads, dd, 0.0, 0.0, tbd)},
      {"fsetp", rate(k_fsetp, blocks, threads, df, 0.0f, 0.0f, tbf)},
      {"isetp64", rate(k_isetp64, blocks, threads, dd, 0.0, 0.0, tbd)},
      {"f2f_d2f", rate(k_d2f, blocks, threads, dd, 0.0, 0.0, tbd)},
      {"f2f_f2d", rate(k_f2d, blocks, threads, dd, 0.0, 0.0, tbf)},
      {"dmin", rate(k_dmin, blocks, threads, dd, 0.0, 0.0, tbd)},
      {"fmin", rate(k_fmin, blocks, threads, df, 0.0f, 0.0f, tbf)},
  };
  const double per = (double)sms * clk_khz * 1e3;
  printf("{\"gpu\": \"%s\", \"clock_mhz_attr\": %.0f", p.name, clk_khz / 1e3);
  for (auto& r : rs) printf(", \"%s\": {\"gops\": %.1f, \"per_sm_clk\": %.1f}", r.n, r.r / 1e9, r.r / per);
  printf("}\n");
  return 0;
}
