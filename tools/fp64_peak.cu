// FP64 / FP32 pipe peak microbenchmark (the FP64 roofline denominator of the
// closed-form stencils; MEASURED_PEAKS.json has HBM and bf16 only).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak            -> one JSON line
//
// Each thread runs ILP independent FMA chains; the grid fills every SM with
// enough warps to hide the pipe latency.  Timed with CUDA events after a
// warm-up; best of 5.  FLOP = 2 per FMA.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kIlp = 8;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kIlp; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;  // keeps the chains live
}

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kIlp; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}

// DSETP + DMNMX-style work (the stencils' comparisons on the FP64 pipe)
__global__ void dmin_kernel(double* out, double a) {
  double x[kIlp];
#pragma unroll
  for (int i = 0; i < kIlp; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kIlp; ++i) x[i] = fmin(x[i], a + it);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kIlp; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

template <typename K, typename... A>
static float best_ms(K kern, int blocks, int threads, A... args) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(args...);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(args...);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount, threads = 256, blocks = sms * 8;
  double* d;
  cudaMalloc(&d, 64);
  const double n = (double)blocks * threads * kIters * kIlp;
  const float t64 = best_ms(dfma_kernel, blocks, threads, d, 0.999999, 1e-7);
  const float t32 = best_ms(ffma_kernel, blocks, threads, (float*)d, 0.999999f, 1e-7f);
  const float tmn = best_ms(dmin_kernel, blocks, threads, d, 0.5);
  const double f64 = 2.0 * n / (t64 * 1e-3) / 1e12, f32 = 2.0 * n / (t32 * 1e-3) / 1e12;
  const double nominal = (double)sms * 64 * 2 * clk_khz * 1e3 / 1e12;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_mhz_attr\": %.0f, \"dfma_tflops\": %.2f, "
         "\"dfma_per_sm_per_clk_at_attr_clock\": %.1f, \"ffma_tflops\": %.2f, "
         "\"dmnmx_gops\": %.1f, \"fp64_nominal_64_per_sm_tflops\": %.2f, \"how\": \"%d blocks x %d "
         "threads x %d iters x %d independent FMA chains, best of 5, CUDA events\"}\n",
         p.name, sms, clk_khz / 1e3, f64, f64 * 1e12 / 2 / sms / (clk_khz * 1e3), f32,
         n / (tmn * 1e-3) / 1e9, nominal, blocks, threads, kIters, kIlp);
  cudaFree(d);
  return 0;
}
