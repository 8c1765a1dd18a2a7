// Non-tensor FMA peaks of the B200 (the roofline denominator of
// the ALU-bound resampling kernels). Each thread runs ILP independent FMA
// chains for ITERS steps; grid = SMs x 8 CTAs of 256 threads, so every
// scheduler has 16 warps to issue from. Reports the best of 10 launches (CUDA
// events) and the SM clock NVML would report is sampled by the caller.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu
//   ./fma_peak        -> JSON line {"dfma_tflops", "ffma_tflops", "ffma2_tflops", ...}
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ILP = 8;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma_kernel(float* out, float a, float b) {
  float x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-9f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float a, float b) {
  float2 x[ILP];
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = make_float2(threadIdx.x * 1e-9f + i, i);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = __ffma2_rn(x[i], a2, b2);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i].x + x[i].y;
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const int ctas = sms * 8, thr = 256;
  double* dd;
  float* df;
  cudaMalloc(&dd, 1024 * sizeof(double));
  cudaMalloc(&df, 1024 * sizeof(float));
  const double n_fma = (double)ctas * thr * ILP * ITERS;
  const float t64 = best_ms([&] { dfma_kernel<<<ctas, thr>>>(dd, 0.999999, 1e-7); });
  const float t32 = best_ms([&] { ffma_kernel<<<ctas, thr>>>(df, 0.999999f, 1e-7f); });
  const float t32x2 = best_ms([&] { ffma2_kernel<<<ctas, thr>>>(df, 0.999999f, 1e-7f); });
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"ctas\": %d, \"threads\": %d, \"ilp\": %d, \"iters\": %d, "
         "\"dfma_ms\": %.4f, \"ffma_ms\": %.4f, \"ffma2_ms\": %.4f, "
         "\"dfma_tflops\": %.3f, \"ffma_tflops\": %.3f, \"ffma2_tflops\": %.3f, "
         "\"dfma_per_sm_per_clk_at_attr_clock\": %.2f, \"attr_clock_mhz\": %.0f, \"err\": \"%s\"}\n",
         sms, ctas, thr, ILP, ITERS, t64, t32, t32x2, 2 * n_fma / (t64 * 1e-3) / 1e12,
         2 * n_fma / (t32 * 1e-3) / 1e12, 4 * n_fma / (t32x2 * 1e-3) / 1e12,
         n_fma / (t64 * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
