// FP64 CUDA-core FMA peak (the decomposition kernels) on the B200 (the three-roof's FP32-pipe denominator,
// SURVEY §8(d)): every thread runs 8 independent DFMA chains, grid = 8 CTAs x 256
// threads per SM, timed with CUDA events after a warm-up.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  fma_loop<<<blocks, threads>>>(out, 2000, 0.9999, 1e-4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_loop<<<blocks, threads>>>(out, iters, 0.9999, 1e-4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
  printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f, \"err\": \"%s\"}\n", flops / (best * 1e-3) / 1e12,
         sms, best, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
