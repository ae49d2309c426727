// Probe of lrs_sym_pinv_kernel (lrs_decomp.cuh): Hadamard-of-Grams V from random factors,
// two runs (determinism), sweeps, and ||V P V - V|| / ||V||.  nvcc ... -o tools/pinv_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../paper_2006_06443_b200/csrc/lrs_decomp.cuh"
using namespace lrs;
int main(int argc, char** argv) {
  const int r = argc > 1 ? atoi(argv[1]) : 128;
  const int rows[4] = {512, 512, 3, 3};
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  double* dg[4];
  for (int m = 0; m < 4; ++m) {
    std::vector<double> f(rows[m] * r), gm(r * r, 0.0);
    for (auto& x : f) x = nd(g);
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        double s = 0;
        for (int i = 0; i < rows[m]; ++i) s += f[i * r + a] * f[i * r + b];
        gm[a * r + b] = s;
      }
    cudaMalloc(&dg[m], r * r * 8);
    cudaMemcpy(dg[m], gm.data(), r * r * 8, cudaMemcpyHostToDevice);
  }
  const int rp = (r + 1) & ~1;
  double *a, *v, *p;
  int* sw;
  cudaMalloc(&a, rp * rp * 8);
  cudaMalloc(&v, rp * rp * 8);
  cudaMalloc(&p, r * r * 8);
  cudaMalloc(&sw, 16);
  const size_t vb = (size_t)rp * rp * 8;
  for (int vsm = 0; vsm < 2; ++vsm) {
    const size_t smem = vsm ? vb : 0;
    if (smem > 210 * 1024) continue;
    cudaFuncSetAttribute(lrs_sym_pinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    std::vector<double> h1(r * r), h2(r * r);
    for (int run = 0; run < 2; ++run) {
      PinvParams q{};
      for (int i = 0; i < 4; ++i) q.g[i] = dg[i];
      q.mode = 0; q.r = r; q.rp = rp; q.a_smem = vsm; q.rcond = 1e-10; q.a = a; q.v = v; q.p = p; q.sweeps = sw;
      q.force_eigen = argc > 2 ? atoi(argv[2]) : 0;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      lrs_sym_pinv_kernel<<<1, kJThreads, smem>>>(q);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int sweeps; cudaMemcpy(&sweeps, sw, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(run ? h2.data() : h1.data(), p, r * r * 8, cudaMemcpyDeviceToHost);
      printf("v_smem %d run %d: %.3f ms, sweeps %d, err %s\n", vsm, run, ms, sweeps, cudaGetErrorString(cudaGetLastError()));
    }
    // V (host) and || V P V - V || / ||V||
    std::vector<double> V(r * r), gh(r * r);
    for (int i = 0; i < r * r; ++i) V[i] = 1.0;
    for (int m = 1; m < 4; ++m) {
      cudaMemcpy(gh.data(), dg[m], r * r * 8, cudaMemcpyDeviceToHost);
      for (int i = 0; i < r * r; ++i) V[i] *= gh[i];
    }
    std::vector<double> VP(r * r, 0.0);
    for (int i = 0; i < r; ++i) for (int k = 0; k < r; ++k) { const double x = V[i * r + k]; for (int j = 0; j < r; ++j) VP[i * r + j] += x * h1[k * r + j]; }
    double num = 0, den = 0;
    for (int i = 0; i < r; ++i) for (int j = 0; j < r; ++j) { double s = 0; for (int k = 0; k < r; ++k) s += VP[i * r + k] * V[k * r + j]; num += (s - V[i * r + j]) * (s - V[i * r + j]); den += V[i * r + j] * V[i * r + j]; }
    int same = 1; for (int i = 0; i < r * r; ++i) same &= h1[i] == h2[i];
    printf("v_smem %d: ||VPV - V||/||V|| = %.3e, deterministic %d\n", vsm, sqrt(num / den), same);
  }
  return 0;
}
