// mma_layout.cu -- dense tcgen05 kind::f16 MMA throughput (M=128, K=16) with the A
// operand in SW128 vs SWIZZLE_NONE K-major layouts (the T1 window of lrs_core.cuh).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_layout tools/mma_layout.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int n, int mode, uint32_t lbo, uint32_t sbo, int rowoff, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 1024);
    const uint32_t idesc = umma_idesc(1u, n, 128u);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint64_t ad;
      if (mode == 0) ad = umma_desc(a + (i & 3) * 32, 128);
      else ad = umma_desc_noswz(a + ((i * rowoff) & 63) * 16 + (i & 3) * 2 * lbo, lbo, sbo);
      mma_bf16(tm, ad, umma_desc(b + (i & 3) * 32, 128), idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 4096;
  struct Cfg { int mode; uint32_t lbo, sbo; int rowoff; const char* what; };
  Cfg cfgs[] = {{0, 0, 0, 0, "SW128 A"},
                {1, 4096, 128, 0, "NONE LBO=4096 SBO=128"},
                {1, 4096, 128, 1, "NONE LBO=4096 SBO=128 row offsets"},
                {1, 4096 + 64, 128, 0, "NONE LBO=4160 SBO=128"},
                {1, 4096 + 16, 128, 0, "NONE LBO=4112 SBO=128"},
                {1, 2048 + 1024 + 512 + 256 + 128 + 16, 128, 0, "NONE LBO=4000 SBO=128"},
                {1, 128, 256, 0, "NONE LBO=128 SBO=256 (K-interleaved)"}};
  for (int n : {64, 128, 256})
    for (const Cfg& c : cfgs) {
      k<<<148, 128, 200 * 1024>>>(n, c.mode, c.lbo, c.sbo, c.rowoff, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      const double cyc = avg / iters;
      printf("N=%3d %-40s %6.1f cycles/MMA -> %6.0f MAC/clk/SM\n", n, c.what, cyc, 128.0 * n * 16 / cyc);
    }
  return 0;
}
