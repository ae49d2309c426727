// mma_env.cu -- MMA issue rate of one warp while other warps of the CTA sleep on an
// mbarrier (the core kernel's epilogue warps), vs alone; TMEM 256 vs 512 columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_env tools/mma_env.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int mode, int cols, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  __shared__ uint32_t addr_s[2];
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); mbar_init(&done, 1); fence_mbar_init();
    addr_s[0] = smem_u32(smem); addr_s[1] = smem_u32(smem + 32768);
  }
  if (threadIdx.x >= 32 && threadIdx.x < 64) tmem_alloc(&slot, cols);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  const int warp = threadIdx.x / 32;
  if (warp == 1) {
    uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    if (mode >= 3) { a = addr_s[0]; b = addr_s[1]; }  // per-thread registers: R2UR before every MMA
    const uint32_t idesc = umma_idesc(1u, 64, 128u);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode == 4) {
        if (threadIdx.x == 32) mma_bf16(tm, umma_desc(a + (i & 3) * 32, 128), umma_desc(b + (i & 3) * 32, 128), idesc, 1u);
      } else {
        if (elect_one()) mma_bf16(tm, umma_desc(a + (i & 3) * 32, 128), umma_desc(b + (i & 3) * 32, 128), idesc, 1u);
        __syncwarp();
      }
    }
    __syncwarp();
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 32) { out[blockIdx.x] = clock64() - t0; mbar_arrive(&done); }
  } else if (warp >= 2 && mode == 1) {
    mbar_wait_sleep(&done, 0);
  } else if (warp >= 2 && mode == 2) {
    mbar_wait(&done, 0);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tm, cols); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 2048;
  const char* names[] = {"others idle at bar.sync", "others mbar_wait_sleep", "others mbar_wait spin",
                         "addresses from smem (R2UR)", "same, lane 0 issues"};
  for (int cols : {256})
    for (int mode = 0; mode < 5; ++mode) {
      k<<<148, 320, 200 * 1024>>>(mode, cols, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      printf("tmem %d cols, %-28s %6.1f cycles/MMA (N=64)\n", cols, names[mode], avg / 148 / iters);
    }
  return 0;
}
