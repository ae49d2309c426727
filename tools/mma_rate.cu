// mma_rate.cu -- tcgen05 MMA issue-to-completion throughput on one SM per CTA:
// dense kind::f16 (K=16) vs 2:4 sparse (K=32 logical), M=128, N in {64,128,256},
// A/B in shared memory (SS).  Operands are garbage (timing only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_rate tools/mma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int n, int sparse, int iters, unsigned long long* out, int bsbo, int nacc, int extra) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t idesc = umma_idesc(1u, n, 128u) | (sparse ? (1u << 2) : 0u);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if ((extra & 1) && (i & 1) == 0) tmem_cp_128x128b(tm + 480, umma_desc_rows16(smem_u32(smem + 65536)));
      if ((extra & 2) && (i & 1) == 1) mma_commit(&bar2);
      if (sparse)
        mma_sp_bf16(tm + (i % nacc) * n, umma_desc(a, 64), umma_desc_sbo(b + (i & 1) * 64, 128, bsbo), idesc | (i & 1), 1u, tm + 480);
      else
        mma_bf16(tm + (i % nacc) * n, umma_desc(a + (i & 3) * 32, 128), umma_desc_sbo(b + (i & 3) * 32, 128, bsbo), idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  for (int extra = 0; extra < 4; ++extra)
  for (int sp = 1; sp < 2; ++sp)
    for (int n : {64, 256})
      for (int nacc : {1}) {
        if (n * nacc > 448) continue;
        const int sbo = 1024;
        k<<<148, 128, 100 * 1024>>>(n, sp, iters, d, sbo, nacc, extra);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double cyc = avg / iters;
        const double kl = sp ? 32 : 16;
        printf("extra=%d (1=cp/2mma, 2=commit/2mma) ", extra); printf("%s N=%3d: %6.1f cycles/MMA  -> %6.0f logical MAC/clk/SM\n", sp ? "sparse" : "dense ", n, cyc,
               128.0 * n * kl / cyc);
      }
  return 0;
}
