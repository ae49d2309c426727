// probe_2cta_rate.cu -- issue rate of 2:4 sparse MMAs (bf16, K = 32 logical per MMA),
// one CTA (M = 128, N = n) vs a CTA pair (cta_group::2: M = 256, N = n, each CTA holding
// n/2 rows of B): cycles per MMA measured on the issuing thread over `iters` back-to-back
// MMAs (operands zero: only the rate matters).  Answers whether the pair form lifts the
// per-SM shared-memory bound of the windowed kernel's MMAs (A 4 KB + B n*64 B per MMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_2cta_rate tools/probe_2cta_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;


template <bool PAIR>
__global__ void rate(int n, int iters, long long* out, int cp_every) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  fence_proxy_async_smem();
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (t < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(&tslot, 512);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t m = PAIR ? 256u : 128u;
  if ((!PAIR || cluster_rank() == 0) && t == 0) {
    const uint32_t idesc = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(n) >> 3) << 17) | ((m >> 4) << 24);
    const uint64_t ad = umma_desc(smem_u32(smem), 64);
    const uint64_t bd = umma_desc(smem_u32(smem) + 8192, 128);
    const uint32_t e = tm + 384;
    long long t0 = clock64();
    const uint64_t ed = umma_desc_rows16(smem_u32(smem) + 49152);
    // blocks of 8 MMAs; a metadata copy before every block (cp_every = 8, into the
    // slots the MMAs read, 4 slots of 8 columns), into unread columns (-8), or none (0)
    for (int blk = 0; blk < iters / 8; ++blk) {
      const uint32_t es = static_cast<uint32_t>(blk & 3) * 8;
      if (cp_every == 8) {
        if (PAIR) tmem_cp_128x256b_2(e + es, ed);
        else tmem_cp_128x256b(e + es, ed);
      } else if (cp_every == -8) {
        if (PAIR) tmem_cp_128x256b_2(tm + 448 + es, ed);
        else tmem_cp_128x256b(tm + 448 + es, ed);
      }
      const uint32_t eu = cp_every == 8 ? e + es : e;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (PAIR)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n}" ::"r"(tm),
                       "l"(ad), "l"(bd), "r"(idesc | (q & 1)), "r"(1u), "r"(eu) : "memory");
        else
          mma_sp_bf16(tm, ad, bd, idesc | (q & 1), 1u, eu);
      }
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                       smem_u32(&bar)), "h"(static_cast<uint16_t>(3)) : "memory");
    else
      mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  __syncwarp();
  if (PAIR && cluster_rank() != 0 && t == 0) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  if (t < 32) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
    else tmem_dealloc(tm, 512);
  }
}

int main(int argc, char** argv) {
  const int iters = 4000;
  long long* d;
  cudaMalloc(&d, 2048 * 8);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int cpe : {0, 8, -8}) {
  printf("-- metadata tcgen05.cp every %d MMAs\n", cpe);
  for (int n : {128, 256}) {
    for (int grid : {148}) {
      rate<false><<<grid, 128, smem>>>(n, iters, d, cpe);
      cudaDeviceSynchronize();
      long long c1;
      cudaMemcpy(&c1, d, 8, cudaMemcpyDeviceToHost);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid == 1 ? 2 : 148);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, rate<true>, n, iters, d, cpe);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      long long c2 = 0;
      cudaMemcpy(&c2, d, 8, cudaMemcpyDeviceToHost);
      printf("N=%3d grid %3s: 1 CTA  M=128 %6.1f cyc/MMA (%5.0f logical MAC/clk/SM) | pair M=256 %6.1f cyc/MMA "
             "(%5.0f logical MAC/clk/SM) %s\n", n, grid == 1 ? "1" : "all", (double)c1 / iters,
             128.0 * n * 32 / ((double)c1 / iters), (double)c2 / iters, 128.0 * n * 32 / ((double)c2 / iters),
             cudaGetErrorString(e));
    }
  }
  }
  return 0;
}
