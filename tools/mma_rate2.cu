// mma_rate2.cu -- cost of one "item" of the fused kernel's MMA loop:
// [tcgen05.cp of 128x16B metadata] + S sparse MMAs (N each) + tcgen05.commit,
// issued by one elected lane of a warp-uniform loop, B start moving per item.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_rate2 tools/mma_rate2.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int n, int nmma, int use_cp, int move_b, int items, unsigned long long* out, int samed, int dowait) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 180 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  for (int i = threadIdx.x; i < 2048 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem + 176 * 1024)[i] = 0x44444444u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); mbar_init(&bar3, 1); mbar_arrive(&bar3); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x < 32) {
    const uint64_t ad = umma_desc(smem_u32(smem + 160 * 1024), 64);
    const uint64_t bd = umma_desc_sbo(smem_u32(smem), 128, 1024);
    const uint64_t ed = umma_desc_rows16(smem_u32(smem + 176 * 1024));
    const uint32_t idesc = umma_idesc(1u, n, 128u) | (1u << 2);
    const long long t0 = clock64();
    for (int i = 0; i < items; ++i) {
      if (dowait) { mbar_wait(&bar3, 0); tc_fence_after(); }
      const uint32_t tapoff = move_b ? static_cast<uint32_t>((i % 9) / 3 * 9 + (i % 3)) * 64u : 0u;
      if (elect_one()) {
        if (use_cp) tmem_cp_128x128b(tm + 480 + 4 * (i % 3), ed);
        for (int m = 0; m < nmma; ++m)
          mma_sp_bf16(samed ? tm : (tm + (m % 2) * 256 % 480), ad + 2 * (m & 1), bd + tapoff + 4 * (m & 1), idesc | (m & 1), 1u,
                      tm + 480 + 4 * (i % 3));
        mma_commit(&bar2);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int items = 2000;
  struct C { int n, nmma, cp, mv, same, wt; } cs[] = {{224, 0, 0, 1, 1, 0}, {224, 0, 1, 1, 1, 0}, {224, 0, 0, 1, 1, 1},
                                                       {224, 2, 1, 1, 1, 0}};
  for (auto c : cs) {
    k<<<148, 128, 200 * 1024>>>(c.n, c.nmma, c.cp, c.mv, items, d, c.same, c.wt);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("wait=%d sameD=%d ", c.wt, c.same); printf("N=%3d mma/item=%d cp=%d moveB=%d: %7.1f cycles/item, %6.1f cycles/MMA, %5.0f logical MAC/clk/SM\n", c.n,
           c.nmma, c.cp, c.mv, avg / items, avg / items / (c.nmma ? c.nmma : 1), 128.0 * c.n * 32 * c.nmma / (avg / items));
  }
  return 0;
}
