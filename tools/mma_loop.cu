// mma_loop.cu -- replicates the core kernel's phase-2 issue loop (warp-wide loop,
// elect_one issue, 4 K steps per tap, A = SWIZZLE_NONE window at a tap row offset,
// B = SW128 weight slot per tap) to time it in isolation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_loop tools/mma_loop.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int n, int mode, int reps, unsigned long long* out, int rnd) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t v = 0x3c003c00u;
    if (rnd) {  // pseudo-random bf16 pairs with magnitudes ~1
      uint32_t h = (i + 1) * 2654435761u;
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      v = (h & 0x807f807fu) | 0x3f003f00u;
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x < 32) {
    const uint32_t t1w = smem_u32(smem), gb = smem_u32(smem + 64 * 1024);
    const uint32_t lbo = 256 * 16;
    const uint32_t idesc = umma_idesc(1u, n, 128u);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int t = 0; t < 9; ++t) {
        const uint32_t tap_off = static_cast<uint32_t>((t / 3) * 16 + (t % 3)) * 16u;
        if (mode == 0) {
          if (elect_one()) {
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tm, umma_desc_noswz(t1w + tap_off + 2 * kk * lbo, lbo, 128u),
                       umma_desc(gb + t * 8192 + kk * 32u, 128), idesc, 1u);
          }
          __syncwarp();
        } else if (mode == 1) {
          if (elect_one()) {
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tm, umma_desc(t1w + 32 * 1024 + kk * 32, 128),
                       umma_desc(gb + t * 8192 + kk * 32u, 128), idesc, 1u);
          }
          __syncwarp();
        } else {
          if (elect_one()) {
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tm, umma_desc_noswz(t1w + 2 * kk * lbo, lbo, 128u),
                       umma_desc(gb + kk * 32u, 128), idesc, 1u);
          }
          __syncwarp();
        }
      }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int reps = 100;
  const char* names[] = {"NONE A + tap offsets, B per tap", "SW128 A, B per tap", "NONE A fixed, B fixed"};
  for (int rnd = 0; rnd < 2; ++rnd)
  for (int n : {64, 128})
    for (int mode = 0; mode < 3; ++mode) {
      k<<<148, 128, 210 * 1024>>>(n, mode, reps, d, rnd);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("%s N=%3d %-36s %6.1f cycles/MMA\n", rnd ? "random" : "ones  ", n, names[mode], avg / (reps * 36));
    }
  return 0;
}
