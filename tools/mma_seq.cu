// mma_seq.cu -- MMA issue sequences of lrs_core.cuh in isolation: where do the ~120
// cycles per N = 64 MMA measured inside the kernel (tools/ctrace.py) come from, against
// 48 in a plain loop (tools/mma_baseoff.cu)?  Variants (each 4096 MMAs, M = 128, N = 64,
// K = 16, SW128 A and B, one thread issues):
//   0 plain loop, one accumulator
//   1 groups of 4 MMAs alternating between 2 accumulators (a1: two M blocks)
//   2 as 1 + tcgen05.commit to an mbarrier after every 8 MMAs (a1: per X chunk)
//   3 as 2 + the issuing warp waits for that commit before the next group (no overlap)
//   4 groups of 4 with a try_wait on an already-completed mbarrier + fence per group
//   5 A operand 16 KB apart per group (a1 blocks), one accumulator
//   6 ONE elect block around the whole loop (groups of 4, running descriptor offsets)
//   7 as 6 with one MMA per loop iteration (no unrolling)
//   8 as 6 while 3 other warps spin on an mbarrier try_wait (the kernels' waiting warps)
//   9 as 8 with the spinning warps backing off (nanosleep between polls)
//  10 the core kernel's a1 loop: per chunk 3 M blocks (16 KB apart, 3 accumulators) x 4 K
//     steps, a commit per chunk, chunks 27 KB apart -- one elected thread
//  11 as 10 with random data instead of a constant
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_seq tools/mma_seq.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int mode, int total, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t v = 0x3c003c00u;
    if (mode == 11) {  // random bf16 pairs with moderate exponents
      uint32_t hsh = static_cast<uint32_t>(i) * 2654435761u;
      hsh ^= hsh >> 13;
      hsh *= 0x5bd1e995u;
      v = (hsh & 0x807F807Fu) | 0x3C003C00u;
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x >= 32 && mode >= 8) {
    // other warps poll a barrier that completes only when the MMA thread is done
    while (!mbar_try_wait(&done, 1))
      if (mode == 9) __nanosleep(200);
  }
  if (threadIdx.x < 32) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = umma_idesc(1u, 64u, 128u);
    const uint64_t ad = umma_desc(a, 128), bd = umma_desc(b, 128);
    // a completed barrier for mode 4
    if (threadIdx.x == 0) mbar_arrive(&done);
    __syncwarp();
    const long long t0 = clock64();
    uint32_t ph = 0;
    if (mode >= 10) {
      if (elect_one()) {
        const uint64_t ud = umma_desc(a + 4 * 27648 - 8192, 128);
        for (int it = 0; it < total / 48; ++it)
          for (int c = 0; c < 4; ++c) {
            const uint64_t xd = ad + static_cast<uint32_t>(c) * (27648u >> 4);
            for (int b1 = 0; b1 < 3; ++b1) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16(tm + b1 * 64u, xd + b1 * 1024u + 2 * kk, ud + 2 * kk, idesc, (c > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&bar);
          }
      }
      __syncwarp();
    } else if (mode >= 6) {
      if (elect_one()) {
        if (mode == 6 || mode >= 8) {
          uint32_t ao = 0;
          for (int g = 0; g < total / 4; ++g) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_bf16(tm, ad + ao + 2 * kk, bd + 2 * kk, idesc, 1u);
            ao = (ao + 1024u) & 4095u;
          }
        } else {
          for (int i = 0; i < total; ++i) mma_bf16(tm, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
        }
      }
      __syncwarp();
    }
    for (int g = 0; g < (mode >= 6 ? 0 : total / 4); ++g) {
      if (mode == 4) {
        mbar_wait(&done, 0);
        tc_fence_after();
      }
      if (elect_one()) {
        const uint32_t d = tm + ((mode >= 1 && mode <= 3) ? (g & 1) * 64u : 0u);
        const uint64_t ab = ad + (mode == 5 ? (g & 3) * 1024u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16(d, ab + 2 * kk, bd + 2 * kk, idesc, 1u);
        if ((mode == 2 || mode == 3) && (g & 1)) mma_commit(&bar);
      }
      __syncwarp();
      if (mode == 3 && (g & 1)) {
        mbar_wait(&bar, ph);
        ph ^= 1u;
      }
    }
    if (elect_one()) mma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 1);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tm, 256);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
  const char* what[] = {"plain loop, one accumulator", "groups of 4, two accumulators",
                        "+ commit per 8 MMAs", "+ wait for each commit", "try_wait + fence per group of 4",
                        "A 16 KB apart per group", "one elect block, groups of 4", "one elect block, 1 per iteration",
                        "6 + 3 warps spinning on try_wait", "6 + 3 warps polling with nanosleep",
                        "core a1 loop (3 blocks, commit/chunk)", "core a1 loop, random data"};
  const int total = 4096;
  for (int mode = 0; mode < 12; ++mode) {
    k<<<148, 128, 201 * 1024>>>(mode, total, d);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("fault mode %d\n", mode);
      return 1;
    }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    printf("mode %d %-36s %6.1f cycles/MMA\n", mode, what[mode], avg / 148 / total);
  }
  return 0;
}
