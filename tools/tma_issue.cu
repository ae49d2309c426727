// tma_issue.cu -- single-thread issue cost of bulk copies: N x cp.async.bulk (1-D, bytes
// each) on one mbarrier, timed from the first issue to the last issue (clock64) and to
// completion.  One CTA per SM, data from a 64 MB buffer (L2 / HBM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_issue tools/tma_issue.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(const uint8_t* src, int nreq, uint32_t bytes, int stride_blocks, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint8_t* base = src + (static_cast<size_t>(blockIdx.x) * 65536 * 4) % (48u << 20);
    mbar_arrive_expect_tx(&bar, nreq * bytes);
    const long long t0 = clock64();
    for (int i = 0; i < nreq; ++i)
      bulk_load(smem_raw + (i * bytes) % (160 * 1024), base + static_cast<size_t>(i) * stride_blocks * bytes, bytes, &bar);
    const long long t1 = clock64();
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  }
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 1, 64 << 20);
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (uint32_t bytes : {2048u, 8192u, 32768u})
    for (int nreq : {1, 4, 16, 64}) {
      for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 128, 200 * 1024>>>(src, nreq, bytes, 3, d);
        cudaDeviceSynchronize();
      }
      unsigned long long h[296];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double is = 0, tot = 0;
      for (int i = 0; i < 148; ++i) { is += h[2 * i]; tot += h[2 * i + 1]; }
      printf("bulk %6u B x %3d: issue %8.1f cyc (%6.1f per request), complete %8.1f cyc, %6.1f B/cyc/SM\n", bytes, nreq,
             is / 148, is / 148 / nreq, tot / 148, nreq * bytes / (tot / 148));
    }
  return 0;
}
