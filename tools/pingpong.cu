// pingpong.cu -- producer/consumer slot ring latency on one SM: the consumer
// (MMA warp) either commits (tcgen05.commit -> mbarrier) or arrives plainly on
// "empty"; the producer waits "empty" and arrives "full".  Reports ns per item.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/pingpong tools/pingpong.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int items, int ns, int use_commit, unsigned long long* out, int extra_mode) {
  __shared__ uint64_t full[8], empty[8];
  __shared__ uint32_t slot_;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&slot_, 32);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const long long t0 = clock64();
  __shared__ uint64_t done;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  __syncthreads();
  if (warp >= 2) {
    // extra warps: 1 = sleep-poll an mbarrier (like the epilogue), 2 = try_wait spin, 0 = exit
    if (extra_mode == 1) mbar_wait_sleep(&done, 0);
    else if (extra_mode == 2) mbar_wait(&done, 0);
  } else if (warp == 0 && lane == 0) {
    for (int it = 0; it < items; ++it) {
      const int s = it % ns;
      if (it >= ns) mbar_wait(&empty[s], ((it / ns) - 1) & 1);
      mbar_arrive(&full[s]);
    }
  } else if (warp == 1) {
    for (int it = 0; it < items; ++it) {
      const int s = it % ns;
      mbar_wait(&full[s], (it / ns) & 1);
      tc_fence_after();
      if (elect_one()) {
        if (use_commit) mma_commit(&empty[s]);
        else mbar_arrive(&empty[s]);
      }
      __syncwarp();
    }
  }
  if (warp == 1 && lane == 0) mbar_arrive(&done);
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(slot_, 32); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  const int items = 4000;
  for (int extra = 0; extra < 3; ++extra)
  for (int commit = 1; commit < 2; ++commit)
    for (int ns : {2, 4}) {
      k<<<148, 320>>>(items, ns, commit, d, extra);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("extra warps mode %d (0 idle, 1 sleep-poll, 2 spin) %s ns=%d: %.0f cycles/item\n", extra, commit ? "tcgen05.commit" : "mbarrier.arrive", ns, avg / items);
    }
  return 0;
}
