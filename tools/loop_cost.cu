// loop_cost.cu -- single-thread cost of the MMA issuer's per-chunk bookkeeping on B200:
// an mbarrier try_wait on an already-complete phase, tcgen05.fence::after_thread_sync,
// a %globaltimer read, tcgen05.commit (with no MMA in flight), ld.shared of a table.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/loop_cost tools/loop_cost.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(int mode, int iters, unsigned long long* out) {
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc(&tslot, 32);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive(&bar[0]);  // phase 0 of bar 0 complete
    unsigned long long acc = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode & 1) mbar_wait(&bar[0], 0);
      if (mode & 2) tc_fence_after();
      if (mode & 4) acc += gtimer();
      if (mode & 8) mma_commit(&bar[1]);
      if (mode & 16) tc_fence_before();
      if (mode & 32) acc += i * 3;
      if (mode & 64) asm volatile("" ::: "memory");
    }
    const long long t1 = clock64();
    out[0] = t1 - t0;
    out[1] = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(0, 32);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const char* names[] = {"", "try_wait(complete)", "fence_after", "wait+fence", "globaltimer", "", "", "wait+fence+timer",
                         "commit", "wait+commit", "", "wait+fence+commit"};
  for (int mode : {0, 32, 64, 1, 2, 3, 4, 7, 8, 9, 11, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      k<<<1, 128>>>(mode, 1000, d);
      cudaDeviceSynchronize();
    }
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %2d %-20s %.1f cycles/iter (%s)\n", mode, mode < 12 ? names[mode] : (mode == 16 ? "fence_before" : "plain"), h[0] / 1000.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
