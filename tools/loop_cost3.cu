// loop_cost3.cu -- single-thread cost of the MMA issuer's per-chunk bookkeeping with every
// loop value in registers (loop bound read from shared memory, see lrs_ptx.cuh smem_param):
// try_wait on a complete mbarrier phase, tcgen05.fence::after_thread_sync, tcgen05.commit,
// mbarrier arrive.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/loop_cost3 tools/loop_cost3.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

template <int MODE>
__global__ void k(int iters, unsigned long long* out) {
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  __shared__ int prm[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    prm[0] = iters;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc(&tslot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 32) {
    const int n = smem_param(prm);
    __shared__ __align__(1024) uint8_t ebuf[4096];
    const uint64_t edesc = umma_desc_rows16(smem_u32(ebuf));
    mbar_arrive(&bar[0]);  // phase 0 of bar 0 complete
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      if (MODE & 1) mbar_wait(&bar[0], 0);
      if (MODE & 2) tc_fence_after();
      if (MODE & 4) mma_commit(&bar[1]);
      if (MODE & 8) mbar_arrive(&bar[2]);
      if (MODE & 16) { while (!mbar_test_wait(&bar[0], 0)) {} }
      if (MODE & 32) { while (!mbar_try_wait(&bar[0], 0)) {} }
      if (MODE & 64) tmem_cp_128x256b(0u, edesc);
      if (MODE & 128) tmem_cp_128x128b(0u, edesc);
    }
    const long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(0, 32);
}

template <int MODE>
void run(const char* name, unsigned long long* d) {
  for (int rep = 0; rep < 2; ++rep) {
    k<MODE><<<1, 128>>>(1000, d);
    cudaDeviceSynchronize();
  }
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.1f cycles/iter (%s)\n", name, h / 1000.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<0>("empty", d);
  run<1>("try_wait (complete phase)", d);
  run<2>("tcgen05.fence::after", d);
  run<3>("wait + fence", d);
  run<4>("tcgen05.commit", d);
  run<7>("wait + fence + commit", d);
  run<8>("mbarrier.arrive", d);
  run<16>("test_wait (complete phase)", d);
  run<32>("bare try_wait loop", d);
  run<18>("test_wait + fence", d);
  run<64>("tcgen05.cp 128x256b", d);
  run<128>("tcgen05.cp 128x128b", d);
  run<64 + 7>("wait+fence+cp256+commit", d);
  return 0;
}
