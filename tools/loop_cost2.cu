// loop_cost2.cu -- why a single-thread loop costs ~280 cycles/iteration: where do the
// other 31 lanes of the issuing warp (and the other warps) wait?
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/loop_cost2 tools/loop_cost2.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__device__ __forceinline__ unsigned long long body(int iters) {
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i * 3;
    asm volatile("" ::: "memory");
  }
  return acc;
}
struct P { int a[64]; };
// variants of loop_cost's empty-loop case: 0 TMEM allocated, 1 a never-taken mbar_wait in the body,
// 2 a never-taken tcgen05.commit in the body, 3 both, 4 neither (kernel has an mbarrier only)
__global__ void kv(int variant, int flag, int iters, unsigned long long* out) {
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (variant == 0 && threadIdx.x < 32) tmem_alloc(&tslot, 32);
  __syncthreads();
  unsigned long long t = 0, acc = 0;
  if (variant == 5) {  // same empty loop, params copied into registers the compiler cannot rematerialize
    int v = variant, f = flag, n = iters;
    asm volatile("" : "+r"(v), "+r"(f), "+r"(n));
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int i = 0; i < n; ++i) {
        acc += i * 3;
        if ((v == 1 || v == 3) && f) mbar_wait(&bar, 0);
        asm volatile("" ::: "memory");
      }
      t = clock64() - t0;
    }
    __syncthreads();
    if (threadIdx.x == 0) { out[0] = t; out[1] = acc; }
    return;
  }
  if (threadIdx.x == 0) {
    mbar_arrive(&bar);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      acc += i * 3;
      if (variant == 5) { /* locals pinned in registers below */ }
      if ((variant == 1 || variant == 3) && flag) mbar_wait(&bar, 0);
      if ((variant == 2 || variant == 3) && flag) mma_commit(&bar);
      asm volatile("" ::: "memory");
    }
    t = clock64() - t0;
  }
  __syncthreads();
  if (variant == 0 && threadIdx.x < 32) tmem_dealloc(0, 32);
  if (threadIdx.x == 0) { out[0] = t; out[1] = acc; }
}
__device__ __forceinline__ unsigned long long body_param(const P& p, int iters, int kind) {
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (kind == 0) acc += p.a[i & 7];            // param-space loads each iteration
    else acc += p.a[5];
    asm volatile("" ::: "memory");
  }
  return acc;
}
__global__ void kp(const __grid_constant__ P p, int kind, int iters, unsigned long long* out) {
  unsigned long long t = 0, acc = 0;
  if (threadIdx.x == 0) { long long t0 = clock64(); acc = body_param(p, iters, kind); t = clock64() - t0; }
  __syncthreads();
  if (threadIdx.x == 0) { out[0] = t; out[1] = acc; }
}

__global__ void k(int mode, int iters, unsigned long long* out) {
  unsigned long long t = 0, acc = 0;
  if (mode == 0) {  // lane 0 alone, lanes 1-31 at __syncwarp, other warps at __syncthreads
    if (threadIdx.x == 0) { long long t0 = clock64(); acc = body(iters); t = clock64() - t0; }
    __syncwarp();
  } else if (mode == 1) {  // whole warp 0 runs the loop
    if (threadIdx.x < 32) { long long t0 = clock64(); acc = body(iters); t = clock64() - t0; }
  } else if (mode == 2) {  // lane 0 alone, lanes 1-31 fall straight through to __syncthreads
    if (threadIdx.x == 0) { long long t0 = clock64(); acc = body(iters); t = clock64() - t0; }
  } else if (mode == 3) {  // lane 0 alone, lanes 1-31 spin on a shared flag
    __shared__ volatile int flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    if (threadIdx.x == 0) { long long t0 = clock64(); acc = body(iters); t = clock64() - t0; flag = 1; }
    else if (threadIdx.x < 32) { while (!flag) { __nanosleep(1000); } }
  }
  __syncthreads();
  if (threadIdx.x == 0) { out[0] = t; out[1] = acc; }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const char* names[] = {"lane 0; lanes 1-31 at __syncwarp", "whole warp", "lane 0; others at __syncthreads",
                         "lane 0; others nanosleep-spin"};
  for (int bs : {32, 320})
    for (int mode = 0; mode < 4; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        k<<<1, bs>>>(mode, 1000, d);
        cudaDeviceSynchronize();
      }
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("block %3d %-36s %.1f cycles/iter\n", bs, names[mode], h[0] / 1000.0);
    }
  for (int v = 0; v < 6; ++v) {
    for (int rep = 0; rep < 2; ++rep) { kv<<<1, 320>>>(v, 0, 1000, d); cudaDeviceSynchronize(); }
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("block 320 variant %d: %.1f cycles/iter\n", v, h[0] / 1000.0);
  }
  P hp;
  for (int i = 0; i < 64; ++i) hp.a[i] = i;
  for (int kind = 0; kind < 2; ++kind) {
    for (int rep = 0; rep < 2; ++rep) { kp<<<1, 320>>>(hp, kind, 1000, d); cudaDeviceSynchronize(); }
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("block 320 param load kind %d (%s): %.1f cycles/iter\n", kind, kind ? "fixed index" : "dynamic index", h[0] / 1000.0);
  }
  return 0;
}
