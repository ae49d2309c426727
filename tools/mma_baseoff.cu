// mma_baseoff.cu -- is a SW128 K-major A operand legal at a start row that is not a
// multiple of the 8-row swizzle atom?  (The T1 window of lrs_core.cuh is read at
// arbitrary row offsets -- one per kernel tap -- and therefore uses SWIZZLE_NONE,
// measured 88 vs 58 cycles per N = 64 MMA in tools/mma_layout.cu.)
// A: 256 rows x 64 bf16 (128 B rows) written in the TMA SW128 pattern (16-B chunk c of
// row r at r*128 + ((c ^ (r & 7)) * 16)); B: 64 x 64; D = A[r0 : r0 + 128] . B^T for
// r0 = 0..15 with the descriptor's base-offset field (bits 49-51) = 0 or (r0 & 7),
// checked against a host product.  Then the MMA rate at odd start rows.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_baseoff tools/mma_baseoff.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(const __nv_bfloat16* ga, const __nv_bfloat16* gb, float* out, int r0, int boff, int iters,
                  unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* sa = smem;               // 256 rows x 128 B
  uint8_t* sb = smem + 256 * 128;   // 64 rows x 128 B
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sa + r * 128 + ((c ^ (r & 7)) * 16)) = reinterpret_cast<const uint4*>(ga)[i];
  }
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sb + r * 128 + ((c ^ (r & 7)) * 16)) = reinterpret_cast<const uint4*>(gb)[i];
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc(1u, 64u, 128u);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = umma_desc(smem_u32(sa) + r0 * 128 + kk * 32, 128);
        ad |= static_cast<uint64_t>(boff & 7) << 49;
        mma_bf16(tm, ad, umma_desc(smem_u32(sb) + kk * 32, 128), idesc, (it > 0 || kk > 0) ? 1u : 0u);
      }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    if (cyc) cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 128) {
    const int w = threadIdx.x >> 5;
    for (int c0 = 0; c0 < 64; c0 += 16) {
      float v[16];
      tmem_ld16(tm + ((w * 32) << 16) + c0, v);
      for (int j = 0; j < 16; ++j) out[threadIdx.x * 64 + c0 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tm, 64);
  }
}

int main() {
  std::vector<__nv_bfloat16> ha(256 * 64), hb(64 * 64);
  std::vector<float> fa(256 * 64), fb(64 * 64);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return static_cast<float>((s >> 9) & 0xFF) / 64.f - 2.f; };
  for (int i = 0; i < 256 * 64; ++i) { ha[i] = __float2bfloat16(rnd()); fa[i] = __bfloat162float(ha[i]); }
  for (int i = 0; i < 64 * 64; ++i) { hb[i] = __float2bfloat16(rnd()); fb[i] = __bfloat162float(hb[i]); }
  __nv_bfloat16 *da, *db;
  float* dout;
  unsigned long long* dc;
  cudaMalloc(&da, ha.size() * 2);
  cudaMalloc(&db, hb.size() * 2);
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMalloc(&dc, 148 * 8);
  cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<float> o(128 * 64);
  for (int mode = 0; mode < 2; ++mode)
    for (int r0 = 0; r0 < 16; ++r0) {
      const int boff = mode ? (r0 & 7) : 0;
      k<<<1, 128, 64 * 1024>>>(da, db, dout, r0, boff, 1, nullptr);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("fault r0=%d\n", r0); return 1; }
      cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int kk = 0; kk < 64; ++kk) ref += static_cast<double>(fa[(r0 + m) * 64 + kk]) * fb[n * 64 + kk];
          maxerr = fmax(maxerr, fabs(ref - o[m * 64 + n]));
        }
      printf("base_offset=%s r0=%2d: max |err| = %g %s\n", mode ? "r0&7" : "0   ", r0, maxerr,
             maxerr < 1e-2 ? "OK" : "WRONG");
    }
  for (int r0 : {0, 1, 3, 8}) {
    k<<<148, 128, 64 * 1024>>>(da, db, dout, r0, r0 & 7, 1024, dc);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    printf("rate r0=%d: %.1f cycles per N=64 MMA\n", r0, avg / 148 / 4096);
  }
  return 0;
}
