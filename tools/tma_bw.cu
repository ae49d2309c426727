// tma_bw.cu -- per-SM inbound bandwidth of the operand loads the 1x1 kernel uses, all
// SMs streaming: each CTA walks position tiles of a [P][256] bf16 matrix (C4's X) and
// loads each 128-position x 256-channel tile (64 KB) into a 3-deep ring, only waiting
// for arrival.  Modes: 0 = four 2-D boxes {64 ch, 128 rows} SW128 (one per 64-channel
// chunk); 1 = one 4-D box {64 ch, 8 rows, 4 chunks, 16 row groups} SW128; 2 = one 1-D
// bulk copy of the contiguous 64 KB; 3 = mode 0 with `share` CTAs reading the same tile
// at the same time (the kernel's channel groups).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lcuda -o tools/tma_bw tools/tma_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"
using namespace lrs;

__global__ void k(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m4, const uint8_t* src,
                  int n_tiles, int mode, int share, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[3];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int cta = mode == 3 ? blockIdx.x / share : blockIdx.x;
  const int step = mode == 3 ? gridDim.x / share : gridDim.x;
  const long long t0 = clock64();
  int it = 0;
  for (int t = cta; t < n_tiles; t += step, ++it) {
    const int s = it % 3;
    if (it >= 3) mbar_wait(&bar[s], ((it / 3) - 1) & 1);
    uint8_t* dst = smem + s * 65536;
    mbar_arrive_expect_tx(&bar[s], 65536);
    if (mode == 0 || mode == 3) {
      for (int c = 0; c < 4; ++c) tma_load_2d(dst + c * 16384, &m2, &bar[s], c * 64, t * 128);
    } else if (mode == 1) {
      tma_load_4d(dst, &m4, &bar[s], 0, 0, 0, t * 16);
    } else {
      bulk_load(dst, src + static_cast<size_t>(t) * 65536, 65536, &bar[s]);
    }
  }
  for (int j = it - 3 < 0 ? 0 : it - 3; j < it; ++j) mbar_wait(&bar[j % 3], (j / 3) & 1);
  out[blockIdx.x] = clock64() - t0;
  out[4096 + blockIdx.x] = it;
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int P = 25088 * 4;  // 4 C4 batches: 51 MB, larger than what L2 keeps warm across modes
  const int n_tiles = P / 128;
  uint8_t* src;
  cudaMalloc(&src, static_cast<size_t>(P) * 512);
  cudaMemset(src, 1, static_cast<size_t>(P) * 512);
  unsigned long long* d;
  cudaMalloc(&d, 8192 * 8);
  PFN enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap m2, m4;
  {
    cuuint64_t dims[2] = {256, (cuuint64_t)P};
    cuuint64_t str[1] = {512};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[4] = {64, 8, 4, (cuuint64_t)P / 8};
    cuuint64_t str[3] = {512, 128, 4096};
    cuuint32_t box[4] = {64, 8, 4, 16}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("4-D map encode failed %d\n", (int)r);
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536 + 1024);
  const char* names[] = {"2-D boxes x4", "4-D box x1", "1-D bulk 64KB", "2-D x4, 8 CTAs share"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      k<<<144, 32, 3 * 65536 + 1024>>>(m2, m4, src, n_tiles, mode, 8, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    unsigned long long h[8192];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0, bytes = 0;
    for (int i = 0; i < 144; ++i) { cyc = cyc > h[i] ? cyc : h[i]; bytes += h[4096 + i] * 65536.0; }
    printf("%-22s: %.0f cycles, %.1f B/clk/SM, %.2f TB/s at 1.965 GHz (%.0f MB)\n", names[mode], cyc,
           bytes / cyc / 144, bytes / (cyc / 1.965e9) / 1e12, bytes / 1e6);
  }
  return 0;
}
