// probe_2cta.cu -- the CTA-pair (cta_group::2) form of the 2:4 sparse MMA on sm_100a:
// tcgen05.mma.sp.cta_group::2.kind::f16 issued by the pair's rank-0 CTA, M = 256 (rows
// 0..127 = CTA 0's A, 128..255 = CTA 1's A, each from its own shared memory at the same
// offset), metadata copied to each CTA's TMEM by one tcgen05.cp.cta_group::2, completion
// signalled to both CTAs by one multicast tcgen05.commit.  Question answered: where must B
// live -- split (each CTA holds N/2 rows: mode 0) or whole in both CTAs (mode 1)?
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_2cta tools/probe_2cta.cu
// usage: probe_2cta [mode]
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2006_06443_b200/csrc/lrs_ptx.cuh"

using namespace lrs;

constexpr int MC = 128, M = 256, N = 64, KL = 64, KC = KL / 2;  // per-CTA rows, logical / stored K

__host__ __device__ inline uint32_t sw64(int r, int b) {
  return (r / 8) * 512 + (r % 8) * 64 + ((((b / 16) ^ ((r % 8) / 2)) & 3) * 16) + (b % 16);
}
__host__ __device__ inline uint32_t sw128(int r, int b) {
  return (r / 8) * 1024 + (r % 8) * 128 + ((((b / 16) ^ (r % 8))) * 16) + (b % 16);
}

// ac: [M][KC] compressed A (rows 0..127 CTA 0, 128..255 CTA 1); b: [N][KL]; e: [M][4] metadata words
__global__ void __cluster_dims__(2, 1, 1) probe(const __nv_bfloat16* ac, const __nv_bfloat16* b, const uint32_t* e,
                                               float* d, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;           // 128 rows x 64 B, SW64 (compressed A, K = 64 logical)
  uint8_t* sb = smem + 8192;    // up to 64 rows x 128 B, SW128 (B, K = 64)
  uint32_t* se = reinterpret_cast<uint32_t*>(smem + 16384);  // [128 lanes][4 words]
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  const uint32_t rank = cluster_rank();
  for (int i = t; i < MC * KC; i += blockDim.x) {
    const int r = i / KC, k = i % KC;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw64(r, k * 2)) = ac[(rank * MC + r) * KC + k];
  }
  const int nb = mode == 0 ? N / 2 : N;          // B rows this CTA holds
  const int b0 = mode == 0 ? rank * (N / 2) : 0;  // first B row
  for (int i = t; i < nb * KL; i += blockDim.x) {
    const int r = i / KL, k = i % KL;
    *reinterpret_cast<__nv_bfloat16*>(sb + sw128(r, k * 2)) = b[(b0 + r) * KL + k];
  }
  for (int i = t; i < MC * 4; i += blockDim.x) se[i] = e[(rank * MC + i / 4) * 4 + i % 4];
  fence_proxy_async_smem();
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' operands, barriers and TMEM ready
  tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t tm_e = tm + 64;
  if (rank == 0 && t == 0) {
    const uint64_t ed = umma_desc_rows16(smem_u32(se));
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(tm_e), "l"(ed) : "memory");
    for (int s = 0; s < 2; ++s) {
      const uint32_t idesc = (static_cast<uint32_t>(s) & 3u) | (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) |
                             ((N >> 3) << 17) | ((M >> 4) << 24);
      const uint64_t ad = umma_desc(smem_u32(sa) + s * 32, 64);
      const uint64_t bd = umma_desc(smem_u32(sb) + s * 64, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n}" ::"r"(tm),
          "l"(ad), "l"(bd), "r"(idesc), "r"(s > 0 ? 1u : 0u), "r"(tm_e)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    const int w = t / 32;
    for (int c = 0; c < N; c += 16) {
      float v[16];
      tmem_ld16(tm + (static_cast<uint32_t>(w * 32) << 16) + c, v);
      for (int i = 0; i < 16; ++i) d[(rank * MC + w * 32 + (t % 32)) * N + c + i] = v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (t < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128) : "memory");
  }
}

static float bf(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  srand(7);
  auto rnd = []() { return (rand() / (float)RAND_MAX) * 2.f - 1.f; };
  std::vector<float> A(M * KL, 0.f), B(N * KL);
  std::vector<int> idx(M * KL / 2);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < KL / 4; ++g) {
      int i0 = rand() % 4, i1 = rand() % 4;
      while (i1 == i0) i1 = rand() % 4;
      if (i0 > i1) std::swap(i0, i1);
      A[r * KL + g * 4 + i0] = bf(rnd());
      A[r * KL + g * 4 + i1] = bf(rnd());
      idx[(r * KL / 4 + g) * 2] = i0;
      idx[(r * KL / 4 + g) * 2 + 1] = i1;
    }
  for (auto& v : B) v = bf(rnd());
  std::vector<float> Dref(M * N, 0.f);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < KL; ++k) s += (double)A[i * KL + k] * B[j * KL + k];
      Dref[i * N + j] = (float)s;
    }
  std::vector<__nv_bfloat16> Ac(M * KC), Bh(N * KL);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < KL / 4; ++g)
      for (int q = 0; q < 2; ++q) Ac[r * KC + g * 2 + q] = __float2bfloat16(A[r * KL + g * 4 + idx[(r * KL / 4 + g) * 2 + q]]);
  for (int i = 0; i < N * KL; ++i) Bh[i] = __float2bfloat16(B[i]);
  // the metadata layout measured for cta_group::1 (lrs_ptx.cuh mma_sp_bf16), per CTA's 128 rows
  std::vector<uint32_t> E(M * 4, 0u);
  for (int mm = 0; mm < M; ++mm)
    for (int G = 0; G < KL / 4; ++G) {
      const int m = mm % MC, c = mm / MC;
      const int i0 = idx[(mm * KL / 4 + G) * 2], i1 = idx[(mm * KL / 4 + G) * 2 + 1];
      const int s = G / 8, gs = G % 8;
      const int lane = m % 8 + 8 * (gs / 4) + 16 * (m / 16);
      const int nibpos = (gs % 4) + 4 * ((m / 8) % 2);
      E[(c * MC + lane) * 4 + s] |= static_cast<uint32_t>(i0 | (i1 << 2)) << (4 * nibpos);
    }
  __nv_bfloat16 *dAc, *dB;
  uint32_t* dE;
  float* dD;
  cudaMalloc(&dAc, Ac.size() * 2);
  cudaMalloc(&dB, Bh.size() * 2);
  cudaMalloc(&dE, E.size() * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dAc, Ac.data(), Ac.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xFF, M * N * 4);
  const int smem = 16384 + 2048 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<2, 128, smem>>>(dAc, dB, dE, dD, mode);
  cudaError_t err = cudaDeviceSynchronize();
  printf("mode %d (%s): launch %s\n", mode, mode == 0 ? "B split N/2 per CTA" : "B whole in both CTAs",
         cudaGetErrorString(err));
  if (err != cudaSuccess) return 1;
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double e0 = 0, e1 = 0, n0 = 0;
  int bad0 = 0, bad1 = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      const double df = D[i * N + j] - Dref[i * N + j];
      (i < MC ? e0 : e1) += df * df;
      n0 += (double)Dref[i * N + j] * Dref[i * N + j];
      if (std::fabs(df) > 1e-3 * (1 + std::fabs(Dref[i * N + j]))) (i < MC ? bad0 : bad1)++;
    }
  printf("rel err rows 0-127 %.3e (bad %d), rows 128-255 %.3e (bad %d)\n", std::sqrt(e0 / n0 * 2), bad0,
         std::sqrt(e1 / n0 * 2), bad1);
  printf("D[0][0..3] %.4f %.4f %.4f %.4f ref %.4f %.4f %.4f %.4f\n", D[0], D[1], D[2], D[3], Dref[0], Dref[1], Dref[2],
         Dref[3]);
  printf("D[200][40..43] %.4f %.4f %.4f %.4f ref %.4f %.4f %.4f %.4f\n", D[200 * N + 40], D[200 * N + 41],
         D[200 * N + 42], D[200 * N + 43], Dref[200 * N + 40], Dref[200 * N + 41], Dref[200 * N + 42],
         Dref[200 * N + 43]);
  return (bad0 + bad1) ? 2 : 0;
}
