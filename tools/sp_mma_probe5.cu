// sp_mma_probe5.cu -- sparse MMA with A in TMEM (tcgen05.mma.sp [a_tmem])  the TMEM metadata layout of the sm_100a 2:4
// sparse tensor-core MMA (tcgen05.mma.sp.cta_group::1.kind::f16, bf16 in, fp32
// accumulate, M = 128, N = 64, K = 64 logical = 2 MMAs of K = 32).
// Metadata words are written straight into TMEM with tcgen05.st (each thread
// owns its lane), so every hypothesis is a plain (lane, column, bit) map.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/sp_probe2 tools/sp_mma_probe2.cu
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

constexpr int M = 128, N = 64, KL = 128, KC = KL / 2;  // logical / stored K
constexpr int ECOLS = 16;                              // metadata columns written per lane

__device__ __forceinline__ void mma_sp_ts(uint32_t d, uint32_t a_tmem, uint64_t bd, uint32_t idesc, uint32_t acc,
                                          uint32_t e) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;\n}" ::"r"(d),
      "r"(a_tmem), "l"(bd), "r"(idesc), "r"(acc), "r"(e)
      : "memory");
}
__device__ __forceinline__ void mma_ts_dense(uint32_t d, uint32_t a_tmem, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a_tmem), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
      "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// sw64 K-major byte offset of (row r, byte b) in a tile of 64-byte rows (8-row atoms of 512 B)
__host__ __device__ inline uint32_t sw64(int r, int b) {
  return (r / 8) * 512 + (r % 8) * 64 + ((((b / 16) ^ ((r % 8) / 2)) & 3) * 16) + (b % 16);
}
// sw128 K-major byte offset of (row r, byte b) in a tile of 128-byte rows
__host__ __device__ inline uint32_t sw128(int r, int b) {
  return (r / 8) * 1024 + (r % 8) * 128 + ((((b / 16) ^ (r % 8))) * 16) + (b % 16);
}

// e_words: [M lanes][ECOLS] metadata words; e_addr[s] = column offset (and lane<<16) of step s
__global__ void probe(const __nv_bfloat16* ac, const __nv_bfloat16* b, const uint32_t* e_words, float* d,
                      uint32_t idlo0, uint32_t idlo1, uint32_t e_addr0, uint32_t e_addr1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;          // 2 x (128 rows x 64 B) (compressed A, K = 64 stored), SW64
  uint8_t* sb = smem + 16384;  // 64 rows x 256 B as 2 SW128 atoms (B, K = 128)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < M * KC; i += blockDim.x) {
    const int r = i / KC, k = i % KC;
    *reinterpret_cast<__nv_bfloat16*>(sa + (k / 32) * 8192 + sw64(r, (k % 32) * 2)) = ac[i];
  }
  for (int i = t; i < N * KL; i += blockDim.x) {
    const int r = i / KL, k = i % KL;
    *reinterpret_cast<__nv_bfloat16*>(sb + (k / 64) * 8192 + sw128(r, (k % 64) * 2)) = b[i];
  }
  fence_proxy_async_smem();
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (t < 32) tmem_alloc(&tslot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t tm_e = tm + 64;  // metadata columns [64, 68)
  uint32_t* se = reinterpret_cast<uint32_t*>(smem + 32768);  // [128 lanes][4 words]
  for (int i = t; i < M * 4; i += blockDim.x) se[i] = e_words[(i / 4) * ECOLS + (i % 4)];
  fence_proxy_async_smem();
  __syncthreads();
  if (idlo0 == 0) {  // tcgen05.st path
    const int w = t / 32, lane = t % 32;
    const int row = w * 32 + lane;
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = i < 4 ? e_words[row * ECOLS + i] : 0u;
    tmem_st8(tm_e + (static_cast<uint32_t>(w * 32) << 16), v);
    tmem_st_wait();
  } else if (t == 0) {
    uint64_t d = 0;
    const uint32_t sa_ = smem_u32(se);
    d |= static_cast<uint64_t>((sa_ >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((e_addr1 >> 4) & 0x3FFFu) << 16;   // LBO (bytes) from argv
    d |= static_cast<uint64_t>((128u >> 4) & 0x3FFFu) << 32;      // SBO = 8 rows x 16 B
    d |= 1ull << 46;
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tm_e), "l"(d) : "memory");
  }
  if (t == 0) {
    // idesc: sparse selector idlo (bits 0-1), sparse enable (bit 2), f32 D (bit 4), bf16 A/B, K-major, N, M
    for (int s = 0; s < (int)idlo1; ++s) {
      const uint32_t idesc = (static_cast<uint32_t>(s % 2) & 3u) | (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) |
                             ((N >> 3) << 17) | ((M >> 4) << 24);
      const uint64_t ad = umma_desc(smem_u32(sa) + (s / 2) * 8192 + (s % 2) * 32, 64);
      const uint64_t bd = umma_desc(smem_u32(sb) + (s / 2) * 8192 + (s % 2) * 64, 128);
      if (e_addr1 == 6 || e_addr1 == 7) mma_sp_ts(tm, tm + 72 + 8 * s, bd, idesc, s > 0 ? 1u : 0u, tm_e + 2 * (s / 2));
      else mma_sp_bf16(tm, ad, bd, idesc, s > 0 ? 1u : 0u, tm_e + e_addr0 * (s / 2));
      (void)ad;
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    const int w = t / 32;
    for (int c = 0; c < N; c += 16) {
      float v[16];
      tmem_ld16(tm + (static_cast<uint32_t>(w * 32) << 16) + c, v);
      for (int i = 0; i < 16; ++i) d[(w * 32 + (t % 32)) * N + c + i] = v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) {
    tc_fence_after();
    tmem_dealloc(tm, 128);
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

struct Hyp {
  const char* name;
  int kind;        // placement family
  int nib_swap;    // nibble = i1 | i0 << 2 instead of i0 | i1 << 2
  uint32_t e0, e1; // step addresses (lane << 16 | col)
  uint32_t id0, id1;  // sparsity selector per step
};

int main(int argc, char** argv) {
  const uint32_t lbo = argc > 1 ? atoi(argv[1]) : 128;
  const uint32_t use_cp = argc > 2 ? atoi(argv[2]) : 0;
  const uint32_t nsteps = argc > 3 ? atoi(argv[3]) : 4;
  const uint32_t astride = argc > 4 ? atoi(argv[4]) : 2;
  srand(5);
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
      for (int k = 0; k < (int)nsteps * 32; ++k) s += (double)A[i * KL + k] * B[j * KL + k];
      Dref[i * N + j] = (float)s;
    }
  std::vector<__nv_bfloat16> Ac(M * KC), Bh(N * KL);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < KL / 4; ++g)
      for (int q = 0; q < 2; ++q) Ac[r * KC + g * 2 + q] = __float2bfloat16(A[r * KL + g * 4 + idx[(r * KL / 4 + g) * 2 + q]]);
  for (int i = 0; i < N * KL; ++i) Bh[i] = __float2bfloat16(B[i]);
  // learned layout: step s = G/8 -> word s; lane = m%8 + 8*((G%8)/4) + 16*(m/16); nibble = (G%4) + 4*((m/8)%2)
  const uint32_t astride_ = astride;
  std::vector<uint32_t> E(M * ECOLS, 0u);
  for (int m = 0; m < M; ++m)
    for (int G = 0; G < KL / 4; ++G) {
      const int i0 = idx[(m * KL / 4 + G) * 2], i1 = idx[(m * KL / 4 + G) * 2 + 1];
      const int s = G / 8, gs = G % 8;
      const int lane = m % 8 + 8 * (gs / 4) + 16 * (m / 16);
      const int nibpos = (gs % 4) + 4 * ((m / 8) % 2);
      E[lane * ECOLS + (s / 2) * astride + (s % 2)] |= static_cast<uint32_t>(i0 | (i1 << 2)) << (4 * nibpos);
    }
  __nv_bfloat16 *dAc, *dB;
  uint32_t* dE;
  float* dD;
  cudaMalloc(&dAc, Ac.size() * 2);
  cudaMalloc(&dB, Bh.size() * 2);
  cudaMalloc(&dE, M * ECOLS * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dAc, Ac.data(), Ac.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  probe<<<1, 128, 48 * 1024>>>(dAc, dB, dE, dD, use_cp, nsteps, astride, lbo);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("lbo %u CUDA error %s\n", lbo, cudaGetErrorString(err)); return 1; }
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int i = 0; i < M * N; ++i) { num += (D[i] - Dref[i]) * (double)(D[i] - Dref[i]); den += (double)Dref[i] * Dref[i]; }
  printf("cp=%u lbo=%u steps=%u addr_stride=%u: relL2 = %.3e\n", use_cp, lbo, nsteps, astride, sqrt(num / den));
  return 0;
}
