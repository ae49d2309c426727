// sp_mma_probe2.cu -- pin down the TMEM metadata layout of the sm_100a 2:4
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

constexpr int M = 128, N = 64, KL = 64, KC = KL / 2;  // logical / stored K
constexpr int ECOLS = 16;                              // metadata columns written per lane

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
  uint8_t* sa = smem;          // 128 rows x 64 B (compressed A, K = 32 stored), SW64
  uint8_t* sb = smem + 8192;   // 64 rows x 128 B (B, K = 64), SW128
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < M * KC; i += blockDim.x) {
    const int r = i / KC, k = i % KC;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw64(r, k * 2)) = ac[i];
  }
  for (int i = t; i < N * KL; i += blockDim.x) {
    const int r = i / KL, k = i % KL;
    *reinterpret_cast<__nv_bfloat16*>(sb + sw128(r, k * 2)) = b[i];
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
  const uint32_t tm_e = tm + 64;  // metadata columns [64, 64 + ECOLS)
  {
    const int w = t / 32, lane = t % 32;
    const int row = w * 32 + lane;
    for (int c = 0; c < ECOLS; c += 8) {
      uint32_t v[8];
      for (int i = 0; i < 8; ++i) v[i] = e_words[row * ECOLS + c + i];
      tmem_st8(tm_e + (static_cast<uint32_t>(w * 32) << 16) + c, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    // idesc: sparse selector idlo (bits 0-1), sparse enable (bit 2), f32 D (bit 4), bf16 A/B, K-major, N, M
    for (int s = 0; s < 2; ++s) {
      const uint32_t idesc = ((s == 0 ? idlo0 : idlo1) & 3u) | (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) |
                             ((N >> 3) << 17) | ((M >> 4) << 24);
      const uint64_t ad = umma_desc(smem_u32(sa) + s * 32, 64);
      const uint64_t bd = umma_desc(smem_u32(sb) + s * 64, 128);
      mma_sp_bf16(tm, ad, bd, idesc, s > 0 ? 1u : 0u, tm_e + (s == 0 ? e_addr0 : e_addr1));
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
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int pmode = argc > 2 ? atoi(argv[2]) : 0;  // 0 random, 1 uniform (0,1), 2 uniform (2,3), 3 by row, 4 by group
  srand(7);
  auto rnd = []() { return (rand() / (float)RAND_MAX) * 2.f - 1.f; };
  std::vector<float> A(M * KL, 0.f), B(N * KL);
  std::vector<int> idx(M * KL / 2);
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < KL / 4; ++g) {
      int i0 = rand() % 4, i1 = rand() % 4;
      while (i1 == i0) i1 = rand() % 4;
      static const int P[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
      if (pmode == 1) { i0 = 0; i1 = 1; }
      if (pmode == 2) { i0 = 2; i1 = 3; }
      if (pmode == 3) { i0 = P[r % 6][0]; i1 = P[r % 6][1]; }
      if (pmode == 4) { i0 = P[g % 6][0]; i1 = P[g % 6][1]; }
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

  __nv_bfloat16 *dAc, *dB;
  uint32_t* dE;
  float* dD;
  cudaMalloc(&dAc, Ac.size() * 2);
  cudaMalloc(&dB, Bh.size() * 2);
  cudaMalloc(&dE, M * ECOLS * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dAc, Ac.data(), Ac.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);

  // kinds:
  //  0  lane = m, word s holds the 8 nibbles of step s (group g of the step at bits 4g)
  //  1  CUTLASS-style atom: lane = m%8 + 16*(m/16), byte kb = k/8 at column (kb%16)/4 + 4*((m/8)%2), byte kb%4
  //  2  like 1 but the (m/8)%2 half goes to lane +8 instead of column +4
  //  3  lane = m, one word for both steps: step s at bits 16*s (nibble g at 4g within 16 bits)?? (K=32 -> 8 nibbles = 32 bits, so
  //     this packs only half; kept as a negative control)
  std::vector<Hyp> hyps = {
      {"lane=m word/step sel=s", 0, 0, 0, 0, 0, 1},
      {"lane=m word/step swap sel=s", 0, 1, 0, 0, 0, 1},
      {"cutlass col+4 sel=s", 1, 0, 0, 0, 0, 1},
      {"cutlass col+4 swap sel=s", 1, 1, 0, 0, 0, 1},
      {"cutlass lane+8 sel=s", 2, 0, 0, 0, 0, 1},
      {"cutlass lane+8 swap sel=s", 2, 1, 0, 0, 0, 1},
      {"lane=m 2 words/step sel=2s", 4, 0, 0, 0, 0, 2},
      {"lane=m 2 words/step swap", 4, 1, 0, 0, 0, 2},
      {"lane=m word/step addr4", 5, 0, 0, 4, 0, 0},
      {"lane=m word/step addr4 swap", 5, 1, 0, 4, 0, 0},
      {"replicate row nibble", 6, 0, 0, 0, 0, 0},
      {"replicate row nibble swap", 6, 1, 0, 0, 0, 0},
      {"group nibble 4g all words", 7, 0, 0, 0, 0, 0},
      {"group nibble 4g all words swap", 7, 1, 0, 0, 0, 0},
      {"replicate row nibble sel=s", 6, 0, 0, 0, 0, 1},
      {"group nibble 4g sel=s", 7, 0, 0, 0, 0, 1},
  };
  int best = -1;
  if (only >= static_cast<int>(hyps.size())) return 3;
  for (size_t h = 0; h < hyps.size(); ++h) {
    if (only >= 0 && static_cast<int>(h) != only) continue;
    const Hyp& H = hyps[h];
    std::vector<uint32_t> E(M * ECOLS, 0u);
    for (int m = 0; m < M; ++m)
      for (int g = 0; g < KL / 4; ++g) {
        const int i0 = idx[(m * KL / 4 + g) * 2], i1 = idx[(m * KL / 4 + g) * 2 + 1];
        const uint32_t nib = H.nib_swap ? (i1 | (i0 << 2)) : (i0 | (i1 << 2));
        const int k = g * 4;
        const int s = k / 32, gs = (k % 32) / 4;  // step, group within step
        int lane = m, col = 0, bit = 0;
        if (H.kind == 0 || H.kind == 5) {
          col = H.kind == 0 ? s : 4 * s;
          bit = 4 * gs;
        } else if (H.kind == 1 || H.kind == 2) {
          const int kb = k / 8;
          lane = m % 8 + 16 * (m / 16) + (H.kind == 2 ? 8 * ((m / 8) % 2) : 0);
          col = (kb % 16) / 4 + (H.kind == 1 ? 4 * ((m / 8) % 2) : 0);
          bit = 8 * (kb % 4) + 4 * ((k / 4) % 2);
        } else if (H.kind == 4) {
          col = 2 * s + gs / 4;
          bit = 8 * (gs % 4);
        }
        if (H.kind == 6) {  // replicate this row's nibble everywhere in its lane (valid for pmode 1-3)
          for (int c = 0; c < ECOLS; ++c) E[m * ECOLS + c] = nib * 0x11111111u;
          continue;
        }
        if (H.kind == 7) {  // nibble of group g at bits 4*(g%8) of every word of every lane (valid for pmode 1,2,4)
          for (int l = 0; l < M; ++l)
            for (int c = 0; c < ECOLS; ++c) E[l * ECOLS + c] = (E[l * ECOLS + c] & ~(0xFu << (4 * (g % 8)))) | (nib << (4 * (g % 8)));
          continue;
        }
        if (H.kind == 8) {  // nibble of group g at bits 4*(g%4) + 16*? : 2-bit fields, index i at 2*(2*(g%8)+q)
          continue;
        }
        E[lane * ECOLS + col] |= nib << bit;
      }
    cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128, 32 * 1024>>>(dAc, dB, dE, dD, H.id0, H.id1, H.e0, H.e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("H%zu %-26s CUDA error %s\n", h, H.name, cudaGetErrorString(err));
      return 1;  // sticky error: the context is gone
    }
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    int bad_rows = 0;
    for (int i = 0; i < M; ++i) {
      double rn = 0, rd = 0;
      for (int j = 0; j < N; ++j) {
        const double e = D[i * N + j] - Dref[i * N + j];
        rn += e * e;
        rd += (double)Dref[i * N + j] * Dref[i * N + j];
      }
      num += rn;
      den += rd;
      if (rn > 1e-6 * rd) ++bad_rows;
    }
    const double rel = sqrt(num / den);
    printf("H%zu %-26s relL2 = %.3e  bad rows %3d  D[0]=%9.4f ref %9.4f\n", h, H.name, rel, bad_rows, D[0], Dref[0]);
    if (rel < 1e-3 && best < 0) best = static_cast<int>(h);
  }
  printf("BEST %d\n", best);
  return 0;
}
