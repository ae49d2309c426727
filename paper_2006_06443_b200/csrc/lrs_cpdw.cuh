// lrs_cpdw.cuh -- stages 2 and 3 of the paper's CP-decomposed convolution
// (§3.3), the two depthwise convolutions over the rank channels:
//
//   Y^B[n, s, m, r] = sum_k  B[k, r] Y^A[n, s*sh + k - ph, m, r]      (k x 1, along H)
//   Y^C[n, s, m, r] = sum_p  C[p, r] Y^B[n, s, m*sw + p - pw, r]      (1 x k, along W)
//
// (the paper writes C_kr in the first line -- a typo, reading #5).  Y^A is
// T1 (the 1x1 projection, computed by the tensor-core GEMM), Y^C is T2, which the
// expansion + sparse kernel consumes exactly as the Tucker-2 core's output.
//
// Memory-bound stencil (2k FMAs per output element against 2 x 16 B of traffic
// per 8 channels): one thread per (output position, 16-byte channel vector); the
// k x k input taps of a position hit L1/L2 (T1 is written just before).  Each
// output keeps the paper's stage order: the k column partial sums Y^B first, then
// their 1 x k combination.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kCpThreads = 256;
constexpr int kCpMaxK = 7;

struct CpDwParams {
  const void* t1;    // [n][h][w][ld] dtype
  void* t2;          // [n][ho][wo][ld] dtype
  const float* b;    // [kh][ld] vertical taps (zero-padded ranks)
  const float* c;    // [kw][ld] horizontal taps
  int n, h, w, ho, wo, ld;
  int kh, kw, sh, sw, ph, pw;
};

template <bool F32>
__global__ void __launch_bounds__(kCpThreads) lrs_cp_dw_kernel(const __grid_constant__ CpDwParams p) {
  constexpr int V = F32 ? 4 : 8;  // channels per 16-byte vector
  pdl_wait();  // T1 comes from the projection kernel launched just before
  pdl_launch_dependents();  // only after the wait: every kernel before us is then complete
  const int nvec = p.ld / V;
  const long long total = static_cast<long long>(p.n) * p.ho * p.wo * nvec;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cv = static_cast<int>(i % nvec);
    long long pos = i / nvec;
    const int wo = static_cast<int>(pos % p.wo);
    pos /= p.wo;
    const int ho = static_cast<int>(pos % p.ho);
    const int n = static_cast<int>(pos / p.ho);
    const int ch = cv * V;
    float out[V];
#pragma unroll
    for (int j = 0; j < V; ++j) out[j] = 0.f;
    for (int x = 0; x < p.kw; ++x) {
      const int wi = wo * p.sw + x - p.pw;
      // Y^B at column wi: the k x 1 stage
      float yb[V];
#pragma unroll
      for (int j = 0; j < V; ++j) yb[j] = 0.f;
      if (wi >= 0 && wi < p.w) {
        for (int y = 0; y < p.kh; ++y) {
          const int hi = ho * p.sh + y - p.ph;
          if (hi < 0 || hi >= p.h) continue;
          const long long off = ((static_cast<long long>(n) * p.h + hi) * p.w + wi) * p.ld + ch;
          float v[V];
          if constexpr (F32) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(p.t1) + off));
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
          } else {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.t1) + off));
            const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              v[2 * j] = __uint_as_float(u[j] << 16);
              v[2 * j + 1] = __uint_as_float(u[j] & 0xFFFF0000u);
            }
          }
          const float* bt = p.b + y * p.ld + ch;
#pragma unroll
          for (int j = 0; j < V; ++j) yb[j] = fmaf(__ldg(bt + j), v[j], yb[j]);
        }
      }
      // the 1 x k stage
      const float* ct = p.c + x * p.ld + ch;
#pragma unroll
      for (int j = 0; j < V; ++j) out[j] = fmaf(__ldg(ct + j), yb[j], out[j]);
    }
    const long long o = ((static_cast<long long>(n) * p.ho + ho) * p.wo + wo) * p.ld + ch;
    if constexpr (F32) {
      *reinterpret_cast<float4*>(static_cast<float*>(p.t2) + o) = make_float4(out[0], out[1], out[2], out[3]);
    } else {
      uint4 q;
      uint32_t* u = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(out[2 * j], out[2 * j + 1]);
        u[j] = *reinterpret_cast<uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.t2) + o) = q;
    }
  }
}

}  // namespace lrs
