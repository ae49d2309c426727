// lrs_spadd.cuh -- a3 + a4 + a5 for fp32 layers on the CUDA cores:
//
//   Y[n, ho, wo, j] = sum_b T2[n, ho, wo, b] U_out[b, j]                                 (a3)
//                   + sum_{e in row j} v_e X[n, ho*s + y_e - p, wo*s + x_e - p, c_e]   (a4)
//
// accumulated in fp32 registers and written to Y once (a5).  The expansion is a
// register-blocked SIMT GEMM over a shared-memory tile of T2 (exact fp32, no tf32
// split); the sparse term is a direct CSR gather over a shared-memory window of X
// whose innermost dimension is 4 IMAGES: one 16-byte shared load then feeds 4
// FMAs that share the nonzero's value -- the layout the round-1 microbenchmark
// (tools/ubench_sparse.cu) measured fastest for fp32 activations.  The window
// is staged by a register transpose of NHWC loads (4 images x 4 channels).
//
// CTA (256 threads): 4 images x `th` output rows x all output columns x 64 output
// channels; warp w owns channels 8w..8w+7, lanes own output positions (<= 2 per
// lane).  Nonzeros are warp-uniform: (value, window byte offset) pairs staged in
// shared memory per input-channel chunk.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kSpThreads = 256;
constexpr int kSpKP = 2;   // output positions per lane
constexpr int kSpRc = 32;  // ranks per staged chunk of the expansion
constexpr uint32_t kSpDenseBytes = kSpRc * 32 * kSpKP * 16 + kSpRc * 64 * 4;  // T2 tile + U_out tile

struct SpaddParams {
  const float* x;
  float* y;
  int n, h, w, cin, ho, wo, cout;
  int kh, kw, sh, sw, ph, pw;
  int th, bands, n_nc;  // output rows per tile, row bands, 64-channel chunks
  int cc, n_cc;         // input channels per staged chunk, chunks
  int wr, wc;           // window rows / cols
  int pitch;            // 16-byte vectors per window row (>= wc; == wo*sw mod 8: conflict-free LDS.128)
  const int2* ent;      // (fp32 value bits, window byte offset)
  const int* ent_ptr;   // [(nc * n_cc + c) * 64 + jl] first entry; [+64] end of the chunk
  int max_ent;          // max entries of one (nc, c) chunk (smem staging)
  uint32_t win_bytes;    // the shared region: max(X window, kSpDenseBytes)
  const float* t;        // T2 (or T1 of the SVD pair) [n][ho][wo][t_ld]
  const float* uo;       // U_out [r][cout] fp32 (rows >= R2 zero)
  int t_ld, r;           // row pitch of T, ranks to sum (multiple of 4)
  int dbg;              // timing experiments (LRS_SPADD_DBG): 1 skip staging, 2 skip gather, 4 skip Y update
  const float2* epi;    // per output channel (scale, bias) of the fused output epilogue, or NULL
  int relu;
};

__global__ void __launch_bounds__(kSpThreads, 2) lrs_spadd_kernel(const __grid_constant__ SpaddParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  float4* win = reinterpret_cast<float4*>(sm);
  int2* ents0 = reinterpret_cast<int2*>(sm + p.win_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bid = blockIdx.x;
  const int nc = bid % p.n_nc;
  bid /= p.n_nc;
  const int band = bid % p.bands;
  const int n0 = (bid / p.bands) * 4;
  const int ho0 = band * p.th;
  const int rows = min(p.th, p.ho - ho0);
  const int npos = rows * p.wo;
  const int jw = nc * 64 + warp * 8;  // first output channel of this warp
  // PDL: T2 is written by the core kernel launched just before (and X by
  // whatever ran before the chain); wait for both before touching either
  pdl_wait();  // the previous kernel's output is visible from here on
  pdl_launch_dependents();  // only after the wait: every kernel before us is then complete

  // window-relative base (in 16-byte vectors) of each of this lane's positions
  int base[kSpKP];
  bool valid[kSpKP];
#pragma unroll
  for (int k = 0; k < kSpKP; ++k) {
    const int q = lane + 32 * k;
    valid[k] = q < npos;
    const int hl = valid[k] ? q / p.wo : 0, wl = valid[k] ? q - (q / p.wo) * p.wo : 0;
    base[k] = hl * p.sh * p.pitch + wl * p.sw;
  }
  float acc[kSpKP][8][4];
#pragma unroll
  for (int k = 0; k < kSpKP; ++k)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[k][jj][i] = 0.f;

  // ---- a3: acc = T2 tile . U_out, rank chunks of kSpRc staged as [rank][position][4 images]
  {
    float4* tt = win;
    const float4* us4 = reinterpret_cast<const float4*>(sm + kSpRc * 32 * kSpKP * 16);
    for (int b0 = 0; b0 < p.r; b0 += kSpRc) {
      const int rcn = min(kSpRc, p.r - b0);
      for (int wi = threadIdx.x; wi < npos * (rcn / 4); wi += kSpThreads) {
        const int b4 = wi / npos, q = wi - b4 * npos;
        const int ho = ho0 + q / p.wo, wo = q - (q / p.wo) * p.wo;
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (n0 + i < p.n)
            v[i] = __ldg(reinterpret_cast<const float4*>(
                p.t + ((static_cast<long long>(n0 + i) * p.ho + ho) * p.wo + wo) * p.t_ld + b0 + 4 * b4));
        }
        float4* dst = tt + (4 * b4) * (32 * kSpKP) + q;
        dst[0] = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
        dst[32 * kSpKP] = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
        dst[64 * kSpKP] = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
        dst[96 * kSpKP] = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
      }
      float4* usw = reinterpret_cast<float4*>(sm + kSpRc * 32 * kSpKP * 16);
      for (int wi = threadIdx.x; wi < rcn * 16; wi += kSpThreads) {
        const int bl = wi >> 4, j = nc * 64 + 4 * (wi & 15);
        usw[wi] = j < p.cout ? __ldg(reinterpret_cast<const float4*>(p.uo + static_cast<long long>(b0 + bl) * p.cout + j))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncthreads();
#pragma unroll 4
      for (int bl = 0; bl < rcn; ++bl) {
        const float4 ua = us4[bl * 16 + warp * 2], ub = us4[bl * 16 + warp * 2 + 1];
        const float u[8] = {ua.x, ua.y, ua.z, ua.w, ub.x, ub.y, ub.z, ub.w};
#pragma unroll
        for (int k = 0; k < kSpKP; ++k) {
          const float4 tv = tt[bl * (32 * kSpKP) + lane + 32 * k];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            acc[k][jj][0] = fmaf(u[jj], tv.x, acc[k][jj][0]);
            acc[k][jj][1] = fmaf(u[jj], tv.y, acc[k][jj][1]);
            acc[k][jj][2] = fmaf(u[jj], tv.z, acc[k][jj][2]);
            acc[k][jj][3] = fmaf(u[jj], tv.w, acc[k][jj][3]);
          }
        }
      }
      __syncthreads();
    }
  }

  const int plane = p.wr * p.pitch;  // vectors per channel
  const int items = p.wr * p.wc * (p.cc / 4);
  int2* ents = ents0;
  for (int c = 0; c < p.n_cc; ++c) {
    const int c0 = c * p.cc;
    // this warp's CSR row bounds of the chunk (lanes 0..8), loaded ahead of the staging
    const int* ptr = p.ent_ptr + (static_cast<long long>(nc) * p.n_cc + c) * 64;
    const int e_begin = __ldg(ptr), e_end = __ldg(ptr + 64);
    const int rb = lane <= 8 ? __ldg(ptr + warp * 8 + lane) - e_begin : 0;
    // ---- stage X[n0..n0+3, window rows/cols, c0..c0+cc) as [c][row][pitch][4 images]
    for (int wi = threadIdx.x; wi < (LRS_XDBG(p.dbg & 1) ? 0 : items); wi += kSpThreads) {
      const int c4 = wi / (p.wr * p.wc), pos = wi - c4 * (p.wr * p.wc);
      const int r = pos / p.wc, col = pos - r * p.wc;
      const int hi = ho0 * p.sh - p.ph + r, wi_ = col - p.pw, ch = c0 + 4 * c4;
      const bool inb = hi >= 0 && hi < p.h && wi_ >= 0 && wi_ < p.w && ch < p.cin;
      float4 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (inb && n0 + i < p.n)
          v[i] = __ldg(reinterpret_cast<const float4*>(
              p.x + ((static_cast<long long>(n0 + i) * p.h + hi) * p.w + wi_) * p.cin + ch));
      }
      float4* dst = win + static_cast<size_t>(4 * c4) * plane + r * p.pitch + col;
      dst[0] = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
      dst[plane] = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
      dst[2 * plane] = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
      dst[3 * plane] = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
    }
    // ---- stage this chunk's nonzeros of the CTA's 64 output channels
    for (int e = e_begin + static_cast<int>(threadIdx.x); e < e_end; e += kSpThreads) ents[e - e_begin] = __ldg(p.ent + e);
    __syncthreads();
    // ---- warp-uniform CSR rows of this warp's 8 channels, two nonzeros per step
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int a = __shfl_sync(0xffffffffu, rb, jj), b = LRS_XDBG(p.dbg & 2) ? a : __shfl_sync(0xffffffffu, rb, jj + 1);
      int e = a;
      for (; e + 2 <= b; e += 2) {
        const int2 en0 = ents[e], en1 = ents[e + 1];
        const float v0 = __int_as_float(en0.x), v1 = __int_as_float(en1.x);
        const float4* s0 = win + (en0.y >> 4);
        const float4* s1 = win + (en1.y >> 4);
        float4 x0[kSpKP], x1[kSpKP];
#pragma unroll
        for (int k = 0; k < kSpKP; ++k) {
          x0[k] = s0[base[k]];
          x1[k] = s1[base[k]];
        }
#pragma unroll
        for (int k = 0; k < kSpKP; ++k) {
          acc[k][jj][0] = fmaf(v0, x0[k].x, acc[k][jj][0]);
          acc[k][jj][1] = fmaf(v0, x0[k].y, acc[k][jj][1]);
          acc[k][jj][2] = fmaf(v0, x0[k].z, acc[k][jj][2]);
          acc[k][jj][3] = fmaf(v0, x0[k].w, acc[k][jj][3]);
          acc[k][jj][0] = fmaf(v1, x1[k].x, acc[k][jj][0]);
          acc[k][jj][1] = fmaf(v1, x1[k].y, acc[k][jj][1]);
          acc[k][jj][2] = fmaf(v1, x1[k].z, acc[k][jj][2]);
          acc[k][jj][3] = fmaf(v1, x1[k].w, acc[k][jj][3]);
        }
      }
      if (e < b) {
        const int2 en = ents[e];
        const float v = __int_as_float(en.x);
        const float4* src = win + (en.y >> 4);
#pragma unroll
        for (int k = 0; k < kSpKP; ++k) {
          const float4 xv = src[base[k]];
          acc[k][jj][0] = fmaf(v, xv.x, acc[k][jj][0]);
          acc[k][jj][1] = fmaf(v, xv.y, acc[k][jj][1]);
          acc[k][jj][2] = fmaf(v, xv.z, acc[k][jj][2]);
          acc[k][jj][3] = fmaf(v, xv.w, acc[k][jj][3]);
        }
      }
    }
    __syncthreads();
  }
  // ---- Y = Y_L + Y_S, written once: each lane owns 8 consecutive channels of its positions
  if (jw >= p.cout || LRS_XDBG(p.dbg & 4)) return;
  if (p.epi != nullptr || p.relu) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const float2 sb = out_epi_load(p.epi, min(jw + jj, p.cout - 1));
#pragma unroll
      for (int k = 0; k < kSpKP; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[k][jj][i] = out_epi(acc[k][jj][i], sb, p.relu);
    }
  }
#pragma unroll
  for (int k = 0; k < kSpKP; ++k) {
    if (!valid[k]) continue;
    const int q = lane + 32 * k;
    const int ho = ho0 + q / p.wo, wo = q - (q / p.wo) * p.wo;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (n0 + i >= p.n) continue;
      float* yp = p.y + ((static_cast<long long>(n0 + i) * p.ho + ho) * p.wo + wo) * p.cout + jw;
      if (jw + 8 <= p.cout) {
        *reinterpret_cast<float4*>(yp) = make_float4(acc[k][0][i], acc[k][1][i], acc[k][2][i], acc[k][3][i]);
        *reinterpret_cast<float4*>(yp + 4) = make_float4(acc[k][4][i], acc[k][5][i], acc[k][6][i], acc[k][7][i]);
      } else {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (jw + jj < p.cout) yp[jj] = acc[k][jj][i];
      }
    }
  }
}

}  // namespace lrs
