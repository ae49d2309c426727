// lrs_tiny.cuh -- the whole fp32 layer in ONE kernel for layers whose weights and
// per-row working set fit in shared memory (C1: batch 1, 64 channels, ranks 16):
//
//   T1[q, a]  = sum_c X[q, c] U_in[c, a]                          (a1)  on the input window
//   T2[p, b]  = sum_{y,x,a} T1[p*s + (y,x) - pad, a] G[a, b, y, x]    (a2)
//   Y[p, j]   = sum_b T2[p, b] U_out[b, j]                           (a3)
//             + sum_{e in row j} v_e X[p*s + (y_e, x_e) - pad, c_e]   (a4)
//
// written to Y once (a5).  At batch 1 the tensor-core chain is three dependent launches
// of a few CTAs each (~35 us of latency for ~14 M MAC); here a CTA owns one image x th
// output rows x tc output columns x all output channels and runs the four stages back to back
// out of shared memory with exact fp32 FMAs (the north star's fp32 bar, no tf32 split).
// T1 is recomputed on the window's halo rows (a1 is the cheapest stage at small ranks).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kTyThreads = 512;

struct TinyParams {
  const float* x;    // [n][h][w][cin]
  float* y;          // [n][ho][wo][cout]
  const float* uin;  // [cin][r1p]   (ranks >= R1 zero)
  const float* g;    // [taps][r1p][r2p]
  const float* uo;   // [r2p][cout]
  const int* rp;     // CSR row_ptr [cout + 1]
  const int* ent_c;  // per nonzero: c | ty << 16 | tx << 24
  const float* ent_v;
  int n, h, w, cin, ho, wo, cout;
  int kh, kw, sh, sw, ph, pw;
  int r1p, r2p, th, bands, wr, wc;
  int tc, cbands;  // output columns per CTA and column bands (CTA = image x row band x column band)
  int cp;          // 1: CP core: g holds B [kh][r1p] then C [kw][r1p], r2p == r1p
  int nnz;
  uint32_t off_t1, off_t2, off_u, off_g, off_uo, off_rp, off_ec, off_ev;  // shared-memory carve-up (bytes)
  const float2* epi;  // per output channel (scale, bias) of the fused output epilogue, or NULL
  int relu;
  // 1: X is not the previous kernel's output (lrs_conv.cu forward_impl): compute at once and
  // wait for the previous kernel only before the first store of Y (the one buffer a previous
  // forward may still be writing)
  int early;
};

__global__ void __launch_bounds__(kTyThreads, 1) lrs_tiny_kernel(const __grid_constant__ TinyParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  float* xs = reinterpret_cast<float*>(sm);              // [cin][wr][wc]
  float* t1 = reinterpret_cast<float*>(sm + p.off_t1);   // [wr*wc][r1p]
  float* t2 = reinterpret_cast<float*>(sm + p.off_t2);   // [th*tc][r2p]
  float* us = reinterpret_cast<float*>(sm + p.off_u);    // [cin][r1p]
  float* gs = reinterpret_cast<float*>(sm + p.off_g);    // [taps][r1p][r2p], or CP: B [kh][r1p], C [kw][r1p]
  float* uos = reinterpret_cast<float*>(sm + p.off_uo);  // [r2p][cout]
  int* rps = reinterpret_cast<int*>(sm + p.off_rp);      // CSR of S in shared memory
  int* ecs = reinterpret_cast<int*>(sm + p.off_ec);
  float* evs = reinterpret_cast<float*>(sm + p.off_ev);
  const int cbi = blockIdx.x % p.cbands, rb = blockIdx.x / p.cbands;
  const int n = rb / p.bands, ho0 = (rb - n * p.bands) * p.th;
  const int wo0 = cbi * p.tc;
  const int rows = min(p.th, p.ho - ho0);
  const int cols = min(p.tc, p.wo - wo0);
  const int taps = p.kh * p.kw;
  const int wrc = p.wr * p.wc;
  // weights first: they do not depend on the previous kernel
  for (int i = threadIdx.x; i < p.cin * p.r1p / 4; i += kTyThreads)
    reinterpret_cast<float4*>(us)[i] = __ldg(reinterpret_cast<const float4*>(p.uin) + i);
  const int gn = p.cp ? (p.kh + p.kw) * p.r1p : taps * p.r1p * p.r2p;
  for (int i = threadIdx.x; i < gn / 4; i += kTyThreads)
    reinterpret_cast<float4*>(gs)[i] = __ldg(reinterpret_cast<const float4*>(p.g) + i);
  for (int i = threadIdx.x; i < p.r2p * p.cout / 4; i += kTyThreads)
    reinterpret_cast<float4*>(uos)[i] = __ldg(reinterpret_cast<const float4*>(p.uo) + i);
  for (int i = threadIdx.x; i <= p.cout; i += kTyThreads) rps[i] = __ldg(p.rp + i);
  for (int i = threadIdx.x; i < p.nnz; i += kTyThreads) {
    ecs[i] = __ldg(p.ent_c + i);
    evs[i] = __ldg(p.ent_v + i);
  }
  if (!p.early) pdl_wait();  // the previous kernel's output is visible from here on
  pdl_launch_dependents();
  // ---- X window [c][row][col] (zero padding), 4 channels per load, 4 loads in flight
  {
    const int nit = wrc * (p.cin / 4);
    for (int i0 = threadIdx.x; i0 < nit; i0 += 4 * kTyThreads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kTyThreads;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < nit) {
          const int c4 = i / wrc, q = i - c4 * wrc;
          const int r = q / p.wc, col = q - r * p.wc;
          const int hi = ho0 * p.sh - p.ph + r, wi = wo0 * p.sw + col - p.pw;
          if (hi >= 0 && hi < p.h && wi >= 0 && wi < p.w)
            v[u] = __ldg(reinterpret_cast<const float4*>(p.x + ((static_cast<long long>(n) * p.h + hi) * p.w + wi) * p.cin) +
                         c4);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kTyThreads;
        if (i < nit) {
          const int c4 = i / wrc, q = i - c4 * wrc;
          xs[(4 * c4 + 0) * wrc + q] = v[u].x;
          xs[(4 * c4 + 1) * wrc + q] = v[u].y;
          xs[(4 * c4 + 2) * wrc + q] = v[u].z;
          xs[(4 * c4 + 3) * wrc + q] = v[u].w;
        }
      }
    }
  }
  __syncthreads();
  // ---- a1: T1 on every window position, 4 ranks per item
  {
    const int ag = p.r1p / 4;
    for (int it = threadIdx.x; it < wrc * ag; it += kTyThreads) {
      const int q = it / ag, a0 = 4 * (it - q * ag);
      // two independent partial sums (even / odd channels): halves the FMA chain
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), acd = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
      for (int c = 0; c < p.cin; c += 2) {
        const float xv = xs[c * wrc + q], xw = xs[(c + 1) * wrc + q];
        const float4 u = *reinterpret_cast<const float4*>(us + c * p.r1p + a0);
        const float4 w = *reinterpret_cast<const float4*>(us + (c + 1) * p.r1p + a0);
        acc.x = fmaf(xv, u.x, acc.x);
        acc.y = fmaf(xv, u.y, acc.y);
        acc.z = fmaf(xv, u.z, acc.z);
        acc.w = fmaf(xv, u.w, acc.w);
        acd.x = fmaf(xw, w.x, acd.x);
        acd.y = fmaf(xw, w.y, acd.y);
        acd.z = fmaf(xw, w.z, acd.z);
        acd.w = fmaf(xw, w.w, acd.w);
      }
      *reinterpret_cast<float4*>(t1 + q * p.r1p + a0) =
          make_float4(acc.x + acd.x, acc.y + acd.y, acc.z + acd.z, acc.w + acd.w);
    }
  }
  __syncthreads();
  // ---- a2: T2 at the tile's output positions, 4 ranks per item
  const int npos = rows * cols;
  if (p.cp) {
    // CP: the paper's two depthwise stages per rank channel, in its
    // order: for each column tap x the k x 1 sum over y with B, then the 1 x k sum with C
    const int bg = p.r1p / 4;
    for (int it = threadIdx.x; it < npos * bg; it += kTyThreads) {
      const int pp = it / bg, a0 = 4 * (it - pp * bg);
      const int hl = pp / cols, wl = pp - hl * cols;
      float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int x = 0; x < p.kw; ++x) {
        float4 yb = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int y = 0; y < p.kh; ++y) {
          const float4 tv = *reinterpret_cast<const float4*>(t1 + ((hl * p.sh + y) * p.wc + wl * p.sw + x) * p.r1p + a0);
          const float4 bv = *reinterpret_cast<const float4*>(gs + y * p.r1p + a0);
          yb.x = fmaf(bv.x, tv.x, yb.x);
          yb.y = fmaf(bv.y, tv.y, yb.y);
          yb.z = fmaf(bv.z, tv.z, yb.z);
          yb.w = fmaf(bv.w, tv.w, yb.w);
        }
        const float4 cv = *reinterpret_cast<const float4*>(gs + (p.kh + x) * p.r1p + a0);
        out.x = fmaf(cv.x, yb.x, out.x);
        out.y = fmaf(cv.y, yb.y, out.y);
        out.z = fmaf(cv.z, yb.z, out.z);
        out.w = fmaf(cv.w, yb.w, out.w);
      }
      *reinterpret_cast<float4*>(t2 + pp * p.r2p + a0) = out;
    }
  } else {
    const int bg = p.r2p / 4;
    for (int it = threadIdx.x; it < npos * bg; it += kTyThreads) {
      const int pp = it / bg, b0 = 4 * (it - pp * bg);
      const int hl = pp / cols, wl = pp - hl * cols;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = 0; t < taps; ++t) {
        const int ty = t / p.kw, tx = t - ty * p.kw;
        const float* tq = t1 + ((hl * p.sh + ty) * p.wc + wl * p.sw + tx) * p.r1p;
        const float* gt = gs + t * p.r1p * p.r2p + b0;
#pragma unroll 4
        for (int a = 0; a < p.r1p; ++a) {
          const float tv = tq[a];
          const float4 gv = *reinterpret_cast<const float4*>(gt + a * p.r2p);
          acc.x = fmaf(tv, gv.x, acc.x);
          acc.y = fmaf(tv, gv.y, acc.y);
          acc.z = fmaf(tv, gv.z, acc.z);
          acc.w = fmaf(tv, gv.w, acc.w);
        }
      }
      *reinterpret_cast<float4*>(t2 + pp * p.r2p + b0) = acc;
    }
  }
  __syncthreads();
  // ---- a3 + a4 + a5: thread = (output channel j, group of positions); Y written once
  if (p.early) pdl_wait();  // before touching Y
  const int pgroups = max(1, kTyThreads / p.cout);
  const int per = (npos + pgroups - 1) / pgroups;
  for (int it = threadIdx.x; it < p.cout * pgroups; it += kTyThreads) {
    const int j = it % p.cout, pg = it / p.cout;
    const int pa = pg * per, pb = min(npos, pa + per);
    for (int pp0 = pa; pp0 < pb; pp0 += 8) {
      float acc[8];
      int qoff[8];  // window offset of each position (tap (0, 0)); divisions hoisted out of the nnz loop
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc[k] = 0.f;
        const int q = min(pp0 + k, pb - 1), hl = q / cols, wl = q - hl * cols;
        qoff[k] = hl * p.sh * p.wc + wl * p.sw;
      }
      for (int b = 0; b < p.r2p; ++b) {
        const float u = uos[b * p.cout + j];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (pp0 + k < pb) acc[k] = fmaf(t2[(pp0 + k) * p.r2p + b], u, acc[k]);
      }
      for (int e = rps[j]; e < rps[j + 1]; ++e) {
        const int cd = ecs[e];
        const float v = evs[e];
        const int c = cd & 0xFFFF, ty = (cd >> 16) & 0xFF, tx = cd >> 24;
        const float* xc = xs + c * wrc + ty * p.wc + tx;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fmaf(v, xc[qoff[k]], acc[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (pp0 + k < pb) {
          const int q = pp0 + k, hl = q / cols, wl = q - hl * cols;
          p.y[((static_cast<long long>(n) * p.ho + ho0 + hl) * p.wo + wo0 + wl) * p.cout + j] =
              out_epi(acc[k], out_epi_load(p.epi, j), p.relu);
        }
      }
    }
  }
}

}  // namespace lrs
