// lrs_core.cuh -- a1 + a2 in one kernel on the sm_100a tensor cores (bf16, stride 1):
//
//   T1[n, h, w, a]    = sum_c X[n, h, w, c] U_in[c, a]                              (a1)
//   T2[n, ho, wo, b]  = sum_{a, y, x} T1[n, ho + y - p, wo + x - p, a] G[a, b, y, x]  (a2)
//
// T1 never leaves the SM: a tile (ipt images x th output rows x full width) first
// computes T1 on its input WINDOW (wr = th + kh - 1 rows x wc = wo + kw - 1 cols,
// zero padding = TMA out-of-bounds fill, and T1 of a zero row is zero because the
// projection has no bias), restages it as bf16 into shared memory, and then runs
// the k x k core convolution from that window: the im2col operand of tap (y, x)
// is the same window at a start offset of y*wc + x rows.  The T1 window uses the
// K-major SWIZZLE_NONE layout (8-row x 16-B core matrices, rows 16 B apart), the
// one canonical layout in which ANY row offset is a legal operand start.
//
// MMA rows are window positions in row-major order, so one M = 128 MMA covers
// several output rows; the kw - 1 padding columns between rows are computed and
// discarded (the same trade as lrs_wconv.cuh).  Output rows of the tile:
// q = hl * wc + wl, valid for wl < wo and hl < rows of the band.
//
// The ipt images of a tile are stacked along the rows (one TMA box {64, wc, wr, ipt}):
// the weight chunks (U_in, G), which every tile streams from L2, are then shared by
// ipt images.  A T2 MMA row m reads T1 rows m + tap offset, so M blocks run across
// the image boundaries; rows whose window position is no output are discarded.
//
// Persistent CTAs walk the tiles.  Warps: 0 TMA producer, 1 MMA issuer,
// 2..9 epilogue (T1 restage, T2 store); TMEM holds T1 and T2 of a tile, double
// buffered when it fits so the T2 epilogue of tile k overlaps tile k+1.  T2 reuses
// the TMEM columns of T1 (the restage has read them before the core MMAs start).
#pragma once
#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kCThreads = 320;
constexpr int kCMaxSlots = 8;

struct CoreParams {
  CUtensorMap tmX;  // X 4-D (C, W, H, N) bf16, box {64, wc, wr, 1}, SW128
  CUtensorMap tmU;  // U_in^T [R1p][Cin] bf16, box {64, R1p}, SW128
  CUtensorMap tmG;  // G^T [R2p][taps * R1p] bf16, box {g_kc, R2p}, swizzle sw_g
  __nv_bfloat16* t2;  // [n * ho * wo][R2p]
  int n, ho, wo, kh, kw, ph, pw;
  int th, bands, n_tiles;
  int ipt;               // images per tile (stacked windows)
  int wr, wc, p1;        // window rows / cols / positions per image
  int nb1, nb2;          // M blocks of T1 (ipt * p1 rows) and of T2 ((ipt - 1) * p1 + (th - 1) * wc + wo rows)
  int n_ck;              // Cin / 64
  int r1p, r2p;
  int g_kc, n_gk;        // G K chunk (elements) and chunks per tap
  uint32_t sw_g;
  uint32_t x_bytes;      // one X box (ipt * wr * wc * 128 B)
  uint32_t x_region;     // X part of a slot (nb1 * 16 KB)
  uint32_t u_bytes, g_bytes;
  uint32_t slot_bytes;
  int ns;
  uint32_t t1_rows;      // rows of the T1 window (LBO = t1_rows * 16 B)
  uint32_t acc_cols;     // TMEM columns per buffer: max(nb1 * R1p, nb2 * R2p)
  int nacc;
  uint32_t tmem_cols;
  uint32_t off_t1, off_bar;
  unsigned long long* trace;  // optional globaltimer stamps (LRS_WCONV_DEBUG builds, tools/ctrace.py)
};

#ifdef LRS_WCONV_DEBUG
#define CTRACE(p, cond, idx) \
  do {                       \
    if ((p).trace && (cond)) (p).trace[idx] = gtimer(); \
  } while (0)
#else
#define CTRACE(p, cond, idx) \
  do {                       \
  } while (0)
#endif

__global__ void __launch_bounds__(kCThreads, 1) lrs_core_kernel(const __grid_constant__ CoreParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;                        // [ns]
  uint64_t* empty = bars + kCMaxSlots;          // [ns]
  uint64_t* t1_full = bars + 2 * kCMaxSlots;    // [2] MMA -> epilogue: T1 accumulated
  uint64_t* t2_full = t1_full + 2;              // [2] MMA -> epilogue: T2 accumulated
  uint64_t* acc_empty = t2_full + 2;            // [2] epilogue -> MMA (8 arrivals)
  uint64_t* t1s_full = acc_empty + 2;           // epilogue -> MMA: T1 window restaged (8 arrivals)
  uint64_t* t1w_empty = t1s_full + 1;           // MMA -> epilogue: core MMAs done reading the window
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t1w_empty + 1);
  const int taps = p.kh * p.kw;

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t1_full[i], 1);
      mbar_init(&t2_full[i], 1);
      mbar_init(&acc_empty[i], 8);
    }
    mbar_init(t1s_full, 8);
    mbar_init(t1w_empty, 1);
    fence_mbar_init();
    tma_prefetch_desc(&p.tmX);
    tma_prefetch_desc(&p.tmU);
    tma_prefetch_desc(&p.tmG);
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  CTRACE(p, threadIdx.x == 0 && blockIdx.x < 2048, 9000 + 2 * blockIdx.x);
  pdl_wait();  // the previous kernel's output is visible from here on
  pdl_launch_dependents();  // only after the wait: every kernel before us is then complete
  CTRACE(p, threadIdx.x == 0 && blockIdx.x == 0, 8190);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int it = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const int g = tile / p.bands, ho0 = (tile - g * p.bands) * p.th;
        for (int c = 0; c < p.n_ck; ++c, ++it) {
          const int s = it % p.ns;
          if (it >= p.ns) mbar_wait(&empty[s], ((it / p.ns) - 1) & 1);
          CTRACE(p, blockIdx.x == 0 && c == 0 && (tile - blockIdx.x) / gridDim.x < 4,
                 8200 + 10 * ((tile - blockIdx.x) / gridDim.x) + 1);
          uint8_t* dst = smem + s * p.slot_bytes;
          mbar_arrive_expect_tx(&full[s], p.x_bytes + p.u_bytes);
          tma_load_4d(dst, &p.tmX, &full[s], c * 64, -p.pw, ho0 - p.ph, g * p.ipt);
          tma_load_2d(dst + p.x_region, &p.tmU, &full[s], c * 64, 0);
        }
        for (int t = 0; t < taps; ++t)
          for (int gk = 0; gk < p.n_gk; ++gk, ++it) {
            const int s = it % p.ns;
            if (it >= p.ns) mbar_wait(&empty[s], ((it / p.ns) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], p.g_bytes);
            tma_load_2d(smem + s * p.slot_bytes + p.x_region, &p.tmG, &full[s], t * p.r1p + gk * p.g_kc, 0);
          }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    const uint32_t idesc1 = umma_idesc(1u, static_cast<uint32_t>(p.r1p), 128u);
    const uint32_t idesc2 = umma_idesc(1u, static_cast<uint32_t>(p.r2p), 128u);
    const uint32_t base = smem_u32(smem);
    const uint32_t t1w = smem_u32(smem + p.off_t1);
    const uint32_t lbo = p.t1_rows * 16u;
    const int gsteps = p.g_kc / 16;
    int it = 0, k = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++k) {
      const int b = p.nacc == 2 ? (k & 1) : 0;
      const int use = p.nacc == 2 ? (k >> 1) : k;
      if (use > 0) {
        mbar_wait(&acc_empty[b], (use - 1) & 1);
        tc_fence_after();
      }
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * p.acc_cols;
      const uint32_t t2c = acc0;  // T2 overwrites T1's columns (restaged already)
      // ---- a1: T1 (window rows) = X window . U_in, K = Cin in 64-channel chunks
      for (int c = 0; c < p.n_ck; ++c, ++it) {
        const int s = it % p.ns;
        mbar_wait(&full[s], (it / p.ns) & 1);
        tc_fence_after();
        CTRACE(p, blockIdx.x == 0 && lane == 0 && k < 4 && c == 0, 8200 + 10 * k + 2);
        const uint32_t xa = base + s * p.slot_bytes;
        if (elect_one()) {
          for (int b1 = 0; b1 < p.nb1; ++b1)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(acc0 + static_cast<uint32_t>(b1 * p.r1p), umma_desc(xa + b1 * 16384u + kk * 32u, 128),
                       umma_desc(xa + p.x_region + kk * 32u, 128), idesc1, (c > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
          if (c == p.n_ck - 1) mma_commit(&t1_full[b]);
        }
        __syncwarp();
      }
      CTRACE(p, blockIdx.x == 0 && lane == 0 && k < 4, 8200 + 10 * k + 3);
      // ---- wait for the bf16 T1 window in shared memory
      mbar_wait(t1s_full, k & 1);
      tc_fence_after();
      CTRACE(p, blockIdx.x == 0 && lane == 0 && k < 4, 8200 + 10 * k + 6);
      // ---- a2: T2 = sum over taps of (window shifted by y*wc + x) . G[tap]
      for (int t = 0; t < taps; ++t) {
        const int ty = t / p.kw, tx = t - ty * p.kw;
        const uint32_t tap_off = static_cast<uint32_t>(ty * p.wc + tx) * 16u;
        for (int gk = 0; gk < p.n_gk; ++gk, ++it) {
          const int s = it % p.ns;
          mbar_wait(&full[s], (it / p.ns) & 1);
          tc_fence_after();
          const uint32_t ga = base + s * p.slot_bytes + p.x_region;
          if (elect_one()) {
            for (int b2 = 0; b2 < p.nb2; ++b2)
              for (int kk = 0; kk < gsteps; ++kk) {
                const uint32_t kslice = static_cast<uint32_t>((gk * p.g_kc) / 8 + 2 * kk);
                mma_bf16(t2c + static_cast<uint32_t>(b2 * p.r2p),
                         umma_desc_noswz(t1w + static_cast<uint32_t>(b2 * 128) * 16u + tap_off + kslice * lbo, lbo,
                                         128u),
                         umma_desc(ga + kk * 32u, p.sw_g), idesc2, (t > 0 || gk > 0 || kk > 0) ? 1u : 0u);
              }
            mma_commit(&empty[s]);
          }
          __syncwarp();
        }
      }
      if (elect_one()) {
        mma_commit(&t2_full[b]);
        mma_commit(t1w_empty);
      }
      __syncwarp();
      CTRACE(p, blockIdx.x == 0 && lane == 0 && k < 4, 8200 + 10 * k + 7);
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int q4 = warp & 3;            // TMEM lane quarter
    const int ehalf = (warp - 2) >> 2;  // which 16-column half of every 32 columns
    const uint32_t t1w = smem_u32(smem + p.off_t1);
    int k = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++k) {
      const int g = tile / p.bands, ho0 = (tile - g * p.bands) * p.th;
      const int rows = min(p.th, p.ho - ho0);
      const int b = p.nacc == 2 ? (k & 1) : 0;
      const int use = p.nacc == 2 ? (k >> 1) : k;
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * p.acc_cols + (static_cast<uint32_t>(q4 * 32) << 16);
      // ---- restage T1 (fp32 TMEM) as bf16 into the SWIZZLE_NONE window
      mbar_wait_sleep(&t1_full[b], use & 1);
      if (k > 0) mbar_wait(t1w_empty, (k - 1) & 1);
      tc_fence_after();
      CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 4);
      for (int b1 = 0; b1 < p.nb1; ++b1) {
        const uint32_t row = static_cast<uint32_t>(b1 * 128 + q4 * 32 + lane);
        for (int c0 = ehalf * 16; c0 < p.r1p; c0 += 32) {
          float v[16];
          tmem_ld16(acc0 + static_cast<uint32_t>(b1 * p.r1p + c0), v);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint4 u;
            uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(v[8 * h + 2 * i], v[8 * h + 2 * i + 1]);
              w[i] = *reinterpret_cast<uint32_t*>(&bb);
            }
            const uint32_t kslice = static_cast<uint32_t>(c0 / 8 + h);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(t1w + (kslice * p.t1_rows + row) * 16u),
                         "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                         : "memory");
          }
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t1s_full);
      CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 5);
      // ---- T2 (fp32 TMEM) -> bf16 rows of global T2
      mbar_wait_sleep(&t2_full[b], use & 1);
      tc_fence_after();
      CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 8);
      for (int b2 = 0; b2 < p.nb2; ++b2) {
        const int q = b2 * 128 + q4 * 32 + lane;
        const int img = q / p.p1, rem = q - img * p.p1;
        const int hl = rem / p.wc, wl = rem - (rem / p.wc) * p.wc;
        const int n = g * p.ipt + img;
        const bool ok = wl < p.wo && hl < rows && img < p.ipt && n < p.n;
        __nv_bfloat16* dst =
            p.t2 + ((static_cast<long long>(ok ? n : 0) * p.ho + ho0 + (ok ? hl : 0)) * p.wo + (ok ? wl : 0)) * p.r2p;
        for (int c0 = ehalf * 16; c0 < p.r2p; c0 += 32) {
          float v[16];
          tmem_ld16(acc0 + static_cast<uint32_t>(b2 * p.r2p + c0), v);
          if (ok) {
            uint4 u[2];
            uint32_t* w = reinterpret_cast<uint32_t*>(u);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
              w[i] = *reinterpret_cast<uint32_t*>(&bb);
            }
            reinterpret_cast<uint4*>(dst + c0)[0] = u[0];
            reinterpret_cast<uint4*>(dst + c0)[1] = u[1];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 9);
    }
  }
  CTRACE(p, threadIdx.x == 64 && blockIdx.x < 2048, 9000 + 2 * blockIdx.x + 1);

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
  }
}

}  // namespace lrs
