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
// T1 window layout: when R1p is a multiple of 64 it is K-major SWIZZLE_128B (64-rank
// chunks of 128-B rows).  The hardware applies the swizzle to absolute shared-memory
// address bits, so a start row that is not a multiple of the 8-row atom is a legal
// operand (tools/mma_baseoff.cu: exact at every row offset with base offset 0), and
// an N = 64 MMA then costs 48 instead of 88 cycles (SWIZZLE_NONE, the fallback for
// other ranks; profiles/r01_mma_layout_swizzle_none.log, r01_mma_baseoff.log).
//
// Shared memory: an X ring (one slot = a 64-channel X box + its U_in chunk; the last
// M block of a box reads past its end into the next slot -- garbage rows whose T1 and
// T2 rows are discarded), a G ring of separate small slots (when all k*k*R1p/g_kc
// chunks fit, G is loaded once per CTA, before the PDL wait: weights do not depend on
// the previous kernel), and the T1 window.
//
// Persistent CTAs walk the tiles.  Warps: 0 TMA producer, 1 MMA issuer,
// 2..9 epilogue (T1 restage, T2 store); TMEM holds T1 and T2 of a tile, double
// buffered when it fits so the T2 epilogue of tile k overlaps tile k+1.  T2 reuses
// the TMEM columns of T1 (the restage has read them before the core MMAs start).
#pragma once
#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kCThreads = 320;
constexpr int kCMaxX = 8;   // X ring slots
constexpr int kCMaxG = 32;  // G ring slots

struct CoreParams {
  CUtensorMap tmX;  // X 4-D (C, W, H, N) bf16, box {64, wc, wr, ipt}, SW128
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
  uint32_t u_off;        // U_in chunk offset inside an X slot (x_bytes rounded up to 1 KB)
  uint32_t u_bytes, g_bytes;
  uint32_t x_slot, g_slot;  // ring slot strides
  int ns_x, ns_g;
  int g_res;             // 1: every G chunk has its own slot, loaded once per CTA
  int unified;           // 1 (streamed G): ONE ring of ns_x slots of x_slot bytes holds the X items
                         // (box + U_in chunk) AND the G items (gpk chunks each), in consumption
                         // order -- a2's G stream gets the X ring's bytes in flight (no G ring)
  int gpk;               // G chunks per unified-ring item (x_slot / g_slot)
  int t1_sw128;          // 1: T1 window K-major SW128 (R1p % 64 == 0), 0: SWIZZLE_NONE
  uint32_t t1_rows;      // rows of the T1 window (multiple of 8)
  uint32_t acc_cols;     // TMEM columns per buffer: max(nb1 * R1p, nb2 * R2p)
  int nacc;
  uint32_t tmem_cols;
  uint32_t off_g, off_t1, off_bar;
  int dbg;           // experiment bits (LRS_CORE_DBG): 1 skip the depthwise loop, 2 skip its T2 stores,
                     // 4 skip the X / U loads, 8 skip the T2 stores, 16 skip the T1 restage stores
                     // (timing only)
  const float* cpb;  // CP core (CPDW kernels): B [kh][R1p], C [kw][R1p] fp32
  const float* cpc;
  unsigned long long* trace;  // optional globaltimer stamps (LRS_WCONV_DEBUG builds, tools/ctrace.py)
  // 1: start computing at once and wait for the previous kernel only before exiting.  The
  // host sets it when X is not an output of the library's previous launch on this stream
  // and T2 alternates between two buffers (lrs_conv.cu forward_impl): the
  // previous forward's fused kernel may still be reading the other T2.
  int early;
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

// Byte offset of the 16-byte piece holding ranks [kel, kel + 8) of T1 window row `row`.
__device__ __forceinline__ uint32_t t1_piece(const CoreParams& p, uint32_t row, uint32_t kel) {
  return p.t1_sw128 ? (kel >> 6) * p.t1_rows * 128u + row * 128u + ((((kel & 63u) >> 3) ^ (row & 7u)) << 4)
                    : ((kel >> 3) * p.t1_rows + row) * 16u;
}

// GS = K steps of 16 per G chunk (g_kc / 16: 4, 2 or 1)
// CPDW: the paper's CP form: no G; after the restage the epilogue warps
// run the two depthwise stages (k x 1 with B, then 1 x k with C, the paper's order) on the
// T1 window and write T2 -- the computation of lrs_cpdw.cuh, with T1 kept on chip.
template <int GS, bool CPDW>
__global__ void __launch_bounds__(kCThreads, 1) lrs_core_kernel(const __grid_constant__ CoreParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full_x = bars;                      // [ns_x]
  uint64_t* empty_x = full_x + kCMaxX;          // [ns_x]
  uint64_t* full_g = empty_x + kCMaxX;          // [ns_g]
  uint64_t* empty_g = full_g + kCMaxG;          // [ns_g]
  uint64_t* t1_full = empty_g + kCMaxG;         // [2] MMA -> epilogue: T1 accumulated
  uint64_t* t2_full = t1_full + 2;              // [2] MMA -> epilogue: T2 accumulated
  uint64_t* acc_empty = t2_full + 2;            // [2] epilogue -> MMA (8 arrivals)
  uint64_t* t1s_full = acc_empty + 2;           // epilogue -> MMA: T1 window restaged (8 arrivals)
  uint64_t* t1w_empty = t1s_full + 1;           // MMA -> epilogue: core MMAs done reading the window
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t1w_empty + 1);
  const int n_g = p.kh * p.kw * p.n_gk;         // G chunks per tile
  // the producer's and MMA issuer's loop scalars, staged in shared memory (a kernel
  // parameter read inside a loop is re-loaded from the constant bank at every use, ~100
  // cycles each on the issue path; tools/loop_cost2.cu)
  int* prm = reinterpret_cast<int*>(smem + p.off_bar + 1024);

  if (threadIdx.x == 0) {
    prm[0] = static_cast<int>(p.acc_cols);
    prm[1] = static_cast<int>(p.bands);
    prm[2] = static_cast<int>(p.g_bytes);
    prm[3] = static_cast<int>(p.g_kc);
    prm[4] = static_cast<int>(p.g_res);
    prm[5] = static_cast<int>(p.g_slot);
    prm[6] = static_cast<int>(p.ipt);
    prm[7] = static_cast<int>(p.kw);
    prm[8] = static_cast<int>(p.n_ck);
    prm[9] = static_cast<int>(p.n_gk);
    prm[10] = static_cast<int>(p.n_tiles);
    prm[11] = static_cast<int>(p.nacc);
    prm[12] = static_cast<int>(p.nb1);
    prm[13] = static_cast<int>(p.nb2);
    prm[14] = static_cast<int>(p.ns_g);
    prm[15] = static_cast<int>(p.ns_x);
    prm[16] = static_cast<int>(p.off_g);
    prm[17] = static_cast<int>(p.off_t1);
    prm[18] = static_cast<int>(p.ph);
    prm[19] = static_cast<int>(p.pw);
    prm[20] = static_cast<int>(p.r1p);
    prm[21] = static_cast<int>(p.r2p);
    prm[22] = static_cast<int>(p.sw_g);
    prm[23] = static_cast<int>(p.t1_rows);
    prm[24] = static_cast<int>(p.t1_sw128);
    prm[25] = static_cast<int>(p.th);
    prm[26] = static_cast<int>(p.u_bytes);
    prm[27] = static_cast<int>(p.u_off);
    prm[28] = static_cast<int>(p.wc);
    prm[29] = static_cast<int>(p.x_bytes);
    prm[30] = static_cast<int>(p.x_slot);
    prm[31] = p.unified;
    prm[32] = p.gpk;
    for (int i = 0; i < p.ns_x; ++i) {
      mbar_init(&full_x[i], 1);
      mbar_init(&empty_x[i], 1);
    }
    for (int i = 0; i < p.ns_g; ++i) {
      mbar_init(&full_g[i], 1);
      mbar_init(&empty_g[i], 1);
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
    if (n_g > 0) tma_prefetch_desc(&p.tmG);
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  CTRACE(p, threadIdx.x == 0 && blockIdx.x < 2048, 9000 + 2 * blockIdx.x);
  // a resident G is requested before the PDL wait (weights do not depend on the previous kernel)
  if (threadIdx.x == 0 && p.g_res) {
    for (int j = 0; j < n_g; ++j) {
      const int t = j / p.n_gk, gk = j - t * p.n_gk;
      mbar_arrive_expect_tx(&full_g[j], p.g_bytes);
      tma_load_2d(smem + p.off_g + j * p.g_slot, &p.tmG, &full_g[j], t * p.r1p + gk * p.g_kc, 0);
    }
  }
  // default: wait, then trigger -- when a kernel starts, every kernel before its predecessor
  // is complete.  early: trigger at once; the wait before exiting keeps the invariant for
  // whoever waits on this grid (its completion implies the previous kernel's).
  if (!p.early) pdl_wait();  // the previous kernel's output is visible from here on
  pdl_launch_dependents();
  CTRACE(p, threadIdx.x == 0 && blockIdx.x == 0, 8190);

  if (warp == 0) {
    const int bands_ = static_cast<int>(smem_param(prm + 1));
    const uint32_t g_bytes_ = static_cast<uint32_t>(smem_param(prm + 2));
    const int g_kc_ = static_cast<int>(smem_param(prm + 3));
    const int g_res_ = static_cast<int>(smem_param(prm + 4));
    const uint32_t g_slot_ = static_cast<uint32_t>(smem_param(prm + 5));
    const int ipt_ = static_cast<int>(smem_param(prm + 6));
    const int n_ck_ = static_cast<int>(smem_param(prm + 8));
    const int n_gk_ = static_cast<int>(smem_param(prm + 9));
    const int n_tiles_ = static_cast<int>(smem_param(prm + 10));
    const int nacc_ = static_cast<int>(smem_param(prm + 11));
    const int ns_g_ = static_cast<int>(smem_param(prm + 14));
    const int ns_x_ = static_cast<int>(smem_param(prm + 15));
    const uint32_t off_g_ = static_cast<uint32_t>(smem_param(prm + 16));
    const int ph_ = static_cast<int>(smem_param(prm + 18));
    const int pw_ = static_cast<int>(smem_param(prm + 19));
    const int r1p_ = static_cast<int>(smem_param(prm + 20));
    const int th_ = static_cast<int>(smem_param(prm + 25));
    const uint32_t u_bytes_ = static_cast<uint32_t>(smem_param(prm + 26));
    const uint32_t u_off_ = static_cast<uint32_t>(smem_param(prm + 27));
    const uint32_t x_bytes_ = static_cast<uint32_t>(smem_param(prm + 29));
    const uint32_t x_slot_ = static_cast<uint32_t>(smem_param(prm + 30));
    const int unified_ = smem_param(prm + 31);
    const int gpk_ = smem_param(prm + 32);
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      // Requests follow the MMA thread's consumption order (a1(k+1) before a2(k) when two
      // TMEM buffers allow the lookahead): a streamed G must never block an X box the
      // MMA thread needs first.
      int ix = 0, ig = 0;
      const int m_tiles = static_cast<int>(blockIdx.x) < n_tiles_
                              ? (n_tiles_ - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                              : 0;
      auto load_x = [&](int k) {
        const int tile = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
        const int g = tile / bands_, ho0 = (tile - g * bands_) * th_;
        for (int c = 0; c < n_ck_; ++c, ++ix) {
          const int s = ix % ns_x_;
          if (ix >= ns_x_) mbar_wait(&empty_x[s], ((ix / ns_x_) - 1) & 1);
          CTRACE(p, blockIdx.x == 0 && c == 0 && k < 4, 8200 + 10 * k + 1);
          uint8_t* dst = smem + s * x_slot_;
          if (LRS_XDBG(p.dbg & 4)) {  // timing experiment: no X / U loads (stale shared memory, wrong T2)
            mbar_arrive(&full_x[s]);
            continue;
          }
          mbar_arrive_expect_tx(&full_x[s], x_bytes_ + u_bytes_);
          tma_load_4d(dst, &p.tmX, &full_x[s], c * 64, -pw_, ho0 - ph_, g * ipt_);
          tma_load_2d(dst + u_off_, &p.tmU, &full_x[s], c * 64, 0);
        }
      };
      auto load_g = [&]() {
        if (g_res_) return;
        if (unified_) {  // G items of gpk chunks in the unified ring, after the X items
          for (int j0 = 0; j0 < n_g; j0 += gpk_, ++ix) {
            const int s = ix % ns_x_;
            if (ix >= ns_x_) mbar_wait(&empty_x[s], ((ix / ns_x_) - 1) & 1);
            const int cnt = min(gpk_, n_g - j0);
            mbar_arrive_expect_tx(&full_x[s], static_cast<uint32_t>(cnt) * g_bytes_);
            for (int q = 0; q < cnt; ++q) {
              const int j = j0 + q, t = j / n_gk_, gk = j - t * n_gk_;
              tma_load_2d(smem + s * x_slot_ + q * g_slot_, &p.tmG, &full_x[s], t * r1p_ + gk * g_kc_, 0);
            }
          }
          return;
        }
        for (int j = 0; j < n_g; ++j, ++ig) {
          const int s = ig % ns_g_;
          if (ig >= ns_g_) mbar_wait(&empty_g[s], ((ig / ns_g_) - 1) & 1);
          const int t = j / n_gk_, gk = j - t * n_gk_;
          mbar_arrive_expect_tx(&full_g[s], g_bytes_);
          tma_load_2d(smem + off_g_ + s * g_slot_, &p.tmG, &full_g[s], t * r1p_ + gk * g_kc_, 0);
        }
      };
      if (!CPDW && nacc_ == 2) {
        if (m_tiles > 0) load_x(0);
        for (int k = 0; k < m_tiles; ++k) {
          if (k + 1 < m_tiles) load_x(k + 1);
          load_g();
        }
      } else {
        for (int k = 0; k < m_tiles; ++k) {
          load_x(k);
          load_g();
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t acc_cols_ = static_cast<uint32_t>(smem_param(prm + 0));
    const int g_kc_ = static_cast<int>(smem_param(prm + 3));
    const int g_res_ = static_cast<int>(smem_param(prm + 4));
    const uint32_t g_slot_ = static_cast<uint32_t>(smem_param(prm + 5));
    const int kw_ = static_cast<int>(smem_param(prm + 7));
    const int n_ck_ = static_cast<int>(smem_param(prm + 8));
    const int n_gk_ = static_cast<int>(smem_param(prm + 9));
    const int n_tiles_ = static_cast<int>(smem_param(prm + 10));
    const int nacc_ = static_cast<int>(smem_param(prm + 11));
    const int nb1_ = static_cast<int>(smem_param(prm + 12));
    const int nb2_ = static_cast<int>(smem_param(prm + 13));
    const int ns_g_ = static_cast<int>(smem_param(prm + 14));
    const int ns_x_ = static_cast<int>(smem_param(prm + 15));
    const uint32_t off_g_ = static_cast<uint32_t>(smem_param(prm + 16));
    const uint32_t off_t1_ = static_cast<uint32_t>(smem_param(prm + 17));
    const int r1p_ = static_cast<int>(smem_param(prm + 20));
    const int r2p_ = static_cast<int>(smem_param(prm + 21));
    const uint32_t sw_g_ = static_cast<uint32_t>(smem_param(prm + 22));
    const uint32_t t1_rows_ = static_cast<uint32_t>(smem_param(prm + 23));
    const int t1_sw128_ = static_cast<int>(smem_param(prm + 24));
    const uint32_t u_off_ = static_cast<uint32_t>(smem_param(prm + 27));
    const int wc_ = static_cast<int>(smem_param(prm + 28));
    const uint32_t x_slot_ = static_cast<uint32_t>(smem_param(prm + 30));
    const int unified_ = smem_param(prm + 31);
    const int gpk_ = smem_param(prm + 32);
    // -------------------------------------------------------------- MMA issuer
    // ONE elected thread runs the whole loop (its mbarrier waits included): an elect +
    // reconvergence per item costs ~240 cycles of issue (tools/mma_seq.cu: 108 vs 48
    // cycles per N = 64 MMA), more than the MMAs it feeds.
    if (elect_one()) {
    // Descriptors are linear in the shared-memory address (start >> 4 in the low 14
    // bits), so every operand is a base descriptor plus a precomputed offset: the issue
    // loop is adds and MMAs (address arithmetic per MMA made it issue-bound).
    const uint32_t idesc1 = umma_idesc(1u, static_cast<uint32_t>(r1p_), 128u);
    const uint32_t idesc2 = umma_idesc(1u, static_cast<uint32_t>(r2p_), 128u);
    const uint32_t base = smem_u32(smem);
    const uint32_t t1w = smem_u32(smem + off_t1_);
    const uint32_t lbo = t1_rows_ * 16u;
    const uint64_t xd0 = umma_desc(base, 128);
    const uint64_t ud0 = umma_desc(base + u_off_, 128);
    const uint64_t gd0 = umma_desc(base + off_g_, sw_g_);
    const uint64_t t1d0 = t1_sw128_ ? umma_desc(t1w, 128) : umma_desc_noswz(t1w, lbo, 128u);
    // T1 window: descriptor units (16 B) per window row, per G chunk of g_kc ranks, per K step of 16
    const uint32_t a_rs = t1_sw128_ ? 8u : 1u;
    const uint32_t a_gs = t1_sw128_ ? t1_rows_ * 8u : static_cast<uint32_t>(g_kc_ / 8) * (lbo >> 4);
    const uint32_t a_ks = t1_sw128_ ? 2u : 2u * (lbo >> 4);
    const uint32_t x16 = x_slot_ >> 4, g16 = g_slot_ >> 4;
    int ix = 0, ig = 0;
    const int m_tiles = static_cast<int>(blockIdx.x) < n_tiles_
                            ? (n_tiles_ - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                            : 0;
    // a1 of tile k into TMEM buffer b(k)
    auto phase_a1 = [&](int k) {
      const int b = nacc_ == 2 ? (k & 1) : 0;
      const int use = nacc_ == 2 ? (k >> 1) : k;
      if (use > 0) {
        mbar_wait(&acc_empty[b], (use - 1) & 1);
        tc_fence_after();
      }
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * acc_cols_;
      // ---- a1: T1 (window rows) = X window . U_in, K = Cin in 64-channel chunks
      for (int c = 0; c < n_ck_; ++c, ++ix) {
        const int s = ix % ns_x_;
        mbar_wait(&full_x[s], (ix / ns_x_) & 1);
        tc_fence_after();
        CTRACE(p, blockIdx.x == 0 && k < 4 && c == 0, 8200 + 10 * k + 2);
        const uint64_t xd = xd0 + static_cast<uint32_t>(s) * x16;
        const uint64_t ud = ud0 + static_cast<uint32_t>(s) * x16;
        {
          for (int b1 = 0; b1 < nb1_; ++b1) {
            const uint32_t d = acc0 + static_cast<uint32_t>(b1 * r1p_);
            const uint64_t xb = xd + static_cast<uint32_t>(b1) * 1024u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_bf16(d, xb + 2 * kk, ud + 2 * kk, idesc1, (c > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty_x[s]);
          if (c == n_ck_ - 1) mma_commit(&t1_full[b]);
        }
      }
      CTRACE(p, blockIdx.x == 0 && k < 4, 8200 + 10 * k + 3);
    };
    // a2 of tile k: T2 over T1's columns of buffer b(k), from the restaged window
    auto phase_a2 = [&](int k) {
      const int b = nacc_ == 2 ? (k & 1) : 0;
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * acc_cols_;
      const uint32_t t2c = acc0;  // T2 overwrites T1's columns (restaged already)
      // ---- wait for the bf16 T1 window in shared memory
      mbar_wait(t1s_full, k & 1);
      tc_fence_after();
      CTRACE(p, blockIdx.x == 0 && k < 4, 8200 + 10 * k + 6);
      // ---- a2: T2 = sum over taps of (window shifted by y*wc + x rows) . G[tap]
      // Operand descriptors advance by running offsets: next G chunk of the tap (+a_gs),
      // next tap column (+a_rs), next tap row (+(wc - kw) rows more).
      const uint32_t a_tap = a_rs - static_cast<uint32_t>(n_gk_ - 1) * a_gs;
      const uint32_t a_row = static_cast<uint32_t>(wc_ - kw_) * a_rs;
      const uint32_t a_b2 = 128u * a_rs;
      if (g_res_) {
        // resident G: one wait per chunk for the CTA's first tile, then one issue block
        if (k == 0)
          for (int j = 0; j < n_g; ++j) mbar_wait(&full_g[j], 0);
        tc_fence_after();
        {
          uint64_t bj = gd0;
          uint32_t aj = 0;  // window offset in 16-B units (uint32 wrap-around of the steps cancels)
          int gk = 0, tx = 0;
          for (int j = 0; j < n_g; ++j) {
            uint64_t ab = t1d0 + aj;
            uint32_t d = t2c;
            for (int b2 = 0; b2 < nb2_; ++b2, ab += a_b2, d += static_cast<uint32_t>(r2p_)) {
#pragma unroll
              for (int kk = 0; kk < GS; ++kk)
                mma_bf16(d, ab + kk * a_ks, bj + 2 * kk, idesc2, (j > 0 || kk > 0) ? 1u : 0u);
            }
            bj += g16;
            if (++gk == n_gk_) {
              gk = 0;
              aj += a_tap;
              if (++tx == kw_) {
                tx = 0;
                aj += a_row;
              }
            } else {
              aj += a_gs;
            }
          }
        }
      } else if (unified_) {
        // streamed G through the unified ring: gpk chunks per item, one commit per item
        const uint64_t gu0 = umma_desc(base, sw_g_);
        uint32_t aj = 0;
        int gk = 0, tx = 0;
        for (int j0 = 0; j0 < n_g; j0 += gpk_, ++ix) {
          const int s = ix % ns_x_;
          mbar_wait(&full_x[s], static_cast<uint32_t>((ix / ns_x_) & 1));
          tc_fence_after();
          const int cnt = min(gpk_, n_g - j0);
          for (int q = 0; q < cnt; ++q) {
            const int j = j0 + q;
            const uint64_t bj = gu0 + ((static_cast<uint32_t>(s) * x_slot_ + static_cast<uint32_t>(q) * g_slot_) >> 4);
            uint64_t ab = t1d0 + aj;
            uint32_t d = t2c;
            for (int b2 = 0; b2 < nb2_; ++b2, ab += a_b2, d += static_cast<uint32_t>(r2p_)) {
#pragma unroll
              for (int kk = 0; kk < GS; ++kk)
                mma_bf16(d, ab + kk * a_ks, bj + 2 * kk, idesc2, (j > 0 || kk > 0) ? 1u : 0u);
            }
            if (++gk == n_gk_) {
              gk = 0;
              aj += a_tap;
              if (++tx == kw_) {
                tx = 0;
                aj += a_row;
              }
            } else {
              aj += a_gs;
            }
          }
          mma_commit(&empty_x[s]);
        }
      } else {
        uint32_t aj = 0;
        int gk = 0, tx = 0;
        for (int j = 0; j < n_g; ++j, ++ig) {
          const int s = ig % ns_g_;
          mbar_wait(&full_g[s], static_cast<uint32_t>((ig / ns_g_) & 1));
          tc_fence_after();
          const uint64_t bj = gd0 + static_cast<uint32_t>(s) * g16;
          {
            uint64_t ab = t1d0 + aj;
            uint32_t d = t2c;
            for (int b2 = 0; b2 < nb2_; ++b2, ab += a_b2, d += static_cast<uint32_t>(r2p_)) {
#pragma unroll
              for (int kk = 0; kk < GS; ++kk)
                mma_bf16(d, ab + kk * a_ks, bj + 2 * kk, idesc2, (j > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&empty_g[s]);
          }
          if (++gk == n_gk_) {
            gk = 0;
            aj += a_tap;
            if (++tx == kw_) {
              tx = 0;
              aj += a_row;
            }
          } else {
            aj += a_gs;
          }
        }
      }
      {
        mma_commit(&t2_full[b]);
        mma_commit(t1w_empty);
      }
      CTRACE(p, blockIdx.x == 0 && k < 4, 8200 + 10 * k + 7);
    };
    if constexpr (CPDW) {
      for (int k = 0; k < m_tiles; ++k) phase_a1(k);
    } else if (nacc_ == 2) {
      // a1 of tile k+1 is issued before a2 of tile k (two TMEM buffers): the epilogue's T1
      // restage of tile k then overlaps the projection MMAs of tile k+1
      if (m_tiles > 0) phase_a1(0);
      for (int k = 0; k < m_tiles; ++k) {
        if (k + 1 < m_tiles) phase_a1(k + 1);
        phase_a2(k);
      }
    } else {
      for (int k = 0; k < m_tiles; ++k) {
        phase_a1(k);
        phase_a2(k);
      }
    }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    const int q4 = warp & 3;            // TMEM lane quarter
    const int ehalf = (warp - 2) >> 2;  // which 16-column half of every 32 columns
    const uint32_t t1w = smem_u32(smem + p.off_t1);
    const int m_tiles = static_cast<int>(blockIdx.x) < p.n_tiles
                            ? (p.n_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                            : 0;
    // restage T1 of tile k (TMEM buffer b(k)) into the window
    auto restage = [&](int k) {
      const int tile = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
      const int g = tile / p.bands, ho0 = (tile - g * p.bands) * p.th;
      const int rows = min(p.th, p.ho - ho0);
      const int b = p.nacc == 2 ? (k & 1) : 0;
      const int use = p.nacc == 2 ? (k >> 1) : k;
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * p.acc_cols + (static_cast<uint32_t>(q4 * 32) << 16);
      (void)g; (void)ho0; (void)rows; (void)use; (void)acc0;
      // ---- restage T1 (fp32 TMEM) as bf16 into the window (rows >= t1_rows are never read).
      // One thread polls (no sleep: this hand-off is on the tile's critical path), the other
      // epilogue threads block in a named barrier; TMEM loads are issued in groups of up
      // to four before one wait.
      if (threadIdx.x == 64) {
        mbar_wait(&t1_full[b], use & 1);
        if (!CPDW && k > 0) mbar_wait(t1w_empty, (k - 1) & 1);
      }
      named_bar_sync(1, kCThreads - 64);
      tc_fence_after();
      CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 4);
      for (int b1 = 0; b1 < p.nb1; ++b1) {
        const uint32_t row = static_cast<uint32_t>(b1 * 128 + q4 * 32 + lane);
        for (int cg = ehalf * 16; cg < p.r1p; cg += 128) {
          uint32_t v[4][16];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (cg + 32 * i < p.r1p) tmem_ld16_nowait(acc0 + static_cast<uint32_t>(b1 * p.r1p + cg + 32 * i), v[i]);
          tmem_ld_wait();
          if (row >= p.t1_rows || LRS_XDBG(p.dbg & 16)) continue;  // experiment: skip the restage stores
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (cg + 32 * i >= p.r1p) break;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint4 u;
              uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                w[e] = pack_bf16x2(__uint_as_float(v[i][8 * h + 2 * e]), __uint_as_float(v[i][8 * h + 2 * e + 1]));
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                               t1w + t1_piece(p, row, static_cast<uint32_t>(cg + 32 * i + 8 * h))),
                           "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                           : "memory");
            }
          }
        }
      }
      if constexpr (!CPDW) {  // the window is restaged: the MMA thread may run a2(k)
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(t1s_full);
        CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 5);
      }
    };
    // CP form: the two depthwise stages of tile k from the window, T2 to HBM
    auto depthwise = [&](int k) {
      const int tile = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
      const int g = tile / p.bands, ho0 = (tile - g * p.bands) * p.th;
      const int rows = min(p.th, p.ho - ho0);
      const int b = p.nacc == 2 ? (k & 1) : 0;
      const int use = p.nacc == 2 ? (k >> 1) : k;
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * p.acc_cols + (static_cast<uint32_t>(q4 * 32) << 16);
      (void)g; (void)ho0; (void)rows; (void)use; (void)acc0;
      {
        // TMEM buffer b is read: the MMA thread may start the tile after next
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
        named_bar_sync(1, kCThreads - 64);  // the whole window is restaged
        CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 5);
        // ---- depthwise stages: item = (output position of the tile, 8 ranks)
        const int nv = p.r1p / 8;
        const int items = LRS_XDBG(p.dbg & 1) ? 0 : p.ipt * rows * p.wo * nv;
        for (int it = threadIdx.x - 64; it < items; it += kCThreads - 64) {
          const int v = it % nv, q = it / nv;
          const int wl = q % p.wo, q2 = q / p.wo;
          const int hl = q2 % rows, img = q2 / rows;
          const int n = g * p.ipt + img;
          if (n >= p.n) continue;
          const int a0 = 8 * v;
          float out[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) out[e] = 0.f;
          for (int x = 0; x < p.kw; ++x) {
            float yb[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) yb[e] = 0.f;
            for (int y = 0; y < p.kh; ++y) {
              const uint32_t row = static_cast<uint32_t>(img * p.p1 + (hl + y) * p.wc + wl + x);
              const uint4 tv = lds_v4(t1w + t1_piece(p, row, static_cast<uint32_t>(a0)));
              const uint32_t tw[4] = {tv.x, tv.y, tv.z, tv.w};
              const float* bt = p.cpb + y * p.r1p + a0;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                yb[2 * e] = fmaf(__ldg(bt + 2 * e), __uint_as_float(tw[e] << 16), yb[2 * e]);
                yb[2 * e + 1] = fmaf(__ldg(bt + 2 * e + 1), __uint_as_float(tw[e] & 0xFFFF0000u), yb[2 * e + 1]);
              }
            }
            const float* ct = p.cpc + x * p.r1p + a0;
#pragma unroll
            for (int e = 0; e < 8; ++e) out[e] = fmaf(__ldg(ct + e), yb[e], out[e]);
          }
          uint4 o;
          o.x = pack_bf16x2(out[0], out[1]);
          o.y = pack_bf16x2(out[2], out[3]);
          o.z = pack_bf16x2(out[4], out[5]);
          o.w = pack_bf16x2(out[6], out[7]);
          if (!LRS_XDBG(p.dbg & 2))
            *reinterpret_cast<uint4*>(p.t2 + ((static_cast<long long>(n) * p.ho + ho0 + hl) * p.wo + wl) * p.r2p + a0) = o;
        }
        named_bar_sync(1, kCThreads - 64);  // the window may be overwritten by the next restage
        CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 9);
      }
    };
    // T2 of tile k: hand the window back to the MMA thread, then TMEM -> HBM
    auto t2_store = [&](int k) {
      const int tile = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
      const int g = tile / p.bands, ho0 = (tile - g * p.bands) * p.th;
      const int rows = min(p.th, p.ho - ho0);
      const int b = p.nacc == 2 ? (k & 1) : 0;
      const int use = p.nacc == 2 ? (k >> 1) : k;
      const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * p.acc_cols + (static_cast<uint32_t>(q4 * 32) << 16);
      (void)g; (void)ho0; (void)rows; (void)use; (void)acc0;
      // ---- T2 (fp32 TMEM) -> bf16 rows of global T2
      if (threadIdx.x == 64) mbar_wait(&t2_full[b], use & 1);
      named_bar_sync(1, kCThreads - 64);
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
        for (int cg = ehalf * 16; cg < p.r2p; cg += 128) {
          uint32_t v[4][16];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (cg + 32 * i < p.r2p) tmem_ld16_nowait(acc0 + static_cast<uint32_t>(b2 * p.r2p + cg + 32 * i), v[i]);
          tmem_ld_wait();
          if (!ok || LRS_XDBG(p.dbg & 8)) continue;  // experiment: skip the T2 stores (wrong T2)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (cg + 32 * i >= p.r2p) break;
            uint4 u[2];
            uint32_t* w = reinterpret_cast<uint32_t*>(u);
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = pack_bf16x2(__uint_as_float(v[i][2 * e]), __uint_as_float(v[i][2 * e + 1]));
            reinterpret_cast<uint4*>(dst + cg + 32 * i)[0] = u[0];
            reinterpret_cast<uint4*>(dst + cg + 32 * i)[1] = u[1];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      CTRACE(p, blockIdx.x == 0 && threadIdx.x == 64 && k < 4, 8200 + 10 * k + 9);
    };
    if constexpr (CPDW) {
      for (int k = 0; k < m_tiles; ++k) {
        restage(k);
        depthwise(k);
      }
    } else if (p.nacc == 2) {
      // matches the MMA order a1(k+1) before a2(k): restage k+1 as soon as a2(k) has read
      // the window, then store T2(k) while the MMA thread runs a2(k+1)
      if (m_tiles > 0) restage(0);
      for (int k = 0; k < m_tiles; ++k) {
        if (k + 1 < m_tiles) restage(k + 1);
        t2_store(k);
      }
    } else {
      for (int k = 0; k < m_tiles; ++k) {
        restage(k);
        t2_store(k);
      }
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
  if (p.early) pdl_wait();
}

}  // namespace lrs
