// lrs_wconv.cuh -- the fused a3 + a4 + a5 kernel on the sm_100a tensor cores:
//
//   Y[n, ho, wo, j] = sum_b T2[n, ho, wo, b] U_out[b, j]                          (a3)
//                   + sum_{c, y, x} S[j, c, y, x] X[n, ho*s + y - p, wo*s + x - p, c]  (a4)
//
// computed transposed, D[j, (ho, wo, n)] in TMEM (M = 128 output channels per
// tile, TMEM lane = channel), and written to Y once (a5).
//
// * The sparse term S runs on the 2:4 sparse tensor-core MMA
//   (tcgen05.mma.sp, kind::f16): at create time every group of 4 consecutive
//   input channels of a (row j, tap) is split into a "main" 2:4 block (its
//   first two nonzeros) and, only where a group holds 3-4 nonzeros, a
//   "residual" 2:4 block; both are exact, so S = S_main + S_res bit for bit.
// * The activation operand B is a shared-memory WINDOW of X per 64-channel
//   chunk, loaded by one TMA box {64 ch, 8 images, window cols, window rows}
//   straight from NHWC X (out-of-bounds = zero padding).  Its 8-row core
//   matrices are the 8 images of one spatial position, so the im2col operand
//   of every kernel tap (y, x) is the same window at a different start
//   address -- the window is loaded once and reused by all k*k taps.
//   Stride s is the descriptor's SBO (s KB between output positions).
// * The dense part (a3) uses the same machinery with a window of T2 (or T1
//   for the SVD pair) at the output positions and U_out^T as A.
//
// Tile: 8 images x th output rows x tcols output columns x 128 channels.
// The tile's outputs are covered by up to kWMaxUnits MMA "units", each one
// N range (<= 256 columns = 8 images x <= 32 positions) with its accumulator
// side by side in TMEM.  At stride 1 a unit spans several output rows: its
// positions run along the window rows with the window width as pitch, so one
// MMA covers rows * window_width positions (the window's padding columns are
// computed and discarded) -- few, wide MMAs, because every MMA re-reads its A
// block from shared memory and has a fixed issue cost.  At stride 2 a unit
// is (part of) one output row.
//
// Persistent: gridDim.x <= #SMs CTAs walk the tiles; the producer and the MMA
// issuer stream windows/items across tile boundaries, and when two tiles'
// accumulators fit in TMEM the epilogue of tile k overlaps the MMAs of k+1.
//
// Warps: 0 = TMA producer, 1 = TMEM allocator + MMA issuer, 2..9 = epilogue
// (warp w drains TMEM lanes 32*(w%4) .., the two warps of a quarter split the
// columns; each transposes 32 columns x 32 channels through a private 2 KB
// shared-memory tile so every lane stores 16 contiguous bytes of Y).
#pragma once
#include "lrs_ptx.cuh"

// Debug experiments (LRS_WCONV_DEBUG builds only): timeline stamps into
// p.trace and the p.dbg bits that skip parts of the pipeline; compiled out of
// production builds so the issue loops carry no extra branches.
#ifdef LRS_WCONV_DEBUG
#define WDBG(p, bits) ((p).dbg & (bits))
#define WTRACE(p) ((p).trace != nullptr)
#else
#define WDBG(p, bits) 0
#define WTRACE(p) false
#endif

namespace lrs {


constexpr int kWThreads = 320;  // warps 0 producer, 1 MMA, 2..9 epilogue (2 per TMEM lane quarter)
constexpr int kWMaxSlots = 6;
constexpr int kWMaxWin = 8;  // window buffers in the ring
constexpr int kWMaxUnits = 8;
constexpr int kWMaxBpi = 4;              // sparse blocks per pipeline item
constexpr uint32_t kSpBlockBytes = 8192;  // one compressed 2:4 block: 128 rows x 64 B
constexpr uint32_t kEBlockBytes = 2048;   // its metadata: 128 lanes x 16 B
constexpr uint32_t kEpiScratch = 2048;   // per epilogue warp: 32 columns x 32 channels bf16

struct WconvParams {
  CUtensorMap tmX;   // X   4-D (C, N, W, H) bf16, box {64, ipw, wc, wr}, SW128
  CUtensorMap tmT;   // T   4-D (R, N, Wo, Ho) bf16, box {t_kc, ipw, tbox_w, th}, swizzle sw_t
  // A operands as ready-made shared-memory images (host-swizzled), fetched with one
  // 1-D bulk copy each: a 2-D TMA box of 128 short rows costs 128 TMA requests and
  // the TMA request rate measured as the producer's bottleneck (tools/wtrace.py)
  const uint8_t* img_sp;     // compressed 2:4 blocks, SW64 image, 8 KB each
  const uint8_t* img_e;      // their metadata, [128 lanes][16 B], 2 KB each
  const uint8_t* img_dense;  // U_out^T (or V^T) blocks [n_mt][n_tk], 128 rows x sw_t B, swizzle sw_t
  // 2:4 blocks are stored in STREAM order -- per (M-tile, chunk): for each tap its main block,
  // then its residual block if it has one -- so every item (bpi consecutive blocks of a
  // window) is ONE bulk copy of A and one of E (2 requests instead of 2 per block)
  const int* stream_off;     // [n_mt * n_ck + 1] first block of each (M-tile, chunk)
  const uint32_t* blk_tap;   // [blocks] tap offset of each block: window position * 1024 >> 4
  void* y;
  int n, ho, wo, cout;
  int kh, kw, sh, sw, ph, pw;
  int ipw;                 // images per window (8, or 4 at stride 1): window rows = (position, image)
  int th, bands, n_mt;
  int tcols, cbands;       // output columns per tile, column bands
  int n_tiles;             // groups * bands * cbands * n_mt (for this forward's n)
  int n_units;
  int u_col[kWMaxUnits];   // first TMEM column (within one accumulator buffer)
  int u_n[kWMaxUnits];     // MMA N (multiple of 16)
  int u_xpos[kWMaxUnits];  // X window position of the unit's first output at tap (0, 0)
  int u_tpos[kWMaxUnits];  // T window position of the unit's first output
  int u_r0[kWMaxUnits];    // first output row (tile-relative)
  int u_wo0[kWMaxUnits];   // first output column (tile-relative)
  int u_pitch[kWMaxUnits]; // columns/8 per output row inside the unit
  int u_nw[kWMaxUnits];    // real output columns per row
  int u_rows[kWMaxUnits];  // output rows covered
  int u_q0[kWMaxUnits];    // first virtual position of the unit (pitch-major: row = q / pitch)
  int tbox_w;              // width of the T window box (its row pitch)
  unsigned long long* trace;  // optional: globaltimer stamps (debug, lrs_conv_debug_trace)
  int dbg;                 // debug experiment bits (0 in production)
  int n_ck, n_tk, t_kc;
  int cpw, n_xw;        // 64-channel chunks per X window (boxes x_win_bytes apart), X windows per tile
  uint32_t sw_t;        // bytes per T window row (t_kc * 2) = its swizzle width
  int wr, wc;
  uint32_t x_win_bytes, t_win_bytes, win_stride;
  int ns;
  int bpi;              // sparse blocks per item (2..kWMaxBpi); A slot = bpi * 8 KB, E slot = bpi * 2 KB
  uint32_t a_slot, e_slot;
  int nwb;              // window buffers (2..kWMaxWin)
  int nacc;             // accumulator buffers in TMEM (1 or 2)
  uint32_t acc_cols;    // TMEM columns of one accumulator buffer
  uint32_t e_col0, tmem_cols;
  int e_slots;             // TMEM metadata slots (<= ns): tcgen05.cp and tcgen05.mma of one thread run in
                           // issue order, so an item's metadata may overwrite that of an item issued before
  uint32_t off_a, off_e, off_epi, off_res, off_bar;
  const float2* epi;    // per output channel (scale, bias) of the fused output epilogue, or NULL
  int relu;
  // overflow gather (n_gk > 0): the entries a 2:4 main block cannot hold (3rd/4th nonzero of a
  // group of 4) are NOT given residual 2:4 blocks -- one per (chunk, tap) with any overflow,
  // each a full MMA pass for ~1 entry -- but become n_gk extra dense K chunks of the tile:
  // G[pos][slot] = X[pos shifted by tap_s][c_s] for the M-tile's distinct (c, tap) slots,
  // gathered by the epilogue warps (idle during the MMAs) into global scratch, TMA-loaded
  // back like a T window, multiplied by the slots' values (img_dense blocks n_tk..)
  CUtensorMap tmG;      // G 4-D (n_mt * gs, N, Wo, Ho) bf16, box {t_kc, ipw, tbox_w, th}, swizzle sw_t
  int n_gk;             // G chunks per M-tile (gs = n_gk * t_kc slots), 0: residual blocks
  int g_ch;             // channels per position of G (n_mt * gs)
  const int* g_tab;     // [n_mt][gs] slot -> c | dy << 16 | dx << 24 (dy, dx = tap), -1 = empty slot
  __nv_bfloat16* g;     // G scratch [N][Ho][Wo][g_ch] (empty slots zeroed once at create)
  const __nv_bfloat16* x;  // this forward's X (the gather reads it)
  int in_h, in_w, c_in;
  // CTA pair (lrs_wconv_kernel<.., PAIR = true>, launched as clusters of 2): the pair's two
  // CTAs own M-tiles 2i and 2i + 1 of the same positions; rank 0 issues cta_group::2 MMAs
  // (M = 256) for both, B split along N (every unit has the same N, a multiple of 16), so
  // rank 1 keeps each window shifted by N/2 rows: shift_x (X windows, 128 B rows) and
  // shift_t (T / G windows, sw_t rows) bytes before its buffer (win_margin bytes reserved)
  int pair;
  uint32_t win_margin, shift_x, shift_t;
  // window order of a tile: -1 = all X windows, then the dense (T, G) ones; >= 0 = that many
  // X windows first, then X and dense windows alternate, so each dense window's load hides
  // behind an X window's k*k taps of MMAs instead of queueing behind another short window
  int ilv;
};

// window p of a tile -> its dense chunk (>= 0: T chunks, then G chunks), or -(1 + its X
// window index)
__device__ __forceinline__ int win_map(int p, int n_xw, int ilv) {
  if (ilv < 0) return p >= n_xw ? p - n_xw : -(1 + p);
  if (p < ilv) return -(1 + p);
  const int q = p - ilv;
  return (q & 1) ? (q >> 1) : -(1 + ilv + (q >> 1));
}

struct TileCoord {
  int mt, n0, ho0, wo0, j0;
};
__device__ __forceinline__ TileCoord tile_coord(const WconvParams& p, int tile) {
  TileCoord c;
  c.mt = tile % p.n_mt;
  tile /= p.n_mt;
  const int cband = tile % p.cbands;
  tile /= p.cbands;
  const int band = tile % p.bands;
  const int grp = tile / p.bands;
  c.n0 = grp * p.ipw;
  c.ho0 = band * p.th;
  c.wo0 = cband * p.tcols;
  c.j0 = c.mt * 128;
  return c;
}

__device__ __forceinline__ TileCoord tile_coord_v(int tile, int n_mt, int cbands, int bands, int th, int tcols,
                                                  int ipw) {
  TileCoord c;
  c.mt = tile % n_mt;
  tile /= n_mt;
  const int cband = tile % cbands;
  tile /= cbands;
  const int band = tile % bands;
  const int grp = tile / bands;
  c.n0 = grp * ipw;
  c.ho0 = band * th;
  c.wo0 = cband * tcols;
  c.j0 = c.mt * 128;
  return c;
}

// G rows of one tile: for each valid output position (image, ho, wo) of the tile and each
// slot s of its M-tile, G[pos][mt * gs + s] = X[n][ho*sh - ph + dy_s][wo*sw - pw + dx_s][c_s]
// (0 outside the image).  Empty slots are never written (zeroed at create).
__device__ __forceinline__ void gather_tile(const WconvParams& p, const TileCoord& tc, int we, int lane) {
  const int gs = p.n_gk * p.t_kc;
  const int gi = p.pair ? (tc.mt >> 1) : tc.mt;  // slot set: the M-tile's, or the pair's union
  int tab[8];  // the lane's slots lane, lane + 32, .. (gs <= 256)
#pragma unroll
  for (int i = 0; i < 8; ++i) tab[i] = (lane + 32 * i < gs) ? __ldg(p.g_tab + gi * gs + lane + 32 * i) : -1;
  const int npos = p.th * p.tcols * p.ipw;
  const __nv_bfloat16* __restrict__ x = p.x;
  __nv_bfloat16* __restrict__ g = p.g + gi * gs;
  for (int pi = we; pi < npos; pi += 8) {
    const int img = pi % p.ipw, q = pi / p.ipw;
    const int r = q / p.tcols, c = q - r * p.tcols;
    const int n = tc.n0 + img, ho = tc.ho0 + r, wo = tc.wo0 + c;
    if (n >= p.n || ho >= p.ho || wo >= p.wo) continue;
    const long long xrow = static_cast<long long>(n) * p.in_h;
    __nv_bfloat16* grow = g + ((static_cast<long long>(n) * p.ho + ho) * p.wo + wo) * p.g_ch;
    __nv_bfloat16 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = __float2bfloat16_rn(0.f);
      if (tab[i] >= 0) {
        const int hi = ho * p.sh - p.ph + ((tab[i] >> 16) & 0xFF), wi = wo * p.sw - p.pw + (tab[i] >> 24);
        if (hi >= 0 && hi < p.in_h && wi >= 0 && wi < p.in_w)
          v[i] = x[((xrow + hi) * p.in_w + wi) * p.c_in + (tab[i] & 0xFFFF)];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (tab[i] >= 0) grow[lane + 32 * i] = v[i];
  }
}

// NU = the layer's exact unit count (1..kWMaxUnits): the MMA issue loops are fully
// unrolled without predicates -- a generic 8-unit loop measured 17-39 % slower
// (instruction fetch of the issuing warp dominates small MMAs).
template <int NU, int BPI, bool PAIR>
__global__ void __launch_bounds__(kWThreads, 1) lrs_wconv_kernel(const __grid_constant__ WconvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* win_full = bars;
  uint64_t* win_empty = bars + kWMaxWin;
  uint64_t* a_full = bars + 2 * kWMaxWin;
  uint64_t* a_empty = a_full + kWMaxSlots;
  uint64_t* acc_full = a_empty + kWMaxSlots;  // [2]
  uint64_t* acc_empty = acc_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const uint32_t slot_info = smem_u32(tmem_slot + 4);  // [kWMaxSlots][kWMaxBpi] u32, written by the producer
  uint64_t* g_ready = bars + 48;  // byte 384: the tile's G chunks are in global memory (8 epilogue warps)
  // pair: rank 0 = MMA issuer for both CTAs; its full barriers also count the peer's relay
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool lead = !PAIR || rank == 0;
  // work units: tiles, or (pair) tile pairs -- M-tiles 2i, 2i + 1 of the same positions
  const int g_id = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int g_n = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);

  if (WTRACE(p) && threadIdx.x == 0 && blockIdx.x < 2048) p.trace[2000 + 3 * blockIdx.x] = gtimer();
  const int nwin = p.n_tk + p.n_gk + p.n_xw;
  // the role loops' scalars, staged in shared memory: a kernel parameter read inside a
  // loop is re-loaded from the constant bank at every use (~100 cycles each on the issue
  // path, tools/loop_cost2.cu); a value loaded from shared memory stays in a register
  int* prm = reinterpret_cast<int*>(smem + p.off_bar + 512);

  if (threadIdx.x == 0) {
    prm[0] = static_cast<int>(p.nwb);
    prm[1] = static_cast<int>(p.n_tiles);
    prm[2] = static_cast<int>(p.n_mt);
    prm[3] = static_cast<int>(p.n_ck);
    prm[4] = static_cast<int>(p.n_xw);
    prm[5] = static_cast<int>(p.n_tk);
    prm[6] = static_cast<int>(p.ns);
    prm[7] = static_cast<int>(p.bpi);
    prm[8] = static_cast<int>(p.cpw);
    prm[9] = static_cast<int>(p.t_kc);
    prm[10] = static_cast<int>(p.x_win_bytes);
    prm[11] = static_cast<int>(p.t_win_bytes);
    prm[12] = static_cast<int>(p.win_stride);
    prm[13] = static_cast<int>(p.a_slot);
    prm[14] = static_cast<int>(p.e_slot);
    prm[15] = static_cast<int>(p.sw);
    prm[16] = static_cast<int>(p.pw);
    prm[17] = static_cast<int>(p.sh);
    prm[18] = static_cast<int>(p.ph);
    prm[19] = static_cast<int>(p.sw_t);
    prm[20] = static_cast<int>(p.e_col0);
    prm[21] = static_cast<int>(p.e_slots);
    prm[22] = static_cast<int>(p.nacc);
    prm[23] = static_cast<int>(p.acc_cols);
    prm[24] = static_cast<int>(p.cbands);
    prm[25] = static_cast<int>(p.bands);
    prm[26] = static_cast<int>(p.th);
    prm[27] = static_cast<int>(p.tcols);
    prm[28] = static_cast<int>(p.off_a);
    prm[29] = static_cast<int>(p.off_e);
    prm[30] = static_cast<int>(p.off_res);
    prm[31] = p.ipw;
    prm[32] = p.n_gk;
    prm[33] = static_cast<int>(p.win_margin);
    prm[34] = static_cast<int>(p.shift_x);
    prm[35] = static_cast<int>(p.shift_t);
    prm[36] = p.ilv;
    const uint32_t nf = (PAIR && rank == 0) ? 2u : 1u;  // + the peer relay's arrival
    for (int i = 0; i < p.nwb; ++i) {
      mbar_init(&win_full[i], nf);
      mbar_init(&win_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8 * nf);  // one arrival per epilogue warp (of both CTAs)
    }
    for (int i = 0; i < p.ns; ++i) {
      mbar_init(&a_full[i], nf);
      mbar_init(&a_empty[i], 1);
    }
    mbar_init(g_ready, 8);
    fence_mbar_init();
    tma_prefetch_desc(&p.tmX);
    tma_prefetch_desc(&p.tmT);
    if (p.n_gk > 0) tma_prefetch_desc(&p.tmG);
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc2(tmem_slot, p.tmem_cols);
    else tmem_alloc(tmem_slot, p.tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  // The CTA owns the whole TMEM of its SM (tmem_cols = 512, one CTA per SM), so
  // the allocation starts at lane 0 / column 0.  Using the literal 0 keeps every
  // TMEM address compile-time uniform (uniform registers in the MMA loop).
  if (threadIdx.x == 32 && *tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0u;
  // PDL: every kernel of this library triggers its dependents only after its own
  // griddepcontrol.wait, so when this grid starts everything before the previous kernel
  // is complete: X, the weights and Y may be touched at once.  Only T2 (T1 for the SVD
  // pair) comes from the previous kernel -- each tile runs its sparse windows first and
  // the producer waits just before the first T window, overlapping the previous kernel.

  if (warp == 0) {
    const int ipw_ = smem_param(prm + 31);
    const int nwb_ = static_cast<int>(smem_param(prm + 0));
    const int n_tiles_ = static_cast<int>(smem_param(prm + 1));
    const int n_mt_ = static_cast<int>(smem_param(prm + 2));
    const int n_ck_ = static_cast<int>(smem_param(prm + 3));
    const int n_xw_ = static_cast<int>(smem_param(prm + 4));
    const int n_tk_ = static_cast<int>(smem_param(prm + 5));
    const int ns_ = static_cast<int>(smem_param(prm + 6));
    const int bpi_ = static_cast<int>(smem_param(prm + 7));
    const int cpw_ = static_cast<int>(smem_param(prm + 8));
    const int t_kc_ = static_cast<int>(smem_param(prm + 9));
    const uint32_t x_win_bytes_ = static_cast<uint32_t>(smem_param(prm + 10));
    const uint32_t t_win_bytes_ = static_cast<uint32_t>(smem_param(prm + 11));
    const uint32_t win_stride_ = static_cast<uint32_t>(smem_param(prm + 12));
    const uint32_t a_slot_ = static_cast<uint32_t>(smem_param(prm + 13));
    const uint32_t e_slot_ = static_cast<uint32_t>(smem_param(prm + 14));
    const int sw_ = static_cast<int>(smem_param(prm + 15));
    const int pw_ = static_cast<int>(smem_param(prm + 16));
    const int sh_ = static_cast<int>(smem_param(prm + 17));
    const int ph_ = static_cast<int>(smem_param(prm + 18));
    const uint32_t sw_t_ = static_cast<uint32_t>(smem_param(prm + 19));
    const uint32_t off_a_ = static_cast<uint32_t>(smem_param(prm + 28));
    const uint32_t off_e_ = static_cast<uint32_t>(smem_param(prm + 29));
    const uint32_t off_res_ = static_cast<uint32_t>(smem_param(prm + 30));
    const int cbands_ = static_cast<int>(smem_param(prm + 24));
    const int bands_ = static_cast<int>(smem_param(prm + 25));
    const int th_ = static_cast<int>(smem_param(prm + 26));
    const int tcols_ = static_cast<int>(smem_param(prm + 27));
    const int n_gk_ = smem_param(prm + 32);
    const int n_dk_ = n_tk_ + n_gk_;  // dense chunks per M-tile (T, then G)
    const int ilv_ = smem_param(prm + 36);
    const uint32_t win_margin_ = static_cast<uint32_t>(smem_param(prm + 33));
    const uint32_t shift_x_ = rank ? static_cast<uint32_t>(smem_param(prm + 34)) : 0u;
    const uint32_t shift_t_ = rank ? static_cast<uint32_t>(smem_param(prm + 35)) : 0u;
    // the M-tile's block stream (chunk starts + per-block tap offsets), staged in shared
    // memory: a global load on the issue path measured ~250 ns each (tools/wtrace.py)
    int* so_s = reinterpret_cast<int*>(smem + off_res_);   // [n_ck + 1], relative to mt0
    uint32_t* tap_s = reinterpret_cast<uint32_t*>(so_s + n_ck_ + 1);
    // CTAs own contiguous tile ranges, M-tile fastest: consecutive tiles of a CTA share
    // their windows; with one ring buffer per window (nwb == nwin) a window still resident
    // from the previous tile is reused instead of re-loaded
    const bool contig = nwb_ == nwin;
    const int n_u = PAIR ? n_tiles_ >> 1 : n_tiles_;
    const int t_begin = contig ? static_cast<int>(static_cast<long long>(g_id) * n_u / g_n) : g_id;
    const int t_end = contig ? static_cast<int>(static_cast<long long>(g_id + 1) * n_u / g_n) : n_u;
    const int t_step = contig ? 1 : g_n;
    auto tile_of = [&](int tu) {
      const int hm = n_mt_ >> 1;
      return PAIR ? (tu / hm) * n_mt_ + 2 * (tu % hm) + static_cast<int>(rank) : tu;
    };
    // CTA start: the first window's TMA goes out at once (it needs no table), and the whole
    // warp stages the first M-tile's block stream -- one thread's ~80 loads had delayed the
    // first window by ~2 us (profiles/r02_wtrace_c3_early.log: issued at 3.3 us)
    int first_mt = -1, first_mt0 = 0;
    bool first_issued = false;
    if (t_begin < t_end) {
      const TileCoord tc0 = tile_coord_v(tile_of(t_begin), n_mt_, cbands_, bands_, th_, tcols_, ipw_);
      if (lane == 0 && n_xw_ > 0 && !WDBG(p, 64)) {
        mbar_arrive_expect_tx(&win_full[0], static_cast<uint32_t>(cpw_) * x_win_bytes_);
        for (int q = 0; q < cpw_; ++q)
          tma_load_4d(smem + win_margin_ - shift_x_ + q * x_win_bytes_, &p.tmX, &win_full[0], q * 64, tc0.n0,
                      tc0.wo0 * sw_ - pw_, tc0.ho0 * sh_ - ph_);
        first_issued = true;
      }
      first_mt = tc0.mt;
      first_mt0 = __ldg(p.stream_off + first_mt * n_ck_);
      for (int i = lane; i <= n_ck_; i += 32) so_s[i] = __ldg(p.stream_off + first_mt * n_ck_ + i) - first_mt0;
      __syncwarp();
      const int len = so_s[n_ck_];
      for (int i = lane; i < len; i += 32) tap_s[i] = __ldg(p.blk_tap + first_mt0 + i);
      __syncwarp();
    }
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int it = 0, wg = 0, buf = 0;
      uint32_t wph = 0, gph = 0;
      int cur_mt = first_mt, mt0 = first_mt0;
      bool waited = false;
      int prev_win = -1;
      for (int tu = t_begin; tu < t_end; tu += t_step) {
        const int tile = tile_of(tu);
        const TileCoord tc = tile_coord_v(tile, n_mt_, cbands_, bands_, th_, tcols_, ipw_);
        const int win_key = tile / n_mt_;
        const bool reuse = nwb_ == nwin && win_key == prev_win;
        prev_win = win_key;
        if (tc.mt != cur_mt) {
          mt0 = __ldg(p.stream_off + tc.mt * n_ck_);
          for (int i = 0; i <= n_ck_; ++i) so_s[i] = __ldg(p.stream_off + tc.mt * n_ck_ + i) - mt0;
          const int len = so_s[n_ck_];
          for (int i = 0; i < len; ++i) tap_s[i] = __ldg(p.blk_tap + mt0 + i);
          cur_mt = tc.mt;
        }
        for (int w = 0; w < nwin; ++w, ++wg) {
          if (wg >= nwb_) mbar_wait(&win_empty[buf], wph ^ 1u);
          const int tk = win_map(w, n_xw_, ilv_);  // >= 0: dense (T, then G) chunk; < 0: X window
          // (pair, rank 1: the window sits N/2 B rows earlier, so the leader's descriptors,
          // which address both CTAs at the same offset, see the unit's second half here)
          uint8_t* wdst = smem + win_margin_ + buf * win_stride_ - (tk >= 0 ? shift_t_ : shift_x_);
          if (WTRACE(p) && blockIdx.x == 0 && wg < 16) p.trace[3600 + wg] = gtimer();
          if (tk >= 0 && !waited) {
            pdl_wait();
            pdl_launch_dependents();
            waited = true;
          }
          if (tk == n_tk_) {  // first G chunk: wait until the epilogue warps gathered this tile
            mbar_wait(g_ready, gph);
            gph ^= 1u;
          }
          if (WDBG(p, 64) || (reuse && tk < n_tk_)) {  // G windows differ per M-tile: never reused
            mbar_arrive(&win_full[buf]);  // window already resident (or timing experiment)
          } else if (tk >= n_tk_) {
            mbar_arrive_expect_tx(&win_full[buf], t_win_bytes_);
            tma_load_4d(wdst, &p.tmG, &win_full[buf], (PAIR ? tc.mt >> 1 : tc.mt) * n_gk_ * t_kc_ + (tk - n_tk_) * t_kc_,
                        tc.n0, tc.wo0, tc.ho0);
          } else if (tk >= 0) {
            mbar_arrive_expect_tx(&win_full[buf], t_win_bytes_);
            tma_load_4d(wdst, &p.tmT, &win_full[buf], tk * t_kc_, tc.n0, tc.wo0, tc.ho0);
          }
          if (tk >= 0) {
            const int slot = it % ns_;
            if (it >= ns_) mbar_wait(&a_empty[slot], ((it / ns_) - 1) & 1);
            mbar_arrive_expect_tx(&a_full[slot], 128u * sw_t_);
            bulk_load(smem + off_a_ + slot * a_slot_,
                      p.img_dense + (static_cast<size_t>(tc.mt) * n_dk_ + tk) * (128u * sw_t_), 128u * sw_t_,
                      &a_full[slot]);
            ++it;
          } else {
            const int c = (-tk - 1) * cpw_;  // first chunk of this X window
            if (!(WDBG(p, 64)) && !reuse && !(first_issued && wg == 0)) {
              mbar_arrive_expect_tx(&win_full[buf], static_cast<uint32_t>(cpw_) * x_win_bytes_);
              for (int q = 0; q < cpw_; ++q)
                tma_load_4d(wdst + q * x_win_bytes_, &p.tmX, &win_full[buf], (c + q) * 64, tc.n0,
                            tc.wo0 * sw_ - pw_, tc.ho0 * sh_ - ph_);
            }
            // this window's blocks in stream order, bpi per item: every item costs an
            // mbarrier hand-off and a tcgen05.commit (~450 cycles, tools/mma_rate2.cu), so
            // items are as large as smem allows; each is one bulk copy of A and one of E
            const int sb = so_s[c], se = so_s[c + cpw_];
            for (int b = sb; b < se; b += bpi_) {
              const int np = min(bpi_, se - b);
              const bool last = b + np >= se;
              const int slot = it % ns_;
              if (WTRACE(p) && blockIdx.x == 0 && it < 64) p.trace[3000 + 3 * it] = gtimer();
              if (it >= ns_) mbar_wait(&a_empty[slot], ((it / ns_) - 1) & 1);
              if (WTRACE(p) && blockIdx.x == 0 && it < 64) p.trace[3000 + 3 * it + 1] = gtimer();
#pragma unroll
              for (int q = 0; q < kWMaxBpi; ++q)
                if (q < np)
                  st_shared_u32(slot_info + 4u * (kWMaxBpi * slot + q),
                                tap_s[b + q] | (q == 0 ? (static_cast<uint32_t>(np) << 28) | (last ? 0x80000000u : 0u)
                                                       : 0u));
              if (WDBG(p, 2)) {
                mbar_arrive(&a_full[slot]);
              } else {
                mbar_arrive_expect_tx(&a_full[slot], static_cast<uint32_t>(np) * (kSpBlockBytes + kEBlockBytes));
                bulk_load(smem + off_a_ + slot * a_slot_, p.img_sp + static_cast<size_t>(mt0 + b) * kSpBlockBytes,
                          static_cast<uint32_t>(np) * kSpBlockBytes, &a_full[slot]);
                bulk_load(smem + off_e_ + slot * e_slot_, p.img_e + static_cast<size_t>(mt0 + b) * kEBlockBytes,
                          static_cast<uint32_t>(np) * kEBlockBytes, &a_full[slot]);
              }
              if (WTRACE(p) && blockIdx.x == 0 && it < 64) p.trace[3000 + 3 * it + 2] = gtimer();
              ++it;
            }
          }
          if (++buf == nwb_) { buf = 0; wph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    const int ipw_ = smem_param(prm + 31);
    const int nwb_ = static_cast<int>(smem_param(prm + 0));
    const int n_tiles_ = static_cast<int>(smem_param(prm + 1));
    const int n_xw_ = static_cast<int>(smem_param(prm + 4));
    const int ns_ = static_cast<int>(smem_param(prm + 6));
    const int bpi_ = static_cast<int>(smem_param(prm + 7));
    const uint32_t win_stride_ = static_cast<uint32_t>(smem_param(prm + 12));
    const uint32_t a_slot_ = static_cast<uint32_t>(smem_param(prm + 13));
    const uint32_t e_slot_ = static_cast<uint32_t>(smem_param(prm + 14));
    const int sw_ = static_cast<int>(smem_param(prm + 15));
    const uint32_t sw_t_ = static_cast<uint32_t>(smem_param(prm + 19));
    const uint32_t e_col0_ = static_cast<uint32_t>(smem_param(prm + 20));
    const int e_slots_ = static_cast<int>(smem_param(prm + 21));
    const int nacc_ = static_cast<int>(smem_param(prm + 22));
    const uint32_t acc_cols_ = static_cast<uint32_t>(smem_param(prm + 23));
    const uint32_t off_a_ = static_cast<uint32_t>(smem_param(prm + 28));
    const uint32_t off_e_ = static_cast<uint32_t>(smem_param(prm + 29));
    const int n_mt_ = static_cast<int>(smem_param(prm + 2));
    const int cbands_ = static_cast<int>(smem_param(prm + 24));
    const int bands_ = static_cast<int>(smem_param(prm + 25));
    const int th_ = static_cast<int>(smem_param(prm + 26));
    const int tcols_ = static_cast<int>(smem_param(prm + 27));
    // -------------------------------------------------------------- MMA issuer
    // ONE elected thread runs the whole loop, its mbarrier waits included: an elect +
    // warp reconvergence around every item cost ~240 cycles of issue each
    // (tools/mma_seq.cu: 108 vs 48 cycles per N = 64 MMA), more than the MMAs it feeds.
    // Descriptors are linear in the start address (14-bit field of addr>>4),
    // so every per-unit descriptor is precomputed once and the inner loop
    // only adds byte offsets >> 4: the single-thread issue loop stays short.
    const uint32_t win0 = smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 33));  // + window margin
    const uint32_t t_pos = static_cast<uint32_t>(ipw_) * sw_t_;  // bytes per position in a T window
    const uint32_t x_pos = 128u * static_cast<uint32_t>(ipw_);     // bytes per position in an X window
    // stride between 8-row core-matrix groups: one position (x stride) of 8 images, or two
    // consecutive positions of 4 images (stride 1 only)
    const uint32_t x_sbo = ipw_ == 8 ? 1024u * static_cast<uint32_t>(sw_) : 1024u;
    const uint32_t t_sbo = 8u * sw_t_;
    uint32_t dcol[NU], idu[NU];
    uint64_t bxd[NU], btd[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      {
        dcol[u] = tmem + static_cast<uint32_t>(p.u_col[u]);
        idu[u] = umma_idesc(1u, static_cast<uint32_t>(p.u_n[u]), PAIR ? 256u : 128u);
        bxd[u] = umma_desc_sbo(win0 + static_cast<uint32_t>(p.u_xpos[u]) * x_pos, 128, x_sbo);
        btd[u] = umma_desc_sbo(win0 + static_cast<uint32_t>(p.u_tpos[u]) * t_pos, sw_t_, t_sbo);
      }
    }
    const uint64_t ad_dense = umma_desc(smem_u32(smem + off_a_), sw_t_);
    const uint64_t ad_sp = umma_desc(smem_u32(smem + off_a_), 64);
    const uint64_t ed0 = umma_desc_rows16(smem_u32(smem + off_e_));
    const uint32_t slot_a16 = a_slot_ >> 4, slot_e16 = e_slot_ >> 4;
    const uint32_t win16 = win_stride_ >> 4;
    const int ksteps = static_cast<int>(sw_t_ / 32);
    int slot = 0, k = 0, buf = 0, eslot = 0;
    uint32_t ph = 0, wph = 0;
    const bool contig = nwb_ == nwin;  // must match the producer's tile order
    const int n_u = PAIR ? n_tiles_ >> 1 : n_tiles_;
    const int t_begin = contig ? static_cast<int>(static_cast<long long>(g_id) * n_u / g_n) : g_id;
    const int t_end = contig ? static_cast<int>(static_cast<long long>(g_id + 1) * n_u / g_n) : n_u;
    const int t_step = contig ? 1 : g_n;
    (void)cbands_; (void)bands_; (void)th_; (void)tcols_; (void)n_mt_;
    const int ilv_m = smem_param(prm + 36);
    if (PAIR && !lead) {
      // ---------------------------------------------------------- pair relay (rank 1)
      // Mirror the leader's consumption order: every window and A/E item this CTA's
      // producer lands is forwarded to the leader's full barrier (count 2 there), whose
      // MMAs read this CTA's shared memory at the same offsets.  Releases (empty
      // barriers) arrive here directly through the leader's multicast commits.
      if (elect_one()) {
        for (int tu = t_begin; tu < t_end; tu += t_step) {
          for (int w = 0; w < nwin; ++w) {
            mbar_wait(&win_full[buf], wph);
            mbar_arrive_remote(&win_full[buf], 0);
            if (win_map(w, n_xw_, ilv_m) >= 0) {
              mbar_wait(&a_full[slot], ph);
              mbar_arrive_remote(&a_full[slot], 0);
              if (++slot == ns_) { slot = 0; ph ^= 1u; }
            } else {
              while (true) {
                mbar_wait(&a_full[slot], ph);
                const uint32_t info0 = ld_shared_u32(slot_info + 4u * kWMaxBpi * slot);
                mbar_arrive_remote(&a_full[slot], 0);
                if (++slot == ns_) { slot = 0; ph ^= 1u; }
                if (info0 >> 31) break;
              }
            }
            if (++buf == nwb_) { buf = 0; wph ^= 1u; }
          }
        }
      }
    } else if (elect_one()) {
    int mi_ = 0;  // item count (debug trace)
    (void)mi_;
    for (int tu = t_begin; tu < t_end; tu += t_step, ++k) {
      const int b = nacc_ == 2 ? (k & 1) : 0;
      const int use = nacc_ == 2 ? (k >> 1) : k;  // previous uses of accumulator b
      if (use > 0) {
        if (PAIR) mbar_wait_cluster(&acc_empty[b], (use - 1) & 1);
        else mbar_wait(&acc_empty[b], (use - 1) & 1);
        tc_fence_after();
      }
      const uint32_t acc0 = static_cast<uint32_t>(b) * acc_cols_;
      if (WTRACE(p) && blockIdx.x == 0 && k < 16) p.trace[100 + 4 * k] = gtimer();
      for (int w = 0; w < nwin; ++w) {
        if (WTRACE(p) && blockIdx.x == 0 && k < 16 && w < 8) p.trace[200 + 16 * k + 2 * w] = gtimer();
        if (PAIR) mbar_wait_cluster(&win_full[buf], wph);
        else mbar_wait(&win_full[buf], wph);
        tc_fence_after();
        if (WTRACE(p) && blockIdx.x == 0 && k < 16 && w < 8) p.trace[200 + 16 * k + 2 * w + 1] = gtimer();
        const uint32_t boff = static_cast<uint32_t>(buf) * win16;
        if (win_map(w, n_xw_, ilv_m) >= 0) {  // dense window: the accumulator already holds a sparse part
          if (PAIR) mbar_wait_cluster(&a_full[slot], ph);
          else mbar_wait(&a_full[slot], ph);
          tc_fence_after();
          const uint64_t ab = ad_dense + slot * slot_a16;
          {
#pragma unroll
            for (int u = 0; u < NU; ++u) {
              {
                for (int kk = 0; kk < ksteps; ++kk) {
                  const uint32_t acc1 = (n_xw_ > 0 || w > 0 || kk > 0) ? 1u : 0u;  // S empty: dense starts the sum
                  if (PAIR) mma_bf16_2(dcol[u] + acc0, ab + 2 * kk, btd[u] + boff + 2 * kk, idu[u], acc1);
                  else mma_bf16(dcol[u] + acc0, ab + 2 * kk, btd[u] + boff + 2 * kk, idu[u], acc1);
                }
              }
            }
            if (PAIR) mma_commit_pair(&a_empty[slot]);
            else mma_commit(&a_empty[slot]);
          }
          if (++slot == ns_) { slot = 0; ph ^= 1u; }
        } else {
          // sparse items of this window: the producer tags each slot with the
          // tap's window offset and whether it is the window's last item; the tile's
          // very first MMA step of each unit starts the accumulator (accumulate = 0)
          bool first = w == 0;
          while (true) {
            if (WTRACE(p) && blockIdx.x == 0 && mi_ < 64) p.trace[3300 + 3 * mi_] = gtimer();
            if (PAIR) mbar_wait_cluster(&a_full[slot], ph);
            else mbar_wait(&a_full[slot], ph);
            tc_fence_after();
            if (WTRACE(p) && blockIdx.x == 0 && mi_ < 64) p.trace[3300 + 3 * mi_ + 1] = gtimer();
            const uint32_t info0 = ld_shared_u32(slot_info + 4u * kWMaxBpi * slot);
            const int nb = static_cast<int>((info0 >> 28) & 7u);
            uint32_t tapv[BPI];
#pragma unroll
            for (int q = 0; q < BPI; ++q)
              tapv[q] = (q == 0 ? info0 : ld_shared_u32(slot_info + 4u * (kWMaxBpi * slot + q))) & 0x0FFFFFFFu;
            const uint32_t et = tmem + e_col0_ + 4u * static_cast<uint32_t>(bpi_) * eslot;
            if (++eslot == e_slots_) eslot = 0;
            const uint64_t ab = ad_sp + slot * slot_a16;
            {
              // metadata of block pairs in one tcgen05.cp.128x256b (blocks 2 KB apart = LBO)
#pragma unroll
              // (an odd last block copies alone: its neighbour's columns may belong to the
              // next metadata slot, or lie past the end of TMEM when items are one block)
              for (int bp = 0; bp < BPI; bp += 2)
                if (bp < nb && !WDBG(p, 5)) {
                  const uint64_t esrc = ed0 + slot * slot_e16 + static_cast<uint32_t>(bp) * (kEBlockBytes >> 4);
                  if (bp + 1 < nb) {
                    if (PAIR) tmem_cp_128x256b_2(et + 4u * static_cast<uint32_t>(bp), esrc);
                    else tmem_cp_128x256b(et + 4u * static_cast<uint32_t>(bp), esrc);
                  } else {
                    if (PAIR) tmem_cp_128x128b_2(et + 4u * static_cast<uint32_t>(bp), esrc);
                    else tmem_cp_128x128b(et + 4u * static_cast<uint32_t>(bp), esrc);
                  }
                }
#pragma unroll
              for (int bi = 0; bi < BPI; ++bi) {
                if (bi < nb) {
                  const uint32_t ebi = et + 4u * static_cast<uint32_t>(bi);
#pragma unroll
                  for (int s2 = 0; s2 < (WDBG(p, 8) ? 1 : 2) && !(WDBG(p, 1)); ++s2) {
#pragma unroll
                    for (int u = 0; u < NU; ++u) {
                      const uint64_t aa = ab + static_cast<uint32_t>(bi) * (kSpBlockBytes >> 4) + 2 * s2;
                      const uint64_t bb = bxd[u] + boff + tapv[bi] + 4 * s2;
                      const uint32_t id = idu[u] | (1u << 2) | static_cast<uint32_t>(s2);
                      const uint32_t acc1 = (first && bi == 0 && s2 == 0) ? 0u : 1u;
                      if (PAIR) mma_sp_bf16_2(dcol[u] + acc0, aa, bb, id, acc1, ebi);
                      else mma_sp_bf16(dcol[u] + acc0, aa, bb, id, acc1, ebi);
                    }
                  }
                }
              }
              if (WDBG(p, 512)) mbar_arrive(&a_empty[slot]);
              else if (PAIR) mma_commit_pair(&a_empty[slot]);
              else mma_commit(&a_empty[slot]);
              if (WTRACE(p) && blockIdx.x == 0 && mi_ < 64) p.trace[3300 + 3 * mi_ + 2] = gtimer();
              ++mi_;
            }
            first = false;
            if (++slot == ns_) { slot = 0; ph ^= 1u; }
            if (info0 >> 31) break;
          }
        }
        if (PAIR) mma_commit_pair(&win_empty[buf]);
        else mma_commit(&win_empty[buf]);
        if (++buf == nwb_) { buf = 0; wph ^= 1u; }
      }
      if (PAIR) mma_commit_pair(&acc_full[b]);
      else mma_commit(&acc_full[b]);
      if (WTRACE(p) && blockIdx.x == 0 && k < 16) p.trace[100 + 4 * k + 1] = gtimer();
    }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    const int q4 = warp & 3;            // TMEM lane quarter
    const int ehalf = (warp - 2) >> 2;  // which half of the columns
    const uint32_t scr = smem_u32(smem + p.off_epi) + static_cast<uint32_t>(warp - 2) * kEpiScratch;
    __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(p.y);
    int k = 0;
    const bool contig = p.nwb == nwin;  // must match the producer's tile order
    const int n_u = PAIR ? p.n_tiles >> 1 : p.n_tiles;
    const int t_begin = contig ? static_cast<int>(static_cast<long long>(g_id) * n_u / g_n) : g_id;
    const int t_end = contig ? static_cast<int>(static_cast<long long>(g_id + 1) * n_u / g_n) : n_u;
    const int t_step = contig ? 1 : g_n;
    // accumulator release: the leader's MMA issuer waits for the epilogues of both CTAs
    auto release = [&](int b) {
      if (PAIR && !lead) mbar_arrive_remote(&acc_empty[b], 0);
      else mbar_arrive(&acc_empty[b]);
    };
    for (int tu = t_begin; tu < t_end; tu += t_step, ++k) {
      const int hm = p.n_mt >> 1;
      const int tile = PAIR ? (tu / hm) * p.n_mt + 2 * (tu % hm) + static_cast<int>(rank) : tu;
      const TileCoord tc = tile_coord(p, tile);
      if (p.n_gk > 0) {
        // overflow gather of this tile (the MMA warp needs it only after the tile's sparse
        // and T chunks): warp e takes positions e, e + 8, ..; lane = slot (64-byte stores)
        gather_tile(p, tc, warp - 2, lane);
        fence_proxy_async_global();  // generic-proxy stores -> the producer's TMA (async proxy) loads
        __syncwarp();
        if (lane == 0) mbar_arrive(g_ready);
      }
      const int b = p.nacc == 2 ? (k & 1) : 0;
      const int use = p.nacc == 2 ? (k >> 1) : k;
      // one thread polls the accumulator barrier, the other epilogue threads block in a
      // named barrier: eight warps spinning on an mbarrier slowed the producer's and the
      // MMA issuer's own barrier traffic (tools/wtrace.py: ~300 ns per hand-off)
      if (threadIdx.x == 64) mbar_wait_sleep(&acc_full[b], use & 1);
      named_bar_sync(2, kWThreads - 64);
      tc_fence_after();
      if (WDBG(p, 16)) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release(b);
        continue;
      }
      if (WTRACE(p) && blockIdx.x == 0 && threadIdx.x == 64 && k < 16) p.trace[100 + 4 * k + 2] = gtimer();
      const uint32_t acc0 = static_cast<uint32_t>(b) * p.acc_cols;
      const int jw = tc.j0 + q4 * 32;  // first channel of this warp
      // store side of the transpose: lane = (column lane/4 of every 8, 8-channel part lane%4);
      // a column is (position, image) with ipw images per position, so the lane's image is
      // fixed and, at ipw 4, lanes 16..31 take the second position of each 8 columns
      const int part = lane & 3, img8 = lane >> 2;
      const int ipw = p.ipw;
      const int img = img8 & (ipw - 1), psub = ipw == 8 ? 0 : (img8 >> 2), ppass = 8 / ipw;
      const int jch = jw + part * 8;
      const bool lane_ok = tc.n0 + img < p.n && jch < p.cout;
      __nv_bfloat16* ybase = y + (static_cast<long long>(lane_ok ? tc.n0 + img : 0) * p.ho * p.wo) * p.cout + jch;
      for (int u = 0; u < p.n_units; ++u) {
        const int pitch = p.u_pitch[u], nw = p.u_nw[u], un = p.u_n[u], rows = p.u_rows[u];
        const int r0 = p.u_r0[u], w0 = p.u_wo0[u], ucol = p.u_col[u], q0 = p.u_q0[u];
        for (int c0 = ehalf * 32; c0 < un; c0 += 64) {
          // 32 columns x this warp's 32 channels -> the scratch tile [32 columns][32 channels]
          // bf16: per 16 lanes x 16 columns one tcgen05.ld.16x256b (already in the m8n8
          // fragment layout) and one transposing stmatrix (each stored row = 8 channels of
          // one column) -- instead of 32 two-byte shared stores per lane
          {
            const int t1 = lane >> 2, mi = lane >> 3, mj = lane & 7;
            const bool epi = p.epi != nullptr || p.relu;
            // all four TMEM loads in flight before one wait (each wait is a TMEM round trip)
            uint32_t r[2][2][8];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int cb = 0; cb < 2; ++cb)
                tmem_ld_16x256b_x2(tmem + (static_cast<uint32_t>(q4 * 32 + 16 * h) << 16) + acc0 +
                                       static_cast<uint32_t>(ucol + c0 + 16 * cb),
                                   r[h][cb]);
            float2 sb[2][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              sb[h][0] = sb[h][1] = make_float2(1.f, 0.f);
              if (epi) {
                sb[h][0] = out_epi_load(p.epi, min(jw + 16 * h + t1, p.cout - 1));
                sb[h][1] = out_epi_load(p.epi, min(jw + 16 * h + t1 + 8, p.cout - 1));
              }
            }
            tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
              for (int cb = 0; cb < 2; ++cb) {
                float f[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[h][cb][i]);
                if (epi) {
                  f[0] = out_epi(f[0], sb[h][0], p.relu);
                  f[1] = out_epi(f[1], sb[h][0], p.relu);
                  f[4] = out_epi(f[4], sb[h][0], p.relu);
                  f[5] = out_epi(f[5], sb[h][0], p.relu);
                  f[2] = out_epi(f[2], sb[h][1], p.relu);
                  f[3] = out_epi(f[3], sb[h][1], p.relu);
                  f[6] = out_epi(f[6], sb[h][1], p.relu);
                  f[7] = out_epi(f[7], sb[h][1], p.relu);
                }
                // scratch row (column col, 8-channel part) at col*64 + (part ^ ((col >> 1) & 3))*16:
                // the 8 rows of one stmatrix phase land in 8 distinct 16-byte bank groups
                const int scol = cb * 16 + (mi >> 1) * 8 + mj, spart = 2 * h + (mi & 1);
                const uint32_t addr = scr + static_cast<uint32_t>(scol * 64 + ((spart ^ ((scol >> 1) & 3)) * 16));
                stmatrix_x4_trans(addr, pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                  pack_bf16x2(f[6], f[7]));
              }
            }
          }
          __syncwarp();
          // lane l, pass q: column col = q*8 + l/4 = output position q0 + (c0 + col) / ipw
          // (stepped without per-store divisions) of image `img`, channels 8*(l%4) .. +7
          {
            const int qv0 = q0 + c0 / ipw + psub;
            int rr = qv0 / pitch, cc = qv0 - rr * pitch;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int col = q * 8 + img8;
              const uint4 val = lds_v4(scr + static_cast<uint32_t>(col * 64 + ((part ^ ((col >> 1) & 3)) * 16)));
              const int ho = tc.ho0 + r0 + rr, wo = tc.wo0 + w0 + cc;
              if (lane_ok && c0 + col < un && cc < nw && rr < rows && ho < p.ho && wo < p.wo)
                *reinterpret_cast<uint4*>(ybase + (static_cast<long long>(ho) * p.wo + wo) * p.cout) = val;
              cc += ppass;
              while (cc >= pitch) {
                cc -= pitch;
                ++rr;
              }
            }
          }
          __syncwarp();
        }
      }
      // this warp's TMEM reads of buffer b are complete (wait::ld above)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release(b);
      if (WTRACE(p) && blockIdx.x == 0 && threadIdx.x == 64 && k < 16) p.trace[100 + 4 * k + 3] = gtimer();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // neither CTA frees TMEM / leaves while the pair still works
  if (WTRACE(p) && threadIdx.x == 0 && blockIdx.x < 2048) p.trace[2000 + 3 * blockIdx.x + 2] = gtimer();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    if (PAIR) tmem_dealloc2(tmem, p.tmem_cols);
    else tmem_dealloc(tmem, p.tmem_cols);
  }
}

}  // namespace lrs
