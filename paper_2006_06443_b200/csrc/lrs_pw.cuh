// lrs_pw.cuh -- the fused a3 + a4 + a5 kernel of 1x1 layers whose L is an SVD pair
// (C4, BASELINE.json configs[3]), channel-stationary on the sm_100a tensor cores:
//
//   Y[p, j] = sum_r T1[p, r] V[r, j]                    (a3; T1 = X U, a1)
//           + sum_c S[j, c] X[p, c]                     (a4, PAPER.md:171-191 at k = 1)
//
// A 1x1 convolution has no spatial neighbourhood: p runs over the n*H*W positions of
// the NHWC tensors, X and T1 are plain row-major matrices and every operand tile is a
// 2-D TMA box.  The layer is HBM-bound by the write of Y (C4: 51 MB of 64 MB), so the
// kernel is built to stream: each CTA owns a fixed group of `mpc` 128-channel M-tiles
// whose weights -- the V^T blocks (A of the dense MMAs) and the exact 2:4 main +
// residual blocks of S (A of the sparse MMAs, tcgen05.mma.sp) -- are loaded into shared
// memory once, with their sparsity metadata copied into TMEM once; the CTA then walks
// its share of the position tiles (bp positions each), streaming X chunks (64
// channels x bp positions) and T1 chunks through a ring, so the only per-tile traffic
// is X and T1 in and Y out.
//
// D[j, p] (TMEM lane = output channel, column = position) is accumulated for all mpc
// M-tiles of a position tile at once, chunk-outer (each X / T1 chunk is released as
// soon as its MMAs for all M-tiles are issued); two accumulator sets alternate, so the
// epilogue of tile k (TMEM -> fp32 output epilogue -> bf16 -> stmatrix transpose ->
// 16-byte stores of Y, written once: a5) overlaps the MMAs of tile k + 1.
//
// Warps: 0 = TMA producer, 1 = TMEM allocator + MMA issuer (one elected thread),
// 2..9 = epilogue (warp w drains TMEM lanes 32 (w % 4) .., the two warps of a quarter
// take alternate 32-column chunks).
#pragma once
#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kPThreads = 320;
constexpr int kPMaxMpc = 4;        // M-tiles per CTA
constexpr int kPMaxCk = 8;         // 64-channel input chunks (Cin <= 512)
constexpr int kPMaxSlots = 16;
constexpr uint32_t kPEpiScratch = 4096;  // per epilogue warp, at most: 2 x [32 positions][32 channels] bf16

struct PwParams {
  CUtensorMap tmX;  // X  2-D [P][Cin] bf16, box {64, bp}, SW128
  CUtensorMap tmT;  // T1 2-D [P][R1p] bf16, box {t_kc, bp}, swizzle sw_t
  CUtensorMap tmY;  // Y  2-D [P][Cout] bf16, box {32, 32}, SW64 (the epilogue's TMA stores)
  const uint8_t* img_w;    // per group: [mpc][n_tk] V^T blocks (128 rows x sw_t B, swizzled), then the
                           // group's 2:4 blocks (8 KB each, SW64) in (m, c, main/residual) order
  const uint8_t* img_e;    // per group: their metadata blocks, [128 lanes][16 B] each (2 KB)
  const uint16_t* tab;     // per group: [mpc][n_ck] first block | count << 12
  void* y;
  const float2* epi;       // per output channel (scale, bias) of the fused output epilogue, or NULL
  int relu;
  int P, cout;             // positions of this forward, output channels
  int n_ck, n_x;           // 64-channel chunks of Cin; X chunks per tile (0 if S is empty)
  int n_tk, t_kc;          // T1 chunks per tile, ranks per chunk
  uint32_t sw_t;           // bytes per T1 chunk row (= its swizzle width)
  int bp;                  // positions per tile (MMA N)
  int mpc, n_groups;       // M-tiles per CTA, channel groups
  int n_pt;                // position tiles of this forward
  uint32_t w_bytes;        // one group's weight image (V^T + 2:4 blocks)
  uint32_t dense_bytes;    // its V^T part (2:4 blocks follow)
  int nblk_max;            // most 2:4 blocks of any group (E staging, TMEM columns)
  int ns;                  // ring slots
  int cpi;                 // chunks per ring item: a slot holds cpi X (or T1) chunks of bp x 128 B, one
                           // mbarrier hand-off and one tcgen05.commit per item (~500 cycles of the
                           // MMA thread's serial loop per hand-off bounded C4's tile rate)
  uint32_t slot_bytes;     // one item slot (cpi * bp * 128)
  uint32_t acc_cols;       // TMEM columns of one accumulator set (mpc * bp)
  uint32_t e_col0;         // first metadata column (2 * acc_cols)
  uint32_t off_e, off_ring, off_epi, off_tab, off_bar;
  int e_slot0;             // first ring slot the metadata staging shares (ns: none); the producer
                           // fills slots >= e_slot0 only after the copies to TMEM completed
  int epi_nbuf;            // epilogue scratch buffers per warp (1 or 2, 2 KB each)
  unsigned long long* trace;  // debug builds: %globaltimer stamps of CTA 0 (lrs_conv_debug_trace)
  int dbg;                    // experiment builds (LRS_PW_DBG): 1 skip Y stores, 2 skip MMAs, 4 skip X/T loads,
                              // 8 skip the proxy fence, 16 skip the stmatrix transposes, 32 skip the TMEM loads
  // projection fused in (lrs_pwf_kernel): T1 = X U computed per position tile from the X
  // chunks already in the ring, restaged as bf16 into shared memory, never written to HBM
  const uint8_t* img_u;    // U_in^T blocks [n_ck][R1p rows x 128 B], SW128 (B of the T1 MMAs)
  uint32_t u_bytes;        // n_ck * R1p * 128
  int r1p;
  uint32_t off_u, off_t1s; // resident U^T; two T1 tiles [n_tk][128 rows][sw_t], swizzle sw_t
  uint32_t t1s_bytes;      // one T1 tile (128 * R1p * 2)
  uint32_t t1_col0;        // TMEM columns of the two T1 accumulators (R1p each)
};

#ifdef LRS_WCONV_DEBUG
#define PTRACE(p, idx) \
  do {                 \
    if ((p).trace && blockIdx.x == 0 && (idx) < 4000) (p).trace[(idx)] = gtimer(); \
  } while (0)
#else
#define PTRACE(p, idx) ((void)0)
#endif

template <int MPC>
__global__ void __launch_bounds__(kPThreads, 1) lrs_pw_kernel(const __grid_constant__ PwParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;                       // [kPMaxSlots]
  uint64_t* empty = bars + kPMaxSlots;         // [kPMaxSlots]
  uint64_t* acc_full = empty + kPMaxSlots;     // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint64_t* w_full = acc_empty + 2;            // weights + metadata staged
  uint64_t* e_done = w_full + 1;               // metadata copied to TMEM: its staging slots are free
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(e_done + 1);
  uint16_t* tab_s = reinterpret_cast<uint16_t*>(smem + p.off_tab);

  const int grp = static_cast<int>(blockIdx.x) % p.n_groups;
  const int li = static_cast<int>(blockIdx.x) / p.n_groups;                       // my index in the group
  const int gctas = (static_cast<int>(gridDim.x) - grp + p.n_groups - 1) / p.n_groups;  // CTAs of my group

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);
    }
    mbar_init(w_full, 1);
    mbar_init(e_done, 1);
    fence_mbar_init();
    tma_prefetch_desc(&p.tmX);
    tma_prefetch_desc(&p.tmT);
    tma_prefetch_desc(&p.tmY);
  }
  if (threadIdx.x < MPC * kPMaxCk) {
    const int m = threadIdx.x / kPMaxCk, c = threadIdx.x % kPMaxCk;
    tab_s[threadIdx.x] = c < p.n_ck ? __ldg(p.tab + (static_cast<size_t>(grp) * MPC + m) * p.n_ck + c) : 0;
  }
  // the scalars of the role loops, staged in shared memory (see smem_param in lrs_ptx.cuh)
  int* prm = reinterpret_cast<int*>(smem + p.off_tab + 256);
  if (threadIdx.x == 0) {
    prm[0] = p.n_pt; prm[1] = p.n_x; prm[2] = p.n_tk; prm[3] = p.ns; prm[4] = p.bp;
    prm[5] = static_cast<int>(p.slot_bytes); prm[6] = static_cast<int>(p.sw_t); prm[7] = static_cast<int>(p.acc_cols);
    prm[8] = p.t_kc; prm[9] = static_cast<int>(p.e_col0); prm[10] = p.relu; prm[11] = p.cout; prm[12] = p.P;
    prm[13] = li; prm[14] = gctas; prm[15] = static_cast<int>(p.off_ring); prm[16] = static_cast<int>(p.dense_bytes);
    prm[17] = p.e_slot0; prm[18] = p.epi_nbuf; prm[19] = p.cpi;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 32 && *tmem_slot != 0u) __trap();  // the CTA owns the whole TMEM (1 CTA / SM)
  constexpr uint32_t tmem = 0u;
  const int n_pt = smem_param(prm + 0), n_x = smem_param(prm + 1), n_tk = smem_param(prm + 2);
  const int ns = smem_param(prm + 3), bp = smem_param(prm + 4);
  const int cpi = smem_param(prm + 19);
  const int nxi = (n_x + cpi - 1) / cpi, nti = (n_tk + cpi - 1) / cpi;  // X / T1 items per tile
  const int nq = nxi + nti;                                             // items per tile
  const uint32_t chunk_bytes = static_cast<uint32_t>(bp) * 128u;        // a chunk's place in its item slot
  const int li_ = smem_param(prm + 13), gct = smem_param(prm + 14);
  const uint32_t slot_bytes = smem_param(prm + 5), sw_t = smem_param(prm + 6), acc_cols = smem_param(prm + 7);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // lane 0 requests the weights (they do not depend on the previous kernel: PDL) and
    // the T1 chunks; the X chunks of a tile are requested by lanes 0 .. n_x-1 at once
    // (one 2-D box each: a single issuing thread measured ~290 ns per 16 KB box)
    if (lane == 0) {
      const int nblk = p.nblk_max;
      mbar_arrive_expect_tx(w_full, p.w_bytes + static_cast<uint32_t>(nblk) * 2048u);
      bulk_load(smem, p.img_w + static_cast<size_t>(grp) * p.w_bytes, p.w_bytes, w_full);
      if (nblk > 0)
        bulk_load(smem + p.off_e, p.img_e + static_cast<size_t>(grp) * nblk * 2048u,
                  static_cast<uint32_t>(nblk) * 2048u, w_full);
    }
    bool waited = false;
    const int t_kc = smem_param(prm + 8);
    const int e_slot0 = smem_param(prm + 17);
    const uint32_t ring = smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 15));
    // item it = round * ns + slot, tracked incrementally (no divisions): lane l < n_x owns
    // the X chunk l of every tile (item k * nq + l), lane 0 also the T1 chunks
    int xs = lane, xr = 0;       // this lane's X item
    int ts = nxi, tr = 0;        // lane 0's first T1 item of the tile
    while (xs >= ns) { xs -= ns; ++xr; }  // (a tile may hold more chunks than the ring has slots)
    while (ts >= ns) { ts -= ns; ++tr; }
    for (int pt = li_; pt < n_pt; pt += gct) {
      const int p0 = pt * bp;
      if (lane < nxi) {
        if (xr > 0) mbar_wait(&empty[xs], (xr - 1) & 1);
        else if (xs >= e_slot0) mbar_wait(e_done, 0);  // the slot still holds metadata staging
        const int c0 = lane * cpi, cn = min(cpi, n_x - c0);
        if (LRS_XDBG(p.dbg & 4)) {
          mbar_arrive(&full[xs]);
        } else {
          mbar_arrive_expect_tx(&full[xs], static_cast<uint32_t>(cn * bp) * 128u);
          for (int j = 0; j < cn; ++j)
            tma_load_2d_s(ring + xs * slot_bytes + j * chunk_bytes, &p.tmX, &full[xs], (c0 + j) * 64, p0);
        }
        xs += nq;
        while (xs >= ns) { xs -= ns; ++xr; }
      }
      __syncwarp();
      if (lane == 0) {
        int s = ts, r = tr;
        for (int ti = 0; ti < nti; ++ti) {
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          else if (s >= e_slot0) mbar_wait(e_done, 0);
          if (!waited) {  // T1 is the previous kernel's output
            pdl_wait();
            pdl_launch_dependents();
            waited = true;
          }
          const int t0 = ti * cpi, tn = min(cpi, n_tk - t0);
          if (LRS_XDBG(p.dbg & 4)) {
            mbar_arrive(&full[s]);
          } else {
            mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(tn * bp) * sw_t);
            for (int j = 0; j < tn; ++j)
              tma_load_2d_s(ring + s * slot_bytes + j * chunk_bytes, &p.tmT, &full[s], (t0 + j) * t_kc, p0);
          }
          if (++s == ns) { s = 0; ++r; }
        }
        ts += nq;
        while (ts >= ns) { ts -= ns; ++tr; }
      }
      __syncwarp();
    }
    if (lane == 0 && !waited) {
      pdl_wait();
      pdl_launch_dependents();
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      PTRACE(p, 0);
      mbar_wait(w_full, 0);
      tc_fence_after();
      PTRACE(p, 1);
      // sparsity metadata of the group's 2:4 blocks -> TMEM, once (block b at e_col0 + 4 b)
      const uint64_t ed = umma_desc_rows16(smem_u32(smem + p.off_e));
      for (int b = 0; b < p.nblk_max; ++b) tmem_cp_128x128b(tmem + p.e_col0 + 4u * b, ed + b * (2048u >> 4));
      mma_commit(e_done);  // arrives once the copies have read the staging (ring slots >= e_slot0)
      const uint32_t e_col0 = smem_param(prm + 9);
      const uint32_t idn = umma_idesc(1u, static_cast<uint32_t>(bp), 128u);
      const uint32_t ids = idn | (1u << 2);
      const uint32_t ring_s = smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 15));
      const uint64_t a_dense0 = umma_desc(smem_u32(smem), sw_t);
      const uint64_t a_sp0 = umma_desc(smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 16)), 64);
      const uint64_t ring0 = umma_desc(ring_s, 128);
      const uint64_t ringt0 = umma_desc(ring_s, sw_t);
      const uint32_t slot16 = slot_bytes >> 4;
      const uint32_t dblk16 = (128u * sw_t) >> 4;
      const int ksteps = static_cast<int>(sw_t / 32);
      int slot = 0, k = 0;
      uint32_t ph = 0;
      for (int pt = li_; pt < n_pt; pt += gct, ++k) {
        const int b = k & 1, use = k >> 1;
        PTRACE(p, 100 + 4 * k);
        if (use > 0) {
          mbar_wait(&acc_empty[b], (use - 1) & 1);
          tc_fence_after();
        }
        PTRACE(p, 101 + 4 * k);
        const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * acc_cols;
        uint32_t started = 0;  // bit m: accumulator of M-tile m holds a partial sum
        for (int q = 0; q < nq; ++q) {
          mbar_wait(&full[slot], ph);
          tc_fence_after();
          PTRACE(p, 2000 + k * nq + q);
          if (LRS_XDBG(p.dbg & 2)) {
          } else if (q < nxi) {
            const int c0 = q * cpi, cn = min(cpi, n_x - c0);
            for (int j = 0; j < cn; ++j) {
              const uint64_t bd = ring0 + slot * slot16 + static_cast<uint32_t>(j) * (chunk_bytes >> 4);
#pragma unroll
              for (int m = 0; m < MPC; ++m) {
                const uint32_t e = tab_s[m * kPMaxCk + c0 + j];
                const int b0 = static_cast<int>(e & 0xFFFu), nb = static_cast<int>(e >> 12);
                for (int bi = 0; bi < nb; ++bi) {
                  const uint64_t ad = a_sp0 + static_cast<uint32_t>(b0 + bi) * (8192u >> 4);
                  const uint32_t et = tmem + e_col0 + 4u * static_cast<uint32_t>(b0 + bi);
#pragma unroll
                  for (int s2 = 0; s2 < 2; ++s2) {
                    mma_sp_bf16(acc0 + static_cast<uint32_t>(m * bp), ad + 2 * s2, bd + 4 * s2,
                                ids | static_cast<uint32_t>(s2), (started >> m) & 1u, et);
                    started |= 1u << m;
                  }
                }
              }
            }
          } else {
            const int t0 = (q - nxi) * cpi, tn = min(cpi, n_tk - t0);
            for (int j = 0; j < tn; ++j) {
              const int tk = t0 + j;
              const uint64_t bd = ringt0 + slot * slot16 + static_cast<uint32_t>(j) * (chunk_bytes >> 4);
#pragma unroll
              for (int m = 0; m < MPC; ++m) {
                const uint64_t ad = a_dense0 + static_cast<uint32_t>(m * n_tk + tk) * dblk16;
                for (int kk = 0; kk < ksteps; ++kk) {
                  mma_bf16(acc0 + static_cast<uint32_t>(m * bp), ad + 2 * kk, bd + 2 * kk, idn, (started >> m) & 1u);
                  started |= 1u << m;
                }
              }
            }
          }
          mma_commit(&empty[slot]);  // the slot is free once these MMAs have read it
          if (++slot == ns) {
            slot = 0;
            ph ^= 1u;
          }
        }
        mma_commit(&acc_full[b]);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    // Per 32-position x 32-channel chunk: tcgen05.ld (m8n8 fragments) -> fused output
    // epilogue -> bf16 -> stmatrix transpose into a [32 positions][32 channels] scratch
    // whose 16-byte chunks are XOR-swizzled exactly as TMA SWIZZLE_64B lays them out,
    // then ONE TMA tensor store of the chunk (positions past P are clipped by the map).
    // Two scratch buffers per warp: a buffer is rewritten only after the store issued
    // from it two chunks ago has read it (bulk wait_group.read 1).
    const int q4 = warp & 3;            // TMEM lane quarter
    const int ehalf = (warp - 2) >> 2;  // which alternate 32-column chunks
    const int epi_nbuf = smem_param(prm + 18);
    const uint32_t scr0 = smem_u32(smem + p.off_epi) + static_cast<uint32_t>((warp - 2) * epi_nbuf) * 2048u;
    const int relu = smem_param(prm + 10), cout = smem_param(prm + 11);
    const bool epi = p.epi != nullptr || relu;
    const int t1 = lane >> 2, mi = lane >> 3, mj = lane & 7;
    int k = 0, nchunk = 0;
    for (int pt = li_; pt < n_pt; pt += gct, ++k) {
      const int b = k & 1, use = k >> 1;
      if (threadIdx.x == 64) mbar_wait(&acc_full[b], use & 1);
      named_bar_sync(2, kPThreads - 64);
      tc_fence_after();
      if (threadIdx.x == 64) PTRACE(p, 102 + 4 * k);
      const uint32_t acc0 = static_cast<uint32_t>(b) * acc_cols;
      const int p0 = pt * bp;
      // the quarter's (M-tile, 32-position) chunks alternate between its two warps over the
      // whole list (a fixed column parity left one warp 4 chunks and the other 2 at bp = 96)
      int mv = 0;
      while (mv < MPC && (grp * MPC + mv) * 128 + q4 * 32 < cout) ++mv;
      const int cpm = bp / 32;
#pragma unroll 1
      for (int i = ehalf; i < mv * cpm; i += 2, ++nchunk) {
        const int m = i / cpm, c0 = (i - m * cpm) * 32;
        const int jw = (grp * MPC + m) * 128 + q4 * 32;  // first channel of this warp
        float2 sb[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          sb[h][0] = sb[h][1] = make_float2(1.f, 0.f);
          if (epi) {
            sb[h][0] = out_epi_load(p.epi, min(jw + 16 * h + t1, cout - 1));
            sb[h][1] = out_epi_load(p.epi, min(jw + 16 * h + t1 + 8, cout - 1));
          }
        }
        {
          uint32_t r[2][2][8] = {};
          if (!LRS_XDBG(p.dbg & 32)) {  // experiment: skip the TMEM loads
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int cb = 0; cb < 2; ++cb)
                tmem_ld_16x256b_x2(tmem + (static_cast<uint32_t>(q4 * 32 + 16 * h) << 16) + acc0 +
                                       static_cast<uint32_t>(m * bp + c0 + 16 * cb),
                                   r[h][cb]);
          }
          const uint32_t scr = scr0 + static_cast<uint32_t>(nchunk % epi_nbuf) * 2048u;
          if (lane == 0) {  // the store that last read this buffer is done with it
            if (epi_nbuf == 2) bulk_wait_read1();
            else bulk_wait_read0();
          }
          tmem_ld_wait();
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int cb = 0; cb < 2; ++cb) {
              float f[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[h][cb][i]);
              if (epi) {
                f[0] = out_epi(f[0], sb[h][0], relu);
                f[1] = out_epi(f[1], sb[h][0], relu);
                f[4] = out_epi(f[4], sb[h][0], relu);
                f[5] = out_epi(f[5], sb[h][0], relu);
                f[2] = out_epi(f[2], sb[h][1], relu);
                f[3] = out_epi(f[3], sb[h][1], relu);
                f[6] = out_epi(f[6], sb[h][1], relu);
                f[7] = out_epi(f[7], sb[h][1], relu);
              }
              // scratch row (position col, 8-channel part) at col*64 + (part ^ ((col >> 1) & 3))*16
              const int scol = cb * 16 + (mi >> 1) * 8 + mj, spart = 2 * h + (mi & 1);
              const uint32_t addr = scr + static_cast<uint32_t>(scol * 64 + ((spart ^ ((scol >> 1) & 3)) * 16));
              if (!LRS_XDBG(p.dbg & 16))  // experiment: skip the transposing stores
              stmatrix_x4_trans(addr, pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                pack_bf16x2(f[6], f[7]));
            }
          }
          if (!LRS_XDBG(p.dbg & 8)) fence_proxy_async_smem();  // the generic-proxy stmatrix writes -> visible to the TMA store
          __syncwarp();
          if (lane == 0 && !LRS_XDBG(p.dbg & 1)) {
            tma_store_2d(&p.tmY, scr, jw, p0 + c0);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      if (threadIdx.x == 64) PTRACE(p, 103 + 4 * k);
    }
    if (lane == 0) bulk_wait0();  // every store of this warp complete before the CTA exits
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace lrs
