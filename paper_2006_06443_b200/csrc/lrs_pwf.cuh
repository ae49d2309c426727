// lrs_pwf.cuh -- the whole 1x1 SVD-pair layer in ONE kernel (C4, BASELINE.json configs[3]):
//
//   T1[p, r] = sum_c X[p, c] U[c, r]                     (a1)
//   Y[p, j]  = sum_r T1[p, r] V[r, j]                    (a3)
//            + sum_c S[j, c] X[p, c]                     (a4, PAPER.md:171-191 at k = 1)
//
// lrs_pw.cuh with the projection fused in: the X chunks of a position tile (128 positions
// x 64 channels, SW128 K-major) that feed the sparse MMAs are also the A operand of the T1
// MMAs (M = 128 positions, N = R1p, K = the chunk's 64 channels; U^T resident in shared
// memory), so X is read once and T1 never touches HBM.  T1 (TMEM lane = position) is
// restaged by the epilogue warps as bf16 into a K-major shared-memory tile that is the B
// operand of the dense MMAs.  Software-pipelined: the MMA issuer runs the X phase (T1 +
// sparse MMAs) of tile k+1 before the dense phase of tile k, so the restage of tile k
// overlaps MMAs; the epilogue restages tile k+1 before draining Y of tile k.
#pragma once
#include "lrs_pw.cuh"

namespace lrs {

template <int MPC>
__global__ void __launch_bounds__(kPThreads, 1) lrs_pwf_kernel(const __grid_constant__ PwParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;                       // [kPMaxSlots] X chunk landed
  uint64_t* empty = bars + kPMaxSlots;         // [kPMaxSlots] X chunk's MMAs done
  uint64_t* acc_full = empty + kPMaxSlots;     // [2] Y accumulator complete
  uint64_t* acc_empty = acc_full + 2;          // [2] Y drained (8 warps)
  uint64_t* t1_full = acc_empty + 2;           // [2] T1 accumulator complete
  uint64_t* t1a_empty = t1_full + 2;           // [2] T1 accumulator read by the restage (8 warps)
  uint64_t* t1s_full = t1a_empty + 2;          // [2] T1 tile restaged in smem (8 warps)
  uint64_t* t1s_empty = t1s_full + 2;          // [2] dense MMAs done reading the T1 tile
  uint64_t* w_full = t1s_empty + 2;            // weights + metadata staged
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);
  uint16_t* tab_s = reinterpret_cast<uint16_t*>(smem + p.off_tab);

  const int grp = static_cast<int>(blockIdx.x) % p.n_groups;
  const int li = static_cast<int>(blockIdx.x) / p.n_groups;
  const int gctas = (static_cast<int>(gridDim.x) - grp + p.n_groups - 1) / p.n_groups;

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);
      mbar_init(&t1_full[i], 1);
      mbar_init(&t1a_empty[i], 8);
      mbar_init(&t1s_full[i], 8);
      mbar_init(&t1s_empty[i], 1);
    }
    mbar_init(w_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&p.tmX);
    tma_prefetch_desc(&p.tmY);
  }
  if (threadIdx.x < MPC * kPMaxCk) {
    const int m = threadIdx.x / kPMaxCk, c = threadIdx.x % kPMaxCk;
    tab_s[threadIdx.x] = c < p.n_ck ? __ldg(p.tab + (static_cast<size_t>(grp) * MPC + m) * p.n_ck + c) : 0;
  }
  int* prm = reinterpret_cast<int*>(smem + p.off_tab + 256);
  if (threadIdx.x == 0) {
    prm[0] = p.n_pt; prm[1] = p.n_x; prm[2] = p.n_tk; prm[3] = p.ns; prm[4] = p.bp;
    prm[5] = static_cast<int>(p.slot_bytes); prm[6] = static_cast<int>(p.sw_t); prm[7] = static_cast<int>(p.acc_cols);
    prm[8] = p.t_kc; prm[9] = static_cast<int>(p.e_col0); prm[10] = p.relu; prm[11] = p.cout; prm[12] = p.P;
    prm[13] = li; prm[14] = gctas; prm[15] = static_cast<int>(p.off_ring); prm[16] = static_cast<int>(p.dense_bytes);
    prm[17] = p.r1p; prm[18] = static_cast<int>(p.t1_col0); prm[19] = static_cast<int>(p.off_u);
    prm[20] = static_cast<int>(p.off_t1s); prm[21] = static_cast<int>(p.t1s_bytes); prm[22] = p.n_ck;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 32 && *tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0u;
  const int n_pt = smem_param(prm + 0), n_ck = smem_param(prm + 22), ns = smem_param(prm + 3);
  const int n_tk = smem_param(prm + 2);
  const int li_ = smem_param(prm + 13), gct = smem_param(prm + 14);
  const uint32_t slot_bytes = smem_param(prm + 5), sw_t = smem_param(prm + 6), acc_cols = smem_param(prm + 7);
  const int r1p = smem_param(prm + 17);
  const uint32_t t1_col0 = smem_param(prm + 18);
  const uint32_t t1s0 = smem_u32(smem) + smem_param(prm + 20), t1s_bytes = smem_param(prm + 21);
  constexpr int BP = 128;  // positions per tile: the M of the T1 MMAs
  // the weights (and U^T) do not depend on the previous kernel: request them first
  if (threadIdx.x == 0) {
    const int nblk = p.nblk_max;
    mbar_arrive_expect_tx(w_full, p.w_bytes + static_cast<uint32_t>(nblk) * 2048u + p.u_bytes);
    bulk_load(smem, p.img_w + static_cast<size_t>(grp) * p.w_bytes, p.w_bytes, w_full);
    bulk_load(smem + p.off_u, p.img_u, p.u_bytes, w_full);
    if (nblk > 0)
      bulk_load(smem + p.off_e, p.img_e + static_cast<size_t>(grp) * nblk * 2048u, static_cast<uint32_t>(nblk) * 2048u,
                w_full);
  }
  // X may be the previous kernel's output and Y may still be written by it: every thread
  // waits for it before touching either
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    const uint32_t ring = smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 15));
    int xs = lane, xr = 0;
    while (xs >= ns) { xs -= ns; ++xr; }
    for (int pt = li_; pt < n_pt; pt += gct) {
      if (lane < n_ck) {
        if (xr > 0) mbar_wait(&empty[xs], (xr - 1) & 1);
        mbar_arrive_expect_tx(&full[xs], static_cast<uint32_t>(BP) * 128u);
        tma_load_2d_s(ring + xs * slot_bytes, &p.tmX, &full[xs], lane * 64, pt * BP);
        xs += n_ck;
        while (xs >= ns) { xs -= ns; ++xr; }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      mbar_wait(w_full, 0);
      tc_fence_after();
      const uint32_t e_col0 = smem_param(prm + 9);
      const uint64_t ed = umma_desc_rows16(smem_u32(smem + p.off_e));
      for (int b = 0; b < p.nblk_max; ++b) tmem_cp_128x128b(tmem + e_col0 + 4u * b, ed + b * (2048u >> 4));
      const uint32_t idn = umma_idesc(1u, static_cast<uint32_t>(BP), 128u);  // Y: M 128 channels, N 128 positions
      const uint32_t ids = idn | (1u << 2);
      const uint32_t id1 = umma_idesc(1u, static_cast<uint32_t>(r1p), 128u);  // T1: M 128 positions, N R1p
      const uint32_t ring_s = smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 15));
      const uint64_t a_dense0 = umma_desc(smem_u32(smem), sw_t);
      const uint64_t a_sp0 = umma_desc(smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 16)), 64);
      const uint64_t ring0 = umma_desc(ring_s, 128);
      const uint64_t u0 = umma_desc(smem_u32(smem) + static_cast<uint32_t>(smem_param(prm + 19)), 128);
      const uint64_t t1b0 = umma_desc(t1s0, sw_t);
      const uint32_t slot16 = slot_bytes >> 4;
      const uint32_t dblk16 = (128u * sw_t) >> 4;
      const uint32_t ublk16 = (static_cast<uint32_t>(r1p) * 128u) >> 4;
      const int ksteps = static_cast<int>(sw_t / 32);
      int slot = 0;
      uint32_t ph = 0;
      uint32_t started[2] = {0u, 0u};  // per Y buffer: bit m = M-tile m holds a partial sum
      // X phase of tile k: per chunk the T1 MMAs (A = X chunk, B = U^T chunk) and the sparse
      // MMAs (A = 2:4 blocks, B = X chunk); T1 complete -> t1_full[b]
      auto x_phase = [&](int k) {
        const int b = k & 1, use = k >> 1;
        if (use > 0) {
          mbar_wait(&acc_empty[b], (use - 1) & 1);
          mbar_wait(&t1a_empty[b], (use - 1) & 1);
          tc_fence_after();
        }
        const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * acc_cols;
        const uint32_t t1acc = tmem + t1_col0 + static_cast<uint32_t>(b * r1p);
        started[b] = 0u;
        for (int c = 0; c < n_ck; ++c) {
          mbar_wait(&full[slot], ph);
          tc_fence_after();
          const uint64_t bd = ring0 + slot * slot16;
          const uint64_t ud = u0 + static_cast<uint32_t>(c) * ublk16;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16(t1acc, bd + 2 * kk, ud + 2 * kk, id1, (c | kk) ? 1u : 0u);
#pragma unroll
          for (int m = 0; m < MPC; ++m) {
            const uint32_t e = tab_s[m * kPMaxCk + c];
            const int b0 = static_cast<int>(e & 0xFFFu), nb = static_cast<int>(e >> 12);
            for (int bi = 0; bi < nb; ++bi) {
              const uint64_t ad = a_sp0 + static_cast<uint32_t>(b0 + bi) * (8192u >> 4);
              const uint32_t et = tmem + e_col0 + 4u * static_cast<uint32_t>(b0 + bi);
#pragma unroll
              for (int s2 = 0; s2 < 2; ++s2) {
                mma_sp_bf16(acc0 + static_cast<uint32_t>(m * BP), ad + 2 * s2, bd + 4 * s2,
                            ids | static_cast<uint32_t>(s2), (started[b] >> m) & 1u, et);
                started[b] |= 1u << m;
              }
            }
          }
          mma_commit(&empty[slot]);
          if (++slot == ns) {
            slot = 0;
            ph ^= 1u;
          }
        }
        mma_commit(&t1_full[b]);
      };
      // dense phase of tile k: Y += V^T T1 (B = the restaged T1 tile)
      auto dense_phase = [&](int k) {
        const int b = k & 1, use = k >> 1;
        mbar_wait(&t1s_full[b], use & 1);
        tc_fence_after();
        const uint32_t acc0 = tmem + static_cast<uint32_t>(b) * acc_cols;
        const uint64_t tb = t1b0 + static_cast<uint32_t>(b) * (t1s_bytes >> 4);
        for (int tk = 0; tk < n_tk; ++tk) {
#pragma unroll
          for (int m = 0; m < MPC; ++m) {
            const uint64_t ad = a_dense0 + static_cast<uint32_t>(m * n_tk + tk) * dblk16;
            for (int kk = 0; kk < ksteps; ++kk) {
              mma_bf16(acc0 + static_cast<uint32_t>(m * BP), ad + 2 * kk, tb + tk * dblk16 + 2 * kk, idn,
                       (started[b] >> m) & 1u);
              started[b] |= 1u << m;
            }
          }
        }
        mma_commit(&t1s_empty[b]);
        mma_commit(&acc_full[b]);
      };
      const int nt = li_ < n_pt ? (n_pt - 1 - li_) / gct + 1 : 0;
      if (nt > 0) x_phase(0);
      for (int k = 0; k < nt; ++k) {
        if (k + 1 < nt) x_phase(k + 1);
        dense_phase(k);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    const int q4 = warp & 3;            // TMEM lane quarter
    const int ehalf = (warp - 2) >> 2;  // Y: alternate 32-column chunks; T1: which half of the ranks
    const uint32_t scr0 = smem_u32(smem + p.off_epi) + static_cast<uint32_t>(warp - 2) * kPEpiScratch;
    const int relu = smem_param(prm + 10), cout = smem_param(prm + 11);
    const bool epi = p.epi != nullptr || relu;
    const int t1 = lane >> 2, mi = lane >> 3, mj = lane & 7;
    const int nt = li_ < n_pt ? (n_pt - 1 - li_) / gct + 1 : 0;
    // restage T1 of tile k: this thread owns position row = 32 q4 + lane and ranks
    // [ehalf * R1p/2, +R1p/2) in steps of 16: TMEM -> bf16 -> 16-byte swizzled stores
    auto restage = [&](int k) {
      const int b = k & 1, use = k >> 1;
      if (lane == 0) {
        mbar_wait(&t1_full[b], use & 1);
        if (use > 0) mbar_wait(&t1s_empty[b], (use - 1) & 1);
      }
      __syncwarp();
      tc_fence_after();
      const uint32_t row = static_cast<uint32_t>(q4 * 32 + lane);
      const uint32_t dst = t1s0 + static_cast<uint32_t>(b) * t1s_bytes;
      const int half = r1p / 2;
      for (int r0 = ehalf * half; r0 < (ehalf + 1) * half; r0 += 16) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q4 * 32) << 16) + t1_col0 + static_cast<uint32_t>(b * r1p + r0), v);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + 8 * h;  // 8 ranks = one 16-byte chunk
          const uint32_t tk = static_cast<uint32_t>(r) / (sw_t / 2), byte = (static_cast<uint32_t>(r) % (sw_t / 2)) * 2;
          const uint32_t chunk = ((byte >> 4) ^ ((row & 7u) / (128u / sw_t))) % (sw_t / 16);
          const uint32_t addr = dst + tk * 128u * sw_t + (row >> 3) * (8u * sw_t) + (row & 7u) * sw_t + chunk * 16u;
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pack_bf16x2(v[8 * h], v[8 * h + 1])),
                       "r"(pack_bf16x2(v[8 * h + 2], v[8 * h + 3])), "r"(pack_bf16x2(v[8 * h + 4], v[8 * h + 5])),
                       "r"(pack_bf16x2(v[8 * h + 6], v[8 * h + 7]))
                       : "memory");
        }
      }
      fence_proxy_async_smem();  // generic-proxy stores -> visible to the MMAs reading the tile
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&t1a_empty[b]);
        mbar_arrive(&t1s_full[b]);
      }
    };
    int nchunk = 0;
    auto drain = [&](int k, int pt) {
      const int b = k & 1, use = k >> 1;
      if (lane == 0) mbar_wait(&acc_full[b], use & 1);
      __syncwarp();
      tc_fence_after();
      const uint32_t acc0 = static_cast<uint32_t>(b) * acc_cols;
      const int p0 = pt * BP;
#pragma unroll 1
      for (int m = 0; m < MPC; ++m) {
        const int jw = (grp * MPC + m) * 128 + q4 * 32;
        if (jw >= cout) break;
        float2 sb[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          sb[h][0] = sb[h][1] = make_float2(1.f, 0.f);
          if (epi) {
            sb[h][0] = out_epi_load(p.epi, min(jw + 16 * h + t1, cout - 1));
            sb[h][1] = out_epi_load(p.epi, min(jw + 16 * h + t1 + 8, cout - 1));
          }
        }
#pragma unroll 1
        for (int c0 = ehalf * 32; c0 < BP; c0 += 64, ++nchunk) {
          uint32_t r[2][2][8];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int cb = 0; cb < 2; ++cb)
              tmem_ld_16x256b_x2(tmem + (static_cast<uint32_t>(q4 * 32 + 16 * h) << 16) + acc0 +
                                     static_cast<uint32_t>(m * BP + c0 + 16 * cb),
                                 r[h][cb]);
          const uint32_t scr = scr0 + static_cast<uint32_t>(nchunk & 1) * 2048u;
          if (lane == 0) bulk_wait_read1();
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
              const int scol = cb * 16 + (mi >> 1) * 8 + mj, spart = 2 * h + (mi & 1);
              const uint32_t addr = scr + static_cast<uint32_t>(scol * 64 + ((spart ^ ((scol >> 1) & 3)) * 16));
              stmatrix_x4_trans(addr, pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                pack_bf16x2(f[6], f[7]));
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&p.tmY, scr, jw, p0 + c0);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    };
    if (nt > 0) restage(0);
    for (int k = 0; k < nt; ++k) {
      if (k + 1 < nt) restage(k + 1);
      drain(k, li_ + k * gct);
    }
    if (lane == 0) bulk_wait0();
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
