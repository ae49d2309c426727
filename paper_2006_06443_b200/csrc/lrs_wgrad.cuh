// lrs_wgrad.cuh -- the weight-gradient contractions of the backward pass (
// PAPER.md:194-195 §3.5 "ordinary back-propagation"; oracle/lrs_backward.py).
//
// Every parameter gradient of W = U_in G U_out + S is a reduction over output (or input)
// positions q of a product of two position-major activations:
//
//   dU_out[b][j]     = sum_q T2[q][b]             dY[q][j]     (taps 1)
//   dG[a][b][tap]    = sum_q T1[shift_tap(q)][a]  dT2[q][b]    (taps k*k)
//   dU_in[c][a]      = sum_q X[q][c]              dT1[q][a]    (taps 1, input grid)
//   dW_S[tap][c][j]  = sum_q X[shift_tap(q)][c]   dY[q][j]     (taps k*k; gathered at S's support)
//
// i.e. C[tap][m][n] = sum_q A_tap[q][m] B[q][n] with BOTH operands M/N-contiguous
// ("MN-major" for tcgen05: the reduction index q is the strided one).  One grouped launch
// serves up to four such problems:
//
//   * CTA = 6 warps: warp 0 lane 0 TMA producer, warp 1 TMEM allocator + lane 0 MMA issuer,
//     warps 2-5 epilogue (one TMEM lane quarter each).  Persistent: one CTA per SM runs a
//     list of work items (problem, tap, M tile of 128, N tile of BN, K split -- a contiguous
//     range of position steps), the lists balanced at create (longest processing time first).
//   * A position step is one 4-D TMA box (64 channels x bw x bh x bi images) of each operand:
//     bw = the full row, bh x bi chosen so bw*bh*bi (the MMA K extent of the step, `kst`)
//     is a multiple of 16.  A's box is displaced by the tap (x - pad_w, y - pad_h); the
//     zero fill of out-of-bounds boxes is the convolution's zero padding, and B's boxes
//     past the last image / row are zero, so ragged tails contribute nothing.
//   * Each 64-channel box lands as kst rows of 128 bytes in the SWIZZLE_128B layout, which
//     is exactly the MN-major SW128 canonical layout of tcgen05 (8 K rows x 64 M/N elements
//     per atom): SBO = 1024 B between 8-row K groups, LBO = kst*128 B between the 64-wide
//     M/N atoms; instruction descriptor bits 15/16 select MN-major A / B.
//   * Accumulator fp32 [128 lanes][BN columns] in TMEM; the epilogue stores the split's
//     partial tile into a per-split slab (fp32); lrs_wgrad_reduce_kernel sums the splits in
//     a fixed order (deterministic) and scatters each gradient entry to its destination
//     (factor layouts, or S's value order for dW_S).
#pragma once
#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kGThreads = 192;
constexpr int kGMaxProblems = 4;

struct WgradProblem {
  CUtensorMap tmA;     // 4-D (C_A, W, H, N) bf16, box (64, bw, bh, bi), SWIZZLE_128B
  CUtensorMap tmB;     // 4-D (C_B, W, H, N) bf16, same box
  float* slab;         // [splits][taps][m_tiles*128][n_tiles*bn] fp32 partial sums
  long long split_stride;  // floats per split
  int taps, kw, pad_h, pad_w;
  int sh, sw;          // stride of the shifted operand A (its box samples every s positions)
  int m_tiles, n_tiles, bn;  // bn in {64, 128, 192, 256}
  int splits;
  int kst;             // positions per step (MMA K of one stage), multiple of 16
  int hsteps;          // row steps per image group: ceil(rows / bh)
  int bh, bi;          // rows / images per step
  int k_steps;         // position steps in total = image groups * hsteps
  uint32_t stage_bytes;  // (2 + bn/64) * kst * 128, 1024-aligned
};

// One work item = (problem, tile, K split); a persistent CTA runs the items of its list
// (items[item_ptr[cta] .. item_ptr[cta + 1]), balanced at create by longest-processing-time
// assignment) back to back: one continuous smem ring over all of its position steps, two
// TMEM accumulators (item i+1's MMAs overlap item i's epilogue).
struct WgradItem {
  uint16_t problem;
  uint16_t split;
  int tile;
};

struct WgradParams {
  WgradProblem pr[kGMaxProblems];
  int n_problems;
  int stages;              // ring depth (max stage_bytes over the problems per slot)
  uint32_t slot_bytes;
  const WgradItem* items;
  const int* item_ptr;     // [grid + 1]
};

// MN-major SWIZZLE_128B descriptor: atoms of 8 K rows x 128 B; lbo = bytes between
// 64-element M/N atoms, sbo = bytes between 8-row K groups
__device__ __forceinline__ uint64_t umma_desc_mn128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

struct WgradItemGeom {
  int pi, split, nt, mt, tap, ty, tx, k_begin, k_end;
};

__device__ __forceinline__ WgradItemGeom wgrad_item(const WgradParams& P, const WgradItem& it) {
  WgradItemGeom g;
  g.pi = it.problem;
  g.split = it.split;
  const WgradProblem& p = P.pr[g.pi];
  int tile = it.tile;
  g.nt = tile % p.n_tiles;
  tile /= p.n_tiles;
  g.mt = tile % p.m_tiles;
  g.tap = tile / p.m_tiles;
  g.ty = g.tap / p.kw;
  g.tx = g.tap - g.ty * p.kw;
  g.k_begin = static_cast<int>((static_cast<long long>(p.k_steps) * g.split) / p.splits);
  g.k_end = static_cast<int>((static_cast<long long>(p.k_steps) * (g.split + 1)) / p.splits);
  return g;
}

// PAIR = true: launched as clusters of 2 CTAs (cta_group::2).  A work item then covers TWO
// M tiles (256 rows): CTA rank r loads its own 128 rows of A and HALF of B's N columns
// (n0 + r * bn/2; tcgen05's pair form splits B along N), so per SM a stage moves (2 + bn/128)
// boxes instead of (2 + bn/64) for the same MACs; the leader (rank 0) issues the M = 256
// MMAs over both CTAs' shared memory, its full barriers count the peer's relayed arrival, its
// multicast commits release both rings and both accumulators; each CTA drains its own 128
// accumulator rows.  (Item tile index: ((tap * m_pairs + pair) * n_tiles + nt).)
template <bool PAIR>
__global__ void __launch_bounds__(kGThreads, 1) lrs_wgrad_kernel(const __grid_constant__ WgradParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = P.stages;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool lead = rank == 0;
  const int gid = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int i_begin = P.item_ptr[gid], i_end = P.item_ptr[gid + 1];

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * P.slot_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tmem_full = bars + 2 * S;       // [2]
  uint64_t* tmem_empty = bars + 2 * S + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

  if (threadIdx.x == 0) {
    const uint32_t nf = (PAIR && lead) ? 2u : 1u;  // + the peer relay's arrival
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], nf);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4 * nf);  // one arrival per epilogue warp (of both CTAs)
    }
    fence_mbar_init();
    for (int i = 0; i < P.n_problems; ++i) {
      tma_prefetch_desc(&P.pr[i].tmA);
      tma_prefetch_desc(&P.pr[i].tmB);
    }
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc2(tmem_slot, 512);
    else tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the recompute kernels before us wrote T1 / T2 / dT2 / dT1
  pdl_launch_dependents();

  auto geom = [&](const WgradItem& it) {
    WgradItemGeom g = wgrad_item(P, it);
    if (PAIR) {  // mt counted the M-tile PAIR: this CTA's tile is 2 mt + rank
      const WgradProblem& p = P.pr[g.pi];
      int tile = it.tile;
      g.nt = tile % p.n_tiles;
      tile /= p.n_tiles;
      const int m_pairs = p.m_tiles >> 1;
      g.mt = 2 * (tile % m_pairs) + static_cast<int>(rank);
      g.tap = tile / m_pairs;
      g.ty = g.tap / p.kw;
      g.tx = g.tap - g.ty * p.kw;
    }
    return g;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int q = 0;  // ring position over all of this CTA's position steps
      for (int ii = i_begin; ii < i_end; ++ii) {
        const WgradItemGeom g = geom(P.items[ii]);
        const WgradProblem& p = P.pr[g.pi];
        const uint32_t atom = static_cast<uint32_t>(p.kst) * 128u;
        const int nb_atoms = PAIR ? (p.bn >> 7) : (p.bn >> 6);  // B boxes this CTA loads
        const uint32_t tx_bytes = static_cast<uint32_t>(2 + nb_atoms) * atom;
        const int m0 = g.mt * 128;
        const int n0 = g.nt * p.bn + (PAIR ? static_cast<int>(rank) * (p.bn >> 1) : 0);
        for (int it = g.k_begin; it < g.k_end; ++it, ++q) {
          const int s = q % S;
          if (q >= S) mbar_wait(&empty[s], ((q / S) - 1) & 1);
          uint8_t* st = smem + s * P.slot_bytes;
          const int ig = it / p.hsteps;
          const int h0 = (it - ig * p.hsteps) * p.bh;
          const int img0 = ig * p.bi;
          mbar_arrive_expect_tx(&full[s], tx_bytes);
          tma_load_4d(st, &p.tmA, &full[s], m0, g.tx - p.pad_w, h0 * p.sh + g.ty - p.pad_h, img0);
          tma_load_4d(st + atom, &p.tmA, &full[s], m0 + 64, g.tx - p.pad_w, h0 * p.sh + g.ty - p.pad_h, img0);
          for (int b = 0; b < nb_atoms; ++b)
            tma_load_4d(st + (2 + b) * atom, &p.tmB, &full[s], n0 + 64 * b, 0, h0, img0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      if (PAIR && !lead) {
        // ---------------------------------------------------------- pair relay (rank 1)
        // every stage this CTA's producer lands is forwarded to the leader's full barrier
        int q = 0;
        for (int ii = i_begin; ii < i_end; ++ii) {
          const WgradItemGeom g = geom(P.items[ii]);
          for (int it = g.k_begin; it < g.k_end; ++it, ++q) {
            const int s = q % S;
            mbar_wait(&full[s], (q / S) & 1);
            mbar_arrive_remote(&full[s], 0);
          }
        }
      } else {
        // ---------------------------------------------------------- MMA issuer
        int q = 0;
        for (int ii = i_begin; ii < i_end; ++ii) {
          const int li = ii - i_begin;
          const int buf = li & 1;
          const WgradItemGeom g = geom(P.items[ii]);
          const WgradProblem& p = P.pr[g.pi];
          const uint32_t atom = static_cast<uint32_t>(p.kst) * 128u;
          // kind::f16, bf16 A/B, fp32 D, M = 128 (256 for the pair), N = bn, A and B MN-major
          const uint32_t idesc =
              umma_idesc(1u, static_cast<uint32_t>(p.bn), PAIR ? 256u : 128u) | (1u << 15) | (1u << 16);
          const int ksub = p.kst >> 4;
          const uint32_t acc_t = tmem + static_cast<uint32_t>(buf * 256);
          if (li >= 2) {  // the epilogue(s) drained this accumulator
            if (PAIR) mbar_wait_cluster(&tmem_empty[buf], ((li >> 1) - 1) & 1);
            else mbar_wait(&tmem_empty[buf], ((li >> 1) - 1) & 1);
          }
          tc_fence_after();
          for (int it = g.k_begin; it < g.k_end; ++it, ++q) {
            const int s = q % S;
            if (PAIR) mbar_wait_cluster(&full[s], (q / S) & 1);
            else mbar_wait(&full[s], (q / S) & 1);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(smem + s * P.slot_bytes);
            const uint32_t b_addr = a_addr + 2u * atom;
            for (int kk = 0; kk < ksub; ++kk) {
              const uint64_t ad = umma_desc_mn128(a_addr + kk * 2048u, atom, 1024u);
              const uint64_t bd = umma_desc_mn128(b_addr + kk * 2048u, atom, 1024u);
              const uint32_t accf = (it > g.k_begin || kk > 0) ? 1u : 0u;
              if (PAIR) mma_bf16_2(acc_t, ad, bd, idesc, accf);
              else mma_bf16(acc_t, ad, bd, idesc, accf);
            }
            if (PAIR) mma_commit_pair(&empty[s]);
            else mma_commit(&empty[s]);
          }
          if (PAIR) mma_commit_pair(&tmem_full[buf]);  // (an item without steps: arrives at once)
          else mma_commit(&tmem_full[buf]);
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int qd = warp & 3;  // TMEM lane quarter of this warp
    const int row = qd * 32 + lane;
    for (int ii = i_begin; ii < i_end; ++ii) {
      const int li = ii - i_begin;
      const int buf = li & 1;
      const WgradItemGeom g = geom(P.items[ii]);
      const WgradProblem& p = P.pr[g.pi];
      const bool any = g.k_end > g.k_begin;
      mbar_wait(&tmem_full[buf], (li >> 1) & 1);
      tc_fence_after();
      const int ld = p.n_tiles * p.bn;
      float* out = p.slab + g.split * p.split_stride +
                   (static_cast<long long>(g.tap) * p.m_tiles * 128 + g.mt * 128 + row) * ld + g.nt * p.bn;
      const uint32_t acc_t = tmem + static_cast<uint32_t>(buf * 256) + (static_cast<uint32_t>(qd * 32) << 16);
      for (int cb = 0; cb < p.bn; cb += 16) {
        float v[16];
        if (any) {
          tmem_ld16(acc_t + cb, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        float4* o = reinterpret_cast<float4*>(out + cb);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && !lead) mbar_arrive_remote(&tmem_empty[buf], 0);
        else mbar_arrive(&tmem_empty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // neither CTA frees TMEM / leaves while the pair still works
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    if (PAIR) tmem_dealloc2(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}

// Zero insertion for the adjoint of a strided convolution: up[n][h][w][:] = src[n][h/s][w/s][:]
// when s divides h and w (and the source position exists), else 0.  16-byte vectors.
__global__ void lrs_zero_insert_kernel(const uint4* src, uint4* up, int n, int hs, int ws, int hu, int wu, int sh,
                                       int sw, int cv /* 16-byte vectors per position */) {
  const long long total = static_cast<long long>(n) * hu * wu * cv;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % cv);
    long long r = e / cv;
    const int w = static_cast<int>(r % wu);
    r /= wu;
    const int hh = static_cast<int>(r % hu);
    const long long img = r / hu;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (hh % sh == 0 && w % sw == 0 && hh / sh < hs && w / sw < ws)
      v = src[((img * hs + hh / sh) * ws + w / sw) * cv + c];
    up[e] = v;
  }
}

// The CP core kind's factor gradients from the embedded dense core's gradient (PAPER.md:158:
// G[a][b][y][x] = [a == b] B[y][a] C[x][a]):  dB[y][r] = sum_x dG[r][r][y][x] C[x][r],
// dC[x][r] = sum_y dG[r][r][y][x] B[y][r].  out = [dB (kh x R) ; dC (kw x R)], the core
// array's layout.  Fixed-order sums.
__global__ void lrs_cp_core_grad_kernel(const float* dg, const float* b, const float* c, int r, int kh, int kw,
                                        float* out) {
  for (int e = threadIdx.x; e < (kh + kw) * r; e += blockDim.x) {
    const int t = e / r, q = e - (e / r) * r;
    const float* dq = dg + (static_cast<long long>(q) * r + q) * kh * kw;  // dG[q][q][.][.]
    float acc = 0.f;
    if (t < kh) {
      for (int x = 0; x < kw; ++x) acc = fmaf(dq[t * kw + x], c[x * r + q], acc);
    } else {
      const int x = t - kh;
      for (int y = 0; y < kh; ++y) acc = fmaf(dq[y * kw + x], b[y * r + q], acc);
    }
    out[e] = acc;
  }
}

// dst[i] = sum_{s < splits} slab[s * split_stride + idx[i]] (fixed order: deterministic);
// one launch covers every gradient of the backward (concatenated index tables).
struct WgradReduceParams {
  const float* slab;
  long long split_stride;
  int splits;
  const long long* idx;
  float* dst;
  int count;
};

constexpr int kGRThreads = 256;

struct WgradReduceSet {
  WgradReduceParams r[kGMaxProblems];
  int n;
  int block_base[kGMaxProblems + 1];
};

__global__ void __launch_bounds__(kGRThreads) lrs_wgrad_reduce_kernel(const __grid_constant__ WgradReduceSet R) {
  int pi = 0;
  for (int i = 1; i < R.n; ++i)
    if (static_cast<int>(blockIdx.x) >= R.block_base[i]) pi = i;
  const WgradReduceParams& r = R.r[pi];
  pdl_wait();
  pdl_launch_dependents();
  const int i = (static_cast<int>(blockIdx.x) - R.block_base[pi]) * kGRThreads + threadIdx.x;
  if (i >= r.count) return;
  const long long off = r.idx[i];
  float acc = 0.f;
  for (int s = 0; s < r.splits; ++s) acc += __ldg(r.slab + s * r.split_stride + off);
  r.dst[i] = acc;
}

}  // namespace lrs
