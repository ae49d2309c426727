// lrs_kernels.cuh -- sm_100a kernels of the compressed convolution Y = conv(X, L + S).
//
// One warp-specialised tcgen05 GEMM engine serves the three dense stages of
// the low-rank chain; its epilogue variant fuses the
// direct CSR sparse convolution (a4) and the final sum/store (a5):
//
//   a1  T1[p, a]  = sum_c X[p, c] U_in[c, a]   AMODE_2D,   EPI_STORE
//   a2  T2[p, b]  = sum_{y,x,a} T1[shift_yx(p), a] G[a,b,y,x] (Tucker-2 core)
//                   implicit GEMM: per tap one 4-D TMA box of T1 (OOB -> 0 = zero padding)
//                                                             AMODE_CONV, EPI_STORE
//   a3+a4+a5  Y[p, j] = sum_b T2[p, b] U_out[b, j]
//                     + sum_{e in row j} v_e X[p + off_e, c_e] (§3.4)
//                                                             AMODE_2D,   EPI_SPARSE
//
// CTA = 12 warps:  warp 0 lane 0  TMA producer (A and B K-chunks into an
// mbarrier ring);  warp 1  TMEM allocator, lane 0 MMA issuer (tcgen05.mma,
// M = 128, accumulator in TMEM, tcgen05.commit frees smem slots);  warps 2-3
// fp32 only: split every A stage into tf32 hi/lo (3xTF32, DESIGN.md reading
// #13);  warps 4-11 epilogue: EPI_STORE drains TMEM -> global rows;
// EPI_SPARSE first runs the CSR sparse term out of a channel-major,
// zero-padded shared-memory window of X (warp-uniform nonzeros, 4 pixels x
// BN/8 output channels per thread), then adds the TMEM accumulator and
// writes Y once.
#pragma once
#include "lrs_ptx.cuh"

namespace lrs {

constexpr int kThreads = 384;
constexpr int kTileM = 128;
enum { EPI_STORE = 0, EPI_SPARSE = 1 };
enum { AMODE_2D = 0, AMODE_CONV = 1 };

struct ConvGeom {
  int n;                 // images in this forward
  int h, w, ho, wo;      // input / output extent
  int kh, kw, sh, sw, ph, pw;
  int nb, th, tiles_h;   // AMODE_CONV tile = nb images x th output rows x all wo
};

struct SparseParams {
  const void* x;          // NHWC X (device)
  int cin;
  const int2* ent;        // (fp32 value bits, smem element offset c_local*wstride + y*wp + x)
  const int* ent_ptr;     // [(nchunk * n_cc + cc) * BN + j_local] -> first entry; +1 sentinel
  int cc;                 // channels per staged chunk (multiple of the 16-byte vector)
  int n_cc;               // number of channel chunks
  int wstride;            // elements per channel row of the window
  int wp;                 // window width in padded columns = (wo-1)*sw + kw
  void* y;                // NHWC Y (device)
  int cout;
  const float2* epi;      // per output channel (scale, bias) of the fused output epilogue, or NULL
  int relu;
};

struct GemmParams {
  CUtensorMap tmA;        // A: 2-D [rows][K] or 4-D NHWC (AMODE_CONV)
  CUtensorMap tmB;        // B: 2-D [N rows (x2: tf32 hi | lo)][K]
  int amode;
  int num_k_iters;        // K chunks in total
  int chunks_per_tap;     // AMODE_CONV: K chunks per kernel tap
  int kc;                 // elements per K chunk (= sw_bytes / elem size)
  uint32_t sw_bytes;      // 128 / 64 / 32: swizzle width = bytes per smem row
  int n_stages;
  int bn;                 // MMA N (columns of this CTA's accumulator)
  int b_lo_row;           // fp32: first row of the lo half of B
  uint32_t a_box_bytes;   // bytes one A TMA box delivers
  uint32_t a_stage_stride;
  uint32_t b_box_bytes;
  uint32_t b_stage_stride;  // per stage; fp32 holds hi box then lo box
  uint32_t tmem_cols;
  int m_total;            // AMODE_2D: valid rows
  ConvGeom g;
  void* out;              // EPI_STORE destination rows
  int out_ld;             // elements per destination row
  int out_cols;           // EPI_STORE: valid destination columns (0: all); N chunk c writes columns c*bn..
  uint32_t smem_sparse_off;
  uint32_t smem_bar_off;
  // 1: compute at once, wait for the previous kernel only before exiting (the projection of
  // a 1x1 SVD pair whose T1 alternates between two buffers; lrs_conv.cu forward_impl)
  int early;
  SparseParams sp;
};

template <bool F32>
struct Elem;
template <>
struct Elem<false> {
  using T = __nv_bfloat16;
  static constexpr int kVec = 8;  // elements per 16 bytes
  __device__ static float to_f(T v) { return __bfloat162float(v); }
};
template <>
struct Elem<true> {
  using T = float;
  static constexpr int kVec = 4;
  __device__ static float to_f(T v) { return v; }
};

// store 16 consecutive fp32 accumulator values as dtype
template <bool F32>
__device__ __forceinline__ void store16(void* dst, const float* v) {
  if constexpr (F32) {
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
    uint4 u[2];
    uint32_t* w = reinterpret_cast<uint32_t*>(u);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&b);
    }
    uint4* d = reinterpret_cast<uint4*>(dst);
    d[0] = u[0];
    d[1] = u[1];
  }
}

// Window of the sparse term for one 128-pixel output tile (AMODE_2D rows,
// linear NHWC output order): the padded input rows every image of the tile
// needs, laid out image after image, wp padded columns each.
struct TileWindow {
  int n_first, nt;
  int lo0, rows0;      // first image: first output row, padded rows
  int rows_full;       // middle images
  int lo_last, rows_last;
  int total_slots;
  __device__ __forceinline__ void init(int m0, const ConvGeom& g, int P) {
    const int howo = g.ho * g.wo;
    const int m_last = min(m0 + kTileM - 1, P - 1);
    n_first = m0 / howo;
    const int n_last = m_last / howo;
    nt = n_last - n_first + 1;
    lo0 = (m0 - n_first * howo) / g.wo;
    const int hi0 = nt == 1 ? (m_last - n_first * howo) / g.wo : g.ho - 1;
    rows0 = (hi0 - lo0) * g.sh + g.kh;
    rows_full = (g.ho - 1) * g.sh + g.kh;
    lo_last = 0;
    const int hi_last = (m_last - n_last * howo) / g.wo;
    rows_last = hi_last * g.sh + g.kh;
    if (nt == 1) {
      total_slots = rows0;
    } else {
      total_slots = rows0 + (nt - 2) * rows_full + rows_last;
    }
  }
  // first padded row (in input-row units + ph) of image t, and its slot base row
  __device__ __forceinline__ int lo(int t) const { return t == 0 ? lo0 : 0; }
  __device__ __forceinline__ int base_row(int t) const {
    return t == 0 ? 0 : rows0 + (t - 1) * rows_full;
  }
};

template <bool F32, int EPI, int BN_SP>
__global__ void __launch_bounds__(kThreads, 1) lrs_gemm_kernel(const __grid_constant__ GemmParams p) {
  using E = Elem<F32>;
  using T = typename E::T;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = p.n_stages;

  uint8_t* a_region = smem;
  uint8_t* alo_region = smem + S * p.a_stage_stride;            // fp32 only
  uint8_t* b_region = smem + (F32 ? 2 : 1) * S * p.a_stage_stride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar_off);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* ready = bars + 2 * S;
  uint64_t* tmem_full = bars + 3 * S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 1);

  // tile coordinates
  const int nchunk = blockIdx.y;
  int m0 = 0, n0 = 0, ho0 = 0;
  if (p.amode == AMODE_CONV) {
    n0 = (blockIdx.x / p.g.tiles_h) * p.g.nb;
    ho0 = (blockIdx.x % p.g.tiles_h) * p.g.th;
  } else {
    m0 = blockIdx.x * kTileM;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&p.tmA);
    tma_prefetch_desc(&p.tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue above overlapped the previous kernel's tail; from here on
  // we read its outputs (and overwrite buffers it may read)
  if (!p.early) pdl_wait();  // the previous kernel's output is visible from here on
  pdl_launch_dependents();  // (default: only after the wait, so every kernel before us is complete)

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      const uint32_t tx = p.a_box_bytes + (F32 ? 2u : 1u) * p.b_box_bytes;
      for (int it = 0; it < p.num_k_iters; ++it) {
        const int s = it % S;
        if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
        uint8_t* a_dst = a_region + s * p.a_stage_stride;
        uint8_t* b_dst = b_region + s * p.b_stage_stride;
        mbar_arrive_expect_tx(&full[s], tx);
        if (p.amode == AMODE_CONV) {
          const int tap = it / p.chunks_per_tap;
          const int ch = it - tap * p.chunks_per_tap;
          const int ty = tap / p.g.kw, tx_ = tap - ty * p.g.kw;
          tma_load_4d(a_dst, &p.tmA, &full[s], ch * p.kc, tx_ - p.g.pw, ho0 * p.g.sh - p.g.ph + ty, n0);
        } else {
          tma_load_2d(a_dst, &p.tmA, &full[s], it * p.kc, m0);
        }
        tma_load_2d(b_dst, &p.tmB, &full[s], it * p.kc, nchunk * p.bn);
        if constexpr (F32) {
          tma_load_2d(b_dst + (p.b_stage_stride >> 1), &p.tmB, &full[s], it * p.kc,
                      p.b_lo_row + nchunk * p.bn);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc = umma_idesc(F32 ? 2u : 1u, static_cast<uint32_t>(p.bn), kTileM);
      const int ksteps = static_cast<int>(p.sw_bytes / 32);
      for (int it = 0; it < p.num_k_iters; ++it) {
        const int s = it % S;
        const uint32_t ph = (it / S) & 1;
        mbar_wait(F32 ? &ready[s] : &full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(a_region + s * p.a_stage_stride);
        const uint32_t b_addr = smem_u32(b_region + s * p.b_stage_stride);
        for (int kk = 0; kk < ksteps; ++kk) {
          const uint64_t ad = umma_desc(a_addr + kk * 32, p.sw_bytes);
          const uint64_t bd = umma_desc(b_addr + kk * 32, p.sw_bytes);
          const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
          if constexpr (F32) {
            const uint32_t alo_addr = smem_u32(alo_region + s * p.a_stage_stride);
            const uint64_t adl = umma_desc(alo_addr + kk * 32, p.sw_bytes);
            const uint64_t bdl = umma_desc(b_addr + (p.b_stage_stride >> 1) + kk * 32, p.sw_bytes);
            mma_tf32(tmem, ad, bd, idesc, acc);   // hi * hi
            mma_tf32(tmem, adl, bd, idesc, 1u);   // lo * hi
            mma_tf32(tmem, ad, bdl, idesc, 1u);   // hi * lo
          } else {
            mma_bf16(tmem, ad, bd, idesc, acc);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
  } else {
    if constexpr (F32) {
      // ------------------------------------------------------------ tf32 hi/lo split
      // warps 2..11: the epilogue warps join the split (they are idle until the
      // accumulator is complete) -- with 2 warps the split was the mainloop's bottleneck
      const int t = threadIdx.x - 64;
      constexpr int nt = kThreads - 64;
      const int n16 = static_cast<int>((kTileM * p.sw_bytes) / 16);
      for (int it = 0; it < p.num_k_iters; ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        uint4* a = reinterpret_cast<uint4*>(a_region + s * p.a_stage_stride);
        uint4* alo = reinterpret_cast<uint4*>(alo_region + s * p.a_stage_stride);
        for (int i = t; i < n16; i += nt) {
          uint4 v = a[i];
          uint4 hi, lo;
          hi.x = v.x & 0xFFFFE000u; hi.y = v.y & 0xFFFFE000u;
          hi.z = v.z & 0xFFFFE000u; hi.w = v.w & 0xFFFFE000u;
          lo.x = __float_as_uint(__uint_as_float(v.x) - __uint_as_float(hi.x));
          lo.y = __float_as_uint(__uint_as_float(v.y) - __uint_as_float(hi.y));
          lo.z = __float_as_uint(__uint_as_float(v.z) - __uint_as_float(hi.z));
          lo.w = __float_as_uint(__uint_as_float(v.w) - __uint_as_float(hi.w));
          a[i] = hi;
          alo[i] = lo;
        }
        fence_proxy_async_smem();
        named_bar_sync(1, nt);
        if (t == 0) mbar_arrive(&ready[s]);
      }
    }
  }
  if (warp >= 4) {
    const int e = warp - 4;      // 0..7
    const int q = warp & 3;      // TMEM lane quarter this warp may access
    if constexpr (EPI == EPI_STORE) {
      // ------------------------------------------------------------ drain T rows
      mbar_wait(tmem_full, 0);
      tc_fence_after();
      const int m = q * 32 + lane;
      long long row = -1;
      if (p.amode == AMODE_CONV) {
        const int per_img = p.g.th * p.g.wo;
        const int nl = m / per_img;
        const int hl = (m - nl * per_img) / p.g.wo;
        const int wl = m - nl * per_img - hl * p.g.wo;
        const int n = n0 + nl, ho = ho0 + hl;
        if (nl < p.g.nb && n < p.g.n && ho < p.g.ho)
          row = (static_cast<long long>(n) * p.g.ho + ho) * p.g.wo + wl;
      } else {
        if (m0 + m < p.m_total) row = m0 + m;
      }
      T* out = reinterpret_cast<T*>(p.out) + nchunk * p.bn;
      const int nblk = p.bn / 16;
      const int cols = p.out_cols ? p.out_cols - nchunk * p.bn : p.bn;
      for (int cb = (e >> 2); cb < nblk; cb += 2) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + cb * 16, v);
        if (row < 0 || cb * 16 >= cols) continue;
        if (cb * 16 + 16 <= cols) {
          store16<F32>(out + row * p.out_ld + cb * 16, v);
        } else {
          for (int i = 0; cb * 16 + i < cols; ++i) out[row * p.out_ld + cb * 16 + i] = static_cast<T>(v[i]);
        }
      }
    } else {
      // ------------------------------------------- a4 sparse term + a5 sum and store
      constexpr int JW = BN_SP / 8;  // output channels per warp
      const SparseParams& sp = p.sp;
      const ConvGeom& g = p.g;
      const int P = g.n * g.ho * g.wo;
      const int tid = threadIdx.x - 128;  // 0..255
      T* xs = reinterpret_cast<T*>(smem + p.smem_sparse_off);
      TileWindow win;
      win.init(m0, g, P);
      const int howo = g.ho * g.wo;
      int qoff[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = m0 + lane + 32 * i;
        qoff[i] = 0;
        if (m < P) {
          const int n = m / howo;
          const int rem = m - n * howo;
          const int ho = rem / g.wo, wo = rem - (rem / g.wo) * g.wo;
          const int t = n - win.n_first;
          qoff[i] = (win.base_row(t) + (ho - win.lo(t)) * g.sh) * sp.wp + wo * g.sw;
        }
      }
      float acc[4][JW];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < JW; ++jj) acc[i][jj] = 0.f;

      const T* xg = reinterpret_cast<const T*>(sp.x);
      constexpr int V = E::kVec;
      const int gpc = sp.cc / V;  // 16-byte groups per pixel per chunk
      for (int cc = 0; cc < sp.n_cc; ++cc) {
        const int c0 = cc * sp.cc;
        // ---- stage X[window, c0:c0+cc] channel-major, zero-padded
        const int nwork = win.total_slots * sp.wp * gpc;
        for (int w = tid; w < nwork; w += 256) {
          const int slot = w / gpc;
          const int grp = w - slot * gpc;
          const int prow = slot / sp.wp;
          const int pcol = slot - prow * sp.wp;
          int t, r;
          if (prow < win.rows0) { t = 0; r = prow; }
          else {
            const int rr = prow - win.rows0;
            t = 1 + rr / win.rows_full;
            r = rr - (t - 1) * win.rows_full;
          }
          const int n = win.n_first + t;
          const int hi = win.lo(t) * g.sh + r - g.ph;
          const int wi = pcol - g.pw;
          const int ch = c0 + grp * V;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (hi >= 0 && hi < g.h && wi >= 0 && wi < g.w && ch < sp.cin)
            v = __ldg(reinterpret_cast<const uint4*>(
                xg + ((static_cast<long long>(n) * g.h + hi) * g.w + wi) * sp.cin + ch));
          const T* vv = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int u = 0; u < V; ++u) xs[(grp * V + u) * sp.wstride + slot] = vv[u];
        }
        named_bar_sync(2, 256);
        // ---- warp-uniform CSR rows: this warp's JW output channels
        const int* ptr = sp.ent_ptr + (static_cast<long long>(nchunk) * sp.n_cc + cc) * BN_SP + e * JW;
#pragma unroll
        for (int jj = 0; jj < JW; ++jj) {
          const int e0 = __ldg(ptr + jj), e1 = __ldg(ptr + jj + 1);
          for (int k = e0; k < e1; ++k) {
            const int2 en = __ldg(sp.ent + k);
            const float v = __int_as_float(en.x);
            const T* base = xs + en.y;
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i][jj] = fmaf(v, E::to_f(base[qoff[i]]), acc[i][jj]);
          }
        }
        named_bar_sync(2, 256);
      }
      // ---- a5: add the low-rank accumulator (TMEM) and write Y once
      mbar_wait(tmem_full, 0);
      tc_fence_after();
      float* yl = reinterpret_cast<float*>(smem + p.smem_sparse_off);  // [128][BN_SP + 1]
      constexpr int LD = BN_SP + 1;
      {
        const int m = q * 32 + lane;
        const int half = BN_SP / 2;
        for (int cb = 0; cb < half / 16; ++cb) {
          const int col = (e >> 2) * half + cb * 16;
          float v[16];
          tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + col, v);
#pragma unroll
          for (int u = 0; u < 16; ++u) yl[m * LD + col + u] = v[u];
        }
      }
      named_bar_sync(2, 256);
      T* yg = reinterpret_cast<T*>(sp.y);
      const int jbase = nchunk * BN_SP + e * JW;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ml = lane + 32 * i;
        const int m = m0 + ml;
        if (m >= P) continue;
        float out[JW];
#pragma unroll
        for (int jj = 0; jj < JW; ++jj)
          out[jj] = out_epi(yl[ml * LD + e * JW + jj] + acc[i][jj],
                            out_epi_load(sp.epi, min(jbase + jj, sp.cout - 1)), sp.relu);
        T* dst = yg + static_cast<long long>(m) * sp.cout + jbase;
#pragma unroll
        for (int b = 0; b < JW / 8; ++b) {
          if (jbase + 8 * b + 8 <= sp.cout) {
            if constexpr (F32) {
              float4* d = reinterpret_cast<float4*>(dst + 8 * b);
              d[0] = make_float4(out[8 * b], out[8 * b + 1], out[8 * b + 2], out[8 * b + 3]);
              d[1] = make_float4(out[8 * b + 4], out[8 * b + 5], out[8 * b + 6], out[8 * b + 7]);
            } else {
              uint4 u;
              uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
              for (int z = 0; z < 4; ++z) {
                __nv_bfloat162 bb = __floats2bfloat162_rn(out[8 * b + 2 * z], out[8 * b + 2 * z + 1]);
                w[z] = *reinterpret_cast<uint32_t*>(&bb);
              }
              *reinterpret_cast<uint4*>(dst + 8 * b) = u;
            }
          } else if (jbase + 8 * b < sp.cout) {
            for (int z = 0; z < 8 && jbase + 8 * b + z < sp.cout; ++z) {
              if constexpr (F32) dst[8 * b + z] = out[8 * b + z];
              else dst[8 * b + z] = __float2bfloat16_rn(out[8 * b + z]);
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
  }
  if (p.early) pdl_wait();  // completion of this grid still implies the previous kernel's
}

}  // namespace lrs
