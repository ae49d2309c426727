// lrs_decomp.cuh -- the low-rank + sparse DECOMPOSITION W ~ L + S on the GPU (
// PAPER.md:124-146 §3.2; oracle/lrs_decomp.py).  fp64 throughout (the ALS normal equations
// are solved by a pseudo-inverse with a 1e-10 relative cutoff).
//
// W is an order-4 tensor [I0][I1][I2][I3] (a conv weight: in, out, kh, kw) with I2*I3 <= 64;
// L is CP rank r: L = sum_r F0[:,r] o F1[:,r] o F2[:,r] o F3[:,r].  One iteration
// of the paper's two-step scheme:
//   1. ALS sweep on T = W - S (modes 0..3 in order):   M = MTTKRP(T, F, m)   lrs_mttkrp*_kernel
//                                                       V = *_{o != m} F_o^T F_o, P = V^+
//                                                                              lrs_sym_pinv_kernel
//                                                       F_m = M P             lrs_cp_update_kernel
//   2. Rsd = W - L  (L reconstructed on the fly)                              lrs_cp_residual_kernel
//   3. S = P_c(Rsd): the n = round(c numel) largest |Rsd| (ties: smaller index) by an exact
//      8-bit-digit radix select over the fp64 bit patterns of |Rsd| and an ordered compaction
//                                                       lrs_radix_hist_kernel / lrs_radix_pick_kernel /
//                                                       lrs_select_flags_kernel / scan / compact
//   4. T = W - S, eps = ||Rsd - S|| / ||W||                                    lrs_decomp_finish_kernel
// MTTKRP is a reduction over the other three modes; it is split over blocks and the partial
// sums are added in a fixed order (deterministic results: the same inputs give the same bits).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lrs {

constexpr int kDThreads = 256;

// ---------------------------------------------------------------- MTTKRP, modes 0 and 1
// M[i][r] = sum_j F_other[j][r] * sum_q T[i, j, q] KR23[q][r] where (i, j) = (i0, i1) for mode
// 0 and (i1, i0) for mode 1, q over the I2*I3 inner entries, KR23[q][r] = F2[q / I3][r] F3[q % I3][r].
// Block (i, chunk): threads over r, a chunk of j; partial sums part[chunk][i][r].
struct MttkrpParams {
  const double* t;         // [I0][I1][Q]
  const double* f[4];
  double* part;            // [nchunk][I_m][R]
  int dims[4];
  int q;                   // I2 * I3
  int r;                   // rank
  int mode;
  int nchunk, chunk;       // chunks of the reduced outer index
};

__global__ void __launch_bounds__(kDThreads) lrs_mttkrp01_kernel(const __grid_constant__ MttkrpParams p) {
  __shared__ double kr[64 * 256 / 4];  // KR23 for this block's r slice (<= 64 x 64) -- see below
  const int i = blockIdx.x;
  const int c = blockIdx.y;
  const int r0 = blockIdx.z * 64;       // r slice of 64 (4 warps x 2 ... threads = 256: 4 j-lanes x 64 r)
  const int rr = threadIdx.x & 63;
  const int jl = threadIdx.x >> 6;      // 0..3
  const int r = r0 + rr;
  const int I2 = p.dims[2], I3 = p.dims[3], Q = p.q;
  for (int e = threadIdx.x; e < Q * 64; e += kDThreads) {
    const int qq = e / 64, x = e % 64;
    const int rx = r0 + x;
    kr[e] = rx < p.r ? p.f[2][(qq / I3) * p.r + rx] * p.f[3][(qq % I3) * p.r + rx] : 0.0;
  }
  __syncthreads();
  (void)I2;
  const int n_other = p.mode == 0 ? p.dims[1] : p.dims[0];
  const double* fo = p.mode == 0 ? p.f[1] : p.f[0];
  const long long s_i = p.mode == 0 ? static_cast<long long>(p.dims[1]) * Q : Q;
  const long long s_j = p.mode == 0 ? Q : static_cast<long long>(p.dims[1]) * Q;
  const int j_begin = c * p.chunk, j_end = min(n_other, j_begin + p.chunk);
  double acc = 0.0;
  if (r < p.r) {
    for (int j = j_begin + jl; j < j_end; j += 4) {
      const double* tp = p.t + i * s_i + j * s_j;
      double inner = 0.0;
      for (int qq = 0; qq < Q; ++qq) inner = fma(__ldg(tp + qq), kr[qq * 64 + rr], inner);
      acc = fma(__ldg(fo + static_cast<long long>(j) * p.r + r), inner, acc);
    }
  }
  // the 4 j-lanes of one r: fixed-order sum through shared memory
  __syncthreads();
  double* red = kr;
  red[threadIdx.x] = acc;
  __syncthreads();
  if (jl == 0 && r < p.r) {
    const double s = ((red[rr] + red[64 + rr]) + red[128 + rr]) + red[192 + rr];
    p.part[(static_cast<long long>(c) * p.dims[p.mode] + i) * p.r + r] = s;
  }
}

// Register-blocked form for Q = QC in {1, 9} (1x1 and 3x3 kernels): a thread owns 4 ranks
// (rr, rr + 64, rr + 128, rr + 192) and keeps their KR23 columns in registers, so each
// broadcast load of T feeds 4 fp64 FMAs; one block covers every rank (R <= 256).  Same
// partial-sum layout and the same fixed-order lane combination as lrs_mttkrp01_kernel.
template <int QC>
__global__ void __launch_bounds__(kDThreads) lrs_mttkrp01q_kernel(const __grid_constant__ MttkrpParams p) {
  __shared__ double red[4][kDThreads];
  const int i = blockIdx.x;
  const int c = blockIdx.y;
  const int rr = threadIdx.x & 63;
  const int jl = threadIdx.x >> 6;
  const int I3 = p.dims[3];
  double kr[QC][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = rr + 64 * k;
#pragma unroll
    for (int qq = 0; qq < QC; ++qq)
      kr[qq][k] = r < p.r ? __ldg(p.f[2] + (qq / I3) * p.r + r) * __ldg(p.f[3] + (qq % I3) * p.r + r) : 0.0;
  }
  const int n_other = p.mode == 0 ? p.dims[1] : p.dims[0];
  const double* fo = p.mode == 0 ? p.f[1] : p.f[0];
  const long long s_i = p.mode == 0 ? static_cast<long long>(p.dims[1]) * QC : QC;
  const long long s_j = p.mode == 0 ? QC : static_cast<long long>(p.dims[1]) * QC;
  const int j_begin = c * p.chunk, j_end = min(n_other, j_begin + p.chunk);
  // stage this block's rows of T (the chunk's j x QC entries) in shared memory with all
  // threads (coalesced for mode 0; QC-element runs for mode 1): the per-j loads in the loop
  // below are then shared-memory broadcasts instead of a dependent global-load chain
  extern __shared__ double tsm[];
  const int nj = j_end - j_begin;
  for (int e = threadIdx.x; e < nj * QC; e += kDThreads) {
    const int jj = e / QC, qq = e - jj * QC;
    tsm[e] = __ldg(p.t + i * s_i + static_cast<long long>(j_begin + jj) * s_j + qq);
  }
  __syncthreads();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
  for (int j = j_begin + jl; j < j_end; j += 4) {
    const double* tp = tsm + (j - j_begin) * QC;
    double tv[QC];
#pragma unroll
    for (int qq = 0; qq < QC; ++qq) tv[qq] = tp[qq];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = rr + 64 * k;
      double inner = 0.0;
#pragma unroll
      for (int qq = 0; qq < QC; ++qq) inner = fma(tv[qq], kr[qq][k], inner);
      if (r < p.r) acc[k] = fma(__ldg(fo + static_cast<long long>(j) * p.r + r), inner, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  if (jl == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = rr + 64 * k;
      if (r >= p.r) continue;
      const double sum = ((red[k][rr] + red[k][64 + rr]) + red[k][128 + rr]) + red[k][192 + rr];
      p.part[(static_cast<long long>(c) * p.dims[p.mode] + i) * p.r + r] = sum;
    }
  }
}

// ---------------------------------------------------------------- MTTKRP, modes 2 and 3
// M[k][r] (mode 2) = sum_{i0,i1} F0[i0][r] F1[i1][r] sum_t T[i0,i1,k,t] F3[t][r]; mode 3 alike
// with (k, t) swapped.  Block (chunk of (i0, i1) pairs, r slice): per-thread registers for the
// <= 8 outputs, fixed-order combination of the 4 pair-lanes; partials part[chunk][I_m][R].
__global__ void __launch_bounds__(kDThreads) lrs_mttkrp23_kernel(const __grid_constant__ MttkrpParams p) {
  __shared__ double red[kDThreads * 8];
  const int c = blockIdx.x;
  const int r0 = blockIdx.z * 64;
  const int rr = threadIdx.x & 63;
  const int pl = threadIdx.x >> 6;
  const int r = r0 + rr;
  const int I2 = p.dims[2], I3 = p.dims[3], Q = p.q;
  const int nout = p.mode == 2 ? I2 : I3;
  const int nin = p.mode == 2 ? I3 : I2;
  const double* fin = p.mode == 2 ? p.f[3] : p.f[2];
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  const long long npairs = static_cast<long long>(p.dims[0]) * p.dims[1];
  const long long b = static_cast<long long>(c) * p.chunk;
  const long long e_end = min(npairs, b + p.chunk);
  // the chunk's rows of T (contiguous: pairs b .. e_end, Q entries each) staged in shared memory
  extern __shared__ double tsm2[];
  const long long nst = (e_end > b ? e_end - b : 0) * Q;
  for (long long e = threadIdx.x; e < nst; e += kDThreads) tsm2[e] = __ldg(p.t + b * Q + e);
  __syncthreads();
  if (r < p.r) {
    double fi[8];
    for (int t = 0; t < nin; ++t) fi[t] = __ldg(fin + t * p.r + r);
    for (long long pr = b + pl; pr < e_end; pr += 4) {
      const int i0 = static_cast<int>(pr / p.dims[1]), i1 = static_cast<int>(pr % p.dims[1]);
      const double g = __ldg(p.f[0] + static_cast<long long>(i0) * p.r + r) * __ldg(p.f[1] + static_cast<long long>(i1) * p.r + r);
      const double* tp = tsm2 + (pr - b) * Q;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < nout) {
          double s = 0.0;
          for (int t = 0; t < nin; ++t) {
            const int qq = p.mode == 2 ? k * I3 + t : t * I3 + k;
            s = fma(tp[qq], fi[t], s);
          }
          acc[k] = fma(g, s, acc[k]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[k * kDThreads + threadIdx.x] = acc[k];
  __syncthreads();
  if (pl == 0 && r < p.r) {
    for (int k = 0; k < nout; ++k) {
      const double* q = red + k * kDThreads;
      const double s = ((q[rr] + q[64 + rr]) + q[128 + rr]) + q[192 + rr];
      p.part[(static_cast<long long>(c) * nout + k) * p.r + r] = s;
    }
  }
}

// part[nchunk][rows][R] -> m[rows][R], chunks added in order
__global__ void lrs_part_sum_kernel(const double* part, int nchunk, long long count, double* m) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += part[c * count + i];
  m[i] = s;
}

// G[a][b] = sum_i F[i][a] F[i][b]  (one Gram matrix)
__global__ void lrs_gram_kernel(const double* f, int rows, int r, double* g) {
  const int a = blockIdx.x, b = threadIdx.x;
  if (b >= r) return;
  double s = 0.0;
  for (int i = 0; i < rows; ++i) s = fma(f[static_cast<long long>(i) * r + a], f[static_cast<long long>(i) * r + b], s);
  g[a * r + b] = s;
}

// ---------------------------------------------------------------- pseudo-inverse (one CTA)
// V = Hadamard product of the three Gram matrices of the other modes (SPD, R x R).  First a
// CERTIFIED Cholesky path (the inverse, when a norm bound proves no eigenvalue falls under the
// cutoff -- the usual case, ~20x cheaper); else the eigen path: cyclic
// Jacobi with the parallel (round-robin) ordering: each round rotates R/2 disjoint (p, q)
// pairs at once (one pass: every 2 x 2 block of a pair of pairs maps to itself, plus the
// eigenvector columns); sweeps until the
// off-diagonal mass is below (1e-13)^2 of the total (at most 40; sums in a fixed order, so the
// sweep count and the bits are deterministic).  A lives in shared memory when it fits
// (R <= 160), the (transposed) eigenvectors in the global workspace.
// P = Q diag(1/lambda for lambda > rcond * max |lambda|) Q^T.
struct PinvParams {
  const double* g[4];
  int mode;
  int r;       // rank
  int rp;      // rank rounded up to even (a dummy index pads odd ranks)
  int a_smem;  // 1: A in dynamic shared memory
  double rcond;
  double* a;   // workspace [rp][rp] (when A is not in shared memory)
  double* v;   // workspace [rp][rp]
  double* p;   // out [r][r]
  int* sweeps; // out (diagnostic)
  double* qt;  // [rp][rp] this mode's eigenvectors (transposed) from its previous call: in if warm, out always
  int warm;    // 1: start from A = Q^T V Q (the normal matrix changes little between sweeps)
  int force_eigen;  // 1: skip the certified Cholesky path (LRS_DECOMP_EIGEN; tests of the eigen path)
  const double* single;  // non-NULL: V = this matrix itself (g / mode unused) -- the Tucker-2 Gram Y^T Y
  int inv_sqrt;          // 1: P = Q diag(lambda^-1/2) Q^T (the Loewdin orthonormaliser; eigen path only)
  int chol_qr;           // 1 (with inv_sqrt): P = L^-T of V = L L^T (Cholesky-QR: Y P orthonormal) when every
                         // pivot exceeds rcond * max_i V_ii, else the Loewdin eigen path
};

constexpr int kJThreads = 512;

// the body, instantiated once with A in shared memory (so every access to it compiles to LDS /
// STS, not generic loads) and once with A in the global workspace
template <bool A_SMEM>
__device__ __forceinline__ void sym_pinv_body(const PinvParams& q, double* A) {
  __shared__ double cs[128][2];
  __shared__ int pairs[128][2];
  __shared__ double wsum[kJThreads / 32][2];
  __shared__ double offn, totn;
  const int n = q.rp, r = q.r;
  // A: the full matrix (shared memory when it fits, else the global workspace); the
  // eigenvectors are kept TRANSPOSED (Vt[k][i] = V[i][k]) so a rotation of columns p, q of V
  // touches two contiguous rows of Vt (coalesced / conflict-free)
  double* Vt = q.v;
  // ---- certified Cholesky path: when every eigenvalue of V exceeds rcond * lambda_max, the
  // pseudo-inverse IS the inverse.  V = L L^T (blocked, in place: lower triangle), X = L^-1
  // (strictly lower part kept TRANSPOSED in the free upper triangle, diagonal 1 / L_ii),
  // P = X^T X -- all in shared memory when A is.  Certificate: lambda_min >= 1 / ||P||_F and
  // lambda_max <= ||V||_F, so 1 / ||P||_F > rcond ||V||_F proves the cutoff drops nothing;
  // otherwise (or at a non-positive pivot) the Jacobi eigensolver below decides.
  if (!q.force_eigen && (!q.inv_sqrt || q.chol_qr)) {
    __shared__ int fail;
    __shared__ double vn2, piv_min;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* L = A;
    if (threadIdx.x == 0) fail = 0;
    double lv = 0.0, ld = 0.0;
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
      const int i = e / r, j = e % r;
      double val = 1.0;
      if (q.single)
        val = q.single[i * r + j];
      else
        for (int o = 0; o < 4; ++o)
          if (o != q.mode) val *= q.g[o][i * r + j];
      L[e] = val;
      lv += val * val;
      if (i == j) ld = fmax(ld, val);
    }
    for (int o = 16; o; o >>= 1) {
      lv += __shfl_xor_sync(0xffffffffu, lv, o);
      ld = fmax(ld, __shfl_xor_sync(0xffffffffu, ld, o));
    }
    if (lane == 0) {
      wsum[warp][0] = lv;
      wsum[warp][1] = ld;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0, dm = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
        t += wsum[w][0];
        dm = fmax(dm, wsum[w][1]);
      }
      vn2 = t;
      piv_min = q.chol_qr ? q.rcond * dm : 0.0;  // Cholesky-QR: a relative pivot floor (oracle orth_cholqr)
    }
    __syncthreads();
    constexpr int NB = 32;
    for (int kb = 0; kb < r; kb += NB) {
      const int nb = min(NB, r - kb);
      // (1) the diagonal block, by warp 0 (lane = row)
      if (warp == 0) {
        for (int k = 0; k < nb; ++k) {
          const int kk = kb + k;
          double d = L[kk * r + kk];
          const bool bad = !(d > piv_min);
          d = sqrt(fmax(d, 0.0));
          __syncwarp();
          if (lane == 0) {
            L[kk * r + kk] = d;
            if (bad) fail = 1;
          }
          if (lane > k && lane < nb) L[(kb + lane) * r + kk] /= d;
          __syncwarp();
          if (lane > k && lane < nb)
            for (int j = k + 1; j <= lane; ++j) L[(kb + lane) * r + kb + j] -= L[(kb + lane) * r + kk] * L[(kb + j) * r + kk];
          __syncwarp();
        }
      }
      __syncthreads();
      if (fail) break;
      // (2) the panel below: rows i >= kb + nb, L[i][kb:kb+nb] <- L[i][kb:kb+nb] L_kk^-T
      for (int i = kb + nb + threadIdx.x; i < r; i += blockDim.x) {
        for (int k = 0; k < nb; ++k) {
          double acc = L[i * r + kb + k];
          for (int m = 0; m < k; ++m) acc -= L[i * r + kb + m] * L[(kb + k) * r + kb + m];
          L[i * r + kb + k] = acc / L[(kb + k) * r + kb + k];
        }
      }
      __syncthreads();
      // (3) the trailing lower triangle: L[i][j] -= sum_m L[i][kb+m] L[j][kb+m]
      const int t0 = kb + nb, m = r - t0;
      for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int i = t0 + e / m, j = t0 + e % m;
        if (j > i) continue;
        double acc = 0.0;
        for (int mm = 0; mm < nb; ++mm) acc = fma(L[i * r + kb + mm], L[j * r + kb + mm], acc);
        L[i * r + j] -= acc;
      }
      __syncthreads();
    }
    if (!fail) {
      // X = L^-1: thread j computes column j; X[i][j] (i > j) is stored at L[j][i]
      for (int j = threadIdx.x; j < r; j += blockDim.x) {
        const double xjj = 1.0 / L[j * r + j];
        for (int i = j + 1; i < r; ++i) {
          double acc = L[i * r + j] * xjj;  // k = j term
          for (int k = j + 1; k < i; ++k) acc = fma(L[i * r + k], L[j * r + k], acc);
          L[j * r + i] = -acc / L[i * r + i];
        }
      }
      __syncthreads();
      if (q.chol_qr) {
        // P = X^T = L^-T (upper triangular): P[k][c] = X[c][k] for c >= k
        for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
          const int k = e / r, c = e % r;
          q.p[e] = c < k ? 0.0 : (c == k ? 1.0 / L[k * r + k] : L[k * r + c]);
        }
        if (q.qt)
          for (int e = threadIdx.x; e < n * n; e += blockDim.x) q.qt[e] = (e / n == e % n) ? 1.0 : 0.0;
        if (q.sweeps && threadIdx.x == 0) *q.sweeps = -2;  // diagnostic: Cholesky-QR
        return;
      }
      // P = X^T X: P[a][b] = sum_{k >= max(a, b)} X[k][a] X[k][b]
      double lp = 0.0;
      for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
        const int a = e / r, bb = e % r;
        if (bb < a) continue;
        auto xk = [&](int k, int c) { return k == c ? 1.0 / L[c * r + c] : L[c * r + k]; };  // X[k][c], k >= c
        double acc = 0.0;
        for (int k = bb; k < r; ++k) acc = fma(xk(k, a), xk(k, bb), acc);
        q.p[a * r + bb] = acc;
        q.p[bb * r + a] = acc;
        lp += (a == bb ? 1.0 : 2.0) * acc * acc;
      }
      for (int o = 16; o; o >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o);
      if (lane == 0) wsum[warp][1] = lp;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += wsum[w][1];
        if (!(1.0 / sqrt(t) > q.rcond * sqrt(vn2))) fail = 1;
      }
      __syncthreads();
      if (!fail) {
        // the mode's warm-start basis restarts from the identity (any orthogonal start is valid)
        if (q.qt)
          for (int e = threadIdx.x; e < n * n; e += blockDim.x) q.qt[e] = (e / n == e % n) ? 1.0 : 0.0;
        if (q.sweeps && threadIdx.x == 0) *q.sweeps = -1;  // diagnostic: the Cholesky path
        return;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    double val = 0.0;
    if (i < r && j < r) {
      val = 1.0;
      if (q.single)
        val = q.single[i * r + j];
      else
        for (int o = 0; o < 4; ++o)
          if (o != q.mode) val *= q.g[o][i * r + j];
    }
    A[e] = val;  // the dummy index of an odd rank: a zero row / column (eigenvalue 0, dropped)
    Vt[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  if (q.warm) {
    // warm start: A <- Q^T A Q with Q the previous eigenvectors of this mode (Vt <- Q^T), so
    // the rotations only have to remove the change since the last sweep
    const double* Qt = q.qt;
    double* T = q.a;  // the global workspace (A itself is in shared memory on this path)
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {  // T = A Q
      const int i = e / n, b = e % n;
      double acc = 0.0;
      for (int j = 0; j < n; ++j) acc = fma(A[i * n + j], Qt[b * n + j], acc);
      T[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {  // A = Q^T T
      const int a = e / n, b = e % n;
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc = fma(Qt[a * n + i], T[i * n + b], acc);
      Vt[e] = acc;  // staged (A is still read above by no one; T done)
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e % n;
      // symmetrise (the two triangles of Q^T A Q differ in rounding)
      A[e] = 0.5 * (Vt[e] + Vt[b * n + a]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Vt[e] = Qt[e];
    __syncthreads();
  }
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    // convergence: off-diagonal mass below (1e-13)^2 of the total (the round-off floor of an
    // n = 256 matrix is ~ (n 1e-16)^2; fixed-order sums)
    double lo = 0.0, lt = 0.0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const double x = A[e] * A[e];
      lt += x;
      if (e / n != e % n) lo += x;
    }
    for (int o = 16; o; o >>= 1) {
      lo += __shfl_xor_sync(0xffffffffu, lo, o);
      lt += __shfl_xor_sync(0xffffffffu, lt, o);
    }
    if ((threadIdx.x & 31) == 0) {
      wsum[threadIdx.x >> 5][0] = lo;
      wsum[threadIdx.x >> 5][1] = lt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sa = 0.0, sb = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
        sa += wsum[w][0];
        sb += wsum[w][1];
      }
      offn = sa;
      totn = sb;
    }
    __syncthreads();
    if (!(offn > 1e-26 * totn)) break;
    for (int round = 0; round < n - 1; ++round) {
      // pairs of this round (circle method: 0 fixed, the rest rotated by `round`)
      for (int k = threadIdx.x; k < n / 2; k += blockDim.x) {
        auto pos = [&](int i) { return i == 0 ? 0 : 1 + ((i - 1 + round) % (n - 1)); };
        int pp = pos(k), qq = pos(n - 1 - k);
        if (pp > qq) {
          const int t = pp;
          pp = qq;
          qq = t;
        }
        pairs[k][0] = pp;
        pairs[k][1] = qq;
        const double apq = A[pp * n + qq];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double theta = (A[qq * n + qq] - A[pp * n + pp]) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
        }
        cs[k][0] = c;
        cs[k][1] = s;
      }
      __syncthreads();
      // A <- P^T A P in ONE pass: the pairs are disjoint, so each 2 x 2 block (rows of pair a,
      // columns of pair b) maps to itself -- a' = J_a^T a J_b; and Vt <- P^T Vt (rows p, q)
      const int nh = n / 2;
      for (int e = threadIdx.x; e < nh * nh; e += blockDim.x) {
        const int ka = e / nh, kb = e % nh;
        const double ca = cs[ka][0], sa = cs[ka][1], cb = cs[kb][0], sb = cs[kb][1];
        if (sa == 0.0 && sb == 0.0) continue;
        const int pa = pairs[ka][0], qa = pairs[ka][1], pb = pairs[kb][0], qb = pairs[kb][1];
        const double x00 = A[pa * n + pb], x01 = A[pa * n + qb], x10 = A[qa * n + pb], x11 = A[qa * n + qb];
        const double r00 = ca * x00 - sa * x10, r01 = ca * x01 - sa * x11;
        const double r10 = sa * x00 + ca * x10, r11 = sa * x01 + ca * x11;
        A[pa * n + pb] = cb * r00 - sb * r01;
        A[pa * n + qb] = sb * r00 + cb * r01;
        A[qa * n + pb] = cb * r10 - sb * r11;
        A[qa * n + qb] = sb * r10 + cb * r11;
      }
      // Vt rows in global memory: all loads of a batch are issued before its stores (the
      // compiler cannot reorder them past possibly aliasing stores), so the L2 latency is paid
      // once per batch rather than once per element
      for (int e0 = threadIdx.x; e0 < nh * n; e0 += 8 * blockDim.x) {
        double vp[8], vq[8];
        int off_p[8], off_q[8];
        double cc[8], ss[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * blockDim.x;
          ss[u] = 0.0;
          if (e < nh * n) {
            const int k = e / n, i = e % n;
            ss[u] = cs[k][1];
            cc[u] = cs[k][0];
            off_p[u] = pairs[k][0] * n + i;
            off_q[u] = pairs[k][1] * n + i;
            if (ss[u] != 0.0) {
              vp[u] = Vt[off_p[u]];
              vq[u] = Vt[off_q[u]];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (ss[u] != 0.0) {
            Vt[off_p[u]] = cc[u] * vp[u] - ss[u] * vq[u];
            Vt[off_q[u]] = ss[u] * vp[u] + cc[u] * vq[u];
          }
        }
      }
      __syncthreads();
    }
  }
  // P = sum_k [lambda_k > rcond * max] V[:, k] V[:, k]^T / lambda_k
  __shared__ double lmax;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < n; ++k) m = fmax(m, fabs(A[k * n + k]));
    lmax = m;
    if (q.sweeps) *q.sweeps = sweep;
  }
  __syncthreads();
  __shared__ double inv[256];
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double lam = A[k * n + k];
    inv[k] = fabs(lam) > q.rcond * lmax ? (q.inv_sqrt ? 1.0 / sqrt(fabs(lam)) : 1.0 / lam) : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += Vt[k * n + i] * Vt[k * n + j] * inv[k];
    q.p[e] = s;
  }
  if (q.qt)
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) q.qt[e] = Vt[e];
}

__global__ void __launch_bounds__(kJThreads) lrs_sym_pinv_kernel(const __grid_constant__ PinvParams q) {
  extern __shared__ double jsm[];
  if (q.a_smem)
    sym_pinv_body<true>(q, jsm);
  else
    sym_pinv_body<false>(q, q.a);
}

// ---------------------------------------------------------------- strided batched fp64 GEMM
// C(b, m, n) = sum_k A(b, m, k) B(b, k, n) with arbitrary element strides (the Tucker-2 mode
// products and subspace steps: every operand is a view of a row-major tensor); C = sub - acc when
// `sub` is set (indexed like C: the residual W - L).  64 x 64 tiles, 256 threads x 4 x 4
// outputs (rows ty + 16 i, columns tx + 16 j), K-tiles of 16 through shared memory; each output
// sums its k in order (deterministic).
struct DgemmParams {
  const double* a;
  const double* b;
  double* c;
  const double* sub;
  int m, n, k;
  long long sam, sak, sab, sbk, sbn, sbb, scm, scn, scb;
};

__global__ void __launch_bounds__(256) lrs_dgemm_kernel(const __grid_constant__ DgemmParams p) {
  __shared__ double as[16][65], bs[16][65];
  const long long bz = blockIdx.z;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const double* A = p.a + bz * p.sab;
  const double* B = p.b + bz * p.sbb;
  const bool a_mfast = p.sam <= p.sak, b_nfast = p.sbn <= p.sbk;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < p.k; k0 += 16) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int kk = a_mfast ? e >> 6 : e & 15, mm = a_mfast ? e & 63 : e >> 4;
      const int gm = m0 + mm, gk = k0 + kk;
      as[kk][mm] = (gm < p.m && gk < p.k) ? A[gm * p.sam + gk * p.sak] : 0.0;
      const int kb = b_nfast ? e >> 6 : e & 15, nn = b_nfast ? e & 63 : e >> 4;
      const int gn = n0 + nn, gkb = k0 + kb;
      bs[kb][nn] = (gn < p.n && gkb < p.k) ? B[gkb * p.sbk + gn * p.sbn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double ar[4], br[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ar[i] = as[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) br[j] = bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(ar[i], br[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= p.n) continue;
      const long long o = bz * p.scb + gm * p.scm + gn * p.scn;
      p.c[o] = p.sub ? p.sub[o] - acc[i][j] : acc[i][j];
    }
  }
}

// F[i][c] = sum_k M[i][k] P[k][c]
__global__ void lrs_cp_update_kernel(const double* m, const double* pm, int rows, int r, double* f) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<long long>(rows) * r) return;
  const int i = static_cast<int>(e / r), c = static_cast<int>(e % r);
  double s = 0.0;
  for (int k = 0; k < r; ++k) s = fma(m[static_cast<long long>(i) * r + k], pm[k * r + c], s);
  f[e] = s;
}

// ---------------------------------------------------------------- residual Rsd = W - L
// block (i0, chunk of i1): the block's F0 row and the KR23 table in shared memory; thread per
// (i1, q) entry; L = sum_r F0[i0][r] F1[i1][r] KR23[q][r]
__global__ void __launch_bounds__(kDThreads) lrs_cp_residual_kernel(const double* w, const double* f0,
                                                                     const double* f1, const double* f2,
                                                                     const double* f3, int i1n, int i3n, int q,
                                                                     int r, double* rsd) {
  extern __shared__ double dsm[];
  double* f0r = dsm;         // [r]
  double* kr = dsm + r;      // [q][r]
  const int i0 = blockIdx.x;
  for (int e = threadIdx.x; e < r; e += blockDim.x) f0r[e] = f0[static_cast<long long>(i0) * r + e];
  __syncthreads();  // kr below reads f0r
  for (int e = threadIdx.x; e < q * r; e += blockDim.x) {
    const int qq = e / r, x = e % r;
    kr[e] = f2[(qq / i3n) * r + x] * f3[(qq % i3n) * r + x] * f0r[x];
  }
  __syncthreads();
  const long long row = static_cast<long long>(i1n) * q;
  for (long long e = static_cast<long long>(blockIdx.y) * blockDim.x + threadIdx.x; e < row;
       e += static_cast<long long>(gridDim.y) * blockDim.x) {
    const int i1 = static_cast<int>(e / q), qq = static_cast<int>(e % q);
    const double* fr = f1 + static_cast<long long>(i1) * r;
    const double* kq = kr + qq * r;
    double s = 0.0;
    for (int x = 0; x < r; ++x) s = fma(__ldg(fr + x), kq[x], s);
    const long long gi = static_cast<long long>(i0) * row + e;
    rsd[gi] = w[gi] - s;
  }
}

// ---------------------------------------------------------------- P_c: exact radix select
// keys = bit patterns of |Rsd| (non-negative doubles order like their uint64 bits).  State:
// st[0] = key prefix found so far, st[1] = its mask, st[2] = entries still needed among keys
// matching the prefix; st[3] = entries strictly above the final key (set by the last pick).
__global__ void lrs_radix_hist_kernel(const double* rsd, long long n, const unsigned long long* st, int shift,
                                      unsigned int* hist) {
  __shared__ unsigned int h[256];
  for (int e = threadIdx.x; e < 256; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const unsigned long long pre = st[0], mask = st[1];
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long k = static_cast<unsigned long long>(__double_as_longlong(fabs(rsd[i])));
    if ((k & mask) == pre) atomicAdd(&h[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += blockDim.x)
    if (h[e]) atomicAdd(&hist[e], h[e]);
}

// one thread: the digit (from the top) at which the count of larger keys reaches `need`
__global__ void lrs_radix_pick_kernel(unsigned long long* st, int shift, unsigned int* hist) {
  unsigned long long need = st[2];
  int d = 255;
  for (; d > 0; --d) {
    if (hist[d] >= need) break;
    need -= hist[d];
  }
  st[0] |= static_cast<unsigned long long>(d) << shift;
  st[1] |= 255ull << shift;
  st[2] = need;  // entries to take among keys equal to the final prefix
  for (int e = 0; e < 256; ++e) hist[e] = 0;
}

// flag[i] = 1 if |Rsd[i]| > K*, or == K* (the selected key) -- the latter count toward the
// ordered tie-break below; eq[i] = 1 for the ties
__global__ void lrs_select_flags_kernel(const double* rsd, long long n, const unsigned long long* st,
                                        unsigned int* gt, unsigned int* eq) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = static_cast<unsigned long long>(__double_as_longlong(fabs(rsd[i])));
  gt[i] = k > st[0] ? 1u : 0u;
  eq[i] = k == st[0] ? 1u : 0u;
}

// exclusive scan helpers (two levels; block = 1024 elements)
constexpr int kScanBlock = 1024;
__global__ void lrs_scan_block_kernel(const unsigned int* in, long long n, unsigned int* out, unsigned int* sums) {
  __shared__ unsigned int s[kScanBlock];
  const long long base = static_cast<long long>(blockIdx.x) * kScanBlock;
  for (int e = threadIdx.x; e < kScanBlock; e += blockDim.x) s[e] = base + e < n ? in[base + e] : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int acc = 0;
    for (int e = 0; e < kScanBlock; ++e) {
      const unsigned int v = s[e];
      s[e] = acc;
      acc += v;
    }
    sums[blockIdx.x] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kScanBlock; e += blockDim.x)
    if (base + e < n) out[base + e] = s[e];
}
__global__ void lrs_scan_sums_kernel(unsigned int* sums, int nb) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned int acc = 0;
    for (int b = 0; b < nb; ++b) {
      const unsigned int v = sums[b];
      sums[b] = acc;
      acc += v;
    }
  }
}

// selection + compaction in index order, T = W - S, and the residual mass of the entries
// S does not take (per-block partials, added in order by lrs_decomp_eps_kernel)
__global__ void lrs_decomp_finish_kernel(const double* w, const double* rsd, long long n,
                                         const unsigned long long* st, const unsigned int* gt,
                                         const unsigned int* eq, const unsigned int* eq_pre,
                                         const unsigned int* eq_sums, unsigned int* sel, double* t,
                                         double* eps_part) {
  __shared__ double red[kDThreads];
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  double rem = 0.0;
  if (i < n) {
    const unsigned long long take_eq = st[2];
    const unsigned int rank_eq = eq_pre[i] + eq_sums[i / kScanBlock];
    const bool s = gt[i] || (eq[i] && rank_eq < take_eq);
    sel[i] = s ? 1u : 0u;
    t[i] = s ? w[i] - rsd[i] : w[i];
    if (!s) rem = rsd[i] * rsd[i];
  }
  red[threadIdx.x] = rem;
  __syncthreads();
  for (int o = kDThreads / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) eps_part[blockIdx.x] = red[0];
}

__global__ void lrs_decomp_compact_kernel(const double* rsd, long long n, const unsigned int* sel,
                                          const unsigned int* pre, const unsigned int* sums, long long* idx,
                                          double* val) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !sel[i]) return;
  const unsigned int o = pre[i] + sums[i / kScanBlock];
  idx[o] = i;
  val[o] = rsd[i];
}

__global__ void lrs_decomp_eps_kernel(const double* part, int nb, double* out) {
  __shared__ double red[kDThreads];
  double s = 0.0;
  // fixed-order: thread t sums blocks t, t + 256, ... in order; then a fixed tree
  for (int b = threadIdx.x; b < nb; b += kDThreads) s += part[b];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kDThreads / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace lrs
