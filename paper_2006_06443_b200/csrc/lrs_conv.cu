// lrs_conv.cu -- host side of the C-ABI declared in include/lrs_conv.h:
// descriptor validation, weight repacking (rank padding, K-major tiles,
// tf32 hi/lo split, per-tile sparse code streams), TMA descriptor encoding,
// kernel launches and stage timing.  See DESIGN.md for the data layout.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/lrs_conv.h"
#include "lrs_kernels.cuh"
#include "lrs_core.cuh"
#include "lrs_cpdw.cuh"
#include "lrs_spadd.cuh"
#include "lrs_tiny.cuh"
#include "lrs_wconv.cuh"
#include "lrs_pw.cuh"
#include "lrs_pwf.cuh"
#include "lrs_wgrad.cuh"
#include "lrs_decomp.cuh"

using namespace lrs;

namespace {

thread_local std::string g_err;

lrs_status fail(lrs_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define LRS_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? LRS_ERR_OUT_OF_MEMORY : LRS_ERR_CUDA, \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);    \
  } while (0)

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

CUtensorMapSwizzle swz(uint32_t sw) {
  return sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                   : (sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// rank-r tensor map; dims/strides innermost first (strides in bytes, r-1 of them);
// sw = 0 means no swizzle
lrs_status encode_t(CUtensorMap* m, CUtensorMapDataType dt, int rank, void* ptr, const uint64_t* dims,
                    const uint64_t* strides, const uint32_t* box, const uint32_t* estr, uint32_t sw) {
  PFN_encodeTiled fn = get_encode();
  if (!fn) return fail(LRS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUresult r = fn(m, dt, rank, ptr, reinterpret_cast<const cuuint64_t*>(dims),
                  reinterpret_cast<const cuuint64_t*>(strides), box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  sw == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE : swz(sw), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LRS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d, rank %d)", (int)r, rank);
  return LRS_OK;
}
lrs_status encode(CUtensorMap* m, bool f32, int rank, void* ptr, const uint64_t* dims,
                  const uint64_t* strides, const uint32_t* box, const uint32_t* estr, uint32_t sw) {
  return encode_t(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, ptr, dims,
                  strides, box, estr, sw);
}

inline int round_up(int a, int b) { return (a + b - 1) / b * b; }
inline uint32_t align1024(uint32_t a) { return (a + 1023u) & ~1023u; }
inline uint32_t pow2_cols(int n) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(n)) c <<= 1;
  return c;
}
// widest swizzle (128/64/32 B) that divides a K extent of `bytes`
uint32_t pick_sw(int bytes) {
  if (bytes >= 128) return 128;
  if (bytes >= 64) return 64;
  return 32;
}

constexpr int kMaxSmem = 232448;  // 227 KB dynamic shared memory per CTA on sm_100

enum KernelId { K_STORE_BF16, K_STORE_F32, K_SP64_BF16, K_SP128_BF16, K_SP64_F32, K_SP128_F32 };

const void* kernel_ptr(KernelId id) {
  switch (id) {
    case K_STORE_BF16: return reinterpret_cast<const void*>(&lrs_gemm_kernel<false, EPI_STORE, 0>);
    case K_STORE_F32: return reinterpret_cast<const void*>(&lrs_gemm_kernel<true, EPI_STORE, 0>);
    case K_SP64_BF16: return reinterpret_cast<const void*>(&lrs_gemm_kernel<false, EPI_SPARSE, 64>);
    case K_SP128_BF16: return reinterpret_cast<const void*>(&lrs_gemm_kernel<false, EPI_SPARSE, 128>);
    case K_SP64_F32: return reinterpret_cast<const void*>(&lrs_gemm_kernel<true, EPI_SPARSE, 64>);
    case K_SP128_F32: return reinterpret_cast<const void*>(&lrs_gemm_kernel<true, EPI_SPARSE, 128>);
  }
  return nullptr;
}

// fused TC kernel instantiation for an exact MMA unit count
// (pair: the CTA-pair form, 1 or 2 units)
const void* wconv_kernel_ptr(int nu, int bpi, bool pair = false) {
#define LRS_WK(U) (bpi == 4 ? reinterpret_cast<const void*>(&lrs_wconv_kernel<U, 4, false>) \
                            : reinterpret_cast<const void*>(&lrs_wconv_kernel<U, 2, false>))
  if (pair) {
    if (nu == 1) return bpi == 4 ? reinterpret_cast<const void*>(&lrs_wconv_kernel<1, 4, true>)
                                 : reinterpret_cast<const void*>(&lrs_wconv_kernel<1, 2, true>);
    return bpi == 4 ? reinterpret_cast<const void*>(&lrs_wconv_kernel<2, 4, true>)
                    : reinterpret_cast<const void*>(&lrs_wconv_kernel<2, 2, true>);
  }
  switch (nu) {
    case 1: return LRS_WK(1);
    case 2: return LRS_WK(2);
    case 3: return LRS_WK(3);
    case 4: return LRS_WK(4);
    case 5: return LRS_WK(5);
    case 6: return LRS_WK(6);
    case 7: return LRS_WK(7);
    default: return LRS_WK(8);
  }
#undef LRS_WK
}

// channel-stationary 1x1 kernel instantiation for mpc M-tiles per CTA (ft: projection fused)
const void* pwf_kernel_ptr(int mpc) {
  switch (mpc) {
    case 1: return reinterpret_cast<const void*>(&lrs_pwf_kernel<1>);
    case 2: return reinterpret_cast<const void*>(&lrs_pwf_kernel<2>);
    case 3: return reinterpret_cast<const void*>(&lrs_pwf_kernel<3>);
    default: return reinterpret_cast<const void*>(&lrs_pwf_kernel<4>);
  }
}
const void* pw_kernel_ptr(int mpc) {
  switch (mpc) {
    case 1: return reinterpret_cast<const void*>(&lrs_pw_kernel<1>);
    case 2: return reinterpret_cast<const void*>(&lrs_pw_kernel<2>);
    case 3: return reinterpret_cast<const void*>(&lrs_pw_kernel<3>);
    default: return reinterpret_cast<const void*>(&lrs_pw_kernel<4>);
  }
}

struct Stage {
  const char* name;
  KernelId kid;
  GemmParams p;
  uint32_t smem;
  int tiles_per_image_or_rows;  // unused helper
};

struct TimingRing {
  std::vector<cudaEvent_t> ev;  // pairs
  int used = 0;
  double ms = 0.0;
  long long count = 0;
};

}  // namespace

// one plan of the channel-stationary 1x1 kernel (build_pw; timed by autotune_pw)
struct PwPlan {
  int mpc = 0, bp = 0, ns = 0, nblk = 0, gpg = 0, ft = 0, epi_nbuf = 2, cpi = 1;
  uint32_t smem = 0, w_bytes = 0;
  double cost = 1e300;
};

struct lrs_conv {
  lrs_conv_desc d;
  int device = 0;
  int sms = 148;
  bool f32 = false, svd = false;
  int esz = 2;
  int ho = 0, wo = 0;
  int r1p = 0, r2p = 0, cout_p = 0, bn = 0;
  // device buffers
  void* w_uin = nullptr;   // [R1p (x2)][Cin]
  void* w_core = nullptr;  // [R2p (x2)][k*k*R1p]
  void* w_uout = nullptr;  // [Cout_p (x2)][R2p or R1p]
  void* t1 = nullptr;
  void* t2 = nullptr;
  int2* ent = nullptr;
  int* ent_ptr = nullptr;
  // stages
  Stage a1{}, a2{}, a3{};
  int kc_a1 = 0;
  uint32_t sw_a1 = 0;
  // X map cache
  const void* xmap_ptr = nullptr;
  int xmap_n = -1;
  CUtensorMap xmap{};
  // host-io staging (lrs_conv_forward_host): device buffers, copy streams, chunk events
  void* hx = nullptr;
  void* hy = nullptr;
  cudaStream_t hs_in = nullptr, hs_out = nullptr;
  cudaEvent_t hev[18] = {};  // [0..7] H2D done, [8..15] forward done, [16] start, [17] D2H done
  // timing
  bool timing = false;
  int skip = 0;  // timing experiments only (LRS_SKIP at create): 1 a1, 2 a2, 4 a3/fused, 8 a4 split
  TimingRing ring[4];
  // fused a3+a4+a5 on the tensor cores (lrs_wconv.cuh), bf16 layers
  bool use_w = false;
  // 1x1 SVD-pair layers: channel-stationary fused a3 + a4 + a5 (lrs_pw.cuh)
  bool use_pw = false;
  bool pw_ft = false;         // ... with the projection a1 fused in (lrs_pwf.cuh): one launch, T1 on chip
  void* pw_u = nullptr;       // U_in^T image of the fused projection
  PwParams pp{};
  uint32_t pw_smem = 0;
  int pw_grid_per_group = 0;  // CTAs per channel group at most
  std::vector<PwPlan> pw_cands;  // the cost model's best few plans (autotune_pw times them)
  int force_wth = 0;             // autotune_w: the band height the windowed kernel's planner must take
  int wth_max = 0;               // the tallest band height the planner found feasible
  void* pw_w = nullptr;       // per-group weight images
  void* pw_e = nullptr;       // per-group metadata images
  void* pw_tab = nullptr;     // per-group block tables
  const void* px_ptr = nullptr;
  int px_n = -1;
  const void* py_ptr = nullptr;
  int py_n = -1;
  WconvParams wp{};
  uint32_t w_smem = 0;
  void* w_as = nullptr;   // compressed 2:4 blocks of S (SW64 shared-memory images)
  void* w_dense_img = nullptr;  // U_out^T blocks (shared-memory images)
  // early-start protocol (core -> fused kernel): T2 and G alternate between two
  // buffers per forward so the next forward's kernels may start while this one finishes
  bool dbuf = false;
  int par = 0;                  // buffer parity of the next forward
  void* t2b = nullptr;          // second T2
  void* t1b = nullptr;          // second T1 (projection -> pointwise kernel)
  bool dbuf_pw = false;         // the early-start protocol on the projection -> pointwise chain
  bool no_early = false;        // LRS_NO_EARLY at create
  CUtensorMap tmT_pw_par[2];    // the pointwise kernel's T1 maps, per buffer
  void* w_gb = nullptr;         // second overflow-gather scratch
  CUtensorMap tmT_par[2], tmG_par[2];
  void* w_gtab = nullptr;       // overflow-gather slot table (WconvParams::g_tab)
  void* w_g = nullptr;          // overflow-gather scratch G
  std::vector<uint8_t> w_ovf;   // build-time: overflow-value blocks
  void* w_e = nullptr;    // their metadata
  int* w_res = nullptr;   // residual block table
  const void* wx_ptr = nullptr;
  int wx_n = -1;
  const void* wy_ptr = nullptr;
  int wy_n = -1;
  int w_main_blocks = 0, w_res_blocks = 0;
  // fp32 layers: a3 GEMM stores Y_L, then the SIMT gather kernel adds Y_S (lrs_spadd.cuh)
  bool use_spadd = false;
  SpaddParams spp{};
  uint32_t sp_smem = 0;
  int2* sp_ent = nullptr;
  int* sp_ptr = nullptr;
  float* sp_uo = nullptr;  // U_out fp32 [R2p][Cout] for the SIMT expansion
  // small fp32 layers: the whole layer in one SIMT kernel (lrs_tiny.cuh)
  bool use_tiny = false;
  TinyParams tp{};
  uint32_t tiny_smem = 0;
  void* tiny_buf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  float2* epi = nullptr;  // fused output epilogue: (scale, bias) per output channel
  // CP core (the paper's form): stages 2-3 as two depthwise convs
  bool cp_core = false;
  float* w_cpb = nullptr;  // [kh][R1p] vertical taps
  float* w_cpc = nullptr;  // [kw][R1p] horizontal taps
  CpDwParams cpp{};
  // bf16 Tucker-2 stride-1 layers: a1 + a2 in one kernel (lrs_core.cuh), T1 stays on chip
  bool use_core = false;
  CoreParams cp{};
  uint32_t core_smem = 0;
  int core_grid = 0;  // CTAs of the core kernel (persistent over its tiles)
  const void* cx_ptr = nullptr;
  int cx_n = -1;
};

namespace {

lrs_status validate(const lrs_conv_desc* d) {
  if (!d) return fail(LRS_ERR_INVALID_ARGUMENT, "desc is NULL");
  if (d->batch_max <= 0 || d->in_h <= 0 || d->in_w <= 0 || d->c_in <= 0 || d->c_out <= 0 ||
      d->kernel_h <= 0 || d->kernel_w <= 0 || d->rank_in <= 0 || d->rank_out <= 0)
    return fail(LRS_ERR_INVALID_ARGUMENT, "all extents must be > 0");
  if (d->stride_h < 1 || d->stride_w < 1) return fail(LRS_ERR_INVALID_ARGUMENT, "stride < 1");
  if (d->pad_h < 0 || d->pad_w < 0) return fail(LRS_ERR_INVALID_ARGUMENT, "pad < 0");
  if (d->dtype != LRS_DTYPE_F32 && d->dtype != LRS_DTYPE_BF16)
    return fail(LRS_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)d->dtype);
  const int ho = (d->in_h + 2 * d->pad_h - d->kernel_h) / d->stride_h + 1;
  const int wo = (d->in_w + 2 * d->pad_w - d->kernel_w) / d->stride_w + 1;
  if (d->in_h + 2 * d->pad_h < d->kernel_h || d->in_w + 2 * d->pad_w < d->kernel_w || ho < 1 || wo < 1)
    return fail(LRS_ERR_INVALID_ARGUMENT, "output extent < 1");
  if (!d->u_in || !d->u_out) return fail(LRS_ERR_INVALID_ARGUMENT, "u_in / u_out is NULL");
  if (d->core_kind != LRS_CORE_TUCKER2 && d->core_kind != LRS_CORE_CP)
    return fail(LRS_ERR_INVALID_ARGUMENT, "unknown core_kind %d", (int)d->core_kind);
  if (d->core_kind == LRS_CORE_CP && (!d->core || d->rank_in != d->rank_out))
    return fail(LRS_ERR_INVALID_ARGUMENT, "a CP core needs core != NULL and rank_in == rank_out");
  if (!d->core) {
    if (d->kernel_h != 1 || d->kernel_w != 1 || d->stride_h != 1 || d->stride_w != 1 ||
        d->pad_h != 0 || d->pad_w != 0)
      return fail(LRS_ERR_INVALID_ARGUMENT, "core == NULL (SVD pair) needs a 1x1, stride 1, pad 0 layer");
    if (d->rank_in != d->rank_out)
      return fail(LRS_ERR_INVALID_ARGUMENT, "core == NULL (SVD pair) needs rank_in == rank_out");
  }
  if (d->nnz < 0) return fail(LRS_ERR_INVALID_ARGUMENT, "nnz < 0");
  if (!d->row_ptr) return fail(LRS_ERR_INVALID_ARGUMENT, "row_ptr is NULL");
  if (d->nnz > 0 && (!d->col_idx || !d->values))
    return fail(LRS_ERR_INVALID_ARGUMENT, "col_idx / values is NULL");
  if (d->row_ptr[0] != 0 || d->row_ptr[d->c_out] != d->nnz)
    return fail(LRS_ERR_INVALID_ARGUMENT, "row_ptr must start at 0 and end at nnz");
  const int64_t ncol = static_cast<int64_t>(d->c_in) * d->kernel_h * d->kernel_w;
  for (int j = 0; j < d->c_out; ++j) {
    if (d->row_ptr[j + 1] < d->row_ptr[j])
      return fail(LRS_ERR_INVALID_ARGUMENT, "row_ptr not monotone at row %d", j);
    for (int64_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) {
      const int32_t c = d->col_idx[e];
      if (c < 0 || c >= ncol) return fail(LRS_ERR_INVALID_ARGUMENT, "col_idx out of range at %lld", (long long)e);
      if (e > d->row_ptr[j] && c <= d->col_idx[e - 1])
        return fail(LRS_ERR_INVALID_ARGUMENT, "columns of row %d not strictly increasing", j);
    }
  }
  // ---- legal but not implemented
  if (d->kernel_h > 7 || d->kernel_w > 7) return fail(LRS_ERR_UNSUPPORTED, "kernel > 7");
  if (d->rank_in > 256 || d->rank_out > 256) return fail(LRS_ERR_UNSUPPORTED, "rank > 256");
  const int vec = d->dtype == LRS_DTYPE_BF16 ? 8 : 4;
  if (d->c_in % vec || d->c_out % vec)
    return fail(LRS_ERR_UNSUPPORTED, "c_in and c_out must be multiples of %d", vec);
  // rows wider than 128 outputs: only the bf16 kernels that band the columns (the fused
  // core, the windowed / pointwise expansion kernels, the CP depthwise kernel) take them;
  // layers that would need the GEMM core convolution are refused after planning
  if (wo > 256) return fail(LRS_ERR_UNSUPPORTED, "output width > 256");
  if (wo > 128 && (d->dtype != LRS_DTYPE_BF16 || d->c_in % 64 != 0))
    return fail(LRS_ERR_UNSUPPORTED, "output width > 128 needs a bf16 layer with c_in %% 64 == 0");
  if (wo * d->stride_w > 256 || d->stride_h * std::min(ho, 128) > 256)
    return fail(LRS_ERR_UNSUPPORTED, "TMA box too wide");
  return LRS_OK;
}

// host value of element i of a dtype array
inline float host_val(const void* a, size_t i, bool f32) {
  if (f32) return static_cast<const float*>(a)[i];
  uint32_t b = static_cast<uint32_t>(static_cast<const uint16_t*>(a)[i]) << 16;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

// pack `rows` x `k` fp32 matrix into the device dtype; fp32 -> [hi rows ; lo rows]
std::vector<uint8_t> pack_matrix(const std::vector<float>& m, int rows, int k, bool f32) {
  std::vector<uint8_t> out;
  if (f32) {
    out.resize(static_cast<size_t>(2) * rows * k * 4);
    float* o = reinterpret_cast<float*>(out.data());
    for (size_t i = 0; i < static_cast<size_t>(rows) * k; ++i) {
      uint32_t b;
      memcpy(&b, &m[i], 4);
      b &= 0xFFFFE000u;
      float hi;
      memcpy(&hi, &b, 4);
      o[i] = hi;
      o[static_cast<size_t>(rows) * k + i] = m[i] - hi;
    }
  } else {
    out.resize(static_cast<size_t>(rows) * k * 2);
    uint16_t* o = reinterpret_cast<uint16_t*>(out.data());
    for (size_t i = 0; i < static_cast<size_t>(rows) * k; ++i) {
      uint32_t b;
      memcpy(&b, &m[i], 4);  // values are bf16-exact (copied from bf16 input)
      o[i] = static_cast<uint16_t>(b >> 16);
    }
  }
  return out;
}

lrs_status upload(void** dst, const std::vector<uint8_t>& h) {
  LRS_CUDA(cudaMalloc(dst, std::max<size_t>(h.size(), 16)));
  if (!h.empty()) LRS_CUDA(cudaMemcpy(*dst, h.data(), h.size(), cudaMemcpyHostToDevice));
  return LRS_OK;
}

// Fill the common GEMM stage fields; returns smem bytes (0 if it does not fit)
uint32_t plan_stage(GemmParams& p, bool f32, int k_bytes_total, uint32_t sw, int bn, int b_lo_row,
                    uint32_t a_box_bytes, uint32_t sparse_bytes) {
  const int esz = f32 ? 4 : 2;
  p.sw_bytes = sw;
  p.kc = static_cast<int>(sw) / esz;
  p.num_k_iters = (k_bytes_total + static_cast<int>(sw) - 1) / static_cast<int>(sw);
  p.bn = bn;
  p.b_lo_row = b_lo_row;
  p.a_box_bytes = a_box_bytes;
  p.a_stage_stride = align1024(kTileM * sw);
  p.b_box_bytes = static_cast<uint32_t>(bn) * sw;
  p.b_stage_stride = align1024(p.b_box_bytes) * (f32 ? 2u : 1u);
  p.tmem_cols = pow2_cols(bn);
  int S = std::min(4, p.num_k_iters);
  for (; S >= 1; --S) {
    uint32_t off = S * p.a_stage_stride * (f32 ? 2u : 1u) + S * p.b_stage_stride;
    off = (off + 15u) & ~15u;
    const uint32_t sparse_off = off;
    off += sparse_bytes;
    off = (off + 15u) & ~15u;
    const uint32_t bar_off = off;
    off += 8u * (3u * S + 1u) + 16u;
    const uint32_t total = off + 1024u;
    if (total <= static_cast<uint32_t>(kMaxSmem)) {
      p.n_stages = S;
      p.smem_sparse_off = sparse_off;
      p.smem_bar_off = bar_off;
      return total;
    }
  }
  return 0;
}

// Every kernel is launched with programmatic stream serialization (PDL): it may
// start while the previous kernel in the stream drains; the kernels call
// griddepcontrol.wait after their prologue (barrier init, TMEM alloc,
// descriptor prefetch) and before touching memory.  Captured into CUDA graphs
// as programmatic edges.
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void* param, size_t smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  #ifdef LRS_EXPERIMENTS
  static const bool no_pdl = getenv("LRS_NO_PDL") != nullptr;  // timing experiments
#else
  constexpr bool no_pdl = false;
#endif
  cfg.numAttrs = no_pdl ? 0 : 1;
  void* args[] = {param};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// the same with clusters of 2 CTAs (the windowed kernel's CTA-pair form)
cudaError_t launch_pdl_pair(const void* fn, dim3 grid, dim3 block, void* param, size_t smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  void* args[] = {param};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// event pair around one launch of stage `si` when timing is on
lrs_status time_begin(lrs_conv* h, int si, cudaStream_t stream, cudaEvent_t* e1) {
  *e1 = nullptr;
  if (!h->timing) return LRS_OK;
  TimingRing& r = h->ring[si];
  if (r.used + 2 > static_cast<int>(r.ev.size())) {
    const size_t old = r.ev.size();
    r.ev.resize(old + 512);
    for (size_t i = old; i < r.ev.size(); ++i) LRS_CUDA(cudaEventCreate(&r.ev[i]));
  }
  *e1 = r.ev[r.used + 1];
  LRS_CUDA(cudaEventRecord(r.ev[r.used], stream));
  r.used += 2;
  return LRS_OK;
}

lrs_status launch(lrs_conv* h, int si, Stage& st, dim3 grid, cudaStream_t stream) {
  cudaEvent_t e1 = nullptr;
  lrs_status s = time_begin(h, si, stream, &e1);
  if (s != LRS_OK) return s;
  LRS_CUDA(launch_pdl(kernel_ptr(st.kid), grid, dim3(kThreads), &st.p, st.smem, stream));
  if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
  return LRS_OK;
}


inline uint16_t bf16_bits_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Small fp32 Tucker-2 layers: the four stages in one SIMT kernel when the weights and one
// output row's window fit in shared memory and the grid (images x row bands) is small --
// the regime where the chain's three dependent launches are pure latency (C1).
lrs_status build_tiny(lrs_conv* h, const lrs_conv_desc* d) {
  if (!h->f32 || h->svd || getenv("LRS_NO_TINY")) return LRS_OK;
  const int cin = d->c_in, cout = d->c_out, kh = d->kernel_h, kw = d->kernel_w;
  const int ho = h->ho, wo = h->wo, sh = d->stride_h, sw = d->stride_w;
  const int r1 = d->rank_in, r2 = d->rank_out;
  const int r1p = round_up(r1, 4), r2p = round_up(r2, 4), taps = kh * kw;
  auto a16 = [](uint32_t b) { return (b + 15u) & ~15u; };
  {  // small layers only: some row band height keeps whole-width CTAs within two waves
    int th0 = 1;
    while (th0 <= ho && static_cast<long long>(d->batch_max) * ((ho + th0 - 1) / th0) > 2LL * h->sms) ++th0;
    if (th0 > ho) return LRS_OK;
  }
  // CTA = image x th output rows x tc output columns.  Pick the tile minimising waves x
  // per-CTA FMAs (the halo is recomputed: a1 runs on the (th + k - 1) x (tc + k - 1)
  // window); a CTA's stages are serial, so at batch 1 (C1) small tiles spread the layer
  // over more SMs.
  const uint32_t us = a16(static_cast<uint32_t>(cin) * r1p * 4);
  const bool cp = h->cp_core;
  const uint32_t gs = a16(static_cast<uint32_t>(cp ? (kh + kw) * r1p : taps * r1p * r2p) * 4);
  const uint32_t uo = a16(static_cast<uint32_t>(r2p) * cout * 4);
  const uint32_t rpb = a16(static_cast<uint32_t>(cout + 1) * 4);
  const uint32_t eb = a16(static_cast<uint32_t>(std::max<int64_t>(d->nnz, 1)) * 4);
  const uint32_t fixed_b = us + gs + uo + rpb + 2 * eb;
  auto tile_bytes = [&](int th_, int tc_, uint32_t* xs_, uint32_t* t1_, uint32_t* t2_) {
    const int wr_ = (th_ - 1) * sh + kh, wc_ = (tc_ - 1) * sw + kw;
    *xs_ = a16(static_cast<uint32_t>(cin) * wr_ * wc_ * 4);
    *t1_ = a16(static_cast<uint32_t>(wr_) * wc_ * r1p * 4);
    *t2_ = a16(static_cast<uint32_t>(th_) * tc_ * r2p * 4);
    return *xs_ + *t1_ + *t2_ + fixed_b;
  };
  const int cb_env = getenv("LRS_TINY_CB") ? atoi(getenv("LRS_TINY_CB")) : 0;  // planner experiments
  double best = 1e300;
  int th = 0, tcb = 0;
  for (int th_ = 1; th_ <= ho; ++th_) {
    for (int cb = 1; cb <= wo; ++cb) {
      if (cb_env && cb != cb_env) continue;
      const int tc_ = (wo + cb - 1) / cb;
      if ((wo + tc_ - 1) / tc_ != cb) continue;
      uint32_t xs_, t1_, t2_;
      const uint32_t tot = tile_bytes(th_, tc_, &xs_, &t1_, &t2_);
      if (tot > static_cast<uint32_t>(kMaxSmem) - 1024u) continue;
      const long long ctas = static_cast<long long>(d->batch_max) * ((ho + th_ - 1) / th_) * cb;
      const int per_sm = 1;  // 512 threads x ~96 registers: one CTA per SM
      if (ctas > 2LL * h->sms * per_sm) continue;  // at most two waves
      const long long waves = (ctas + static_cast<long long>(h->sms) * per_sm - 1) / (static_cast<long long>(h->sms) * per_sm);
      const int wr_ = (th_ - 1) * sh + kh, wc_ = (tc_ - 1) * sw + kw;
      const double fma = static_cast<double>(wr_) * wc_ * r1p * cin +
                         static_cast<double>(th_) * tc_ * (cp ? kw * (kh + 1) * r1p : taps * r1p * r2p) +
                         static_cast<double>(th_) * tc_ * (static_cast<double>(r2p) * cout + static_cast<double>(d->nnz));
      const double cost = static_cast<double>(waves) * (fma / kTyThreads + 1500.0);  // + per-CTA load latency
      if (cost < best * 0.999) {
        best = cost;
        th = th_;
        tcb = tc_;
      }
    }
  }
  if (!th) return LRS_OK;
  const int wr = (th - 1) * sh + kh;
  const int wc = (tcb - 1) * sw + kw;
  TinyParams& q = h->tp;
  memset(&q, 0, sizeof(q));
  uint32_t xs, t1, t2;
  const uint32_t total = tile_bytes(th, tcb, &xs, &t1, &t2);
  if (cin % 4 || cout % 4) return LRS_OK;
  q.off_t1 = xs; q.off_t2 = xs + t1; q.off_u = xs + t1 + t2; q.off_g = q.off_u + us; q.off_uo = q.off_g + gs;
  q.off_rp = q.off_uo + uo; q.off_ec = q.off_rp + rpb; q.off_ev = q.off_ec + eb;
  q.nnz = static_cast<int>(d->nnz);
  const bool f32 = true;
  std::vector<float> u(static_cast<size_t>(cin) * r1p, 0.f),
      g(static_cast<size_t>(cp ? (kh + kw) * r1p : taps * r1p * r2p), 0.f), o(static_cast<size_t>(r2p) * cout, 0.f);
  for (int c = 0; c < cin; ++c)
    for (int a = 0; a < r1; ++a) u[static_cast<size_t>(c) * r1p + a] = host_val(d->u_in, (size_t)c * r1 + a, f32);
  if (cp) {  // core = B [kh][R] then C [kw][R] (include/lrs_conv.h LRS_CORE_CP)
    for (int y = 0; y < kh + kw; ++y)
      for (int a = 0; a < r1; ++a) g[static_cast<size_t>(y) * r1p + a] = host_val(d->core, (size_t)y * r1 + a, f32);
  } else {
    for (int a = 0; a < r1; ++a)
      for (int b = 0; b < r2; ++b)
        for (int t = 0; t < taps; ++t)
          g[(static_cast<size_t>(t) * r1p + a) * r2p + b] = host_val(d->core, ((size_t)a * r2 + b) * taps + t, f32);
  }
  for (int b = 0; b < r2; ++b)
    for (int j = 0; j < cout; ++j) o[static_cast<size_t>(b) * cout + j] = host_val(d->u_out, (size_t)b * cout + j, f32);
  std::vector<int> rp(static_cast<size_t>(cout) + 1), ec(static_cast<size_t>(std::max<int64_t>(d->nnz, 1)), 0);
  std::vector<float> ev(ec.size(), 0.f);
  for (int j = 0; j <= cout; ++j) rp[j] = static_cast<int>(d->row_ptr[j]);
  for (int64_t e = 0; e < d->nnz; ++e) {
    const int col = d->col_idx[e], c = col / taps, t = col % taps;
    ec[e] = c | ((t / kw) << 16) | ((t % kw) << 24);
    ev[e] = d->values[e];
  }
  auto up = [&](void** dst, const void* src, size_t bytes) {
    std::vector<uint8_t> b(bytes);
    memcpy(b.data(), src, bytes);
    return upload(dst, b);
  };
  lrs_status st;
  if ((st = up(&h->tiny_buf[0], u.data(), u.size() * 4)) != LRS_OK) return st;
  if ((st = up(&h->tiny_buf[1], g.data(), g.size() * 4)) != LRS_OK) return st;
  if ((st = up(&h->tiny_buf[2], o.data(), o.size() * 4)) != LRS_OK) return st;
  if ((st = up(&h->tiny_buf[3], rp.data(), rp.size() * 4)) != LRS_OK) return st;
  if ((st = up(&h->tiny_buf[4], ec.data(), ec.size() * 4)) != LRS_OK) return st;
  if ((st = up(&h->tiny_buf[5], ev.data(), ev.size() * 4)) != LRS_OK) return st;
  q.uin = static_cast<const float*>(h->tiny_buf[0]);
  q.g = static_cast<const float*>(h->tiny_buf[1]);
  q.uo = static_cast<const float*>(h->tiny_buf[2]);
  q.rp = static_cast<const int*>(h->tiny_buf[3]);
  q.ent_c = static_cast<const int*>(h->tiny_buf[4]);
  q.ent_v = static_cast<const float*>(h->tiny_buf[5]);
  q.h = d->in_h; q.w = d->in_w; q.cin = cin; q.ho = ho; q.wo = wo; q.cout = cout;
  q.kh = kh; q.kw = kw; q.sh = sh; q.sw = sw; q.ph = d->pad_h; q.pw = d->pad_w;
  q.r1p = r1p; q.r2p = r2p; q.th = th; q.bands = (ho + th - 1) / th; q.wr = wr; q.wc = wc;
  q.tc = tcb; q.cbands = (wo + tcb - 1) / tcb;
  q.cp = cp ? 1 : 0;
  h->tiny_smem = total;
  h->use_tiny = true;
  if (getenv("LRS_VERBOSE"))
    fprintf(stderr, "[lrs] tiny: th=%d bands=%d tc=%d cbands=%d wr=%d wc=%d smem=%u\n", th, q.bands, tcb, q.cbands, wr,
            wc, total);
  return LRS_OK;
}

// a1 + a2 fused (lrs_core.cuh).  A plan is (ipt images per tile, th output rows per
// tile, grid): tile = ipt images x th rows, within TMEM (max(T1, T2) columns <= 512) and
// shared memory (X ring >= 2 slots, G ring >= 2 slots, the T1 window).  The model cost
// is waves x bytes a tile moves into shared memory (its X windows + the U_in and G
// chunks it streams); autotune_core then times the best few plans on the device.
struct CoreGeom {
  int cin, kh, kw, ho, wo, wc, r1p, r2p, g_kc, taps, n_g;
  bool cp;
  uint32_t u_bytes, g_bytes, g_slot, avail;
};

static CoreGeom core_geom(const lrs_conv* h, const lrs_conv_desc* d) {
  CoreGeom G;
  G.cin = d->c_in; G.kh = d->kernel_h; G.kw = d->kernel_w; G.ho = h->ho; G.wo = h->wo;
  G.wc = h->wo + G.kw - 1; G.r1p = h->r1p; G.r2p = h->r2p;
  G.g_kc = G.r1p % 64 == 0 ? 64 : (G.r1p % 32 == 0 ? 32 : 16);
  G.taps = G.kh * G.kw;
  G.cp = h->cp_core;
  G.n_g = G.cp ? 0 : G.taps * (G.r1p / G.g_kc);  // the CP form has no dense core to stream
  G.u_bytes = static_cast<uint32_t>(G.r1p) * 128u;
  G.g_bytes = G.cp ? 0u : static_cast<uint32_t>(G.r2p * G.g_kc * 2);
  G.g_slot = align1024(G.g_bytes);
  G.avail = static_cast<uint32_t>(kMaxSmem) - 1024u - 2048u;  // alignment slack, barriers
  return G;
}

// Shared-memory layout of one (ipt, th): X ring (ns_x slots), G ring (ns_g), T1 window.
// gmode 0: G resident when it fits (one X slot less if needed); 1: G streamed through a
// small ring so the X ring is as deep as the tile's chunks (X boxes arrive earlier).
static bool core_layout(const CoreGeom& G, int ipt, int th, CoreParams& q, int gmode = 0) {
  const int wr = th + G.kh - 1, p1 = wr * G.wc;
  if (wr > 256) return false;
  q.nb1 = (ipt * p1 + 127) / 128;
  q.nb2 = ((ipt - 1) * p1 + (th - 1) * G.wc + G.wo + 127) / 128;
  q.acc_cols = static_cast<uint32_t>(std::max(q.nb1 * G.r1p, q.nb2 * G.r2p));
  if (q.acc_cols > 512) return false;
  q.t1_rows = static_cast<uint32_t>((q.nb2 * 128 + (G.kh - 1) * G.wc + G.kw - 1 + 7) & ~7);
  const uint32_t t1_bytes = align1024(q.t1_rows * static_cast<uint32_t>(G.r1p) * 2u);
  q.x_bytes = static_cast<uint32_t>(ipt * wr * G.wc) * 128u;
  q.u_off = align1024(q.x_bytes);
  q.x_slot = q.u_off + G.u_bytes;
  // the last M block of the last X slot reads up to nb1 * 16 KB from the slot start
  const uint32_t x_tail =
      static_cast<uint32_t>(q.nb1) * 16384u > q.x_slot ? static_cast<uint32_t>(q.nb1) * 16384u - q.x_slot : 0u;
  if (t1_bytes + x_tail + 2 * q.x_slot + 2 * G.g_slot > G.avail) return false;
  const uint32_t left = G.avail - t1_bytes - x_tail;
  const int n_ck = G.cin / 64;
  // all X chunks of a tile if possible, then as much of G as fits (all of it: resident)
  q.ns_x = std::min(kCMaxX, std::max(2, n_ck));
  while (q.ns_x > 2 && q.ns_x * q.x_slot + 2 * G.g_slot > left) --q.ns_x;
  q.ns_g = G.n_g == 0 ? 0
                      : static_cast<int>(std::min<uint32_t>(static_cast<uint32_t>(std::min(kCMaxG, G.n_g)),
                                                            (left - q.ns_x * q.x_slot) / G.g_slot));
  if (gmode == 1 && G.n_g > 0) {
    q.ns_x = std::min(kCMaxX, std::max(2, n_ck));
    while (q.ns_x > 2 && q.ns_x * q.x_slot + 2 * G.g_slot > left) --q.ns_x;
    q.ns_g = static_cast<int>(std::min<uint32_t>(std::min<uint32_t>(4u, static_cast<uint32_t>(G.n_g)),
                                                 (left - q.ns_x * q.x_slot) / G.g_slot));
  } else if (q.ns_g < G.n_g) {  // prefer a resident G over a full X ring when one X slot less makes room
    const int ns_x2 = std::max(2, q.ns_x - 1);
    if (G.n_g <= kCMaxG && static_cast<uint32_t>(ns_x2) * q.x_slot + G.n_g * G.g_slot <= left) {
      q.ns_x = ns_x2;
      q.ns_g = G.n_g;
    }
  }
  q.g_res = q.ns_g == G.n_g ? 1 : 0;
  q.unified = 0;
  q.gpk = 0;
  if (!q.g_res && G.n_g > 0 && G.g_slot <= q.x_slot && !getenv("LRS_CORE_SPLIT_RING")) {
    // streamed G: one ring for X and G items (lrs_core.cuh CoreParams::unified); its slots
    // are X slots, a G item packs as many chunks as one holds
    const int ns_u = std::min<int>(kCMaxX, static_cast<int>(left / q.x_slot));
    if (ns_u >= 2) {
      q.unified = 1;
      q.gpk = static_cast<int>(q.x_slot / G.g_slot);
      q.ns_x = ns_u;
      q.ns_g = 0;
    }
  }
  q.off_g = static_cast<uint32_t>(q.ns_x) * q.x_slot + x_tail;
  q.off_t1 = q.off_g + static_cast<uint32_t>(q.ns_g) * G.g_slot;
  q.off_bar = q.off_t1 + t1_bytes;
  return true;
}

// Feasible (model cost, ipt, th) for a grid of `grid` CTAs, cheapest first.
static std::vector<std::tuple<double, int, int>> core_candidates(const lrs_conv* h, const lrs_conv_desc* d,
                                                                 int grid) {
  const CoreGeom G = core_geom(h, d);
  std::vector<std::tuple<double, int, int>> v;
  const int ipt_env = getenv("LRS_CORE_IPT") ? atoi(getenv("LRS_CORE_IPT")) : 0;  // planner experiments
  const int th_env = getenv("LRS_CORE_TH") ? atoi(getenv("LRS_CORE_TH")) : 0;
  for (int ipt = 1; ipt <= 8; ++ipt) {
    if (ipt_env && ipt != ipt_env) continue;
    for (int th = 1; th <= G.ho; ++th) {
      if (th_env && th != th_env) continue;
      CoreParams q;
      memset(&q, 0, sizeof(q));
      if (!core_layout(G, ipt, th, q)) continue;
      const int p1 = (th + G.kh - 1) * G.wc;
      const int bands = (G.ho + th - 1) / th;
      const long long tiles = static_cast<long long>((d->batch_max + ipt - 1) / ipt) * bands;
      const double bytes = static_cast<double>(ipt) * p1 * G.cin * 2 + static_cast<double>(G.cin) * G.r1p * 2 +
                           (G.cp ? 0.0 : static_cast<double>(G.taps) * G.r1p * G.r2p * 2) + 8192.0;
      v.emplace_back(static_cast<double>((tiles + grid - 1) / grid) * bytes, ipt, th);
    }
  }
  std::stable_sort(v.begin(), v.end(),
                   [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b) * 0.999; });
  return v;
}

// Fill h->cp for one plan (the tensor maps of U_in and G are plan-independent and kept).
static void apply_core_plan(lrs_conv* h, const lrs_conv_desc* d, int ipt, int th, int grid, int gmode = 0) {
  const CoreGeom G = core_geom(h, d);
  CoreParams& c = h->cp;
  const CUtensorMap tmU = c.tmU, tmG = c.tmG;
  unsigned long long* trace = c.trace;
  memset(&c, 0, sizeof(c));
  c.tmU = tmU;
  c.tmG = tmG;
  c.trace = trace;
  core_layout(G, ipt, th, c, gmode);
  c.n = d->batch_max; c.ho = G.ho; c.wo = G.wo; c.kh = G.kh; c.kw = G.kw; c.ph = d->pad_h; c.pw = d->pad_w;
  c.th = th; c.bands = (G.ho + th - 1) / th; c.ipt = ipt; c.wr = th + G.kh - 1; c.wc = G.wc; c.p1 = c.wr * G.wc;
  c.n_ck = G.cin / 64;
  c.r1p = G.r1p; c.r2p = G.r2p; c.g_kc = G.g_kc; c.n_gk = G.cp ? 0 : G.r1p / G.g_kc;  // CP: no G chunks
  c.sw_g = static_cast<uint32_t>(G.g_kc * 2);
  c.u_bytes = G.u_bytes;
  c.g_bytes = G.g_bytes;
  c.g_slot = G.g_slot;
  c.t1_sw128 = (G.r1p % 64 == 0 && !getenv("LRS_CORE_T1_NOSWZ")) ? 1 : 0;
  c.cpb = h->w_cpb;
  c.cpc = h->w_cpc;
  #ifdef LRS_EXPERIMENTS
  if (const char* e = getenv("LRS_CORE_DBG")) c.dbg = atoi(e);
#endif
  c.nacc = 2 * c.acc_cols <= 512 ? 2 : 1;
  uint32_t tc = 32;
  while (tc < c.nacc * c.acc_cols) tc <<= 1;
  c.tmem_cols = tc;
  h->core_smem = c.off_bar + 2048u + 1024u;
  h->core_grid = std::max(1, std::min(h->sms, grid));
  h->cx_ptr = nullptr;  // the X tensor map's box depends on the plan
  if (getenv("LRS_VERBOSE"))
    fprintf(stderr,
            "[lrs] core: th=%d ipt=%d bands=%d wr=%d wc=%d nb1=%d nb2=%d acc=%u nacc=%d ns_x=%d ns_g=%d g_res=%d "
            "unified=%d gpk=%d t1_sw128=%d t1_rows=%u smem=%u grid<=%d\n",
            th, ipt, c.bands, c.wr, G.wc, c.nb1, c.nb2, c.acc_cols, c.nacc, c.ns_x, c.ns_g, c.g_res, c.unified, c.gpk,
            c.t1_sw128, c.t1_rows, h->core_smem, h->core_grid);
}

lrs_status build_core(lrs_conv* h, const lrs_conv_desc* d) {
  const int cin = d->c_in, kh = d->kernel_h, kw = d->kernel_w;
  const int r1p = h->r1p, r2p = h->r2p;
  if (h->f32 || h->svd || d->stride_h != 1 || d->stride_w != 1 || cin % 64 != 0 || getenv("LRS_NO_CORE"))
    return LRS_OK;
  const int wc = h->wo + kw - 1;
  if (wc > 256 || r1p > 256 || r2p > 256) return LRS_OK;
  int grid = h->sms;
  if (const char* e = getenv("LRS_CORE_GRID")) grid = std::max(1, std::min(h->sms, atoi(e)));
  const auto cand = core_candidates(h, d, grid);
  if (cand.empty()) return LRS_OK;
  const CoreGeom G = core_geom(h, d);
  CoreParams& c = h->cp;
  memset(&c, 0, sizeof(c));
  lrs_status st;
  {
    uint64_t dims[2] = {static_cast<uint64_t>(cin), static_cast<uint64_t>(r1p)};
    uint64_t strides[1] = {static_cast<uint64_t>(cin) * 2};
    uint32_t box[2] = {64, static_cast<uint32_t>(r1p)};
    uint32_t estr[2] = {1, 1};
    if ((st = encode_t(&c.tmU, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, h->w_uin, dims, strides, box, estr, 128)) != LRS_OK)
      return st;
  }
  if (!G.cp) {
    uint64_t dims[2] = {static_cast<uint64_t>(kh * kw * r1p), static_cast<uint64_t>(r2p)};
    uint64_t strides[1] = {static_cast<uint64_t>(kh * kw * r1p) * 2};
    uint32_t box[2] = {static_cast<uint32_t>(G.g_kc), static_cast<uint32_t>(r2p)};
    uint32_t estr[2] = {1, 1};
    if ((st = encode_t(&c.tmG, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, h->w_core, dims, strides, box, estr,
                       static_cast<uint32_t>(G.g_kc * 2))) != LRS_OK)
      return st;
  }
  apply_core_plan(h, d, std::get<1>(cand[0]), std::get<2>(cand[0]), grid,
                  getenv("LRS_CORE_GSTREAM") ? 1 : 0);  // planner experiments
  h->use_core = true;
  return LRS_OK;
}

// fp32 sparse term (lrs_spadd.cuh): tile = 4 images x th output rows x 64 output
// channels, X window of cc input channels in shared memory; nonzeros regrouped per
// (64-channel chunk, input-channel chunk, output channel) as (value, window offset).
// Leaves h->use_spadd false if the layer does not suit the kernel.
lrs_status build_spadd(lrs_conv* h, const lrs_conv_desc* d) {
  const int cin = d->c_in, cout = d->c_out, kh = d->kernel_h, kw = d->kernel_w;
  const int ho = h->ho, wo = h->wo, sh = d->stride_h, sw = d->stride_w;
  if (cin % 4 != 0 || wo > 32 * kSpKP) return LRS_OK;
  SpaddParams& q = h->spp;
  memset(&q, 0, sizeof(q));
  const int npos_max = 32 * kSpKP;
  int th = std::max(1, std::min(ho, npos_max / wo));
  const int bands = (ho + th - 1) / th;
  th = (ho + bands - 1) / bands;
  const int wr = (th - 1) * sh + kh, wc = (wo - 1) * sw + kw;
  // row pitch with sh*pitch == sw*wo (mod 8): lane q then reads vector sw*q (mod 8), so the
  // 8 lanes of an LDS.128 phase hit distinct banks across row wraps (stride 1)
  int pitch = wc;
  if (th > 1)
    for (int t = wc; t < wc + 8; ++t)
      if ((sh * t - sw * wo) % 8 == 0) {
        pitch = t;
        break;
      }
  const int plane = wr * pitch;
  const int n_nc = (cout + 63) / 64;
  const int kk = kh * kw;
  // channel chunk: window + staged nonzeros within ~110 KB so two CTAs share an SM
  const uint32_t budget = 110 * 1024;
  int cc = std::min(round_up(cin, 4), static_cast<int>((96 * 1024) / (plane * 16)) / 4 * 4);
  if (cc < 4) return LRS_OK;
  std::vector<int> ptr;
  std::vector<int2> ent;
  int n_cc = 0, max_ent = 0;
  for (;;) {
    n_cc = (cin + cc - 1) / cc;
    ptr.assign(static_cast<size_t>(n_nc) * n_cc * 64 + 1, 0);
    ent.clear();
    max_ent = 0;
    for (int nc = 0; nc < n_nc; ++nc)
      for (int c = 0; c < n_cc; ++c) {
        const size_t first = ent.size();
        for (int jl = 0; jl < 64; ++jl) {
          const int j = nc * 64 + jl;
          ptr[(static_cast<size_t>(nc) * n_cc + c) * 64 + jl] = static_cast<int>(ent.size());
          if (j >= cout) continue;
          for (int64_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) {
            const int col = d->col_idx[e];
            const int ch = col / kk, tap = col % kk;
            if (ch / cc != c) continue;
            const int ty = tap / kw, tx = tap % kw;
            int2 v;
            const float val = d->values[e];
            memcpy(&v.x, &val, 4);
            v.y = (((ch - c * cc) * wr + ty) * pitch + tx) * 16;
            ent.push_back(v);
          }
        }
        max_ent = std::max(max_ent, static_cast<int>(ent.size() - first));
      }
    ptr.back() = static_cast<int>(ent.size());
    const uint32_t need = std::max(static_cast<uint32_t>(cc) * plane * 16, kSpDenseBytes) +
                          static_cast<uint32_t>(max_ent) * 8;
    if (need <= budget) break;
    if (cc <= 4) return LRS_OK;
    cc = std::max(4, cc / 2 / 4 * 4);
  }
  q.h = d->in_h; q.w = d->in_w; q.cin = cin; q.ho = ho; q.wo = wo; q.cout = cout;
  q.kh = kh; q.kw = kw; q.sh = sh; q.sw = sw; q.ph = d->pad_h; q.pw = d->pad_w;
  q.th = th; q.bands = bands; q.n_nc = n_nc; q.cc = cc; q.n_cc = n_cc; q.wr = wr; q.wc = wc;
  q.pitch = pitch;
  q.max_ent = max_ent;
  #ifdef LRS_EXPERIMENTS
  if (const char* e = getenv("LRS_SPADD_DBG")) q.dbg = atoi(e);
#endif
  q.win_bytes = std::max(static_cast<uint32_t>(cc) * plane * 16, kSpDenseBytes);
  h->sp_smem = q.win_bytes + static_cast<uint32_t>(std::max(max_ent, 1)) * 8;
  if (h->sp_smem > 113 * 1024u) return LRS_OK;  // keep two CTAs per SM
  std::vector<uint8_t> pe(ptr.size() * 4), ee(std::max<size_t>(ent.size(), 1) * 8, 0);
  memcpy(pe.data(), ptr.data(), pe.size());
  if (!ent.empty()) memcpy(ee.data(), ent.data(), ent.size() * 8);
  lrs_status st;
  void* pp = nullptr;
  void* pee = nullptr;
  if ((st = upload(&pp, pe)) != LRS_OK) return st;
  h->sp_ptr = static_cast<int*>(pp);
  if ((st = upload(&pee, ee)) != LRS_OK) return st;
  h->sp_ent = static_cast<int2*>(pee);
  q.ent = h->sp_ent;
  q.ent_ptr = h->sp_ptr;
  h->use_spadd = true;
  if (getenv("LRS_VERBOSE"))
    fprintf(stderr, "[lrs] spadd: th=%d bands=%d wr=%d wc=%d pitch=%d cc=%d n_cc=%d n_nc=%d max_ent=%d smem=%u\n", th, bands,
            wr, wc, pitch, cc, n_cc, n_nc, max_ent, h->sp_smem);
  return LRS_OK;
}

// S -> exact 2:4 main + residual blocks (bf16 values, RNE) with their TMEM metadata:
// every group of 4 consecutive input channels of a (row j, tap) keeps its first two
// nonzeros in the main block of (M-tile, 64-channel chunk, tap) and, only where the group
// holds 3-4 nonzeros, the rest in a residual block (S = S_main + S_res exactly).
// as: [blocks][128 rows][32] bf16 bits (row-major, unswizzled); ee: [blocks][128 lanes][4]
// u32 metadata words; main block of key (mt * n_ck + c) * taps + t has index key, its
// residual block res_tab[key] (-1 if none).
// With `gather`, a group's 3rd/4th nonzero goes to ovf[M-tile] (row, channel, tap, value)
// instead of a residual block (the overflow-gather form, lrs_wconv.cuh WconvParams::n_gk).
struct Ovf {
  int m, ch, t;
  float v;
};
struct Split24 {
  std::vector<uint16_t> as;
  std::vector<uint32_t> ee;
  std::vector<int> res_tab;
  std::vector<std::vector<Ovf>> ovf;
  int nblk_main = 0, nres = 0;
};

Split24 split_24(const lrs_conv_desc* d, int n_mt, int n_ck, int taps, bool gather = false) {
  const int cout = d->c_out;
  Split24 S;
  const int nblk_main = n_mt * n_ck * taps;
  S.nblk_main = nblk_main;
  std::vector<uint16_t>& as = S.as;
  std::vector<uint32_t>& ee = S.ee;
  std::vector<int>& res_tab = S.res_tab;
  as.assign(static_cast<size_t>(nblk_main) * 128 * 32, 0);
  ee.assign(static_cast<size_t>(nblk_main) * 128 * 4, 0x44444444u);
  res_tab.assign(nblk_main, -1);
  if (gather) S.ovf.assign(n_mt, {});
  int nres = 0;
  std::vector<float> dense(static_cast<size_t>(n_ck) * taps * 64);
  auto put = [&](int blk, int m, int grp, int i0, int i1, float v0, float v1) {
    as[(static_cast<size_t>(blk) * 128 + m) * 32 + 2 * grp] = bf16_bits_rne(v0);
    as[(static_cast<size_t>(blk) * 128 + m) * 32 + 2 * grp + 1] = bf16_bits_rne(v1);
    const int st = grp / 8, gs = grp % 8;
    const int lane = m % 8 + 8 * (gs / 4) + 16 * (m / 16);
    const int nib = (gs % 4) + 4 * ((m / 8) % 2);
    uint32_t& w = ee[(static_cast<size_t>(blk) * 128 + lane) * 4 + st];
    w = (w & ~(0xFu << (4 * nib))) | (static_cast<uint32_t>(i0 | (i1 << 2)) << (4 * nib));
  };
  auto put_list = [&](int blk, int m, int grp, const int* idx, const float* val, int cnt) {
    if (cnt == 0) return;  // block pre-filled with zeros and the (0,1) pattern
    if (cnt == 1) {
      if (idx[0] < 3) put(blk, m, grp, idx[0], idx[0] + 1, val[0], 0.f);
      else put(blk, m, grp, 2, 3, 0.f, val[0]);
    } else {
      put(blk, m, grp, idx[0], idx[1], val[0], val[1]);
    }
  };
  for (int j = 0; j < cout; ++j) {
    const int64_t e0 = d->row_ptr[j], e1 = d->row_ptr[j + 1];
    if (e0 == e1) continue;
    std::fill(dense.begin(), dense.end(), 0.f);
    for (int64_t e = e0; e < e1; ++e) {
      const int col = d->col_idx[e];
      const int ch = col / taps, t = col % taps;
      dense[(static_cast<size_t>(ch / 64) * taps + t) * 64 + ch % 64] = d->values[e];
    }
    const int mt = j / 128, m = j % 128;
    for (int c = 0; c < n_ck; ++c)
      for (int t = 0; t < taps; ++t) {
        const float* b = &dense[(static_cast<size_t>(c) * taps + t) * 64];
        const int key = (mt * n_ck + c) * taps + t;
        for (int grp = 0; grp < 16; ++grp) {
          int idx[4];
          float val[4];
          int cnt = 0;
          for (int i = 0; i < 4; ++i)
            if (b[4 * grp + i] != 0.f) {
              idx[cnt] = i;
              val[cnt] = b[4 * grp + i];
              ++cnt;
            }
          put_list(key, m, grp, idx, val, std::min(cnt, 2));
          if (cnt > 2 && gather) {
            for (int i = 2; i < cnt; ++i) S.ovf[mt].push_back({m, c * 64 + 4 * grp + idx[i], t, val[i]});
          } else if (cnt > 2) {
            if (res_tab[key] < 0) {
              res_tab[key] = nblk_main + nres++;
              as.resize(as.size() + 128 * 32, 0);
              ee.resize(ee.size() + 128 * 4, 0x44444444u);
            }
            put_list(res_tab[key], m, grp, idx + 2, val + 2, cnt - 2);
          }
        }
      }
  }
  S.nres = nres;
  return S;
}

// K-major operand image with 8-row swizzle atoms: byte offset of (row r, byte `byte`)
// in a tile of rows of sw bytes (the layout TMA writes with SWIZZLE_<sw>B)
inline int swz_off(int r, int byte, int sw) {
  return (r / 8) * (8 * sw) + (r % 8) * sw + ((((byte / 16) ^ ((r % 8) / (128 / sw))) % (sw / 16)) * 16) + byte % 16;
}

// Fused a3+a4+a5 on the tensor cores (lrs_wconv.cuh): choose the tile geometry,
// split S into exact 2:4 main + residual blocks with their TMEM metadata, and
// encode the static tensor maps.  Leaves h->use_w false if the layer does not fit.
lrs_status build_wconv(lrs_conv* h, const lrs_conv_desc* d, const ConvGeom& g) {
  const int cin = d->c_in, cout = d->c_out, kh = d->kernel_h, kw = d->kernel_w;
  const int ho = h->ho, wo = h->wo;
  const int taps = kh * kw;
  const int n_ck = cin / 64;
  const int n_mt = (cout + 127) / 128;
  const int rp = h->r2p;  // K of the dense part: R2, or R of the SVD pair
  const bool ering = getenv("LRS_WCONV_ERING") != nullptr;  // experiment: metadata ring smaller than the A ring
  const int t_kc = rp < 64 ? rp : 64;
  if (rp % t_kc) return LRS_OK;
  if (n_ck * kh * kw > 1024) return LRS_OK;  // residual table staged in shared memory
  const int n_tk = rp / t_kc;
  const uint32_t sw_t = static_cast<uint32_t>(t_kc) * 2u;
  const bool s1 = g.sh == 1 && g.sw == 1;
  struct Unit { int col, n, xpos, tpos, r0, wo0, pitch, nw, rows, q0; };
  // MMA units covering a tile of th output rows x tc output columns (see lrs_wconv.cuh);
  // wcw = window width, tbw = T window row pitch
  auto make_units = [&](int th, int tc, int wcw, int tbw, int ipw, std::vector<Unit>& us) -> int {
    us.clear();
    int col = 0;
    if (s1) {
      // stride 1: the tile's outputs are positions q = r * wcw + c of the window
      // (c >= tc are the window's padding columns, computed and discarded); a unit
      // is a run of <= 256 / ipw consecutive positions (N <= 256), whatever rows it spans
      const int npos = (th - 1) * wcw + tc;
      const int per = 256 / ipw;
      for (int q0 = 0; q0 < npos; q0 += per) {
        const int np = std::min(per, npos - q0);
        Unit u{col, round_up(ipw * np, 16), q0, q0, 0, 0, wcw, tc, th, q0};
        us.push_back(u);
        col += u.n;
      }
    } else {
      const int nsplit = (tc + 31) / 32;
      const int wsplit = (tc + nsplit - 1) / nsplit;
      for (int r = 0; r < th; ++r)
        for (int q = 0; q < nsplit; ++q) {
          const int wo0 = q * wsplit, nw = std::min(wsplit, tc - wo0);
          Unit u{col, round_up(8 * nw, 16), r * g.sh * wcw + wo0 * g.sw, r * tbw + wo0, r, wo0, nw, nw, 1, 0};
          us.push_back(u);
          col += u.n;
        }
    }
    return col;
  };
  std::vector<Unit> units, best_units;
  int best_th = 0, best_ns = 0, best_tc = 0, best_wc = 0, best_tbw = 0, best_nwb = 2, best_bpi = 2, best_ipw = 8;
  int best_pair = 0;
  uint32_t best_margin = 0, best_shift_x = 0, best_shift_t = 0;
  // ---- S -> exact 2:4 main + residual blocks (bf16 values, RNE), TMEM metadata; the
  // overflow lists (for the gather form) when any group holds 3+ nonzeros
  Split24 S24 = split_24(d, n_mt, n_ck, taps);
  Split24 Gv;
  if (S24.nres > 0) Gv = split_24(d, n_mt, n_ck, taps, true);
  // distinct (channel, tap) slots of the overflow entries per group of M-tiles (one M-tile,
  // or the CTA pair's two: their MMAs share the B operand, so the G slots are the union)
  auto group_slots = [&](int per) {
    std::vector<std::vector<std::pair<int, int>>> sl((n_mt + per - 1) / per);
    if (S24.nres > 0)
      for (int mt = 0; mt < n_mt; ++mt)
        for (const Ovf& o : Gv.ovf[mt]) {
          auto& v = sl[mt / per];
          if (std::find(v.begin(), v.end(), std::make_pair(o.ch, o.t)) == v.end()) v.emplace_back(o.ch, o.t);
        }
    return sl;
  };
  const char* gather_env = getenv("LRS_WCONV_GATHER");  // plan override: 0 = residual blocks, 1 = gather
  const char* pair_env = getenv("LRS_WCONV_PAIR");      // plan override: 0 = never, 1 = whenever feasible
  const bool pair_force = pair_env && atoi(pair_env) == 1;
  // the pair form needs identical block streams in both CTAs: no residual blocks (the
  // overflow gather replaces them, with the union of the pair's slots, <= 256)
  // (opt-in: exact and at the 2:4 tensor rate in isolation, tools/probe_2cta_rate.cu, but its
  // item stream measured slower at C3 -- 86.9 vs 55.5 us, profiles/r02_ablate_pair_c3.log -- so
  // the cost model does not take it unless LRS_WCONV_PAIR=1)
  bool pair_data = n_mt % 2 == 0 && pair_force && !ering;
  std::vector<std::vector<std::pair<int, int>>> pair_slots;
  if (pair_data && S24.nres > 0) {
    if (gather_env && atoi(gather_env) == 0) pair_data = false;
    pair_slots = group_slots(2);
    size_t mx = 0;
    for (const auto& v : pair_slots) mx = std::max(mx, v.size());
    if ((mx + t_kc - 1) / t_kc * t_kc > 256) pair_data = false;
  }
  long long best_cost = 1LL << 60;
  uint32_t best_stride = 0, best_xw = 0, best_tw = 0, best_total = 0, best_acc = 0;
  // chunks per X window: several 64-channel boxes in one window buffer share one
  // pipeline hand-off (the per-window round trip dominated C4's timeline); the largest
  // that fits wins
  int best_cpw = 1;
  const int cpw_env = getenv("LRS_WCONV_CPW") ? atoi(getenv("LRS_WCONV_CPW")) : 0;
  // ("largest that fits" shrank the tiles and lost badly at C2/C3, so only 1x1 layers --
  // no halo, small windows -- take cpw > 1; C4: 49.0 -> 47.0 us)
  // images per window: 8 (one 8-row core matrix = the 8 images of one position), or 4 at
  // stride 1 (a core matrix = 2 positions x 4 images; a tap then moves the operand start by
  // 512 B, which SW128 allows): half-size windows leave room for a deeper A/E item ring --
  // the small-image layers (C3: 9 x 9 windows of 82 KB) are otherwise held to two items in flight
  // (measured: no config is faster at ipw 4 -- C3 77.5 -> 85.6 us with a 4-deep ring, C2 22 -> 25 us,
  // profiles/r02_ablate_ipw.log -- so 4 is a plan option for LRS_WCONV_IPW=4 only)
  const int ipw_env = getenv("LRS_WCONV_IPW") ? atoi(getenv("LRS_WCONV_IPW")) : 8;  // plan override (tests)
  for (int ipw : {8, 4}) {
  if ((ipw != ipw_env && !pair_data) || (ipw == 4 && !s1)) continue;
  bool found_ipw = false;
  for (int cpw = 8; cpw >= 1 && !found_ipw; cpw /= 2) {
  if (n_ck % cpw || (cpw_env ? cpw != cpw_env : (taps > 1 && cpw != 1))) continue;
  const int cb_env = getenv("LRS_WCONV_CB") ? atoi(getenv("LRS_WCONV_CB")) : 0;  // planner experiments
  for (int cb = cb_env ? cb_env : 1; cb <= 16 && !found_ipw; ++cb) {  // column bands: as few as fit
    const int tc = (wo + cb - 1) / cb;
    if (cb > 1 && (wo + tc - 1) / tc != cb) continue;
    const int wcw = (tc - 1) * g.sw + kw;
    const int tbw = s1 ? wcw : tc;
    if (wcw > 256) continue;
    const int th_env = h->force_wth ? h->force_wth  // autotune_w's candidate
                                    : (getenv("LRS_WCONV_TH") ? atoi(getenv("LRS_WCONV_TH")) : 0);  // planner experiments
    for (int th = std::min(ho, 64); th >= 1; --th) {
      if (th_env && th != th_env) continue;
      const int acc = make_units(th, tc, wcw, tbw, ipw, units);
      if (static_cast<int>(units.size()) > kWMaxUnits) continue;
      const int wr = (th - 1) * g.sh + kh;
      if (wr > 256) continue;
      const int ns_max = getenv("LRS_WCONV_NS") ? atoi(getenv("LRS_WCONV_NS")) : kWMaxSlots;
      const int bpi_max = getenv("LRS_WCONV_BPI") ? atoi(getenv("LRS_WCONV_BPI")) : kWMaxBpi;
      // (blocks per item, slots): prefer big items, then more slots; but when the layer has
      // several M-tiles, first look for a candidate that keeps ALL of a tile's windows in
      // smem (window reuse across the CTA's consecutive M-tiles)
      // (one-block items {1, ns} are taken only when bpi_max (LRS_WCONV_BPI) asks for them)
      const int cand[][2] = {{4, 3}, {4, 2}, {2, 4}, {2, 3}, {2, 2}, {1, 6}, {1, 5}, {1, 4}, {1, 3}};
      // (opt-in: measured slower on C4, 49.4 vs 45.7 us -- the window loads are not its bottleneck)
      int want_all = (n_mt > 1 && n_tk + (d->nnz > 0 ? n_ck / cpw : 0) <= kWMaxWin && getenv("LRS_WCONV_REUSE")) ? 1 : 0;
      // pair: the CTA-pair form (every unit the same N, a multiple of 16, <= 2 units)
      bool same_n = units.size() <= 2;
      for (const Unit& u : units) same_n = same_n && u.n == units[0].n && u.n % 16 == 0;
      for (int pair = 0; pair < 2; ++pair) {
      if (pair == 0 && ipw != ipw_env) continue;
      if (pair == 1 && !(pair_data && same_n)) continue;
      // window margin of the pair's rank 1 (it keeps each window N/2 B rows earlier)
      const uint32_t x_sbo_b = ipw == 8 ? 1024u * static_cast<uint32_t>(g.sw) : 1024u;
      const uint32_t p_shift_x = pair ? static_cast<uint32_t>(units[0].n / 16) * x_sbo_b : 0u;
      const uint32_t p_shift_t = pair ? static_cast<uint32_t>(units[0].n / 2) * sw_t : 0u;
      const uint32_t margin = align1024(std::max(p_shift_x, p_shift_t));
      for (int pass = 0; pass < 2; ++pass) {
      const bool need_all = pass == 0 && want_all;
      if (pass == 1 && !want_all) break;
      bool found = false;
      for (const auto& cnd : cand) {
        const int bpi = cnd[0], ns = cnd[1];
        if (bpi > bpi_max || ns > ns_max || (bpi == 1 && bpi_max != 1)) continue;
        // an A slot also holds one dense U_out^T block (128 rows x sw_t B) of the T windows
        const uint32_t a_slot = std::max<uint32_t>(static_cast<uint32_t>(bpi) * kSpBlockBytes, 128u * sw_t);
        const uint32_t e_slot = static_cast<uint32_t>(bpi) * kEBlockBytes;
        const int es_need = ering ? 1 : ns;  // TMEM metadata slots the plan needs at least
        if (acc + 4 * bpi * es_need > 512) continue;
        const uint32_t pos_b = 128u * ipw;  // bytes per window position
        const uint32_t xw = static_cast<uint32_t>(wr) * wcw * pos_b;  // one chunk's box
        const uint32_t tw = static_cast<uint32_t>(th) * tbw * ipw * sw_t;
        // slack: positions read past the end of a window by the last (padded) MMA rows
        long long last_x = 0, last_t = 0;
        for (const Unit& u : units) {
          last_x = std::max<long long>(last_x, u.xpos + static_cast<long long>(kh - 1) * wcw + (kw - 1) +
                                                   static_cast<long long>(u.n / ipw - 1) * g.sw);
          last_t = std::max<long long>(last_t, u.tpos + u.n / ipw - 1);
        }
        const long long slack_x = std::max(0LL, last_x + 1 - static_cast<long long>(wr) * wcw) * pos_b +
                                  static_cast<long long>(cpw - 1) * xw;  // the window's other boxes
        const long long slack_t = std::max(0LL, last_t + 1 - static_cast<long long>(th) * tbw) * ipw * sw_t;
        const uint32_t stride =
            align1024(static_cast<uint32_t>(std::max<long long>(xw + slack_x, tw + slack_t))) + margin;
        // the M-tile's block stream: chunk starts + a tap offset per (main or residual) block
        const uint32_t res_bytes = (static_cast<uint32_t>(n_ck + 1 + 2 * n_ck * taps) * 4u + 127u) & ~127u;
        const uint32_t fixed = ns * (a_slot + e_slot) + 8 * kEpiScratch + res_bytes + 1024 + 1024;
        const int nwb_min = getenv("LRS_WCONV_NWB1") ? 1 : 2;  // experiment: a single window buffer
        if (static_cast<uint32_t>(nwb_min) * stride + fixed > static_cast<uint32_t>(kMaxSmem)) continue;
        int nwb = nwb_min;
        while (nwb < 4 && (nwb + 1) * stride + fixed <= static_cast<uint32_t>(kMaxSmem)) ++nwb;
        // one buffer per window of a tile when they all fit: windows are then reused by
        // the CTA's next tile of the same images / band (the next M-tile)
        const int nwin_t = n_tk + (d->nnz > 0 ? n_ck / cpw : 0);  // the kernel's windows per tile
        const bool all_fit = static_cast<uint32_t>(nwin_t) * stride + fixed <= static_cast<uint32_t>(kMaxSmem);
        if (need_all && !all_fit) continue;
        if (need_all) nwb = nwin_t;
        const uint32_t total = nwb * stride + fixed;
        // cost model (cycles, measured with tools/mma_rate2 and tools/wtrace on B200): a
        // sparse MMA costs max(~100 issue, (A 4 KB + B N*64 B) / 128 B/clk smem), an item
        // (one tap of a 64-channel chunk: 2 MMA steps per unit) adds ~200; CTAs run in
        // waves of one per SM.
        long long item = 450 / bpi;  // per-block share of the item's hand-off + commit
        // (pair: ~N/2 cycles per MMA -- the 2:4 tensor rate, B split between the two SMs'
        // shared memories, tools/probe_2cta_rate.cu)
        for (const Unit& u : units)
          item += 2 * (pair ? std::max<long long>(50, u.n / 2) : std::max<long long>(100, (4096 + 64LL * u.n) / 128));
        const long long ctas = static_cast<long long>((d->batch_max + ipw - 1) / ipw) * ((ho + th - 1) / th) * cb * n_mt;
        const long long waves = (ctas + h->sms - 1) / h->sms;
        // waves x per-tile cost: the tile's blocks x per-block cost, plus the epilogue
        // (~30 cycles per accumulator column, measured with tools/wtrace) unless two
        // accumulators fit in TMEM and it overlaps the next tile's MMAs
        const long long tile_mma = static_cast<long long>(n_tk + n_ck * taps) * item;
        const bool dbl = 2 * acc + 4 * bpi * es_need <= 512;
        long long cost = waves * (tile_mma + (dbl ? 0LL : 30LL * acc));
        if (pair && pair_force) cost /= 1000;
        if (cost < best_cost) {
          best_pair = pair;
          best_margin = margin;
          best_shift_x = p_shift_x;
          best_shift_t = p_shift_t;
          best_cost = cost;
          best_th = th;
          best_ns = ns;
          best_tc = tc;
          best_wc = wcw;
          best_tbw = tbw;
          best_stride = stride;
          best_xw = xw;
          best_tw = tw;
          best_total = total;
          best_nwb = nwb;
          best_bpi = bpi;
          best_acc = static_cast<uint32_t>(acc);
          best_units = units;
          best_cpw = cpw;
          best_ipw = ipw;
        }
        found = true;
        found_ipw = true;
        h->wth_max = std::max(h->wth_max, th);
        break;
      }
      if (found) break;
      }  // pass
      }  // pair
    }
  }
  }  // cpw
  }  // ipw
  if (!best_th) return LRS_OK;
  const int cpw = best_cpw;
  const int ipw = best_ipw;
  const int th = best_th;
  const int wc = best_wc, tbox_w = best_tbw, tcols = best_tc;

  // overflow gather instead of residual blocks when the residual MMAs cost more than the
  // G chunks: a residual block is 2 sparse MMA steps (each the time of a dense K = 16 step)
  // per unit, a G chunk t_kc / 16 dense steps, plus ~8 steps for the gather hand-off; the
  // pair form always takes it (its two CTAs' block streams must be identical)
  int n_gk = 0;
  const int gper = best_pair ? 2 : 1;  // M-tiles per slot group
  const int n_grp = (n_mt + gper - 1) / gper;
  std::vector<int> g_tab;
  if (S24.nres > 0 && !(gather_env && atoi(gather_env) == 0)) {
    const auto slots = best_pair ? pair_slots : group_slots(1);
    size_t mx = 0;
    for (const auto& v : slots) mx = std::max(mx, v.size());
    const int gk = static_cast<int>((mx + t_kc - 1) / t_kc);
    const bool pays = 2.0 * S24.nres / n_mt > gk * (t_kc / 16.0) + 8.0;
    if (gk * t_kc <= 256 && (best_pair || pays || (gather_env && atoi(gather_env) == 1))) {
      n_gk = gk;
      const int gs = gk * t_kc;
      g_tab.assign(static_cast<size_t>(n_grp) * gs, -1);
      for (int gi = 0; gi < n_grp; ++gi)
        for (size_t si = 0; si < slots[gi].size(); ++si) {
          const int t = slots[gi][si].second;
          g_tab[gi * gs + si] = slots[gi][si].first | ((t / kw) << 16) | ((t % kw) << 24);
        }
      // the overflow values as dense U blocks: row m of M-tile mt, column = its group's slot index
      h->w_ovf.assign(static_cast<size_t>(n_mt) * gk * 128 * sw_t, 0);
      for (int mt = 0; mt < n_mt; ++mt)
        for (const Ovf& o : Gv.ovf[mt]) {
          const auto& v = slots[mt / gper];
          const int si = static_cast<int>(std::find(v.begin(), v.end(), std::make_pair(o.ch, o.t)) - v.begin());
          const uint16_t bits = bf16_bits_rne(o.v);
          memcpy(&h->w_ovf[(static_cast<size_t>(mt) * gk + si / t_kc) * 128 * sw_t + swz_off(o.m, 2 * (si % t_kc), sw_t)],
                 &bits, 2);
        }
      S24 = std::move(Gv);
    }
  }
  if (best_pair && S24.nres > 0) return fail(LRS_ERR_UNSUPPORTED, "CTA-pair plan with residual blocks");
  const int nblk_main = S24.nblk_main;
  const int nres = S24.nres;
  std::vector<uint16_t>& as = S24.as;
  std::vector<uint32_t>& ee = S24.ee;
  std::vector<int>& res_tab = S24.res_tab;
  h->w_main_blocks = nblk_main;
  h->w_res_blocks = nres;
  const int nblk = nblk_main + nres;
  // stream order: per (M-tile, chunk), per tap its main block then its residual block, so
  // the kernel fetches each item (consecutive blocks of a window) with one bulk copy
  std::vector<int> order, stream_off(static_cast<size_t>(n_mt) * n_ck + 1, 0);
  std::vector<uint32_t> blk_tap;
  order.reserve(nblk);
  blk_tap.reserve(nblk);
  for (int mt = 0; mt < n_mt; ++mt)
    for (int c = 0; c < n_ck; ++c) {
      stream_off[static_cast<size_t>(mt) * n_ck + c] = static_cast<int>(order.size());
      for (int t = 0; t < taps; ++t) {
        const int key = (mt * n_ck + c) * taps + t;
        const uint32_t tap16 = static_cast<uint32_t>((t / kw) * wc + (t % kw)) * (8u * ipw) +  // (pos*128*ipw)>>4
                               static_cast<uint32_t>(c % cpw) * (best_xw >> 4);          // the chunk's box
        order.push_back(key);
        blk_tap.push_back(tap16);
        if (res_tab[key] >= 0) {
          order.push_back(res_tab[key]);
          blk_tap.push_back(tap16);
        }
      }
    }
  stream_off.back() = static_cast<int>(order.size());
  lrs_status st;
  // shared-memory images of the A operands (swizzle applied here, 1-D bulk copies in the kernel)
  {
    std::vector<uint8_t> b(static_cast<size_t>(nblk) * kSpBlockBytes, 0);
    std::vector<uint8_t> e(static_cast<size_t>(nblk) * kEBlockBytes);
    for (int pos = 0; pos < nblk; ++pos) {
      const int blk = order[pos];
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 32; ++k)
          memcpy(&b[static_cast<size_t>(pos) * kSpBlockBytes + swz_off(m, 2 * k, 64)],
                 &as[(static_cast<size_t>(blk) * 128 + m) * 32 + k], 2);
      memcpy(&e[static_cast<size_t>(pos) * kEBlockBytes], &ee[static_cast<size_t>(blk) * 128 * 4], kEBlockBytes);
    }
    if ((st = upload(&h->w_as, b)) != LRS_OK) return st;
    if ((st = upload(&h->w_e, e)) != LRS_OK) return st;
    // stream tables: [n_mt * n_ck + 1] chunk starts, then [nblk] tap offsets, one buffer
    std::vector<uint8_t> r((stream_off.size() + blk_tap.size()) * 4);
    memcpy(r.data(), stream_off.data(), stream_off.size() * 4);
    memcpy(r.data() + stream_off.size() * 4, blk_tap.data(), blk_tap.size() * 4);
    void* rp_ = nullptr;
    if ((st = upload(&rp_, r)) != LRS_OK) return st;
    h->w_res = static_cast<int*>(rp_);
    // dense A: U_out^T rows (output channels) x R chunks, the layer's bf16 values
    const int r2 = h->svd ? d->rank_in : d->rank_out;
    // per M-tile: n_tk U_out^T chunks, then n_gk overflow-value chunks (G mode)
    const int n_dk = n_tk + n_gk;
    std::vector<uint8_t> dn(static_cast<size_t>(n_mt) * n_dk * 128 * sw_t, 0);
    for (int mt = 0; mt < n_mt; ++mt) {
      for (int kc = 0; kc < n_tk; ++kc)
        for (int m = 0; m < 128; ++m) {
          const int j = mt * 128 + m;
          if (j >= cout) continue;
          for (int e2 = 0; e2 < t_kc; ++e2) {
            const int bb = kc * t_kc + e2;
            if (bb >= r2) continue;
            const uint16_t bits = static_cast<const uint16_t*>(d->u_out)[static_cast<size_t>(bb) * cout + j];
            memcpy(&dn[(static_cast<size_t>(mt) * n_dk + kc) * 128 * sw_t + swz_off(m, 2 * e2, sw_t)], &bits, 2);
          }
        }
      if (n_gk)
        memcpy(&dn[(static_cast<size_t>(mt) * n_dk + n_tk) * 128 * sw_t],
               &h->w_ovf[static_cast<size_t>(mt) * n_gk * 128 * sw_t], static_cast<size_t>(n_gk) * 128 * sw_t);
    }
    if ((st = upload(&h->w_dense_img, dn)) != LRS_OK) return st;
    h->w_ovf.clear();
    h->w_ovf.shrink_to_fit();
    if (n_gk) {
      std::vector<uint8_t> tb(g_tab.size() * 4);
      memcpy(tb.data(), g_tab.data(), tb.size());
      if ((st = upload(&h->w_gtab, tb)) != LRS_OK) return st;
      const size_t gb = static_cast<size_t>(d->batch_max) * ho * wo * n_grp * n_gk * t_kc * 2;
      LRS_CUDA(cudaMalloc(&h->w_g, gb));
      LRS_CUDA(cudaMemset(h->w_g, 0, gb));  // empty slots stay 0
    }
  }
  WconvParams& w = h->wp;
  memset(&w, 0, sizeof(w));
#if defined(LRS_EXPERIMENTS) || defined(LRS_WCONV_DEBUG)
  if (const char* e = getenv("LRS_WCONV_DBG")) w.dbg = atoi(e);  // experiment bits (debug builds only)
#endif
  w.img_sp = static_cast<const uint8_t*>(h->w_as);
  w.img_e = static_cast<const uint8_t*>(h->w_e);
  w.img_dense = static_cast<const uint8_t*>(h->w_dense_img);
  {
    void* src = h->svd ? h->t1 : h->t2;
    const uint64_t bm = static_cast<uint64_t>(d->batch_max);
    uint64_t dims[4] = {static_cast<uint64_t>(rp), bm, static_cast<uint64_t>(wo), static_cast<uint64_t>(ho)};
    uint64_t strides[3] = {static_cast<uint64_t>(ho) * wo * rp * 2, static_cast<uint64_t>(rp) * 2,
                           static_cast<uint64_t>(wo) * rp * 2};
    uint32_t box[4] = {static_cast<uint32_t>(t_kc), static_cast<uint32_t>(ipw), static_cast<uint32_t>(tbox_w),
                       static_cast<uint32_t>(th)};
    uint32_t estr[4] = {1, 1, 1, 1};
    if ((st = encode_t(&w.tmT, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, src, dims, strides, box, estr, sw_t)) != LRS_OK)
      return st;
  }
  if (n_gk) {
    const uint64_t bm = static_cast<uint64_t>(d->batch_max);
    const uint64_t gch = static_cast<uint64_t>(n_grp) * n_gk * t_kc;
    uint64_t dims[4] = {gch, bm, static_cast<uint64_t>(wo), static_cast<uint64_t>(ho)};
    uint64_t strides[3] = {static_cast<uint64_t>(ho) * wo * gch * 2, gch * 2, static_cast<uint64_t>(wo) * gch * 2};
    uint32_t box[4] = {static_cast<uint32_t>(t_kc), static_cast<uint32_t>(ipw), static_cast<uint32_t>(tbox_w),
                       static_cast<uint32_t>(th)};
    uint32_t estr[4] = {1, 1, 1, 1};
    if ((st = encode_t(&w.tmG, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, h->w_g, dims, strides, box, estr, sw_t)) != LRS_OK)
      return st;
    w.n_gk = n_gk;
    w.g_ch = static_cast<int>(gch);
    w.g_tab = static_cast<const int*>(h->w_gtab);
    w.g = static_cast<__nv_bfloat16*>(h->w_g);
    w.in_h = d->in_h;
    w.in_w = d->in_w;
    w.c_in = cin;
  }
  w.stream_off = h->w_res;
  w.blk_tap = reinterpret_cast<const uint32_t*>(h->w_res + stream_off.size());
  w.ho = ho;
  w.wo = wo;
  w.cout = cout;
  w.kh = kh;
  w.kw = kw;
  w.sh = g.sh;
  w.sw = g.sw;
  w.ph = g.ph;
  w.pw = g.pw;
  w.ipw = ipw;
  w.th = th;
  w.bands = (ho + th - 1) / th;
  w.tcols = tcols;
  w.cbands = (wo + tcols - 1) / tcols;
  w.n_mt = n_mt;
  w.n_units = static_cast<int>(best_units.size());
  for (int i = 0; i < w.n_units; ++i) {
    const Unit& u = best_units[i];
    w.u_col[i] = u.col;
    w.u_n[i] = u.n;
    w.u_xpos[i] = u.xpos;
    w.u_tpos[i] = u.tpos;
    w.u_r0[i] = u.r0;
    w.u_wo0[i] = u.wo0;
    w.u_pitch[i] = u.pitch;
    w.u_nw[i] = u.nw;
    w.u_rows[i] = u.rows;
    w.u_q0[i] = u.q0;
  }
  w.tbox_w = tbox_w;
  w.n_ck = n_ck;
  w.cpw = cpw;
  w.n_xw = d->nnz > 0 ? n_ck / cpw : 0;  // an empty S needs no X windows at all (LR-only layers)
  // k x k layers interleave the dense windows with the last X windows (1 x 1 layers keep
  // them at the end: one tap per X window hides nothing, and the pointwise kernel's
  // summation order stays the windowed kernel's)
  w.ilv = (taps > 1 && w.n_xw >= n_tk + n_gk && !getenv("LRS_WCONV_DENSE_LAST")) ? w.n_xw - (n_tk + n_gk) : -1;
  w.n_tk = n_tk;
  w.t_kc = t_kc;
  w.sw_t = sw_t;
  w.wr = (th - 1) * g.sh + kh;
  w.wc = wc;
  w.x_win_bytes = best_xw;
  w.t_win_bytes = best_tw;
  w.win_stride = best_stride;
  w.ns = best_ns;
  w.pair = best_pair;
  w.win_margin = best_margin;
  w.shift_x = best_shift_x;
  w.shift_t = best_shift_t;
  const uint32_t acc = best_acc;
  w.acc_cols = acc;
  w.bpi = best_bpi;
  w.a_slot = std::max<uint32_t>(static_cast<uint32_t>(best_bpi) * kSpBlockBytes, 128u * sw_t);
  w.e_slot = static_cast<uint32_t>(best_bpi) * kEBlockBytes;
  // double-buffered accumulators (epilogue overlaps MMAs) when two fit next to the metadata columns
  w.nacc = (2 * acc + 4 * best_bpi * (ering ? 1 : best_ns) <= 512) ? 2 : 1;
  w.e_col0 = w.nacc * acc;
  w.e_slots = std::max(1, std::min<int>(best_ns, static_cast<int>((512 - w.nacc * acc) / (4 * best_bpi))));
  w.tmem_cols = 512;  // whole TMEM: base address 0 (lrs_wconv_kernel relies on it)
  w.nwb = best_nwb;
  w.off_a = best_nwb * best_stride;
  w.off_e = w.off_a + best_ns * w.a_slot;
  w.off_epi = w.off_e + best_ns * w.e_slot;
  w.off_res = w.off_epi + 8 * kEpiScratch;  // block stream of the tile's M-tile
  w.off_bar = w.off_res + ((static_cast<uint32_t>(n_ck + 1 + 2 * n_ck * taps) * 4u + 127u) & ~127u);
  h->w_smem = best_total;
  h->use_w = true;
  if (getenv("LRS_VERBOSE"))
    fprintf(stderr, "lrs_wconv plan: ipw %d th %d tcols %d units %d acc %u nacc %d ns %d bpi %d nwb %d cpw %d win %u B smem %u B tiles/img-group %d residual blocks %d gather chunks %d\n",
            ipw, th, tcols, w.n_units, acc, w.nacc, w.ns, w.bpi, w.nwb, cpw, best_stride, best_total, w.bands * w.cbands * w.n_mt,
            nres, n_gk);
  if (getenv("LRS_VERBOSE") && best_pair)
    fprintf(stderr, "lrs_wconv plan: CTA pairs (cta_group::2), unit N %d, window margin %u B\n", best_units[0].n,
            best_margin);
  return LRS_OK;
}

// 1x1 SVD-pair layers (bf16, stride 1, pad 0, c_in % 64 == 0): plan the channel-stationary
// fused kernel (lrs_pw.cuh), build the per-group weight images, encode nothing per call
// yet (X / T1 maps depend on n).  Leaves h->use_pw false if the layer does not fit.
lrs_status build_pw(lrs_conv* h, const lrs_conv_desc* d, const PwPlan* force = nullptr) {
  if (h->f32 || !h->svd || d->c_in % 64 != 0 || getenv("LRS_NO_PW")) return LRS_OK;
  const int cin = d->c_in, cout = d->c_out;
  const int n_ck = cin / 64;
  if (n_ck > kPMaxCk) return LRS_OK;
  const int r1p = h->r1p;
  const int t_kc = r1p < 64 ? r1p : 64;
  if (r1p % t_kc) return LRS_OK;
  const int n_tk = r1p / t_kc;
  const uint32_t sw_t = static_cast<uint32_t>(t_kc) * 2u;
  const int n_mt = (cout + 127) / 128;
  const int n_x = d->nnz > 0 ? n_ck : 0;
  Split24 S = d->nnz > 0 ? split_24(d, n_mt, n_ck, 1) : Split24{};
  const long long p_max = static_cast<long long>(d->batch_max) * d->in_h * d->in_w;
  const int mpc_env = getenv("LRS_PW_MPC") ? atoi(getenv("LRS_PW_MPC")) : 0;  // plan overrides (tests)
  const int bp_env = getenv("LRS_PW_BP") ? atoi(getenv("LRS_PW_BP")) : 0;
  // ft: the projection fused in (lrs_pwf.cuh) -- needs 128-position tiles (the M of the T1
  // MMAs), R1p a multiple of 32 (the restage splits the ranks over two warps in steps of 16)
  // and the X chunks even without a sparse term.  It saves the a1 launch and T1's HBM round
  // trip but measured slower at C4 (33.9 vs 25.9 us: U^T, two T1 tiles and the restage
  // leave a ring of ~1 tile, so every tile's X loads wait for the previous tile's MMAs;
  // profiles/r02_ablate_pwf_c4.log), so it is a plan option: LRS_PW_FT=1
  const bool ft_ok = r1p % 32 == 0 && r1p <= 256 && getenv("LRS_PW_FT") && atoi(getenv("LRS_PW_FT")) == 1;
  using Plan = PwPlan;
  const int cpi_env = getenv("LRS_PW_CPI") ? atoi(getenv("LRS_PW_CPI")) : 0;  // plan override
  Plan best;
  std::vector<Plan> all;
  if (force) best = *force;
  for (int ft = ft_ok ? 1 : 0; ft >= 0 && !best.mpc; --ft) {
  for (int mpc = std::min(kPMaxMpc, n_mt); mpc >= 1; --mpc) {
    if (mpc_env && mpc != mpc_env) continue;
    const int G = (n_mt + mpc - 1) / mpc;
    if (G > h->sms) continue;
    // blocks per group: every (M-tile, chunk) has its main block, plus residual blocks
    int nblk = 0;
    if (n_x)
      for (int g = 0; g < G; ++g) {
        int nb = 0;
        for (int m = 0; m < mpc; ++m)
          for (int c = 0; c < n_ck; ++c) {
            const int mt = g * mpc + m;
            nb += 1 + ((mt < n_mt && S.res_tab[mt * n_ck + c] >= 0) ? 1 : 0);
          }
        nblk = std::max(nblk, nb);
      }
    for (int bp : {128, 96, 64}) {  // multiples of 32: the epilogue stores 32-position TMA boxes
    for (int cpi : {4, 2, 1}) {     // chunks per ring item (one hand-off each)
      if ((bp_env && bp != bp_env) || (ft && bp != 128)) continue;
      if ((cpi_env && cpi != cpi_env) || (ft && cpi != 1) || (cpi > 1 && cpi > std::max(n_x, n_tk))) continue;
      const uint32_t acc = static_cast<uint32_t>(mpc * bp);
      // TMEM: two accumulator sets (+ two T1 accumulators when fused) and the metadata
      const uint32_t t1cols = ft ? 2u * static_cast<uint32_t>(r1p) : 0u;
      if (2 * acc + t1cols + 4u * nblk > 512) continue;
      const uint32_t dense = static_cast<uint32_t>(mpc * n_tk) * 128u * sw_t;
      const uint32_t w_bytes = dense + static_cast<uint32_t>(nblk) * 8192u;
      const uint32_t e_bytes = static_cast<uint32_t>(nblk) * 2048u;
      const uint32_t slot = static_cast<uint32_t>(cpi * bp) * 128u;
      const uint32_t u_bytes = ft ? static_cast<uint32_t>(n_ck * r1p) * 128u : 0u;
      const uint32_t t1s = ft ? 2u * 128u * static_cast<uint32_t>(r1p) * 2u : 0u;
      // (fused: the metadata staging shares the second T1 tile, first written after the copy)
      const uint32_t e_stage = (ft && e_bytes <= t1s / 2) ? 0u : align1024(e_bytes);
      // the two-kernel form stages the metadata in the ring's last slots (free once copied to
      // TMEM) and takes one epilogue scratch buffer per warp when that buys another ring slot
      const uint32_t e_ring = ft ? e_stage : 0u;
      const uint32_t base = align1024(w_bytes) + align1024(u_bytes) + align1024(t1s) + e_ring + 1024 /*tab*/ +
                            1024 /*bars*/ + 1024 /*align*/;
      const int nbuf_env = getenv("LRS_PW_EPIBUF") ? atoi(getenv("LRS_PW_EPIBUF")) : 0;  // plan override
      int epi_nbuf = ft ? 2 : (nbuf_env ? nbuf_env : 2);
      if (base + 8u * 2048u * epi_nbuf >= static_cast<uint32_t>(kMaxSmem)) continue;
      int ns = static_cast<int>((kMaxSmem - base - 8u * 2048u * epi_nbuf) / slot);
      if (!ft && !nbuf_env && epi_nbuf == 2 && ns < kPMaxSlots &&
          static_cast<int>((kMaxSmem - base - 8u * 2048u) / slot) > ns) {
        epi_nbuf = 1;
        ns = static_cast<int>((kMaxSmem - base - 8u * 2048u) / slot);
      }
      ns = std::min(ns, kPMaxSlots);
      if (!ft && ns * slot < e_bytes) continue;  // the staging must fit in the ring
      const uint32_t fixed = base + 8u * 2048u * epi_nbuf;
      // slots are released chunk by chunk (tcgen05.commit after each chunk's MMAs), but the
      // producer lanes request a tile's chunks in parallel, so the ring must hold a whole
      // tile: with fewer slots two lanes would wait on two phases of one slot's mbarrier at
      // once, and a parity wait cannot tell phase r from phase r + 2
      const int nq = ft ? n_ck : (n_x + cpi - 1) / cpi + (n_tk + cpi - 1) / cpi;  // ring items per tile
      if (ns < nq) continue;
      // cost (cycles per CTA): tiles x max(MMA, operand inflow, the group's share of the HBM
      // write of Y); sparse MMA ~ (A 4 KB + B bp*64 B) / 128 B/clk, dense ~ (4 KB + bp*32 B) / 128
      const int gpg = h->sms / G;
      const long long n_pt = (p_max + bp - 1) / bp;
      const long long tiles = (n_pt + gpg - 1) / gpg;
      const double sp = std::max(100.0, (4096.0 + 64.0 * bp) / 128.0), dn = std::max(50.0, (4096.0 + 32.0 * bp) / 128.0);
      const double mma = static_cast<double>(nblk) * 2 * sp + mpc * n_tk * (sw_t / 32.0) * dn;
      const double in = (static_cast<double>(n_x) * bp * 128 + n_tk * bp * sw_t) / 60.0;
      const double out = static_cast<double>(bp) * mpc * 128 * 2 * (G * gpg) / 3300.0;  // ~3.3 KB/clk of HBM writes
      const double shallow = ns < nq + 2 ? 1.25 : 1.0;
      // + the MMA thread's serial hand-off per ring item (wait ~160 + commit ~50 + loop:
      // ~500 cycles measured, tools/loop_cost3.cu, tools/ptrace.py)
      const double cost =
          static_cast<double>(tiles) * std::max(mma + 500.0 * nq, std::max(in, out)) * shallow + 400.0 * mpc;
      Plan c;
      c.cost = cost; c.mpc = mpc; c.bp = bp; c.ns = ns; c.nblk = nblk; c.gpg = gpg;
      c.w_bytes = w_bytes; c.ft = ft; c.epi_nbuf = epi_nbuf; c.cpi = cpi;
      c.smem = fixed + static_cast<uint32_t>(ns) * slot;
      all.push_back(c);
      if (cost < best.cost) best = c;
    }
    }  // cpi
  }
  }  // ft
  if (!best.mpc) return LRS_OK;
  if (!force) {  // the best few distinct (mpc, bp, cpi) plans for the create-time timing
    std::stable_sort(all.begin(), all.end(), [](const Plan& a, const Plan& b) { return a.cost < b.cost; });
    h->pw_cands.clear();
    for (const Plan& c : all)
      if (h->pw_cands.size() < 4) h->pw_cands.push_back(c);
  }
  // a re-applied plan (autotune_pw) replaces the previous one's images
  for (void** b : {&h->pw_w, &h->pw_e, &h->pw_tab, &h->pw_u})
    if (*b) {
      cudaFree(*b);
      *b = nullptr;
    }
  h->px_ptr = nullptr;  // tensor-map boxes depend on bp
  h->py_ptr = nullptr;
  const int mpc = best.mpc, G = (n_mt + mpc - 1) / mpc, nblk = best.nblk;
  // ---- per-group images: [mpc][n_tk] V^T blocks, then the 2:4 blocks; metadata; tables
  std::vector<uint8_t> wimg(static_cast<size_t>(G) * best.w_bytes, 0);
  std::vector<uint8_t> eimg(static_cast<size_t>(G) * std::max(nblk, 1) * 2048u, 0x44);
  std::vector<uint16_t> tab(static_cast<size_t>(G) * mpc * n_ck, 0);
  const uint32_t dense = static_cast<uint32_t>(mpc * n_tk) * 128u * sw_t;
  const int r1 = d->rank_in;
  for (int g = 0; g < G; ++g) {
    uint8_t* wg = &wimg[static_cast<size_t>(g) * best.w_bytes];
    for (int m = 0; m < mpc; ++m)
      for (int tk = 0; tk < n_tk; ++tk)
        for (int r = 0; r < 128; ++r) {
          const int j = (g * mpc + m) * 128 + r;
          if (j >= cout) continue;
          for (int e2 = 0; e2 < t_kc; ++e2) {
            const int bb = tk * t_kc + e2;
            if (bb >= r1) continue;
            const uint16_t bits = static_cast<const uint16_t*>(d->u_out)[static_cast<size_t>(bb) * cout + j];
            memcpy(wg + static_cast<size_t>(m * n_tk + tk) * 128 * sw_t + swz_off(r, 2 * e2, static_cast<int>(sw_t)),
                   &bits, 2);
          }
        }
    if (!n_x) continue;
    int nb = 0;
    for (int m = 0; m < mpc; ++m)
      for (int c = 0; c < n_ck; ++c) {
        const int mt = g * mpc + m;
        const int first = nb;
        int keys[2] = {-1, -1}, cnt = 1;
        if (mt < n_mt) {
          keys[0] = mt * n_ck + c;
          if (S.res_tab[keys[0]] >= 0) keys[cnt++] = S.res_tab[keys[0]];
        }
        for (int q = 0; q < cnt; ++q, ++nb) {
          uint8_t* blk = wg + dense + static_cast<size_t>(nb) * 8192;
          uint8_t* eb = &eimg[(static_cast<size_t>(g) * nblk + nb) * 2048];
          if (keys[q] < 0) continue;  // an M-tile past c_out: zero block (its Y is never stored)
          for (int r = 0; r < 128; ++r)
            for (int k = 0; k < 32; ++k)
              memcpy(blk + swz_off(r, 2 * k, 64), &S.as[(static_cast<size_t>(keys[q]) * 128 + r) * 32 + k], 2);
          memcpy(eb, &S.ee[static_cast<size_t>(keys[q]) * 128 * 4], 2048);
        }
        tab[(static_cast<size_t>(g) * mpc + m) * n_ck + c] = static_cast<uint16_t>(first | (cnt << 12));
      }
  }
  lrs_status st;
  if ((st = upload(&h->pw_w, wimg)) != LRS_OK) return st;
  if ((st = upload(&h->pw_e, eimg)) != LRS_OK) return st;
  {
    std::vector<uint8_t> tb(tab.size() * 2);
    memcpy(tb.data(), tab.data(), tb.size());
    if ((st = upload(&h->pw_tab, tb)) != LRS_OK) return st;
  }
  if (best.ft) {  // U_in^T blocks [n_ck][R1p rows x 128 B] (64 channels per row), SW128
    std::vector<uint8_t> ui(static_cast<size_t>(n_ck) * r1p * 128, 0);
    for (int c = 0; c < n_ck; ++c)
      for (int r = 0; r < r1; ++r)
        for (int k = 0; k < 64; ++k) {
          const uint16_t bits = static_cast<const uint16_t*>(d->u_in)[static_cast<size_t>(c * 64 + k) * r1 + r];
          memcpy(&ui[static_cast<size_t>(c) * r1p * 128 + swz_off(r, 2 * k, 128)], &bits, 2);
        }
    if ((st = upload(&h->pw_u, ui)) != LRS_OK) return st;
  }
  PwParams& q = h->pp;
  memset(&q, 0, sizeof(q));
  q.img_w = static_cast<const uint8_t*>(h->pw_w);
  q.img_e = static_cast<const uint8_t*>(h->pw_e);
  q.tab = static_cast<const uint16_t*>(h->pw_tab);
  q.cout = cout;
  q.n_ck = n_ck;
  q.n_x = n_x;
  q.n_tk = n_tk;
  q.t_kc = t_kc;
  q.sw_t = sw_t;
  q.bp = best.bp;
  q.mpc = mpc;
  q.n_groups = G;
  q.w_bytes = best.w_bytes;
  q.dense_bytes = dense;
  q.nblk_max = nblk;
  q.ns = best.ns;
  q.cpi = best.cpi;
  q.slot_bytes = static_cast<uint32_t>(best.cpi * best.bp) * 128u;
  q.acc_cols = static_cast<uint32_t>(mpc * best.bp);
  if (best.ft) {
    q.r1p = r1p;
    q.u_bytes = static_cast<uint32_t>(n_ck * r1p) * 128u;
    q.img_u = static_cast<const uint8_t*>(h->pw_u);
    q.t1s_bytes = 128u * static_cast<uint32_t>(r1p) * 2u;
    q.t1_col0 = 2 * q.acc_cols;
    q.e_col0 = q.t1_col0 + 2u * static_cast<uint32_t>(r1p);
    q.off_u = align1024(best.w_bytes);
    q.off_t1s = q.off_u + align1024(q.u_bytes);
    const uint32_t e_bytes = static_cast<uint32_t>(nblk) * 2048u;
    const bool e_shared = e_bytes <= q.t1s_bytes;
    q.off_e = e_shared ? q.off_t1s + q.t1s_bytes : q.off_t1s + align1024(2 * q.t1s_bytes);
    q.off_ring = q.off_t1s + align1024(2 * q.t1s_bytes) + (e_shared ? 0u : align1024(e_bytes));
    q.e_slot0 = best.ns;
    q.epi_nbuf = 2;
  } else {
    q.e_col0 = 2 * q.acc_cols;
    q.off_ring = align1024(best.w_bytes);
    // the metadata staging occupies the ring's last slots until its copies to TMEM complete
    const uint32_t e_bytes = static_cast<uint32_t>(nblk) * 2048u;
    const int ke = static_cast<int>((e_bytes + q.slot_bytes - 1) / q.slot_bytes);
    q.e_slot0 = best.ns - ke;
    q.off_e = q.off_ring + static_cast<uint32_t>(q.e_slot0) * q.slot_bytes;
    q.epi_nbuf = best.epi_nbuf;
  }
  q.off_epi = q.off_ring + static_cast<uint32_t>(best.ns) * q.slot_bytes;
  q.off_tab = q.off_epi + 8u * 2048u * static_cast<uint32_t>(q.epi_nbuf);
  q.off_bar = q.off_tab + 1024;
  q.relu = 0;
#ifdef LRS_EXPERIMENTS
  if (const char* e = getenv("LRS_PW_DBG")) q.dbg = atoi(e);
#endif
  h->pw_smem = best.smem;
  h->pw_grid_per_group = best.gpg;
  h->w_main_blocks = n_x ? n_mt * n_ck : 0;
  h->w_res_blocks = S.nres;
  h->use_pw = true;
  h->pw_ft = best.ft != 0;
  if (getenv("LRS_VERBOSE"))
    fprintf(stderr, "[lrs] pw plan: fused a1 %d mpc %d groups %d bp %d ns %d cpi %d epi bufs %d blocks/group %d ctas/group %d smem %u B\n",
            best.ft, mpc, G, best.bp, best.ns, best.cpi, best.epi_nbuf, nblk, best.gpg, best.smem);
  return LRS_OK;
}
}  // namespace

extern "C" {

const char* lrs_conv_last_error(void) { return g_err.c_str(); }

// The early-start protocol for core -> fused-kernel layers: a second T2 (and overflow-gather
// scratch) with the fused kernel's tensor maps for both, so forward f + 1's core kernel can
// run while forward f's fused kernel still reads its T2 (LRS_NO_EARLY=1: off).
static lrs_status setup_early(lrs_conv* h, const lrs_conv_desc* d) {
  h->no_early = getenv("LRS_NO_EARLY") != nullptr;
  if (h->use_pw && !h->pw_ft && !getenv("LRS_NO_EARLY")) {
    // the projection GEMM -> pointwise kernel chain: T1 alternates between two buffers
    const size_t t1_bytes = static_cast<size_t>(d->batch_max) * d->in_h * d->in_w * h->r1p * h->esz;
    if (!h->t1b && cudaMalloc(&h->t1b, t1_bytes) != cudaSuccess) {
      cudaGetLastError();
      h->t1b = nullptr;
      return LRS_OK;  // no room: keep the single-buffer protocol
    }
    h->dbuf_pw = true;
    return LRS_OK;
  }
  if (!h->use_core || !h->use_w || h->svd || getenv("LRS_NO_EARLY")) return LRS_OK;
  WconvParams& w = h->wp;
  const size_t t2_bytes = static_cast<size_t>(d->batch_max) * h->ho * h->wo * h->r2p * h->esz;
  if (cudaMalloc(&h->t2b, t2_bytes) != cudaSuccess) {
    cudaGetLastError();
    h->t2b = nullptr;
    return LRS_OK;  // no room: keep the single-buffer protocol
  }
  h->tmT_par[0] = w.tmT;
  lrs_status st;
  const uint64_t bm = static_cast<uint64_t>(d->batch_max), rp = static_cast<uint64_t>(h->r2p);
  const uint64_t ho = static_cast<uint64_t>(h->ho), wo = static_cast<uint64_t>(h->wo);
  const uint32_t box[4] = {static_cast<uint32_t>(w.t_kc), static_cast<uint32_t>(w.ipw), static_cast<uint32_t>(w.tbox_w),
                           static_cast<uint32_t>(w.th)};
  const uint32_t estr[4] = {1, 1, 1, 1};
  {
    uint64_t dims[4] = {rp, bm, wo, ho};
    uint64_t strides[3] = {ho * wo * rp * 2, rp * 2, wo * rp * 2};
    if ((st = encode_t(&h->tmT_par[1], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, h->t2b, dims, strides,
                       const_cast<uint32_t*>(box), const_cast<uint32_t*>(estr), w.sw_t)) != LRS_OK)
      return st;
  }
  if (w.n_gk) {
    const uint64_t gch = static_cast<uint64_t>(w.g_ch);
    const size_t gb = bm * ho * wo * gch * 2;
    LRS_CUDA(cudaMalloc(&h->w_gb, gb));
    LRS_CUDA(cudaMemset(h->w_gb, 0, gb));
    h->tmG_par[0] = w.tmG;
    uint64_t dims[4] = {gch, bm, wo, ho};
    uint64_t strides[3] = {ho * wo * gch * 2, gch * 2, wo * gch * 2};
    if ((st = encode_t(&h->tmG_par[1], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, h->w_gb, dims, strides,
                       const_cast<uint32_t*>(box), const_cast<uint32_t*>(estr), w.sw_t)) != LRS_OK)
      return st;
  }
  h->dbuf = true;
  return LRS_OK;
}

// Output range of the library's last forward on each (device, stream): a forward whose X
// overlaps it must not start before that forward's last kernel completes (early = 0).
std::mutex g_out_mu;
std::map<std::pair<int, cudaStream_t>, std::pair<uintptr_t, uintptr_t>> g_last_out;

bool x_after_previous_output(int dev, cudaStream_t s, const void* x, size_t xbytes) {
  std::lock_guard<std::mutex> lk(g_out_mu);
  auto it = g_last_out.find({dev, s});
  if (it == g_last_out.end()) return false;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(x), hi = lo + xbytes;
  return lo < it->second.second && it->second.first < hi;
}

void record_output(int dev, cudaStream_t s, const void* y, size_t ybytes) {
  std::lock_guard<std::mutex> lk(g_out_mu);
  const uintptr_t lo = reinterpret_cast<uintptr_t>(y);
  g_last_out[{dev, s}] = {lo, lo + ybytes};
}

// Time the best few core plans on the device (after every kernel is built): for the
// full grid and, when the expansion + sparse kernel leaves SMs free, for a grid of
// exactly those SMs -- the two kernels of consecutive forwards are then co-resident and
// overlap under PDL (C2: the core on 36 SMs while the fused kernel's sparse windows run
// on the other 112).  Each plan runs back-to-back forwards on zero-filled scratch
// buffers of batch_max images; the fastest stays.  LRS_NO_AUTOTUNE=1 keeps the model's
// choice; any LRS_CORE_* override disables the tuning.
// best_us (optional): the winning plan's time per forward, or -1 when nothing was timed.
static lrs_status autotune_core(lrs_conv* h, const lrs_conv_desc* d, float* best_us = nullptr) {
  if (best_us) *best_us = -1.f;
  if (!h->use_core || getenv("LRS_NO_AUTOTUNE") || getenv("LRS_CORE_IPT") || getenv("LRS_CORE_TH") ||
      getenv("LRS_CORE_GRID") || h->skip)
    return LRS_OK;
  const int n = d->batch_max;
  std::vector<std::tuple<int, int, int, int>> plans;  // (ipt, th, grid, gmode)
  std::vector<int> grids{h->sms};
  if (h->use_w) {
    const WconvParams& w = h->wp;
    const long long wt = static_cast<long long>((n + w.ipw - 1) / w.ipw) * w.bands * w.cbands * w.n_mt;
    const int free_sms = h->sms - static_cast<int>(std::min<long long>(wt, h->sms));
    if (free_sms >= 16) grids.push_back(free_sms);
  }
  for (int g : grids) {
    const auto cand = core_candidates(h, d, g);
    const CoreGeom G = core_geom(h, d);
    for (size_t i = 0; i < cand.size() && i < 4; ++i) {
      plans.emplace_back(std::get<1>(cand[i]), std::get<2>(cand[i]), g, 0);
      CoreParams q0, q1;
      memset(&q0, 0, sizeof(q0));
      memset(&q1, 0, sizeof(q1));
      core_layout(G, std::get<1>(cand[i]), std::get<2>(cand[i]), q0, 0);
      if (core_layout(G, std::get<1>(cand[i]), std::get<2>(cand[i]), q1, 1) && q1.ns_x > q0.ns_x)
        plans.emplace_back(std::get<1>(cand[i]), std::get<2>(cand[i]), g, 1);  // deeper X ring, G streamed
    }
  }
  if (plans.size() <= 1) return LRS_OK;
  const size_t xb = static_cast<size_t>(n) * d->in_h * d->in_w * d->c_in * 2;
  const size_t yb = static_cast<size_t>(n) * h->ho * h->wo * d->c_out * 2;
  void *xs = nullptr, *ys = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  lrs_status st = LRS_OK;
  const CoreParams keep = h->cp;
  const uint32_t keep_smem = h->core_smem;
  const int keep_grid = h->core_grid;
  float best = 1e30f;
  int bi = -1;
  bool ready = true;
  {
    cudaError_t e = cudaMalloc(&xs, xb);
    if (e == cudaSuccess) e = cudaMalloc(&ys, yb);
    if (e == cudaErrorMemoryAllocation) {
      // no room for the scratch (huge batch_max): keep the cost model's plan, not an error
      cudaGetLastError();
      ready = false;
      if (getenv("LRS_VERBOSE")) fprintf(stderr, "[lrs] autotune skipped: no memory for %zu B of scratch\n", xb + yb);
    } else {
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreate(&e0);
      if (e == cudaSuccess) e = cudaEventCreate(&e1);
      if (e == cudaSuccess) e = cudaMemsetAsync(xs, 0, xb, s);
      if (e != cudaSuccess) {  // a driver error is an error (only an OOM keeps the model's plan)
        st = fail(LRS_ERR_CUDA, "autotune setup: %s", cudaGetErrorString(e));
        ready = false;
      }
    }
  }
  for (size_t i = 0; ready && st == LRS_OK && i < plans.size(); ++i) {
    apply_core_plan(h, d, std::get<0>(plans[i]), std::get<1>(plans[i]), std::get<2>(plans[i]), std::get<3>(plans[i]));
    for (int r = 0; r < 3 && st == LRS_OK; ++r) st = lrs_conv_forward(h, xs, ys, n, s);
    if (st != LRS_OK) break;
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10 && st == LRS_OK; ++r) st = lrs_conv_forward(h, xs, ys, n, s);
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) st = fail(LRS_ERR_CUDA, "autotune: %s", cudaGetErrorString(cudaGetLastError()));
    float ms = 0.f;
    if (st == LRS_OK) cudaEventElapsedTime(&ms, e0, e1);
    if (getenv("LRS_VERBOSE"))
      fprintf(stderr, "[lrs] autotune core ipt=%d th=%d grid=%d gmode=%d: %.2f us/forward\n", std::get<0>(plans[i]),
              std::get<1>(plans[i]), std::get<2>(plans[i]), std::get<3>(plans[i]), ms * 100.f);
    if (st == LRS_OK && ms < best) {
      best = ms;
      bi = static_cast<int>(i);
    }
  }
  if (ready && st == LRS_OK && bi >= 0) {
    apply_core_plan(h, d, std::get<0>(plans[bi]), std::get<1>(plans[bi]), std::get<2>(plans[bi]), std::get<3>(plans[bi]));
    if (best_us) *best_us = best * 100.f;  // 10 forwards per timing
  } else {
    h->cp = keep;
    h->core_smem = keep_smem;
    h->core_grid = keep_grid;
    h->cx_ptr = nullptr;
  }
  h->wx_ptr = nullptr;  // tensor maps cached for the scratch X
  h->xmap_ptr = nullptr;
  if (s) cudaStreamSynchronize(s);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  if (xs) cudaFree(xs);
  if (ys) cudaFree(ys);
  return st;
}

// The windowed kernel's buffers and plan state, freed before autotune_w rebuilds it
static void free_wconv(lrs_conv* h) {
  for (void** b : {&h->w_as, &h->w_e, &h->w_dense_img, &h->w_gtab, &h->w_g, &h->t2b, &h->w_gb})
    if (*b) {
      cudaFree(*b);
      *b = nullptr;
    }
  if (h->w_res) {
    cudaFree(h->w_res);
    h->w_res = nullptr;
  }
  h->use_w = false;
  h->dbuf = false;
  h->par = 0;
  h->wx_ptr = nullptr;  // the X map's box depends on the band height
}

// Time the windowed kernel's band height: the cost model's choice against the tallest band
// that fits (one tile per image group per M-tile), each with the core kernel's plan tuned
// for it (autotune_core: the co-resident grid depends on the windowed kernel's tile count).
// The model prices MMA issue and item hand-offs per block; at C3 with 128 images per GPU (the
// 2-GPU shard) it picked 2-row bands (45.6 us) where 7-row bands with a co-resident core run
// 42.7 us (profiles/r02_ablate_wconv_th_small_batch.log).  Every band height computes the same
// products in the same order per output (tests/test_gpu_sparse_tc.py).  Any LRS_WCONV_* plan
// override or LRS_NO_AUTOTUNE keeps the model's plan.  *core_tuned: autotune_core has run.
static lrs_status autotune_w(lrs_conv* h, const lrs_conv_desc* d, const ConvGeom& g, bool* core_tuned) {
  *core_tuned = false;
  if (!h->use_w || getenv("LRS_NO_AUTOTUNE") || getenv("LRS_WCONV_TH") || getenv("LRS_WCONV_IPW") ||
      getenv("LRS_WCONV_PAIR") || getenv("LRS_WCONV_BPI") || getenv("LRS_WCONV_NS") || getenv("LRS_WCONV_CB") || h->skip)
    return LRS_OK;
  const int th0 = h->wp.th, thx = h->wth_max;
  if (thx <= th0) return LRS_OK;
  const int n = d->batch_max;
  const size_t xb = static_cast<size_t>(n) * d->in_h * d->in_w * d->c_in * 2;
  const size_t yb = static_cast<size_t>(n) * h->ho * h->wo * d->c_out * 2;
  void *xs = nullptr, *ys = nullptr;
  cudaError_t e = cudaMalloc(&xs, xb);
  if (e == cudaSuccess) e = cudaMalloc(&ys, yb);
  if (e == cudaErrorMemoryAllocation) {  // no room for the scratch: keep the model's plan
    cudaGetLastError();
    if (xs) cudaFree(xs);
    return LRS_OK;
  }
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  lrs_status st = LRS_OK;
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  if (e == cudaSuccess) e = cudaMemsetAsync(xs, 0, xb, s);
  if (e != cudaSuccess) st = fail(LRS_ERR_CUDA, "autotune setup: %s", cudaGetErrorString(e));
  const int cand[2] = {th0, thx};
  float best = 1e30f;
  int bi = -1, built = th0;
  for (int i = 0; i < 2 && st == LRS_OK; ++i) {
    if (cand[i] != built) {
      free_wconv(h);
      h->force_wth = cand[i];
      st = build_wconv(h, d, g);
      h->force_wth = 0;
      built = cand[i];
      if (st != LRS_OK) break;
      if (!h->use_w) continue;  // not feasible after all
      h->wp.epi = h->epi;
      h->wp.relu = d->out_relu ? 1 : 0;
      if ((st = setup_early(h, d)) != LRS_OK) break;
    }
    float us = -1.f;
    if ((st = autotune_core(h, d, &us)) != LRS_OK) break;  // the core plan for this band height
    if (us < 0.f) {  // no core plan to time: time the forward as it is
      for (int r = 0; r < 3 && st == LRS_OK; ++r) st = lrs_conv_forward(h, xs, ys, n, s);
      if (st != LRS_OK) break;
      cudaEventRecord(e0, s);
      for (int r = 0; r < 10 && st == LRS_OK; ++r) st = lrs_conv_forward(h, xs, ys, n, s);
      cudaEventRecord(e1, s);
      if (cudaEventSynchronize(e1) != cudaSuccess)
        st = fail(LRS_ERR_CUDA, "autotune: %s", cudaGetErrorString(cudaGetLastError()));
      float ms = 0.f;
      if (st == LRS_OK) cudaEventElapsedTime(&ms, e0, e1);
      us = ms * 100.f;
    }
    if (getenv("LRS_VERBOSE")) fprintf(stderr, "[lrs] autotune wconv th=%d: %.2f us/forward\n", cand[i], us);
    if (st == LRS_OK && us < best) {
      best = us;
      bi = i;
    }
  }
  if (st == LRS_OK && bi >= 0 && cand[bi] != built) {
    free_wconv(h);
    h->force_wth = cand[bi];
    st = build_wconv(h, d, g);
    h->force_wth = 0;
    if (st == LRS_OK) {
      h->wp.epi = h->epi;
      h->wp.relu = d->out_relu ? 1 : 0;
      st = setup_early(h, d);
    }
    if (st == LRS_OK) st = autotune_core(h, d);
  }
  *core_tuned = st == LRS_OK;
  if (s) cudaStreamSynchronize(s);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  if (xs) cudaFree(xs);
  if (ys) cudaFree(ys);
  if (st == LRS_OK && !h->use_w) st = fail(LRS_ERR_UNSUPPORTED, "autotune: the windowed kernel's plan vanished");
  return st;
}

// Time the pointwise kernel's best few plans (build_pw's cost-model candidates) on the
// device like autotune_core and keep the fastest: the model's tile-rate terms were off by
// up to 15 % between neighbouring plans at C4 (profiles/r02_ablate_pw_cpi_c4.log).  Every
// plan computes the same bits (tests/test_gpu_pw.py).  Any LRS_PW_* override or
// LRS_NO_AUTOTUNE keeps the model's plan.
static lrs_status autotune_pw(lrs_conv* h, const lrs_conv_desc* d) {
  if (!h->use_pw || h->pw_cands.size() < 2 || getenv("LRS_NO_AUTOTUNE") || getenv("LRS_PW_MPC") ||
      getenv("LRS_PW_BP") || getenv("LRS_PW_CPI") || getenv("LRS_PW_EPIBUF") || getenv("LRS_PW_FT") || h->skip)
    return LRS_OK;
  const int n = d->batch_max;
  const size_t xb = static_cast<size_t>(n) * d->in_h * d->in_w * d->c_in * 2;
  const size_t yb = static_cast<size_t>(n) * h->ho * h->wo * d->c_out * 2;
  void *xs = nullptr, *ys = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  lrs_status st = LRS_OK;
  cudaError_t e = cudaMalloc(&xs, xb);
  if (e == cudaSuccess) e = cudaMalloc(&ys, yb);
  if (e == cudaErrorMemoryAllocation) {  // no room for the scratch: keep the model's plan
    cudaGetLastError();
    if (xs) cudaFree(xs);
    return LRS_OK;
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  if (e == cudaSuccess) e = cudaMemsetAsync(xs, 0, xb, s);
  if (e != cudaSuccess) st = fail(LRS_ERR_CUDA, "autotune setup: %s", cudaGetErrorString(e));
  const std::vector<PwPlan> cands = h->pw_cands;
  float best = 1e30f;
  int bi = -1;
  for (size_t i = 0; st == LRS_OK && i < cands.size(); ++i) {
    if ((st = build_pw(h, d, &cands[i])) != LRS_OK) break;
    h->pp.epi = h->epi;
    h->pp.relu = d->out_relu ? 1 : 0;
    for (int r = 0; r < 3 && st == LRS_OK; ++r) st = lrs_conv_forward(h, xs, ys, n, s);
    if (st != LRS_OK) break;
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10 && st == LRS_OK; ++r) st = lrs_conv_forward(h, xs, ys, n, s);
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) st = fail(LRS_ERR_CUDA, "autotune: %s", cudaGetErrorString(cudaGetLastError()));
    float ms = 0.f;
    if (st == LRS_OK) cudaEventElapsedTime(&ms, e0, e1);
    if (getenv("LRS_VERBOSE"))
      fprintf(stderr, "[lrs] autotune pw mpc=%d bp=%d cpi=%d: %.2f us/forward\n", cands[i].mpc, cands[i].bp,
              cands[i].cpi, ms * 100.f);
    if (st == LRS_OK && ms < best) {
      best = ms;
      bi = static_cast<int>(i);
    }
  }
  if (st == LRS_OK && bi >= 0 && (st = build_pw(h, d, &cands[bi])) == LRS_OK) {
    h->pp.epi = h->epi;
    h->pp.relu = d->out_relu ? 1 : 0;
  }
  if (s) cudaStreamSynchronize(s);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  if (xs) cudaFree(xs);
  if (ys) cudaFree(ys);
  return st;
}

lrs_status lrs_conv_create(const lrs_conv_desc* d, int device, lrs_conv** out) {
  if (!out) return fail(LRS_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  lrs_status st = validate(d);
  if (st != LRS_OK) return st;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRS_ERR_CUDA, "no CUDA device available (there is no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(LRS_ERR_INVALID_ARGUMENT, "device %d out of range", device);
  int prev = 0;
  LRS_CUDA(cudaGetDevice(&prev));
  LRS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  LRS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    cudaSetDevice(prev);
    return fail(LRS_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a only",
                device, prop.major, prop.minor);
  }

  lrs_conv* h = new lrs_conv();
  h->d = *d;
  h->d.u_in = h->d.core = h->d.u_out = nullptr;
  h->d.row_ptr = nullptr;
  h->d.col_idx = nullptr;
  h->d.values = nullptr;
  h->device = device;
  h->sms = prop.multiProcessorCount;
  #ifdef LRS_EXPERIMENTS
  if (const char* e = getenv("LRS_SKIP")) h->skip = atoi(e);  // stage skips: timing bisection only (wrong Y)
#endif
  h->f32 = d->dtype == LRS_DTYPE_F32;
  h->svd = d->core == nullptr;
  h->cp_core = d->core_kind == LRS_CORE_CP;
  h->esz = h->f32 ? 4 : 2;
  const bool f32 = h->f32;
  const int esz = h->esz;
  const int cin = d->c_in, cout = d->c_out, kh = d->kernel_h, kw = d->kernel_w;
  const int H = d->in_h, W = d->in_w;
  h->ho = (H + 2 * d->pad_h - kh) / d->stride_h + 1;
  h->wo = (W + 2 * d->pad_w - kw) / d->stride_w + 1;
  const int ho = h->ho, wo = h->wo;
  const int r1 = d->rank_in, r2 = h->svd ? d->rank_in : d->rank_out;
  // ranks padded to the MMA granularity; a rank consumed as the K of a TMEM-window
  // operand (T2, or T1 of the SVD pair) is padded to 16, 32 or a multiple of 64
  auto t_round = [](int r) { return r <= 16 ? 16 : (r <= 32 ? 32 : round_up(r, 64)); };
  // LRS_NO_SPTC: no 2:4 sparse tensor-core kernels -- bf16 layers take engine 0 (the a3 GEMM
  // with the SIMT CSR sparse term in its epilogue), the head-to-head of DESIGN §5
  const bool bf16_w = !f32 && cin % 64 == 0 && !getenv("LRS_NO_SPTC");
  h->r1p = (bf16_w && h->svd) ? t_round(r1) : round_up(r1, 16);
  h->r2p = h->svd ? h->r1p : (bf16_w ? t_round(r2) : round_up(r2, 16));
  if (h->cp_core) h->r1p = h->r2p = std::max(h->r1p, h->r2p);  // T1 and T2 share one row pitch
  h->bn = cout <= 64 ? 64 : 128;
  h->cout_p = bf16_w ? round_up(cout, 128) : round_up(cout, h->bn);
  const int r1p = h->r1p, r2p = h->r2p, bn = h->bn, cout_p = h->cout_p;
  const long long pin_max = static_cast<long long>(d->batch_max) * H * W;
  const long long p_max = static_cast<long long>(d->batch_max) * ho * wo;

  auto cleanup_fail = [&](lrs_status s) {
    lrs_conv_destroy(h);
    cudaSetDevice(prev);
    return s;
  };

  // ---------------------------------------------------------------- weights
  {
    std::vector<float> m(static_cast<size_t>(r1p) * cin, 0.f);  // U_in^T [R1p][Cin]
    for (int c = 0; c < cin; ++c)
      for (int a = 0; a < r1; ++a) m[static_cast<size_t>(a) * cin + c] = host_val(d->u_in, (size_t)c * r1 + a, f32);
    if ((st = upload(&h->w_uin, pack_matrix(m, r1p, cin, f32))) != LRS_OK) return cleanup_fail(st);
  }
  if (h->cp_core) {
    // CP factors: core = B [kernel_h][R] followed by C [kernel_w][R] (dtype), kept fp32 [k][R1p]
    std::vector<float> b(static_cast<size_t>(kh) * r1p, 0.f), c(static_cast<size_t>(kw) * r1p, 0.f);
    for (int y = 0; y < kh; ++y)
      for (int a = 0; a < r1; ++a) b[static_cast<size_t>(y) * r1p + a] = host_val(d->core, (size_t)y * r1 + a, f32);
    for (int x = 0; x < kw; ++x)
      for (int a = 0; a < r1; ++a)
        c[static_cast<size_t>(x) * r1p + a] = host_val(d->core, (size_t)(kh + x) * r1 + a, f32);
    std::vector<uint8_t> bb(b.size() * 4), cb(c.size() * 4);
    memcpy(bb.data(), b.data(), bb.size());
    memcpy(cb.data(), c.data(), cb.size());
    void* pb = nullptr;
    void* pc = nullptr;
    if ((st = upload(&pb, bb)) != LRS_OK) return cleanup_fail(st);
    h->w_cpb = static_cast<float*>(pb);
    if ((st = upload(&pc, cb)) != LRS_OK) return cleanup_fail(st);
    h->w_cpc = static_cast<float*>(pc);
  } else if (!h->svd) {
    const int kk = kh * kw;
    std::vector<float> m(static_cast<size_t>(r2p) * kk * r1p, 0.f);  // G^T [R2p][tap*R1p + a]
    for (int a = 0; a < r1; ++a)
      for (int b = 0; b < r2; ++b)
        for (int t = 0; t < kk; ++t)
          m[static_cast<size_t>(b) * kk * r1p + static_cast<size_t>(t) * r1p + a] =
              host_val(d->core, ((size_t)a * r2 + b) * kk + t, f32);
    if ((st = upload(&h->w_core, pack_matrix(m, r2p, kk * r1p, f32))) != LRS_OK) return cleanup_fail(st);
  }
  {
    std::vector<float> m(static_cast<size_t>(cout_p) * r2p, 0.f);  // U_out^T [Cout_p][R2p]
    for (int b = 0; b < r2; ++b)
      for (int j = 0; j < cout; ++j) m[static_cast<size_t>(j) * r2p + b] = host_val(d->u_out, (size_t)b * cout + j, f32);
    if ((st = upload(&h->w_uout, pack_matrix(m, cout_p, r2p, f32))) != LRS_OK) return cleanup_fail(st);
  }
  // ---------------------------------------------------------------- scratch
  if (cudaMalloc(&h->t1, static_cast<size_t>(pin_max) * r1p * esz) != cudaSuccess)
    return cleanup_fail(fail(LRS_ERR_OUT_OF_MEMORY, "T1 scratch allocation failed"));
  if (!h->svd && cudaMalloc(&h->t2, static_cast<size_t>(p_max) * r2p * esz) != cudaSuccess)
    return cleanup_fail(fail(LRS_ERR_OUT_OF_MEMORY, "T2 scratch allocation failed"));

  // ---------------------------------------------------------------- a1: T1 = X U_in
  {
    GemmParams& p = h->a1.p;
    memset(&p, 0, sizeof(p));
    const uint32_t sw = pick_sw(cin * esz);
    h->sw_a1 = sw;
    h->kc_a1 = static_cast<int>(sw) / esz;
    h->a1.smem = plan_stage(p, f32, cin * esz, sw, r1p, r1p, kTileM * sw, 0);
    if (!h->a1.smem) return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "a1 does not fit in shared memory"));
    p.amode = AMODE_2D;
    p.out = h->t1;
    p.out_ld = r1p;
    uint64_t dims[2] = {static_cast<uint64_t>(cin), static_cast<uint64_t>(r1p) * (f32 ? 2 : 1)};
    uint64_t strides[1] = {static_cast<uint64_t>(cin) * esz};
    uint32_t box[2] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(r1p)};
    uint32_t estr[2] = {1, 1};
    if ((st = encode(&p.tmB, f32, 2, h->w_uin, dims, strides, box, estr, sw)) != LRS_OK) return cleanup_fail(st);
    h->a1.name = "a1_proj";
    h->a1.kid = f32 ? K_STORE_F32 : K_STORE_BF16;
  }
  ConvGeom g{};
  g.h = H; g.w = W; g.ho = ho; g.wo = wo; g.kh = kh; g.kw = kw;
  g.sh = d->stride_h; g.sw = d->stride_w; g.ph = d->pad_h; g.pw = d->pad_w;
  // ---------------------------------------------------------------- a2: T2 = conv(T1, G)
  if (h->cp_core) {
    CpDwParams& q = h->cpp;
    q.t1 = h->t1;
    q.t2 = h->t2;
    q.b = h->w_cpb;
    q.c = h->w_cpc;
    q.h = H; q.w = W; q.ho = ho; q.wo = wo; q.ld = r1p;
    q.kh = kh; q.kw = kw; q.sh = d->stride_h; q.sw = d->stride_w; q.ph = d->pad_h; q.pw = d->pad_w;
  } else if (!h->svd) {
    GemmParams& p = h->a2.p;
    memset(&p, 0, sizeof(p));
    // K chunks must not straddle taps: the swizzle width has to divide R1p * esz
    const uint32_t sw = (r1p * esz) % 128 == 0 ? 128u : ((r1p * esz) % 64 == 0 ? 64u : 32u);
    if (wo > kTileM) {
      // the GEMM core convolution tiles whole output rows (<= 128 outputs): a wider layer
      // must take the fused core kernel (refused below if it does not)
      g.th = 1;
      g.nb = 1;
    } else if (ho * wo <= kTileM) {
      g.th = ho;
      g.nb = kTileM / (ho * wo);
    } else {
      g.nb = 1;
      const int thmax = kTileM / wo;
      const int ntiles = (ho + thmax - 1) / thmax;
      g.th = (ho + ntiles - 1) / ntiles;
    }
    g.tiles_h = (ho + g.th - 1) / g.th;
    const uint32_t a_box = static_cast<uint32_t>(g.nb * g.th * wo) * sw;
    const int kbytes = kh * kw * r1p * esz;
    h->a2.smem = plan_stage(p, f32, kbytes, sw, r2p, r2p, a_box, 0);
    if (!h->a2.smem) return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "a2 does not fit in shared memory"));
    p.chunks_per_tap = (r1p * esz) / static_cast<int>(sw);
    p.amode = AMODE_CONV;
    p.out = h->t2;
    p.out_ld = r2p;
    {
      uint64_t dims[4] = {static_cast<uint64_t>(r1p), static_cast<uint64_t>(W), static_cast<uint64_t>(H),
                          static_cast<uint64_t>(d->batch_max)};
      uint64_t strides[3] = {static_cast<uint64_t>(r1p) * esz, static_cast<uint64_t>(W) * r1p * esz,
                             static_cast<uint64_t>(H) * W * r1p * esz};
      uint32_t box[4] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(wo * g.sw),
                         static_cast<uint32_t>(g.th * g.sh), static_cast<uint32_t>(g.nb)};
      uint32_t estr[4] = {1, static_cast<uint32_t>(g.sw), static_cast<uint32_t>(g.sh), 1};
      if ((st = encode(&p.tmA, f32, 4, h->t1, dims, strides, box, estr, sw)) != LRS_OK) return cleanup_fail(st);
    }
    {
      uint64_t dims[2] = {static_cast<uint64_t>(kh * kw * r1p), static_cast<uint64_t>(r2p) * (f32 ? 2 : 1)};
      uint64_t strides[1] = {static_cast<uint64_t>(kh * kw * r1p) * esz};
      uint32_t box[2] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(r2p)};
      uint32_t estr[2] = {1, 1};
      if ((st = encode(&p.tmB, f32, 2, h->w_core, dims, strides, box, estr, sw)) != LRS_OK) return cleanup_fail(st);
    }
    h->a2.name = "a2_core";
    h->a2.kid = f32 ? K_STORE_F32 : K_STORE_BF16;
  }
  if ((st = build_core(h, d)) != LRS_OK) return cleanup_fail(st);
  if (wo > kTileM && !h->svd && !h->cp_core && !h->use_core)
    return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "output width > 128 needs the fused core kernel (stride 1)"));
  if ((st = build_tiny(h, d)) != LRS_OK) return cleanup_fail(st);
  // ---------------------------------------------------------------- a3+a4+a5
  if (bf16_w && h->svd && (st = build_pw(h, d)) != LRS_OK) return cleanup_fail(st);
  if (bf16_w && !h->use_pw) {
    if ((st = build_wconv(h, d, g)) != LRS_OK) return cleanup_fail(st);
  }
  if (!h->use_w && f32 && !getenv("LRS_F32_FUSED")) {
    if ((st = build_spadd(h, d)) != LRS_OK) return cleanup_fail(st);
  }
  if (h->use_spadd) {
    // a3 + a4 + a5 in lrs_spadd_kernel: U_out as plain fp32 [R2p][Cout] (zero rows past R2)
    std::vector<float> m(static_cast<size_t>(r2p) * cout, 0.f);
    for (int b = 0; b < r2; ++b)
      for (int j = 0; j < cout; ++j) m[static_cast<size_t>(b) * cout + j] = host_val(d->u_out, (size_t)b * cout + j, f32);
    std::vector<uint8_t> mb(m.size() * 4);
    memcpy(mb.data(), m.data(), mb.size());
    void* pu = nullptr;
    if ((st = upload(&pu, mb)) != LRS_OK) return cleanup_fail(st);
    h->sp_uo = static_cast<float*>(pu);
    SpaddParams& q = h->spp;
    q.t = static_cast<const float*>(h->svd ? h->t1 : h->t2);
    q.t_ld = r2p;
    q.r = r2p;
    q.uo = h->sp_uo;
  } else if (!h->use_w && !h->use_pw) {
    GemmParams& p = h->a3.p;
    memset(&p, 0, sizeof(p));
    const int kdim = r2p;  // K of the expansion (R2, or R for the SVD pair)
    const uint32_t sw = pick_sw(kdim * esz);
    // sparse window geometry: max padded rows over all tiles of batch_max images
    const int wp = (wo - 1) * g.sw + kw;
    int rows_max = 1;
    {
      const long long howo = static_cast<long long>(ho) * wo;
      for (long long m0 = 0; m0 < p_max; m0 += kTileM) {
        const long long m_last = std::min(m0 + kTileM - 1, p_max - 1);
        const long long n_first = m0 / howo, n_last = m_last / howo;
        const int nt = static_cast<int>(n_last - n_first + 1);
        const int lo0 = static_cast<int>((m0 - n_first * howo) / wo);
        const int hi0 = nt == 1 ? static_cast<int>((m_last - n_first * howo) / wo) : ho - 1;
        const int rows0 = (hi0 - lo0) * g.sh + kh;
        const int rows_full = (ho - 1) * g.sh + kh;
        const int hi_last = static_cast<int>((m_last - n_last * howo) / wo);
        const int rows_last = hi_last * g.sh + kh;
        const int tot = nt == 1 ? rows0 : rows0 + (nt - 2) * rows_full + rows_last;
        rows_max = std::max(rows_max, tot);
      }
    }
    int wstride = rows_max * wp;
    if (wstride % 2 == 0) wstride += 1;
    const int vec = f32 ? 4 : 8;
    const int budget = 64 * 1024;
    int cc = (budget / (wstride * esz)) / vec * vec;
    cc = std::min(cc, round_up(cin, vec));
    if (cc < vec) return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "sparse window does not fit in shared memory"));
    const int n_cc = (cin + cc - 1) / cc;
    const uint32_t sparse_bytes = std::max<uint32_t>(static_cast<uint32_t>(cc) * wstride * esz,
                                                     static_cast<uint32_t>(kTileM) * (bn + 1) * 4);
    h->a3.smem = plan_stage(p, f32, kdim * esz, sw, bn, cout_p, kTileM * sw, sparse_bytes);
    if (!h->a3.smem) return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "a3 does not fit in shared memory"));
    p.amode = AMODE_2D;
    p.sp.cin = cin;
    p.sp.cc = cc;
    p.sp.n_cc = n_cc;
    p.sp.wstride = wstride;
    p.sp.wp = wp;
    p.sp.cout = cout;
    {
      void* src = h->svd ? h->t1 : h->t2;
      uint64_t dims[2] = {static_cast<uint64_t>(kdim), static_cast<uint64_t>(p_max)};
      uint64_t strides[1] = {static_cast<uint64_t>(kdim) * esz};
      uint32_t box[2] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(kTileM)};
      uint32_t estr[2] = {1, 1};
      if ((st = encode(&p.tmA, f32, 2, src, dims, strides, box, estr, sw)) != LRS_OK) return cleanup_fail(st);
    }
    {
      uint64_t dims[2] = {static_cast<uint64_t>(kdim), static_cast<uint64_t>(cout_p) * (f32 ? 2 : 1)};
      uint64_t strides[1] = {static_cast<uint64_t>(kdim) * esz};
      uint32_t box[2] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(bn)};
      uint32_t estr[2] = {1, 1};
      if ((st = encode(&p.tmB, f32, 2, h->w_uout, dims, strides, box, estr, sw)) != LRS_OK) return cleanup_fail(st);
    }
    // per (Cout chunk, channel chunk, output channel) code streams
    const int n_chunks = cout_p / bn;
    std::vector<int> ptr(static_cast<size_t>(n_chunks) * n_cc * bn + 1, 0);
    std::vector<int2> ent;
    ent.reserve(static_cast<size_t>(d->nnz));
    const int kk = kh * kw;
    for (int nc = 0; nc < n_chunks; ++nc)
      for (int c = 0; c < n_cc; ++c)
        for (int jl = 0; jl < bn; ++jl) {
          const int j = nc * bn + jl;
          ptr[(static_cast<size_t>(nc) * n_cc + c) * bn + jl] = static_cast<int>(ent.size());
          if (j >= cout) continue;
          for (int64_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) {
            const int col = d->col_idx[e];
            const int ch = col / kk, tap = col % kk;
            if (ch / cc != c) continue;
            const int ty = tap / kw, tx = tap % kw;
            int2 v;
            float val = d->values[e];
            memcpy(&v.x, &val, 4);
            v.y = (ch - c * cc) * wstride + ty * wp + tx;
            ent.push_back(v);
          }
        }
    ptr.back() = static_cast<int>(ent.size());
    std::vector<uint8_t> pe(ptr.size() * 4), ee(std::max<size_t>(ent.size(), 1) * 8, 0);
    memcpy(pe.data(), ptr.data(), pe.size());
    if (!ent.empty()) memcpy(ee.data(), ent.data(), ent.size() * 8);
    void* pp = nullptr;
    void* pee = nullptr;
    if ((st = upload(&pp, pe)) != LRS_OK) return cleanup_fail(st);
    h->ent_ptr = static_cast<int*>(pp);
    if ((st = upload(&pee, ee)) != LRS_OK) return cleanup_fail(st);
    h->ent = static_cast<int2*>(pee);
    p.sp.ent = h->ent;
    p.sp.ent_ptr = h->ent_ptr;
    h->a3.name = "a345_expand_sparse";
    h->a3.kid = f32 ? (bn == 64 ? K_SP64_F32 : K_SP128_F32) : (bn == 64 ? K_SP64_BF16 : K_SP128_BF16);
  }
  h->a1.p.g = g;
  h->a2.p.g = g;
  h->a3.p.g = g;
  // ---------------------------------------------------------------- fused output epilogue
  if (d->out_scale || d->out_bias) {
    std::vector<float> sb(static_cast<size_t>(cout) * 2);
    for (int j = 0; j < cout; ++j) {
      sb[2 * j] = d->out_scale ? d->out_scale[j] : 1.f;
      sb[2 * j + 1] = d->out_bias ? d->out_bias[j] : 0.f;
    }
    std::vector<uint8_t> b(sb.size() * 4);
    memcpy(b.data(), sb.data(), b.size());
    void* pe = nullptr;
    if ((st = upload(&pe, b)) != LRS_OK) return cleanup_fail(st);
    h->epi = static_cast<float2*>(pe);
  }
  const int relu = d->out_relu ? 1 : 0;
  h->wp.epi = h->epi;
  h->wp.relu = relu;
  h->pp.epi = h->epi;
  h->pp.relu = relu;
  h->spp.epi = h->epi;
  h->spp.relu = relu;
  h->tp.epi = h->epi;
  h->tp.relu = relu;
  h->a3.p.sp.epi = h->epi;
  h->a3.p.sp.relu = relu;
  for (int k = 0; k < 6; ++k) {
    cudaError_t e = cudaFuncSetAttribute(kernel_ptr(static_cast<KernelId>(k)),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    if (e != cudaSuccess)
      return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)));
  }
  for (const void* fn : {reinterpret_cast<const void*>(&lrs_core_kernel<4, false>),
                         reinterpret_cast<const void*>(&lrs_core_kernel<2, false>),
                         reinterpret_cast<const void*>(&lrs_core_kernel<1, false>),
                         reinterpret_cast<const void*>(&lrs_core_kernel<1, true>),
                         reinterpret_cast<const void*>(&lrs_tiny_kernel)}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    if (e != cudaSuccess) return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)));
  }
  for (const void* fn : {reinterpret_cast<const void*>(&lrs_spadd_kernel), pw_kernel_ptr(1), pw_kernel_ptr(2),
                         pw_kernel_ptr(3), pw_kernel_ptr(4), pwf_kernel_ptr(1), pwf_kernel_ptr(2), pwf_kernel_ptr(3),
                         pwf_kernel_ptr(4)}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    if (e != cudaSuccess) return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)));
  }
  for (int u = 1; u <= kWMaxUnits; ++u)
    for (int b = 2; b <= 4; b += 2)
      for (int pr = 0; pr < (u <= 2 ? 2 : 1); ++pr) {
        cudaError_t e = cudaFuncSetAttribute(wconv_kernel_ptr(u, b, pr != 0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kMaxSmem);
        if (e != cudaSuccess)
          return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)));
      }
  if ((st = setup_early(h, d)) != LRS_OK) return cleanup_fail(st);
  bool core_tuned = false;
  if ((st = autotune_w(h, d, g, &core_tuned)) != LRS_OK) return cleanup_fail(st);
  if (!core_tuned && (st = autotune_core(h, d)) != LRS_OK) return cleanup_fail(st);
  if ((st = autotune_pw(h, d)) != LRS_OK) return cleanup_fail(st);
  cudaSetDevice(prev);
  *out = h;
  return LRS_OK;
}

}  // extern "C"

namespace {
// Restores the caller's current device on every exit path of an ABI call.
struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  cudaError_t enter(int device) {
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return e;
    if (prev != device) {
      e = cudaSetDevice(device);
      switched = e == cudaSuccess;
    }
    return e;
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};

// The launches of one forward on the handle's (current) device; arguments validated.
lrs_status forward_impl(lrs_conv* h, const void* x, void* y, int32_t n, cudaStream_t stream) {
  const bool f32 = h->f32;
  const int esz = h->esz;
  const lrs_conv_desc& d = h->d;
  lrs_status st = LRS_OK;
  if (h->xmap_ptr != x || h->xmap_n != n) {
    uint64_t dims[2] = {static_cast<uint64_t>(d.c_in), static_cast<uint64_t>(n) * d.in_h * d.in_w};
    uint64_t strides[1] = {static_cast<uint64_t>(d.c_in) * esz};
    uint32_t box[2] = {static_cast<uint32_t>(h->kc_a1), static_cast<uint32_t>(kTileM)};
    uint32_t estr[2] = {1, 1};
    if ((st = encode(&h->xmap, f32, 2, const_cast<void*>(x), dims, strides, box, estr, h->sw_a1)) != LRS_OK)
      return st;
    h->xmap_ptr = x;
    h->xmap_n = n;
  }
  const long long pin = static_cast<long long>(n) * d.in_h * d.in_w;
  const long long P = static_cast<long long>(n) * h->ho * h->wo;
  if (h->use_tiny) {
    TinyParams& q = h->tp;
    q.x = static_cast<const float*>(x);
    q.y = static_cast<float*>(y);
    q.n = n;
    // early start unless X may be the previous kernel's output (the registry of the
    // library's last output on this stream); LRS_NO_EARLY=1 at create disables it
    q.early = (!h->no_early &&
               !x_after_previous_output(h->device, stream, x, static_cast<size_t>(n) * d.in_h * d.in_w * d.c_in * esz))
                  ? 1 : 0;
    cudaEvent_t e1 = nullptr;
    if ((st = time_begin(h, 2, stream, &e1)) != LRS_OK) return st;
    LRS_CUDA(launch_pdl(reinterpret_cast<const void*>(&lrs_tiny_kernel), dim3(static_cast<unsigned>(n * q.bands * q.cbands)),
                        dim3(kTyThreads), &q, h->tiny_smem, stream));
    if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
    return LRS_OK;
  }
  if (h->use_core && !(h->skip & 1)) {
    CoreParams& c = h->cp;
    if (h->cx_ptr != x || h->cx_n != n) {
      uint64_t dims[4] = {static_cast<uint64_t>(d.c_in), static_cast<uint64_t>(d.in_w), static_cast<uint64_t>(d.in_h),
                          static_cast<uint64_t>(n)};
      uint64_t strides[3] = {static_cast<uint64_t>(d.c_in) * 2, static_cast<uint64_t>(d.in_w) * d.c_in * 2,
                             static_cast<uint64_t>(d.in_h) * d.in_w * d.c_in * 2};
      uint32_t box[4] = {64, static_cast<uint32_t>(c.wc), static_cast<uint32_t>(c.wr), static_cast<uint32_t>(c.ipt)};
      uint32_t estr[4] = {1, 1, 1, 1};
      if ((st = encode_t(&c.tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, estr,
                         128)) != LRS_OK)
        return st;
      h->cx_ptr = x;
      h->cx_n = n;
    }
    c.n = n;
    c.t2 = static_cast<__nv_bfloat16*>(h->t2);
    c.early = 0;
    if (h->dbuf) {
      // this forward's buffers; early start unless X may still be written by the previous
      // kernel on the stream (the library's last forward there produced it)
      const int par = h->par;
      h->par ^= 1;
      c.t2 = static_cast<__nv_bfloat16*>(par ? h->t2b : h->t2);
      h->wp.tmT = h->tmT_par[par];
      if (h->wp.n_gk) {
        h->wp.tmG = h->tmG_par[par];
        h->wp.g = static_cast<__nv_bfloat16*>(par ? h->w_gb : h->w_g);
      }
      const size_t xbytes = static_cast<size_t>(n) * d.in_h * d.in_w * d.c_in * esz;
      c.early = x_after_previous_output(h->device, stream, x, xbytes) ? 0 : 1;
    }
    c.n_tiles = ((n + c.ipt - 1) / c.ipt) * c.bands;
    const unsigned grid = static_cast<unsigned>(std::min(c.n_tiles, h->core_grid));
    cudaEvent_t e1 = nullptr;
    if ((st = time_begin(h, 0, stream, &e1)) != LRS_OK) return st;
    const void* kfn = h->cp_core    ? reinterpret_cast<const void*>(&lrs_core_kernel<1, true>)
                      : c.g_kc == 64 ? reinterpret_cast<const void*>(&lrs_core_kernel<4, false>)
                      : c.g_kc == 32 ? reinterpret_cast<const void*>(&lrs_core_kernel<2, false>)
                                     : reinterpret_cast<const void*>(&lrs_core_kernel<1, false>);
    LRS_CUDA(launch_pdl(kfn, dim3(grid), dim3(kCThreads), &c, h->core_smem, stream));
    if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
  }
  // a1
  h->a1.p.tmA = h->xmap;
  h->a1.p.m_total = static_cast<int>(pin);
  h->a1.p.g.n = n;
  int pw_par = 0;
  h->a1.p.early = 0;
  h->a1.p.out = h->t1;
  if (h->dbuf_pw) {
    // the projection of forward f+1 may run while the pointwise kernel of f still reads the
    // other T1 (same protocol as the core kernel's T2 above)
    pw_par = h->par;
    h->par ^= 1;
    h->a1.p.out = pw_par ? h->t1b : h->t1;
    const size_t xbytes = static_cast<size_t>(pin) * d.c_in * esz;
    h->a1.p.early = x_after_previous_output(h->device, stream, x, xbytes) ? 0 : 1;
  }
  if (!h->use_core && !h->pw_ft && !(h->skip & 1) &&
      (st = launch(h, 0, h->a1, dim3(static_cast<unsigned>((pin + kTileM - 1) / kTileM)), stream)) != LRS_OK)
    return st;
  if (h->use_pw) {
    PwParams& q = h->pp;
    if (h->px_ptr != x || h->px_n != n) {
      {
        uint64_t dims[2] = {static_cast<uint64_t>(d.c_in), static_cast<uint64_t>(pin)};
        uint64_t strides[1] = {static_cast<uint64_t>(d.c_in) * 2};
        uint32_t box[2] = {64, static_cast<uint32_t>(q.bp)};
        uint32_t estr[2] = {1, 1};
        if ((st = encode_t(&q.tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
                           128)) != LRS_OK)
          return st;
      }
      if (!h->pw_ft) {
        uint64_t dims[2] = {static_cast<uint64_t>(h->r1p), static_cast<uint64_t>(pin)};
        uint64_t strides[1] = {static_cast<uint64_t>(h->r1p) * 2};
        uint32_t box[2] = {static_cast<uint32_t>(q.t_kc), static_cast<uint32_t>(q.bp)};
        uint32_t estr[2] = {1, 1};
        for (int b = 0; b < (h->dbuf_pw ? 2 : 1); ++b)
          if ((st = encode_t(&h->tmT_pw_par[b], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b ? h->t1b : h->t1, dims, strides,
                             box, estr, q.sw_t)) != LRS_OK)
            return st;
      }
      h->px_ptr = x;
      h->px_n = n;
    }
    if (h->py_ptr != y || h->py_n != n) {
      uint64_t dims[2] = {static_cast<uint64_t>(d.c_out), static_cast<uint64_t>(pin)};
      uint64_t strides[1] = {static_cast<uint64_t>(d.c_out) * 2};
      uint32_t box[2] = {32, 32};
      uint32_t estr[2] = {1, 1};
      if ((st = encode_t(&q.tmY, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, estr, 64)) != LRS_OK)
        return st;
      h->py_ptr = y;
      h->py_n = n;
    }
    if (!h->pw_ft) q.tmT = h->tmT_pw_par[pw_par];
    q.y = y;
    q.P = static_cast<int>(pin);
    q.n_pt = static_cast<int>((pin + q.bp - 1) / q.bp);
    const int per_group = std::max(1, std::min(h->pw_grid_per_group, q.n_pt));
    cudaEvent_t e1 = nullptr;
    if ((st = time_begin(h, 2, stream, &e1)) != LRS_OK) return st;
    LRS_CUDA(launch_pdl(h->pw_ft ? pwf_kernel_ptr(q.mpc) : pw_kernel_ptr(q.mpc),
                        dim3(static_cast<unsigned>(per_group * q.n_groups)), dim3(kPThreads), &q, h->pw_smem, stream));
    if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
    return LRS_OK;
  }
  // a2
  if (h->cp_core && !h->use_core && !(h->skip & 2)) {
    CpDwParams& q = h->cpp;
    q.n = n;
    const long long items = static_cast<long long>(n) * h->ho * h->wo * (q.ld / (f32 ? 4 : 8));
    const unsigned grid = static_cast<unsigned>(std::min<long long>((items + kCpThreads - 1) / kCpThreads, 16LL * h->sms));
    cudaEvent_t e1 = nullptr;
    if ((st = time_begin(h, 1, stream, &e1)) != LRS_OK) return st;
    LRS_CUDA(launch_pdl(f32 ? reinterpret_cast<const void*>(&lrs_cp_dw_kernel<true>)
                            : reinterpret_cast<const void*>(&lrs_cp_dw_kernel<false>),
                        dim3(grid), dim3(kCpThreads), &q, 0, stream));
    if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
  } else if (!h->svd && !h->use_core && !(h->skip & 2)) {
    h->a2.p.g.n = n;
    const int tiles = ((n + h->a2.p.g.nb - 1) / h->a2.p.g.nb) * h->a2.p.g.tiles_h;
    if ((st = launch(h, 1, h->a2, dim3(tiles), stream)) != LRS_OK) return st;
  }
  // a3 + a4 + a5
  if (h->use_w && (h->skip & 4)) return LRS_OK;
  if (h->use_w) {
    WconvParams& w = h->wp;
    if (h->wx_ptr != x || h->wx_n != n) {
      uint64_t dims[4] = {static_cast<uint64_t>(d.c_in), static_cast<uint64_t>(n), static_cast<uint64_t>(d.in_w),
                          static_cast<uint64_t>(d.in_h)};
      uint64_t strides[3] = {static_cast<uint64_t>(d.in_h) * d.in_w * d.c_in * 2, static_cast<uint64_t>(d.c_in) * 2,
                             static_cast<uint64_t>(d.in_w) * d.c_in * 2};
#if defined(LRS_EXPERIMENTS) || defined(LRS_WCONV_DEBUG)
      if (w.dbg & 32) strides[0] = 128;  // timing experiment: contiguous 1 KB per position (wrong data)
#endif
      uint32_t box[4] = {64, static_cast<uint32_t>(w.ipw), static_cast<uint32_t>(w.wc), static_cast<uint32_t>(w.wr)};
      uint32_t estr[4] = {1, 1, 1, 1};
      if ((st = encode_t(&w.tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box,
                         estr, 128)) != LRS_OK)
        return st;
      h->wx_ptr = x;
      h->wx_n = n;
    }
    w.n = n;
    w.y = y;
    w.x = static_cast<const __nv_bfloat16*>(x);
    w.n_tiles = ((n + w.ipw - 1) / w.ipw) * w.bands * w.cbands * w.n_mt;
    const unsigned grid = w.pair ? 2u * static_cast<unsigned>(std::min(w.n_tiles / 2, h->sms / 2))
                                 : static_cast<unsigned>(std::min(w.n_tiles, h->sms));
    cudaEvent_t e1 = nullptr;
    if ((st = time_begin(h, 2, stream, &e1)) != LRS_OK) return st;
    if (w.pair)
      LRS_CUDA(launch_pdl_pair(wconv_kernel_ptr(w.n_units, w.bpi, true), dim3(grid), dim3(kWThreads), &w, h->w_smem,
                               stream));
    else
      LRS_CUDA(launch_pdl(wconv_kernel_ptr(w.n_units, w.bpi), dim3(grid), dim3(kWThreads), &w, h->w_smem, stream));
    if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
    return LRS_OK;
  }
  h->a3.p.m_total = static_cast<int>(P);
  h->a3.p.g.n = n;
  h->a3.p.sp.x = x;
  h->a3.p.sp.y = y;
  if (!h->use_spadd && !(h->skip & 4) &&
      (st = launch(h, 2, h->a3,
                   dim3(static_cast<unsigned>((P + kTileM - 1) / kTileM), h->cout_p / h->bn), stream)) != LRS_OK)
    return st;
  if (h->use_spadd && !(h->skip & 4)) {
    SpaddParams& q = h->spp;
    q.x = static_cast<const float*>(x);
    q.y = static_cast<float*>(y);
    q.n = n;
    const unsigned grid = static_cast<unsigned>(((n + 3) / 4) * q.bands * q.n_nc);
    cudaEvent_t e1 = nullptr;
    if ((st = time_begin(h, 2, stream, &e1)) != LRS_OK) return st;
    LRS_CUDA(launch_pdl(reinterpret_cast<const void*>(&lrs_spadd_kernel), dim3(grid), dim3(kSpThreads), &q,
                        h->sp_smem, stream));
    if (e1) LRS_CUDA(cudaEventRecord(e1, stream));
  }
  return LRS_OK;
}

}  // namespace

extern "C" {

lrs_status lrs_conv_forward(const lrs_conv* hc, const void* x, void* y, int32_t n, void* stream_) {
  // host state (tensor-map caches, per-call launch parameters) is updated here: see the
  // header's note on concurrent host calls
  lrs_conv* h = const_cast<lrs_conv*>(hc);
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (n < 0 || n > h->d.batch_max) return fail(LRS_ERR_INVALID_ARGUMENT, "n=%d outside [0, %d]", n, h->d.batch_max);
  if (n == 0) return LRS_OK;
  if (!x || !y) return fail(LRS_ERR_INVALID_ARGUMENT, "x / y is NULL");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15))
    return fail(LRS_ERR_INVALID_ARGUMENT, "x / y must be 16-byte aligned");
  DeviceGuard g;
  LRS_CUDA(g.enter(h->device));
  const lrs_status st = forward_impl(h, x, y, n, static_cast<cudaStream_t>(stream_));
  if (st == LRS_OK)
    record_output(h->device, static_cast<cudaStream_t>(stream_), y,
                  static_cast<size_t>(n) * h->ho * h->wo * h->d.c_out * h->esz);
  return st;
}

lrs_status lrs_conv_forward_host(lrs_conv* h, const void* x_host, void* y_host, int32_t n, void* stream_) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (n < 0 || n > h->d.batch_max) return fail(LRS_ERR_INVALID_ARGUMENT, "n=%d outside [0, %d]", n, h->d.batch_max);
  if (n == 0) return LRS_OK;
  if (!x_host || !y_host) return fail(LRS_ERR_INVALID_ARGUMENT, "x_host / y_host is NULL");
  DeviceGuard g;
  LRS_CUDA(g.enter(h->device));
  const size_t xi = static_cast<size_t>(h->d.in_h) * h->d.in_w * h->d.c_in * h->esz;  // bytes per image
  const size_t yi = static_cast<size_t>(h->ho) * h->wo * h->d.c_out * h->esz;
  if (!h->hx) LRS_CUDA(cudaMalloc(&h->hx, xi * h->d.batch_max));
  if (!h->hy) LRS_CUDA(cudaMalloc(&h->hy, yi * h->d.batch_max));
  if (!h->hs_in) {
    LRS_CUDA(cudaStreamCreateWithFlags(&h->hs_in, cudaStreamNonBlocking));
    LRS_CUDA(cudaStreamCreateWithFlags(&h->hs_out, cudaStreamNonBlocking));
    for (auto& e : h->hev) LRS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  // Pipeline in chunks of >= 8 images (the fused kernel's image groups): the copy of
  // chunk i+1 in, the forward of chunk i and the copy of chunk i-1 out overlap (the copy
  // engines run both directions concurrently).  Every stream starts after the caller's
  // prior work on `stream`, and `stream` ends after the last copy out, so the call keeps
  // single-stream semantics -- also when a step fails midway: the error path still joins
  // both copy streams into `stream` before returning, so no copy outlives the call's
  // stream order.
  const int nch = std::max(1, std::min(4, n / 8));
  const uint8_t* xs = static_cast<const uint8_t*>(x_host);
  uint8_t* ys = static_cast<uint8_t*>(y_host);
  uint8_t* dx = static_cast<uint8_t*>(h->hx);
  uint8_t* dy = static_cast<uint8_t*>(h->hy);
  LRS_CUDA(cudaEventRecord(h->hev[16], stream));
  LRS_CUDA(cudaStreamWaitEvent(h->hs_in, h->hev[16], 0));
  LRS_CUDA(cudaStreamWaitEvent(h->hs_out, h->hev[16], 0));
  lrs_status st = LRS_OK;
  auto step = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && st == LRS_OK)
      st = fail(e == cudaErrorMemoryAllocation ? LRS_ERR_OUT_OF_MEMORY : LRS_ERR_CUDA, "forward_host %s: %s", what,
                cudaGetErrorString(e));
    return st == LRS_OK;
  };
  for (int i = 0; i < nch && st == LRS_OK; ++i) {
    const int i0 = static_cast<int>(static_cast<long long>(n) * i / nch) / 8 * 8;
    const int i1 = i + 1 == nch ? n : static_cast<int>(static_cast<long long>(n) * (i + 1) / nch) / 8 * 8;
    if (i1 <= i0) continue;
    if (!step(cudaMemcpyAsync(dx + i0 * xi, xs + i0 * xi, (i1 - i0) * xi, cudaMemcpyHostToDevice, h->hs_in), "H2D"))
      break;
    if (!step(cudaEventRecord(h->hev[i], h->hs_in), "event")) break;
    if (!step(cudaStreamWaitEvent(stream, h->hev[i], 0), "wait")) break;
    if ((st = forward_impl(h, dx + i0 * xi, dy + i0 * yi, i1 - i0, stream)) != LRS_OK) break;
    if (!step(cudaEventRecord(h->hev[8 + i], stream), "event")) break;
    if (!step(cudaStreamWaitEvent(h->hs_out, h->hev[8 + i], 0), "wait")) break;
    step(cudaMemcpyAsync(ys + i0 * yi, dy + i0 * yi, (i1 - i0) * yi, cudaMemcpyDeviceToHost, h->hs_out), "D2H");
  }
  // join: `stream` waits for both copy streams (also on the error path)
  cudaError_t e1 = cudaEventRecord(h->hev[17], h->hs_out);
  if (e1 == cudaSuccess) e1 = cudaStreamWaitEvent(stream, h->hev[17], 0);
  cudaError_t e2 = cudaEventRecord(h->hev[16], h->hs_in);
  if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(stream, h->hev[16], 0);
  step(e1, "join");
  step(e2, "join");
  return st;
}

lrs_status lrs_conv_destroy(lrs_conv* h) {
  if (!h) return LRS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  void* bufs[] = {h->w_uin, h->w_core, h->w_uout, h->t1, h->t2, h->ent, h->ent_ptr, h->hx, h->hy,
                  h->w_as, h->w_e, h->w_res, h->w_dense_img, h->w_gtab, h->w_g, h->t2b, h->w_gb, h->t1b, h->sp_ent, h->sp_ptr, h->w_cpb, h->w_cpc,
                  h->sp_uo, h->epi, h->pw_w, h->pw_e, h->pw_tab, h->pw_u};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (void* b : h->tiny_buf)
    if (b) cudaFree(b);
  if (h->hs_in) {
    cudaStreamSynchronize(h->hs_in);
    cudaStreamSynchronize(h->hs_out);
    cudaStreamDestroy(h->hs_in);
    cudaStreamDestroy(h->hs_out);
    for (auto e : h->hev) cudaEventDestroy(e);
  }
  for (auto& r : h->ring)
    for (auto e : r.ev) cudaEventDestroy(e);
  cudaSetDevice(prev);
  delete h;
  return LRS_OK;
}

lrs_status lrs_conv_output_shape(const lrs_conv* h, int32_t* out_h, int32_t* out_w) {
  if (!h || !out_h || !out_w) return fail(LRS_ERR_INVALID_ARGUMENT, "NULL argument");
  *out_h = h->ho;
  *out_w = h->wo;
  return LRS_OK;
}

int32_t lrs_conv_launches_per_forward(const lrs_conv* h) {
  if (h && (h->use_tiny || h->pw_ft)) return 1;
  return h ? (h->svd ? 2 : 3) - (h->use_core ? 1 : 0) : 0;
}

lrs_status lrs_conv_set_timing(lrs_conv* h, int32_t enable) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->timing = enable != 0;
  return LRS_OK;
}

lrs_status lrs_conv_stage_times(lrs_conv* h, float* ms, int64_t* counts, int32_t max_stages,
                                int32_t* n_stages, int32_t reset) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  for (int s = 0; s < 4; ++s) {
    TimingRing& r = h->ring[s];
    for (int i = 0; i + 1 < r.used; i += 2) {
      LRS_CUDA(cudaEventSynchronize(r.ev[i + 1]));
      float t = 0.f;
      LRS_CUDA(cudaEventElapsedTime(&t, r.ev[i], r.ev[i + 1]));
      r.ms += t;
      r.count += 1;
    }
    r.used = 0;
  }
  if (n_stages) *n_stages = 4;
  for (int s = 0; s < 4 && s < max_stages; ++s) {
    if (ms) ms[s] = static_cast<float>(h->ring[s].ms);
    if (counts) counts[s] = h->ring[s].count;
  }
  if (reset)
    for (auto& r : h->ring) {
      r.ms = 0.0;
      r.count = 0;
    }
  return LRS_OK;
}

const char* lrs_conv_stage_name(const lrs_conv* h, int32_t stage) {
  static const char* names[] = {"a1_proj", "a2_core", "a345_expand_sparse", "a4_sparse_add"};
  if (stage == 0 && h && h->use_core) return h->cp_core ? "a12_proj_cp" : "a12_proj_core";
  if (stage == 1 && h && h->cp_core) return "a2_cp_depthwise";
  return (stage >= 0 && stage < 4) ? names[stage] : "";
}

int32_t lrs_conv_sparse_engine(const lrs_conv* h, int32_t* main_blocks, int32_t* residual_blocks) {
  if (!h) return -1;
  const bool tc = h->use_w || h->use_pw;
  if (main_blocks) *main_blocks = tc ? h->w_main_blocks : 0;
  if (residual_blocks) *residual_blocks = tc ? h->w_res_blocks : 0;
  return tc ? 1 : (h->use_tiny ? 3 : (h->use_spadd ? 2 : 0));
}

int32_t lrs_conv_cta_pairs(const lrs_conv* h) {
  if (!h) return -1;
  return h->use_w && !h->use_pw ? h->wp.pair : 0;
}

int32_t lrs_conv_overflow_chunks(const lrs_conv* h) {
  if (!h) return -1;
  return h->use_w && !h->use_pw ? h->wp.n_gk : 0;
}

int32_t lrs_conv_expand_kernel(const lrs_conv* h) {
  if (!h) return -1;
  return h->use_pw ? 2 : (h->use_w ? 1 : 0);
}

int32_t lrs_conv_core_fused(const lrs_conv* h) { return h ? (h->use_core ? 1 : 0) : -1; }

lrs_status lrs_sparse_from_slices(int32_t c_in, int32_t c_out, int32_t kernel_h, int32_t kernel_w,
                                  const int64_t* slice_ptr, const void* packed, int32_t packed_bytes,
                                  const float* values, int64_t* row_ptr, int32_t* col_idx, float* values_out) {
  if (c_in <= 0 || c_out <= 0 || kernel_h <= 0 || kernel_w <= 0)
    return fail(LRS_ERR_INVALID_ARGUMENT, "all extents must be > 0");
  if (packed_bytes != 2 && packed_bytes != 4) return fail(LRS_ERR_INVALID_ARGUMENT, "packed_bytes must be 2 or 4");
  if (!slice_ptr || !row_ptr) return fail(LRS_ERR_INVALID_ARGUMENT, "slice_ptr / row_ptr is NULL");
  if (slice_ptr[0] != 0) return fail(LRS_ERR_INVALID_ARGUMENT, "slice_ptr[0] != 0");
  for (int i = 0; i < c_in; ++i)
    if (slice_ptr[i + 1] < slice_ptr[i]) return fail(LRS_ERR_INVALID_ARGUMENT, "slice_ptr not monotone at %d", i);
  const int64_t nnz = slice_ptr[c_in];
  if (nnz > 0 && (!packed || !values || !col_idx || !values_out))
    return fail(LRS_ERR_INVALID_ARGUMENT, "NULL entry array");
  const int64_t taps = static_cast<int64_t>(kernel_h) * kernel_w;
  if (packed_bytes == 2 && static_cast<int64_t>(c_out) * taps > 65536)
    return fail(LRS_ERR_INVALID_ARGUMENT, "c_out * kernel taps > 65536 needs 4-byte packed indices");
  // decode: packed = j * taps + tap (tap = ky * kernel_w + kx), slice i = input channel
  std::vector<int64_t> cnt(static_cast<size_t>(c_out) + 1, 0);
  std::vector<std::pair<int32_t, int32_t>> jc(static_cast<size_t>(nnz));  // (row j, col)
  for (int i = 0; i < c_in; ++i)
    for (int64_t e = slice_ptr[i]; e < slice_ptr[i + 1]; ++e) {
      const int64_t pk = packed_bytes == 2 ? static_cast<const uint16_t*>(packed)[e]
                                           : static_cast<const uint32_t*>(packed)[e];
      const int64_t j = pk / taps, tap = pk % taps;
      if (j >= c_out) return fail(LRS_ERR_INVALID_ARGUMENT, "packed index %lld decodes to row %lld >= c_out",
                                  (long long)pk, (long long)j);
      jc[static_cast<size_t>(e)] = {static_cast<int32_t>(j), static_cast<int32_t>(i * taps + tap)};
      ++cnt[static_cast<size_t>(j) + 1];
    }
  for (int j = 0; j < c_out; ++j) cnt[j + 1] += cnt[j];
  for (int j = 0; j <= c_out; ++j) row_ptr[j] = cnt[j];
  std::vector<int64_t> fillp(cnt.begin(), cnt.end() - 1);
  std::vector<std::pair<int32_t, float>> tmp(static_cast<size_t>(nnz));
  for (int64_t e = 0; e < nnz; ++e) {
    const int32_t j = jc[static_cast<size_t>(e)].first;
    tmp[static_cast<size_t>(fillp[j]++)] = {jc[static_cast<size_t>(e)].second, values[e]};
  }
  for (int j = 0; j < c_out; ++j) {
    auto b = tmp.begin() + cnt[j], en = tmp.begin() + cnt[j + 1];
    std::sort(b, en, [](const std::pair<int32_t, float>& u, const std::pair<int32_t, float>& v) {
      return u.first < v.first;
    });
    for (auto it = b; it != en; ++it) {
      if (it != b && it->first == (it - 1)->first)
        return fail(LRS_ERR_INVALID_ARGUMENT, "duplicate entry (row %d, col %d)", j, it->first);
      const int64_t e = it - tmp.begin();
      col_idx[e] = it->first;
      values_out[e] = it->second;
    }
  }
  return LRS_OK;
}

lrs_status lrs_conv_debug_trace(lrs_conv* h, void* dev_buf) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->wp.trace = static_cast<unsigned long long*>(dev_buf);
  h->cp.trace = static_cast<unsigned long long*>(dev_buf);  // core kernel: indices 8190..13095
  h->pp.trace = static_cast<unsigned long long*>(dev_buf);  // pointwise kernel: indices 0..3999
#if defined(LRS_EXPERIMENTS) || defined(LRS_WCONV_DEBUG)
  if (const char* e = getenv("LRS_WCONV_DBG")) h->wp.dbg = atoi(e);
#endif
  return LRS_OK;
}

lrs_status lrs_conv_debug_buffer(const lrs_conv* h, int32_t which, const void** ptr, int32_t* ld) {
  if (!h || !ptr || !ld) return fail(LRS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (which == 0) {
    *ptr = (h->dbuf_pw && h->par == 0) ? h->t1b : h->t1;  // the buffer the last forward wrote
    *ld = h->r1p;
  } else if (which == 1) {
    *ptr = (h->dbuf && h->par == 0) ? h->t2b : h->t2;  // the buffer the last forward wrote
    *ld = h->r2p;
  } else {
    return fail(LRS_ERR_INVALID_ARGUMENT, "which must be 0 or 1");
  }
  return LRS_OK;
}

}  // extern "C"

// the backward pass (include/lrs_conv.h "Backward pass"); shares this unit's helpers
#include "lrs_backward.cuh"
// the low-rank + sparse decomposition (include/lrs_conv.h "Decomposition")
#include "lrs_decomp_host.cuh"
