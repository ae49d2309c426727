// lrs_backward.cuh -- host side of the backward pass (include/lrs_conv.h "Backward pass";
// SURVEY §8(f) f3; §3.5).  Included at the end of lrs_conv.cu so it shares
// the translation unit's helpers (TMA encoding, GEMM stage planning, PDL launches).
//
//   backward_data:     dX = forward of the transposed layer on dY (an lrs_conv handle)
//   backward_weights:  T1 = X U_in, T2 = conv(T1, G), dT2 = dY U_out^T,
//                      dT1 = conv(dT2, G') (G' = G transposed + flipped, pad k-1-p)   -- lrs_gemm_kernel
//                      dU_out, dG, dU_in, dW_S: one grouped lrs_wgrad_kernel launch  -- lrs_wgrad.cuh
//                      split sums gathered into the gradient layouts                  -- lrs_wgrad_reduce_kernel
//   (SVD pair: T1 = X U, dT1 = dY V^T; dV, dU, dW_S.)

struct lrs_conv_bwd {
  int device = 0;
  int sms = 148;
  lrs_conv_desc d{};
  bool svd = false;
  int kh = 1, kw = 1, H = 0, W = 0, ho = 0, wo = 0, cin = 0, cout = 0, r1 = 0, r2 = 0, r1p = 0, r2p = 0;
  int sh = 1, sw = 1;   // stride
  // the paper's CP core kind: run as its Tucker-2 embedding (diagonal core G[a][a][y][x] =
  // B[y][a] C[x][a]); dG goes to dg_int and lrs_cp_core_grad_kernel folds it into dB, dC
  bool cp = false;
  float* cp_b = nullptr;   // B [kh][R] fp32
  float* cp_c = nullptr;   // C [kw][R] fp32
  float* dg_int = nullptr; // dG [R][R][kh][kw] fp32
  int hu = 0, wu = 0;   // extent of the zero-inserted gradient grid (= ho, wo at stride 1)
  void* dy_up = nullptr;   // zero-inserted dY  [batch_max][hu][wu][Cout] (stride > 1)
  void* dt2_up = nullptr;  // zero-inserted dT2 [batch_max][hu][wu][R2p]  (stride > 1)
  int batch_max = 0;
  long long nnz = 0;
  lrs_conv* tr = nullptr;  // the transposed layer (dX = its forward of dY)
  // weights (bf16, row-major B operands of lrs_gemm_kernel)
  void* w_uin = nullptr;   // U_in^T  [R1p][Cin]          T1 = X U_in
  void* w_core = nullptr;  // G^T     [R2p][kk*R1p]       T2 = conv(T1, G)
  void* w_uout = nullptr;  // U_out   [R2p][Cout]         dT2 = dY U_out^T   (SVD: dT1 = dY V^T)
  void* w_coret = nullptr; // G'^T    [R1p][kk*R2p]       dT1 = conv(dT2, G')
  // scratch (bf16): T1 [Pin][R1p], T2 [P][R2p], dT2 [P][R2p], dT1 [Pin][R1p]
  void* t1 = nullptr;
  void* t2 = nullptr;
  void* dt2 = nullptr;
  void* dt1 = nullptr;
  float* slab = nullptr;
  size_t slab_floats = 0;
  long long* idx = nullptr;  // gather tables of the reduction, per problem
  Stage g_t1{}, g_t2{}, g_dt2{}, g_dt1{};
  int kc_x = 0, kc_dy = 0;
  uint32_t sw_x = 0, sw_dy = 0;
  // grouped weight-gradient launch
  WgradParams wp{};
  WgradParams wpp{};        // the CTA-pair launch (lrs_wgrad_kernel<true>)
  int wg_ctas_l[2] = {0, 0};   // per launch: CTAs (solo) / clusters (pair)
  uint32_t wg_smem_l[2] = {0, 0};
  void* wg_items_l[2] = {nullptr, nullptr};  // WgradItem lists of the persistent CTAs / pairs
  void* wg_ptr_l[2] = {nullptr, nullptr};
  double wg_max_load = 0;    // the most loaded CTA's work / the mean (LPT balance)
  // which operand of each problem is which (rebuilt per call: pointer / n dependent maps)
  struct Opnd {
    int kind;      // 0 X, 1 dY, 2 T1, 3 T2, 4 dT2, 5 dT1
    int ch;        // channel pitch
    int h, w;      // grid
  };
  Opnd opa[kGMaxProblems], opb[kGMaxProblems];
  int box_bw[kGMaxProblems], box_bh[kGMaxProblems], box_bi[kGMaxProblems];
  int dst_of[kGMaxProblems];  // 0 d_u_out, 1 d_core, 2 d_u_in, 3 d_values
  WgradReduceSet rs{};
  int rs_blocks = 0;
  // lrs_conv_backward: the recompute GEMMs (T1, T2, dT2) run on a side stream concurrently
  // with the transposed layer's forward (fork / join events; graph-capturable)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool use_side = false;
  // stage timing (lrs_conv_bwd_set_timing): bwd_t1, bwd_t2, bwd_dt2, bwd_dt1, wgrad, wgrad_reduce
  bool timing = false;
  TimingRing ring[6];
  // lrs_conv_backward: dT1 taken from the transposed layer's forward (its T2, or T1 for an
  // SVD pair) instead of recomputed; nullptr = the handle's own dT1
  const void* dt1_ext = nullptr;
  const void* cdt1 = nullptr;
  // per-call map caches
  const void* cx = nullptr;
  const void* cdy = nullptr;
  int cn = -1;
};

namespace {

// the GEMM core-convolution tile (lrs_gemm_kernel AMODE_CONV): nb images x th rows x all wo
void conv_tile(ConvGeom& g) {
  if (g.ho * g.wo <= kTileM) {
    g.th = g.ho;
    g.nb = kTileM / (g.ho * g.wo);
  } else {
    g.nb = 1;
    const int thmax = kTileM / g.wo;
    const int ntiles = (g.ho + thmax - 1) / thmax;
    g.th = (g.ho + ntiles - 1) / ntiles;
  }
  g.tiles_h = (g.ho + g.th - 1) / g.th;
}

// a2-style implicit-GEMM conv stage: out[P][n_p] = conv(in [N][g.h][g.w][k_p], Bmat [n_p][kk*k_p])
lrs_status plan_conv_stage(Stage& s, ConvGeom g, int k_p, int n_p, void* in, void* bmat, void* out, int batch_max) {
  GemmParams& p = s.p;
  memset(&p, 0, sizeof(p));
  const uint32_t sw = (k_p * 2) % 128 == 0 ? 128u : ((k_p * 2) % 64 == 0 ? 64u : 32u);
  conv_tile(g);
  const uint32_t a_box = static_cast<uint32_t>(g.nb * g.th * g.wo) * sw;
  const int kk = g.kh * g.kw;
  s.smem = plan_stage(p, false, kk * k_p * 2, sw, n_p, n_p, a_box, 0);
  if (!s.smem) return fail(LRS_ERR_UNSUPPORTED, "backward: a conv GEMM stage does not fit in shared memory");
  p.chunks_per_tap = (k_p * 2) / static_cast<int>(sw);
  p.amode = AMODE_CONV;
  p.out = out;
  p.out_ld = n_p;
  p.g = g;
  lrs_status st;
  {
    uint64_t dims[4] = {static_cast<uint64_t>(k_p), static_cast<uint64_t>(g.w), static_cast<uint64_t>(g.h),
                        static_cast<uint64_t>(batch_max)};
    uint64_t strides[3] = {static_cast<uint64_t>(k_p) * 2, static_cast<uint64_t>(g.w) * k_p * 2,
                           static_cast<uint64_t>(g.h) * g.w * k_p * 2};
    uint32_t box[4] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(g.wo * g.sw),
                       static_cast<uint32_t>(g.th * g.sh), static_cast<uint32_t>(g.nb)};
    uint32_t estr[4] = {1, static_cast<uint32_t>(g.sw), static_cast<uint32_t>(g.sh), 1};  // stride: traversal
    if ((st = encode(&p.tmA, false, 4, in, dims, strides, box, estr, sw)) != LRS_OK) return st;
  }
  {
    uint64_t dims[2] = {static_cast<uint64_t>(kk * k_p), static_cast<uint64_t>(n_p)};
    uint64_t strides[1] = {static_cast<uint64_t>(kk * k_p) * 2};
    uint32_t box[2] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(n_p)};
    uint32_t estr[2] = {1, 1};
    if ((st = encode(&p.tmB, false, 2, bmat, dims, strides, box, estr, sw)) != LRS_OK) return st;
  }
  s.kid = K_STORE_BF16;
  return LRS_OK;
}

// 1x1 projection stage: out[M][n_p] = A[M][k] Bmat[n_p][k]^T; A's map is encoded per call
lrs_status plan_proj_stage(Stage& s, int k, int n_p, void* bmat, void* out, uint32_t* sw_out, int* kc_out) {
  GemmParams& p = s.p;
  memset(&p, 0, sizeof(p));
  const uint32_t sw = pick_sw(k * 2);
  s.smem = plan_stage(p, false, k * 2, sw, n_p, n_p, kTileM * sw, 0);
  if (!s.smem) return fail(LRS_ERR_UNSUPPORTED, "backward: a projection GEMM stage does not fit in shared memory");
  p.amode = AMODE_2D;
  p.out = out;
  p.out_ld = n_p;
  uint64_t dims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(n_p)};
  uint64_t strides[1] = {static_cast<uint64_t>(k) * 2};
  uint32_t box[2] = {static_cast<uint32_t>(p.kc), static_cast<uint32_t>(n_p)};
  uint32_t estr[2] = {1, 1};
  lrs_status st = encode(&p.tmB, false, 2, bmat, dims, strides, box, estr, sw);
  if (st != LRS_OK) return st;
  s.kid = K_STORE_BF16;
  *sw_out = sw;
  *kc_out = p.kc;
  return LRS_OK;
}

lrs_status encode_proj_a(GemmParams& p, const void* a, long long rows, int k, uint32_t sw, int kc) {
  uint64_t dims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(rows)};
  uint64_t strides[1] = {static_cast<uint64_t>(k) * 2};
  uint32_t box[2] = {static_cast<uint32_t>(kc), static_cast<uint32_t>(kTileM)};
  uint32_t estr[2] = {1, 1};
  p.m_total = static_cast<int>(rows);
  return encode(&p.tmA, false, 2, const_cast<void*>(a), dims, strides, box, estr, sw);
}

// position step of a weight-gradient problem over a grid of rows x w positions per image:
// box (64, w, bh, bi) with w*bh*bi % 16 == 0 (the MMA K of a stage), at least 2 stages of
// (2 + bn/64) boxes in shared memory; least padding waste, then the largest step
bool pick_wgrad_step(int rows, int w, int n_img, int bn, int* bh_out, int* bi_out, int* stages_out) {
  const uint32_t budget = static_cast<uint32_t>(kMaxSmem) - 2048u;
  double best = 1e300;
  bool found = false;
  for (int bh = 1; bh <= rows; ++bh)
    for (int bi = 1; bi <= 256; ++bi) {  // images past n_img are out of bounds: zero, counted as waste
      const int kst = w * bh * bi;
      if (kst % 16 || kst > 256) continue;
      const uint32_t stage = static_cast<uint32_t>(2 + bn / 64) * kst * 128u;
      const int stages = std::min<int>(4, static_cast<int>(budget / stage));
      if (stages < 2) continue;
      const double waste = (static_cast<double>((rows + bh - 1) / bh) * bh / rows) *
                           (static_cast<double>((n_img + bi - 1) / bi) * bi / n_img);
      // per-step overheads favour longer steps; slots over 96 KB leave a 2-deep ring for
      // every problem of the grouped launch (one slot size), so they pay a penalty
      const double cost = waste * (1.0 + 32.0 / kst) * (stage > 96u * 1024u ? 1.25 : 1.0);
      if (cost < best) {
        best = cost;
        *bh_out = bh;
        *bi_out = bi;
        *stages_out = stages;
        found = true;
      }
    }
  return found;
}

lrs_status bwd_alloc(void** p, size_t bytes, const char* what) {
  if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess)
    return fail(LRS_ERR_OUT_OF_MEMORY, "backward: %s allocation failed", what);
  return LRS_OK;
}

const void* bwd_operand_ptr(const lrs_conv_bwd* h, int kind, const void* x, const void* dy) {
  switch (kind) {
    case 0: return x;
    case 1: return dy;
    case 2: return h->t1;
    case 3: return h->t2;
    case 4: return h->dt2;
    default: return h->dt1_ext ? h->dt1_ext : h->dt1;
  }
}

// per-call: the pointer- and n-dependent tensor maps
lrs_status bwd_encode_call(lrs_conv_bwd* h, const void* x, const void* dy, int n) {
  if (h->cx == x && h->cdy == dy && h->cn == n && h->cdt1 == h->dt1_ext) return LRS_OK;
  lrs_status st;
  const long long pin = static_cast<long long>(n) * h->H * h->W;
  const long long P = static_cast<long long>(n) * h->ho * h->wo;
  if (x && (st = encode_proj_a(h->g_t1.p, x, pin, h->cin, h->sw_x, h->kc_x)) != LRS_OK) return st;
  if (dy && (st = encode_proj_a(h->g_dt2.p, dy, P, h->cout, h->sw_dy, h->kc_dy)) != LRS_OK) return st;
  h->g_t1.p.g.n = n;
  h->g_dt2.p.g.n = n;
  h->g_t2.p.g.n = n;
  h->g_dt1.p.g.n = n;
  for (int i = 0; i < h->wp.n_problems; ++i) {
    WgradProblem& q = h->wp.pr[i];
    for (int ab = 0; ab < 2; ++ab) {
      const lrs_conv_bwd::Opnd& o = ab ? h->opb[i] : h->opa[i];
      const void* ptr = bwd_operand_ptr(h, o.kind, x, dy);
      uint64_t dims[4] = {static_cast<uint64_t>(o.ch), static_cast<uint64_t>(o.w), static_cast<uint64_t>(o.h),
                          static_cast<uint64_t>(n)};
      uint64_t strides[3] = {static_cast<uint64_t>(o.ch) * 2, static_cast<uint64_t>(o.w) * o.ch * 2,
                             static_cast<uint64_t>(o.h) * o.w * o.ch * 2};
      // the shifted operand of a strided layer is sampled every s positions (TMA traversal stride)
      const uint32_t ssw = ab ? 1u : static_cast<uint32_t>(q.sw), ssh = ab ? 1u : static_cast<uint32_t>(q.sh);
      uint32_t box[4] = {64, static_cast<uint32_t>(h->box_bw[i]) * ssw, static_cast<uint32_t>(h->box_bh[i]) * ssh,
                         static_cast<uint32_t>(h->box_bi[i])};
      uint32_t estr[4] = {1, ssw, ssh, 1};
      if ((st = encode_t(ab ? &q.tmB : &q.tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims,
                         strides, box, estr, 128)) != LRS_OK)
        return st;
    }
    const int hsteps = (h->opb[i].h + q.bh - 1) / q.bh;
    q.hsteps = hsteps;
    q.k_steps = ((n + q.bi - 1) / q.bi) * hsteps;
  }
  h->cx = x;
  h->cdy = dy;
  h->cn = n;
  h->cdt1 = h->dt1_ext;
  return LRS_OK;
}

}  // namespace

namespace {
lrs_status bwd_weights_impl(lrs_conv_bwd* h, const void* x, const void* dy, int32_t n, const lrs_conv_grads* gr,
                            void* stream_);
// dY (or dT2) -> its zero-inserted grid for the stride-s adjoint (a plain launch: the next
// kernel, PDL or not, starts after it completes)
lrs_status bwd_zero_insert(const lrs_conv_bwd* h, const void* src, void* up, int n, int c, cudaStream_t s) {
  const int cv = c / 8;
  const long long total = static_cast<long long>(n) * h->hu * h->wu * cv;
  const unsigned grid = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 8LL * h->sms));
  lrs_zero_insert_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(up), n, h->ho,
                                              h->wo, h->hu, h->wu, h->sh, h->sw, cv);
  LRS_CUDA(cudaGetLastError());
  return LRS_OK;
}

}  // namespace

extern "C" {

lrs_status lrs_conv_bwd_destroy(lrs_conv_bwd* h) {
  if (!h) return LRS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  void* bufs[] = {h->w_uin, h->w_core, h->w_uout, h->w_coret, h->t1, h->t2, h->dt2, h->dt1, h->slab, h->idx,
                  h->dy_up, h->dt2_up, h->cp_b, h->cp_c, h->dg_int,
                  h->wg_items_l[0], h->wg_ptr_l[0], h->wg_items_l[1], h->wg_ptr_l[1]};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (h->tr) lrs_conv_destroy(h->tr);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (auto& r : h->ring)
    for (auto e : r.ev) cudaEventDestroy(e);
  cudaSetDevice(prev);
  delete h;
  return LRS_OK;
}

lrs_status lrs_conv_bwd_create(const lrs_conv_desc* d, int device, lrs_conv_bwd** out) {
  if (!out) return fail(LRS_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  lrs_status st = validate(d);
  if (st != LRS_OK) return st;
  if (d->dtype != LRS_DTYPE_BF16) return fail(LRS_ERR_UNSUPPORTED, "backward: bf16 layers only");
  // the CP core kind (the paper's own decomposition): its Tucker-2 embedding, a
  // diagonal core G[a][b][y][x] = [a == b] B[y][a] C[x][a] (bf16, RNE of the fp32 product)
  std::vector<uint16_t> cp_emb;
  std::vector<float> cp_bf, cp_cf;
  lrs_conv_desc d_emb;
  const bool is_cp = d->core && d->core_kind == LRS_CORE_CP;
  if (is_cp) {
    const int R = d->rank_in, kh_ = d->kernel_h, kw_ = d->kernel_w;
    cp_bf.resize(static_cast<size_t>(kh_) * R);
    cp_cf.resize(static_cast<size_t>(kw_) * R);
    for (int y = 0; y < kh_; ++y)
      for (int a = 0; a < R; ++a) cp_bf[static_cast<size_t>(y) * R + a] = host_val(d->core, static_cast<size_t>(y) * R + a, false);
    for (int x = 0; x < kw_; ++x)
      for (int a = 0; a < R; ++a)
        cp_cf[static_cast<size_t>(x) * R + a] = host_val(d->core, static_cast<size_t>(kh_ + x) * R + a, false);
    cp_emb.assign(static_cast<size_t>(R) * R * kh_ * kw_, 0);
    for (int a = 0; a < R; ++a)
      for (int y = 0; y < kh_; ++y)
        for (int x = 0; x < kw_; ++x)
          cp_emb[((static_cast<size_t>(a) * R + a) * kh_ + y) * kw_ + x] =
              bf16_bits_rne(cp_bf[static_cast<size_t>(y) * R + a] * cp_cf[static_cast<size_t>(x) * R + a]);
    d_emb = *d;
    d_emb.core = cp_emb.data();
    d_emb.core_kind = LRS_CORE_TUCKER2;
    d = &d_emb;
  }
  if (d->stride_h > 4 || d->stride_w > 4) return fail(LRS_ERR_UNSUPPORTED, "backward: stride > 4");
  if (d->out_scale || d->out_bias || d->out_relu)
    return fail(LRS_ERR_UNSUPPORTED, "backward: no fused output epilogue (back-propagate through it in the caller)");
  if (d->in_w > kTileM) return fail(LRS_ERR_UNSUPPORTED, "backward: in_w > 128");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRS_ERR_CUDA, "no CUDA device available (there is no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(LRS_ERR_INVALID_ARGUMENT, "device %d out of range", device);
  DeviceGuard dg;
  LRS_CUDA(dg.enter(device));
  cudaDeviceProp prop;
  LRS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(LRS_ERR_UNSUPPORTED, "device %d is not sm_100", device);

  lrs_conv_bwd* h = new lrs_conv_bwd();
  h->cp = is_cp;
  auto cleanup_fail = [&](lrs_status s) {
    lrs_conv_bwd_destroy(h);
    return s;
  };
  h->device = device;
  h->sms = prop.multiProcessorCount;
  h->d = *d;
  h->svd = d->core == nullptr;
  h->kh = d->kernel_h;
  h->kw = d->kernel_w;
  h->H = d->in_h;
  h->W = d->in_w;
  h->sh = d->stride_h;
  h->sw = d->stride_w;
  h->ho = (d->in_h + 2 * d->pad_h - d->kernel_h) / h->sh + 1;
  h->wo = (d->in_w + 2 * d->pad_w - d->kernel_w) / h->sw + 1;
  // at stride s the adjoint convolutions run on zero-inserted gradients: dY_up[n][ho*s][wo*s]
  // = dY[n][ho][wo], extent (out - 1) s + 1 + r with r = (in + 2p - k) mod s, so that the
  // stride-1 transposed convolution (pad k-1-p) returns exactly the input extent
  h->hu = (h->ho - 1) * h->sh + 1 + (d->in_h + 2 * d->pad_h - d->kernel_h) % h->sh;
  h->wu = (h->wo - 1) * h->sw + 1 + (d->in_w + 2 * d->pad_w - d->kernel_w) % h->sw;
  h->cin = d->c_in;
  h->cout = d->c_out;
  h->r1 = d->rank_in;
  h->r2 = h->svd ? d->rank_in : d->rank_out;
  h->r1p = round_up(h->r1, 16);
  h->r2p = h->svd ? h->r1p : round_up(h->r2, 16);
  h->batch_max = d->batch_max;
  h->nnz = d->nnz;
  const int kh = h->kh, kw = h->kw, kk = kh * kw, cin = h->cin, cout = h->cout;
  const int r1 = h->r1, r2 = h->r2, r1p = h->r1p, r2p = h->r2p;
  const long long pin_max = static_cast<long long>(d->batch_max) * h->H * h->W;
  const long long p_max = static_cast<long long>(d->batch_max) * h->ho * h->wo;
  if (h->wo > kTileM) return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "backward: output width > 128"));

  // ------------------------------------------------ the transposed layer (dX = its forward)
  {
    std::vector<uint16_t> ui(static_cast<size_t>(cout) * r2), uo(static_cast<size_t>(r1) * cin), g;
    auto bits = [&](const void* a, size_t i) { return static_cast<const uint16_t*>(a)[i]; };
    for (int j = 0; j < cout; ++j)
      for (int b = 0; b < r2; ++b) ui[static_cast<size_t>(j) * r2 + b] = bits(d->u_out, static_cast<size_t>(b) * cout + j);
    for (int a = 0; a < r1; ++a)
      for (int c = 0; c < cin; ++c) uo[static_cast<size_t>(a) * cin + c] = bits(d->u_in, static_cast<size_t>(c) * r1 + a);
    if (!h->svd) {
      g.resize(static_cast<size_t>(r2) * r1 * kk);
      for (int b = 0; b < r2; ++b)
        for (int a = 0; a < r1; ++a)
          for (int y = 0; y < kh; ++y)
            for (int x = 0; x < kw; ++x)
              g[((static_cast<size_t>(b) * r1 + a) * kh + y) * kw + x] =
                  bits(d->core, ((static_cast<size_t>(a) * r2 + b) * kh + (kh - 1 - y)) * kw + (kw - 1 - x));
    }
    // S' by input channel: entry (c, j, y, x, v) -> row c, col (j*kh + kh-1-y)*kw + kw-1-x
    std::vector<std::vector<std::pair<int32_t, float>>> rows(cin);
    for (int j = 0; j < cout; ++j)
      for (int64_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) {
        const int col = d->col_idx[e];
        const int c = col / kk, t = col % kk, y = t / kw, x = t % kw;
        rows[c].push_back({(j * kh + (kh - 1 - y)) * kw + (kw - 1 - x), d->values[e]});
      }
    std::vector<int64_t> rp(cin + 1, 0);
    std::vector<int32_t> ci;
    std::vector<float> va;
    ci.reserve(static_cast<size_t>(d->nnz));
    va.reserve(static_cast<size_t>(d->nnz));
    for (int c = 0; c < cin; ++c) {
      std::sort(rows[c].begin(), rows[c].end());
      for (auto& e : rows[c]) {
        ci.push_back(e.first);
        va.push_back(e.second);
      }
      rp[c + 1] = static_cast<int64_t>(ci.size());
    }
    lrs_conv_desc t = *d;
    t.in_h = h->hu;
    t.in_w = h->wu;
    t.stride_h = 1;
    t.stride_w = 1;
    t.c_in = cout;
    t.c_out = cin;
    t.pad_h = kh - 1 - d->pad_h;
    t.pad_w = kw - 1 - d->pad_w;
    t.rank_in = r2;
    t.rank_out = h->svd ? r2 : r1;
    t.u_in = ui.data();
    t.core = h->svd ? nullptr : g.data();
    t.u_out = uo.data();
    t.row_ptr = rp.data();
    t.col_idx = ci.empty() ? nullptr : ci.data();
    t.values = va.empty() ? nullptr : va.data();
    if (t.pad_h < 0 || t.pad_w < 0)
      return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "backward: pad > kernel - 1 (the transposed layer would crop)"));
    if ((st = lrs_conv_create(&t, device, &h->tr)) != LRS_OK) return cleanup_fail(st);
  }

  // ------------------------------------------------ recompute weights (bf16 B operands)
  auto val = [&](const void* a, size_t i) { return host_val(a, i, false); };
  {
    std::vector<float> m(static_cast<size_t>(r1p) * cin, 0.f);  // U_in^T
    for (int c = 0; c < cin; ++c)
      for (int a = 0; a < r1; ++a) m[static_cast<size_t>(a) * cin + c] = val(d->u_in, static_cast<size_t>(c) * r1 + a);
    if ((st = upload(&h->w_uin, pack_matrix(m, r1p, cin, false))) != LRS_OK) return cleanup_fail(st);
  }
  {
    std::vector<float> m(static_cast<size_t>(r2p) * cout, 0.f);  // U_out [R2p][Cout]
    for (int b = 0; b < r2; ++b)
      for (int j = 0; j < cout; ++j) m[static_cast<size_t>(b) * cout + j] = val(d->u_out, static_cast<size_t>(b) * cout + j);
    if ((st = upload(&h->w_uout, pack_matrix(m, r2p, cout, false))) != LRS_OK) return cleanup_fail(st);
  }
  if (!h->svd) {
    std::vector<float> m(static_cast<size_t>(r2p) * kk * r1p, 0.f);  // G^T [R2p][tap*R1p + a]
    std::vector<float> mt(static_cast<size_t>(r1p) * kk * r2p, 0.f);  // G'^T [R1p][tap'*R2p + b]
    for (int a = 0; a < r1; ++a)
      for (int b = 0; b < r2; ++b)
        for (int t = 0; t < kk; ++t) {
          const float v = val(d->core, (static_cast<size_t>(a) * r2 + b) * kk + t);
          m[static_cast<size_t>(b) * kk * r1p + static_cast<size_t>(t) * r1p + a] = v;
          const int y = t / kw, x = t % kw;
          const int tf = (kh - 1 - y) * kw + (kw - 1 - x);  // G'[b][a][tf] = G[a][b][t]
          mt[static_cast<size_t>(a) * kk * r2p + static_cast<size_t>(tf) * r2p + b] = v;
        }
    if ((st = upload(&h->w_core, pack_matrix(m, r2p, kk * r1p, false))) != LRS_OK) return cleanup_fail(st);
    if ((st = upload(&h->w_coret, pack_matrix(mt, r1p, kk * r2p, false))) != LRS_OK) return cleanup_fail(st);
  }
  // ------------------------------------------------ scratch
  if ((st = bwd_alloc(&h->t1, static_cast<size_t>(pin_max) * r1p * 2, "T1")) != LRS_OK) return cleanup_fail(st);
  if ((st = bwd_alloc(&h->dt1, static_cast<size_t>(pin_max) * r1p * 2, "dT1")) != LRS_OK) return cleanup_fail(st);
  if (!h->svd) {
    if ((st = bwd_alloc(&h->t2, static_cast<size_t>(p_max) * r2p * 2, "T2")) != LRS_OK) return cleanup_fail(st);
    if ((st = bwd_alloc(&h->dt2, static_cast<size_t>(p_max) * r2p * 2, "dT2")) != LRS_OK) return cleanup_fail(st);
  }
  if (h->cp) {
    std::vector<uint8_t> bb(cp_bf.size() * 4), cb(cp_cf.size() * 4);
    memcpy(bb.data(), cp_bf.data(), bb.size());
    memcpy(cb.data(), cp_cf.data(), cb.size());
    void* p1 = nullptr;
    void* p2 = nullptr;
    if ((st = upload(&p1, bb)) != LRS_OK) return cleanup_fail(st);
    h->cp_b = static_cast<float*>(p1);
    if ((st = upload(&p2, cb)) != LRS_OK) return cleanup_fail(st);
    h->cp_c = static_cast<float*>(p2);
    if ((st = bwd_alloc(reinterpret_cast<void**>(&h->dg_int), static_cast<size_t>(r1) * r2 * kk * 4, "dG")) != LRS_OK)
      return cleanup_fail(st);
  }
  if (h->sh > 1 || h->sw > 1) {
    const size_t pu = static_cast<size_t>(d->batch_max) * h->hu * h->wu;
    if ((st = bwd_alloc(&h->dy_up, pu * cout * 2, "dY_up")) != LRS_OK) return cleanup_fail(st);
    if (!h->svd && (st = bwd_alloc(&h->dt2_up, pu * r2p * 2, "dT2_up")) != LRS_OK) return cleanup_fail(st);
  }
  // ------------------------------------------------ recompute GEMM stages
  if ((st = plan_proj_stage(h->g_t1, cin, r1p, h->w_uin, h->t1, &h->sw_x, &h->kc_x)) != LRS_OK) return cleanup_fail(st);
  h->g_t1.name = "bwd_t1";
  if ((st = plan_proj_stage(h->g_dt2, cout, r2p, h->w_uout, h->svd ? h->dt1 : h->dt2, &h->sw_dy, &h->kc_dy)) != LRS_OK)
    return cleanup_fail(st);
  h->g_dt2.name = h->svd ? "bwd_dt1" : "bwd_dt2";
  if (!h->svd) {
    ConvGeom g{};
    g.h = h->H; g.w = h->W; g.ho = h->ho; g.wo = h->wo; g.kh = kh; g.kw = kw;
    g.sh = h->sh; g.sw = h->sw; g.ph = d->pad_h; g.pw = d->pad_w;
    if ((st = plan_conv_stage(h->g_t2, g, r1p, r2p, h->t1, h->w_core, h->t2, d->batch_max)) != LRS_OK) return cleanup_fail(st);
    h->g_t2.name = "bwd_t2";
    ConvGeom gt{};
    gt.h = h->hu; gt.w = h->wu; gt.ho = h->H; gt.wo = h->W; gt.kh = kh; gt.kw = kw;
    gt.sh = 1; gt.sw = 1; gt.ph = kh - 1 - d->pad_h; gt.pw = kw - 1 - d->pad_w;
    void* dt1_in = (h->sh > 1 || h->sw > 1) ? h->dt2_up : h->dt2;
    if ((st = plan_conv_stage(h->g_dt1, gt, r2p, r1p, dt1_in, h->w_coret, h->dt1, d->batch_max)) != LRS_OK)
      return cleanup_fail(st);
    h->g_dt1.name = "bwd_dt1";
  }

  // ------------------------------------------------ the weight-gradient problems
  // (operand kinds: 0 X, 1 dY, 2 T1, 3 T2, 4 dT2, 5 dT1)
  struct Prob {
    int akind, ach, bkind, bch, m, n, taps, grid_in;  // grid_in: 1 = positions of the input grid
    int dst;
  };
  std::vector<Prob> probs;
  if (h->svd) {
    probs.push_back({2, r1p, 1, cout, r1, cout, 1, 0, 0});  // dV = T1^T dY      -> d_u_out
    probs.push_back({0, cin, 5, r1p, cin, r1, 1, 1, 2});    // dU = X^T dT1      -> d_u_in
  } else {
    probs.push_back({3, r2p, 1, cout, r2, cout, 1, 0, 0});  // dU_out = T2^T dY
    probs.push_back({2, r1p, 4, r2p, r1, r2, kk, 0, 1});    // dG (A = T1 shifted by the tap)
    probs.push_back({0, cin, 5, r1p, cin, r1, 1, 1, 2});    // dU_in = X^T dT1
  }
  if (d->nnz > 0) probs.push_back({0, cin, 1, cout, cin, cout, kk, 0, 3});  // dW_S at S's support
  const int np = static_cast<int>(probs.size());
  // LRS_WGRAD_PAIR=1: the CTA-pair form (exact, measured SLOWER -- C3 95.7 vs 84.8 us, C2 43.7 vs
  // 29.6 us -- so opt-in)
  const bool pair_on = getenv("LRS_WGRAD_PAIR") != nullptr;
  h->wp.n_problems = np;
  std::vector<double> work(np);
  std::vector<int> tiles(np), ksteps_max(np), stage_count(np);
  for (int i = 0; i < np; ++i) {
    const Prob& pr = probs[i];
    WgradProblem& q = h->wp.pr[i];
    // the CTA-pair form (opt-in) needs an even number of 128-row M tiles and N tiles of 128
    // or 256 (each CTA loads half of B in 64-wide boxes): small problems are padded (the
    // out-of-range rows / columns load as zeros and are never gathered) so that ONE balanced
    // pair launch covers every problem
    const int bn_cap = getenv("LRS_WGRAD_BN") ? std::max(64, atoi(getenv("LRS_WGRAD_BN")) / 64 * 64) : 256;  // plan override
    const int bn = pair_on ? std::min(256, round_up(pr.n, 128)) : std::min(bn_cap, round_up(pr.n, 64));  // pair: 2 x 64k
    q.bn = bn;
    q.n_tiles = (pr.n + bn - 1) / bn;
    q.m_tiles = pair_on ? round_up((pr.m + 127) / 128, 2) : (pr.m + 127) / 128;
    q.taps = pr.taps;
    q.kw = pr.taps == 1 ? 1 : kw;
    q.pad_h = pr.taps == 1 ? 0 : d->pad_h;
    q.pad_w = pr.taps == 1 ? 0 : d->pad_w;
    q.sh = pr.taps == 1 ? 1 : h->sh;  // the shifted operand (T1 / X) is sampled at the stride
    q.sw = pr.taps == 1 ? 1 : h->sw;
    const int gh = pr.grid_in ? h->H : h->ho, gw = pr.grid_in ? h->W : h->wo;
    int bh = 0, bi = 0, stages = 0;
    if (!pick_wgrad_step(gh, gw, d->batch_max, bn, &bh, &bi, &stages))
      return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "backward: no weight-gradient step fits a %d-wide row", gw));
    q.bh = bh;
    q.bi = bi;
    q.kst = gw * bh * bi;
    q.stage_bytes = static_cast<uint32_t>(2 + bn / 64) * q.kst * 128u;
    stage_count[i] = stages;
    q.hsteps = (gh + bh - 1) / bh;
    q.k_steps = ((d->batch_max + bi - 1) / bi) * q.hsteps;
    h->box_bw[i] = gw;
    h->box_bh[i] = bh;
    h->box_bi[i] = bi;
    h->opa[i] = {pr.akind, pr.ach, pr.akind == 0 || pr.akind == 2 || pr.akind == 5 ? h->H : h->ho,
                 pr.akind == 0 || pr.akind == 2 || pr.akind == 5 ? h->W : h->wo};
    h->opb[i] = {pr.bkind, pr.bch, gh, gw};
    h->dst_of[i] = pr.dst;
    tiles[i] = pr.taps * q.m_tiles * q.n_tiles;
    ksteps_max[i] = q.k_steps;
    work[i] = static_cast<double>(tiles[i]) * q.k_steps * q.kst * (2 + bn / 64);
  }
  // K splits and the persistent schedule: items (problem, tile, split) of about equal work,
  // assigned longest-first to the least-loaded unit (LPT): one CTA per item
  // (lrs_wgrad_kernel<false>), or with LRS_WGRAD_PAIR every problem in ONE launch of CTA PAIRS
  // (cta_group::2: an item covers 2 M tiles, each CTA loads half of B; lrs_wgrad_kernel<true>;
  // the problems were padded to fit above).  Per launch, the granularity g (items per unit) trades balance against the split
  // slabs the reduction reads back: the model time = the most loaded unit's operand bytes at
  // ~60 B/clk per SM (TMA inbound, profiles/r02_tma_bw.log) + the slab bytes written and read
  // at ~5 TB/s.
  struct Sched {
    std::vector<int> splits;
    std::vector<std::vector<WgradItem>> lists;
    std::vector<double> load;
    size_t slab = 0;
    double t = 1e300;
  };
  std::vector<int> pairp(np);
  for (int i = 0; i < np; ++i) {
    const WgradProblem& q = h->wp.pr[i];
    pairp[i] = (pair_on && q.m_tiles % 2 == 0 && q.bn >= 128) ? 1 : 0;
  }
  std::vector<int> splits_of(np, 1);
  auto schedule = [&](int pair, Sched& best) {
    const int units = pair ? h->sms / 2 : h->sms;
    double total = 0;
    for (int i = 0; i < np; ++i)
      if (pairp[i] == pair) total += work[i] * (pair ? (2.0 + h->wp.pr[i].bn / 128) / (2.0 + h->wp.pr[i].bn / 64) : 1.0);
    if (total <= 0) return;
    for (double g : {1.0, 1.5, 2.0, 3.0, 4.0}) {
      Sched sc;
      sc.splits.assign(np, 1);
      const double item_work = total / (g * units);
      std::vector<std::pair<double, WgradItem>> items;
      for (int i = 0; i < np; ++i) {
        if (pairp[i] != pair) continue;
        const WgradProblem& q = h->wp.pr[i];
        const int ut = pair ? tiles[i] / 2 : tiles[i];  // items per split
        const double per_step = static_cast<double>(q.kst) * (2 + q.bn / (pair ? 128 : 64));  // per CTA
        int splits = static_cast<int>(std::lround(per_step * q.k_steps * ut / (ut * item_work)));
        splits = std::max(1, std::min(splits, ksteps_max[i]));
        sc.splits[i] = splits;
        sc.slab += static_cast<size_t>(splits) * q.taps * q.m_tiles * 128 * q.n_tiles * q.bn;
        for (int t = 0; t < ut; ++t)
          for (int sp = 0; sp < splits; ++sp) {
            WgradItem it;
            it.problem = static_cast<uint16_t>(i);
            it.split = static_cast<uint16_t>(sp);
            it.tile = t;
            const long long kb = static_cast<long long>(q.k_steps) * sp / splits;
            const long long ke = static_cast<long long>(q.k_steps) * (sp + 1) / splits;
            items.push_back({static_cast<double>(ke - kb) * per_step, it});
          }
      }
      std::stable_sort(items.begin(), items.end(),
                       [](const std::pair<double, WgradItem>& x, const std::pair<double, WgradItem>& y) {
                         return x.first > y.first;
                       });
      const int grid = std::min<int>(units, static_cast<int>(items.size()));
      sc.lists.assign(grid, {});
      sc.load.assign(grid, 0.0);
      for (auto& it : items) {
        const int c = static_cast<int>(std::min_element(sc.load.begin(), sc.load.end()) - sc.load.begin());
        sc.load[c] += it.first;
        sc.lists[c].push_back(it.second);
      }
      const double mk = *std::max_element(sc.load.begin(), sc.load.end()) * 128.0 / (60.0 * 1.965e9);
      sc.t = mk + 2.0 * sc.slab * 4.0 / 5e12;
      if (sc.t < best.t) best = std::move(sc);
    }
  };
  Sched sch[2];
  schedule(0, sch[0]);
  schedule(1, sch[1]);
  for (int i = 0; i < np; ++i) splits_of[i] = sch[pairp[i]].splits.empty() ? 1 : sch[pairp[i]].splits[i];
  size_t slab_off = 0;
  std::vector<size_t> slab_at(np);
  for (int i = 0; i < np; ++i) {
    WgradProblem& q = h->wp.pr[i];
    q.splits = splits_of[i];
    q.split_stride = static_cast<long long>(q.taps) * q.m_tiles * 128 * q.n_tiles * q.bn;
    slab_at[i] = slab_off;
    slab_off += static_cast<size_t>(q.splits) * q.split_stride;
  }
  h->wg_max_load = 0;
  for (int L = 0; L < 2; ++L) {
    WgradParams& wpL = L ? h->wpp : h->wp;
    if (L) wpL = h->wp;  // the same problems (maps refreshed per call), its own items
    const int grid = static_cast<int>(sch[L].lists.size());
    h->wg_ctas_l[L] = grid;
    if (grid == 0) continue;
    uint32_t slot = 0;
    for (int i = 0; i < np; ++i)
      if (pairp[i] == L) {
        const WgradProblem& q = h->wp.pr[i];
        slot = std::max(slot, static_cast<uint32_t>(2 + q.bn / (L ? 128 : 64)) * q.kst * 128u);
      }
    const int stages = std::min<int>(4, static_cast<int>((static_cast<uint32_t>(kMaxSmem) - 2048u) / slot));
    if (stages < 2) return cleanup_fail(fail(LRS_ERR_UNSUPPORTED, "backward: weight-gradient stages do not fit"));
    std::vector<WgradItem> flat;
    std::vector<int> ptr(grid + 1, 0);
    for (int c = 0; c < grid; ++c) {
      for (auto& it : sch[L].lists[c]) flat.push_back(it);
      ptr[c + 1] = static_cast<int>(flat.size());
    }
    std::vector<uint8_t> b(flat.size() * sizeof(WgradItem)), pb(ptr.size() * 4);
    memcpy(b.data(), flat.data(), b.size());
    memcpy(pb.data(), ptr.data(), pb.size());
    void* p1 = nullptr;
    void* p2 = nullptr;
    if ((st = upload(&p1, b)) != LRS_OK) return cleanup_fail(st);
    h->wg_items_l[L] = p1;
    if ((st = upload(&p2, pb)) != LRS_OK) return cleanup_fail(st);
    h->wg_ptr_l[L] = p2;
    wpL.items = static_cast<const WgradItem*>(p1);
    wpL.item_ptr = static_cast<const int*>(p2);
    wpL.slot_bytes = slot;
    wpL.stages = stages;
    h->wg_smem_l[L] = static_cast<uint32_t>(stages) * slot + 8u * (2u * stages + 4u) + 16u + 1024u;
    double tot = 0;
    for (double v : sch[L].load) tot += v;
    h->wg_max_load = std::max(h->wg_max_load, *std::max_element(sch[L].load.begin(), sch[L].load.end()) / (tot / grid));
  }
  h->slab_floats = slab_off;
  if ((st = bwd_alloc(reinterpret_cast<void**>(&h->slab), slab_off * 4, "weight-gradient slabs")) != LRS_OK)
    return cleanup_fail(st);
  // gather tables: gradient element -> slab offset of split 0
  std::vector<long long> idx;
  std::vector<int> counts(np), idx_at(np);
  for (int i = 0; i < np; ++i) {
    const WgradProblem& q = h->wp.pr[i];
    const long long ld = static_cast<long long>(q.n_tiles) * q.bn;
    const long long mrows = static_cast<long long>(q.m_tiles) * 128;
    idx_at[i] = static_cast<int>(idx.size());
    const size_t s0 = slab_at[i];
    switch (probs[i].dst) {
      case 0:  // [m = b][n = j]
      case 2:  // [m = c][n = a]
        for (int m = 0; m < probs[i].m; ++m)
          for (int n = 0; n < probs[i].n; ++n) idx.push_back(static_cast<long long>(s0) + m * ld + n);
        break;
      case 1:  // dG [a][b][y][x] from [tap][a][b]
        for (int a = 0; a < r1; ++a)
          for (int b = 0; b < r2; ++b)
            for (int t = 0; t < kk; ++t) idx.push_back(static_cast<long long>(s0) + (t * mrows + a) * ld + b);
        break;
      default:  // dvalues[e] from dW_S [tap][c][j]
        for (int j = 0; j < cout; ++j)
          for (int64_t e = d->row_ptr[j]; e < d->row_ptr[j + 1]; ++e) {
            const int col = d->col_idx[e];
            const int c = col / kk, t = col % kk;
            idx.push_back(static_cast<long long>(s0) + (t * mrows + c) * ld + j);
          }
        break;
    }
    counts[i] = static_cast<int>(idx.size()) - idx_at[i];
  }
  {
    std::vector<uint8_t> b(idx.size() * 8);
    memcpy(b.data(), idx.data(), b.size());
    void* p = nullptr;
    if ((st = upload(&p, b)) != LRS_OK) return cleanup_fail(st);
    h->idx = static_cast<long long*>(p);
  }
  h->rs.n = np;
  int blocks = 0;
  for (int i = 0; i < np; ++i) {
    WgradProblem& q = h->wp.pr[i];
    q.slab = h->slab + slab_at[i];
    WgradReduceParams& r = h->rs.r[i];
    r.slab = h->slab;
    r.split_stride = q.split_stride;
    r.splits = q.splits;
    r.idx = h->idx + idx_at[i];
    r.count = counts[i];
    r.dst = nullptr;
    h->rs.block_base[i] = blocks;
    blocks += (counts[i] + kGRThreads - 1) / kGRThreads;
  }
  h->rs.block_base[np] = blocks;
  h->rs_blocks = blocks;
  if (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess)
    return cleanup_fail(fail(LRS_ERR_CUDA, "backward: side stream / event creation failed"));
  for (const void* fn : {reinterpret_cast<const void*>(&lrs_wgrad_kernel<false>),
                         reinterpret_cast<const void*>(&lrs_wgrad_kernel<true>), kernel_ptr(K_STORE_BF16)}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    if (e != cudaSuccess) return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)));
  }
  if (getenv("LRS_VERBOSE")) {
    for (int i = 0; i < np; ++i) {
      const WgradProblem& q = h->wp.pr[i];
      fprintf(stderr, "lrs bwd: problem %d dst %d taps %d m_tiles %d n_tiles %d bn %d kst %d (bh %d bi %d) "
              "splits %d k_steps %d\n", i, probs[i].dst, q.taps, q.m_tiles, q.n_tiles, q.bn, q.kst, q.bh,
              q.bi, q.splits, q.k_steps);
    }
    fprintf(stderr, "lrs bwd: weight gradients: %d solo CTAs (%d stages x %u B) + %d CTA pairs (%d stages x %u B), "
            "max load %.3f x mean, slabs %.1f MB, reduce %d blocks\n", h->wg_ctas_l[0], h->wp.stages, h->wp.slot_bytes,
            h->wg_ctas_l[1], h->wpp.stages, h->wpp.slot_bytes, h->wg_max_load, h->slab_floats * 4.0 / 1e6, h->rs_blocks);
  }
  *out = h;
  return LRS_OK;
}

lrs_status lrs_conv_backward_data(lrs_conv_bwd* h, const void* dy, void* dx, int32_t n, void* stream) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (h->dy_up && n > 0 && n <= h->batch_max) {
    if (!dy || !dx) return fail(LRS_ERR_INVALID_ARGUMENT, "dy / dx is NULL");
    DeviceGuard dg;
    LRS_CUDA(dg.enter(h->device));
    lrs_status st = bwd_zero_insert(h, dy, h->dy_up, n, h->cout, static_cast<cudaStream_t>(stream));
    if (st != LRS_OK) return st;
    return lrs_conv_forward(h->tr, h->dy_up, dx, n, stream);
  }
  return lrs_conv_forward(h->tr, dy, dx, n, stream);
}

lrs_status lrs_conv_backward_weights(lrs_conv_bwd* h, const void* x, const void* dy, int32_t n,
                                     const lrs_conv_grads* gr, void* stream_) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->dt1_ext = nullptr;
  return bwd_weights_impl(h, x, dy, n, gr, stream_);
}

lrs_status lrs_conv_backward(lrs_conv_bwd* h, const void* x, const void* dy, void* dx, int32_t n,
                             const lrs_conv_grads* gr, void* stream_) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (n > 0 && n <= h->batch_max) {
    DeviceGuard dg;
    LRS_CUDA(dg.enter(h->device));
    LRS_CUDA(cudaEventRecord(h->ev_fork, static_cast<cudaStream_t>(stream_)));  // before the transposed forward
  }
  lrs_status st = lrs_conv_backward_data(h, dy, dx, n, stream_);
  if (st != LRS_OK || n == 0) {
    if (st == LRS_OK) st = bwd_weights_impl(h, x, dy, n, gr, stream_);
    return st;
  }
  // the transposed layer's forward just computed dT1 (its T2; T1 for an SVD pair) in the
  // scratch buffer of this forward's parity; it stays intact until its forward after next
  const void* buf = nullptr;
  int32_t ld = 0;
  const bool have = h->svd ? !h->tr->pw_ft : true;
  h->dt1_ext = nullptr;
  if (have && lrs_conv_debug_buffer(h->tr, h->svd ? 0 : 1, &buf, &ld) == LRS_OK && ld == h->r1p) h->dt1_ext = buf;
  h->use_side = true;
  st = bwd_weights_impl(h, x, dy, n, gr, stream_);
  h->use_side = false;
  h->dt1_ext = nullptr;
  return st;
}

}  // extern "C"

namespace {
lrs_status bwd_weights_impl(lrs_conv_bwd* h, const void* x, const void* dy, int32_t n, const lrs_conv_grads* gr,
                            void* stream_) {
  if (n < 0 || n > h->batch_max) return fail(LRS_ERR_INVALID_ARGUMENT, "n=%d outside [0, %d]", n, h->batch_max);
  if (!gr) return fail(LRS_ERR_INVALID_ARGUMENT, "grads is NULL");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  DeviceGuard dg;
  LRS_CUDA(dg.enter(h->device));
  // CP: dG is reduced into the internal buffer and folded into dB, dC afterwards
  const float* dsts[4] = {gr->d_u_out, (h->cp && gr->d_core) ? h->dg_int : gr->d_core, gr->d_u_in, gr->d_values};
  if (n > 0 && (!x || !dy)) return fail(LRS_ERR_INVALID_ARGUMENT, "x / dy is NULL");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(dy) & 15))
    return fail(LRS_ERR_INVALID_ARGUMENT, "x / dy must be 16-byte aligned");
  if (n == 0) {
    // no positions: every gradient is zero
    const size_t sizes[4] = {static_cast<size_t>(h->r2) * h->cout,
                             h->cp ? static_cast<size_t>(h->kh + h->kw) * h->r1
                                   : static_cast<size_t>(h->r1) * h->r2 * h->kh * h->kw,
                             static_cast<size_t>(h->cin) * h->r1, static_cast<size_t>(h->nnz)};
    const float* user[4] = {gr->d_u_out, gr->d_core, gr->d_u_in, gr->d_values};
    for (int i = 0; i < 4; ++i)
      if (user[i] && sizes[i] && !(i == 1 && h->svd))
        LRS_CUDA(cudaMemsetAsync(const_cast<float*>(user[i]), 0, sizes[i] * 4, stream));
    return LRS_OK;
  }
  lrs_status st = bwd_encode_call(h, x, dy, n);
  if (st != LRS_OK) return st;
  const long long pin = static_cast<long long>(n) * h->H * h->W;
  const long long P = static_cast<long long>(n) * h->ho * h->wo;
  // the recompute GEMMs: on the side stream when lrs_conv_backward forked it (they do not
  // read dT1, so they overlap the transposed layer's forward), else in order on `stream`
  const cudaStream_t rstream = h->use_side ? h->side : stream;
  if (h->use_side) LRS_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  // an event pair around a launch of stage si when timing is on
  auto timed = [&](int si, auto&& fn, cudaStream_t ts) -> lrs_status {
    cudaEvent_t e1 = nullptr;
    if (h->timing) {
      TimingRing& r = h->ring[si];
      if (r.used + 2 > static_cast<int>(r.ev.size())) {
        const size_t old = r.ev.size();
        r.ev.resize(old + 256);
        for (size_t i = old; i < r.ev.size(); ++i) LRS_CUDA(cudaEventCreate(&r.ev[i]));
      }
      e1 = r.ev[r.used + 1];
      LRS_CUDA(cudaEventRecord(r.ev[r.used], ts));
      r.used += 2;
    }
    LRS_CUDA(fn());
    if (e1) LRS_CUDA(cudaEventRecord(e1, ts));
    return LRS_OK;
  };
  auto launch_stage = [&](Stage& s, dim3 grid) -> lrs_status {
    const int si = &s == &h->g_t1 ? 0 : (&s == &h->g_t2 ? 1 : (&s == &h->g_dt2 ? 2 : 3));
    return timed(si, [&] { return launch_pdl(kernel_ptr(s.kid), grid, dim3(kThreads), &s.p, s.smem, rstream); },
                 rstream);
  };
  // recompute the chain's activations and back-propagate through it
  if ((st = launch_stage(h->g_t1, dim3(static_cast<unsigned>((pin + kTileM - 1) / kTileM)))) != LRS_OK) return st;
  if (!h->svd) {
    const ConvGeom& g = h->g_t2.p.g;
    if ((st = launch_stage(h->g_t2, dim3(static_cast<unsigned>(((n + g.nb - 1) / g.nb) * g.tiles_h)))) != LRS_OK)
      return st;
  }
  if ((!h->svd || !h->dt1_ext) &&
      (st = launch_stage(h->g_dt2, dim3(static_cast<unsigned>((P + kTileM - 1) / kTileM)))) != LRS_OK)
    return st;
  if (!h->svd && !h->dt1_ext) {
    if (h->dt2_up && (st = bwd_zero_insert(h, h->dt2, h->dt2_up, n, h->r2p, rstream)) != LRS_OK) return st;
    const ConvGeom& g = h->g_dt1.p.g;
    if ((st = launch_stage(h->g_dt1, dim3(static_cast<unsigned>(((n + g.nb - 1) / g.nb) * g.tiles_h)))) != LRS_OK)
      return st;
  }
  if (h->use_side) {  // join: the weight gradients need the recompute AND the transposed forward
    LRS_CUDA(cudaEventRecord(h->ev_join, h->side));
    LRS_CUDA(cudaStreamWaitEvent(stream, h->ev_join, 0));
  }
  // the grouped weight-gradient launch; split counts were sized at batch_max (a smaller n
  // keeps them: a split may then own no position step and stores zeros)
  if ((st = timed(4, [&] {
         cudaError_t e = cudaSuccess;
         if (h->wg_ctas_l[0] > 0)
           e = launch_pdl(reinterpret_cast<const void*>(&lrs_wgrad_kernel<false>),
                          dim3(static_cast<unsigned>(h->wg_ctas_l[0])), dim3(kGThreads), &h->wp, h->wg_smem_l[0], stream);
         if (e == cudaSuccess && h->wg_ctas_l[1] > 0) {
           for (int i = 0; i < h->wp.n_problems; ++i) h->wpp.pr[i] = h->wp.pr[i];  // this call's maps
           e = launch_pdl_pair(reinterpret_cast<const void*>(&lrs_wgrad_kernel<true>),
                               dim3(static_cast<unsigned>(2 * h->wg_ctas_l[1])), dim3(kGThreads), &h->wpp,
                               h->wg_smem_l[1], stream);
         }
         return e;
       }, stream)) != LRS_OK)
    return st;
  // split sums -> gradients (problems whose output the caller skipped are not gathered)
  WgradReduceSet rs = h->rs;
  int blocks = 0, k = 0;
  for (int i = 0; i < h->rs.n; ++i) {
    const float* dst = dsts[h->dst_of[i]];
    if (!dst) continue;
    rs.r[k] = h->rs.r[i];
    rs.r[k].dst = const_cast<float*>(dst);
    rs.block_base[k] = blocks;
    blocks += (rs.r[k].count + kGRThreads - 1) / kGRThreads;
    ++k;
  }
  rs.n = k;
  rs.block_base[k] = blocks;
  if (blocks > 0 && (st = timed(5, [&] {
                       return launch_pdl(reinterpret_cast<const void*>(&lrs_wgrad_reduce_kernel),
                                         dim3(static_cast<unsigned>(blocks)), dim3(kGRThreads), &rs, 0, stream);
                     }, stream)) != LRS_OK)
    return st;
  if (h->cp && gr->d_core) {
    lrs_cp_core_grad_kernel<<<1, 256, 0, stream>>>(h->dg_int, h->cp_b, h->cp_c, h->r1, h->kh, h->kw, gr->d_core);
    LRS_CUDA(cudaGetLastError());
  }
  return LRS_OK;
}

}  // namespace

extern "C" {

lrs_status lrs_conv_bwd_set_timing(lrs_conv_bwd* h, int32_t enable) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->timing = enable != 0;
  return lrs_conv_set_timing(h->tr, enable);
}

lrs_status lrs_conv_bwd_stage_times(lrs_conv_bwd* h, float* ms, int64_t* counts, int32_t max_stages,
                                    int32_t* n_stages, int32_t reset) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  float tms[4];
  int64_t tcnt[4];
  int32_t tn = 0;
  lrs_status st = lrs_conv_stage_times(h->tr, tms, tcnt, 4, &tn, reset);
  if (st != LRS_OK) return st;
  for (int s = 0; s < 6; ++s) {
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
  if (n_stages) *n_stages = 10;
  for (int s = 0; s < 10 && s < max_stages; ++s) {
    if (ms) ms[s] = s < 6 ? static_cast<float>(h->ring[s].ms) : tms[s - 6];
    if (counts) counts[s] = s < 6 ? h->ring[s].count : tcnt[s - 6];
  }
  if (reset)
    for (auto& r : h->ring) {
      r.ms = 0.0;
      r.count = 0;
    }
  return LRS_OK;
}

const char* lrs_conv_bwd_stage_name(const lrs_conv_bwd* h, int32_t stage) {
  static const char* names[] = {"bwd_t1", "bwd_t2", "bwd_dt2", "bwd_dt1", "wgrad", "wgrad_reduce"};
  static const char* dx_names[] = {"dx_a1_proj", "dx_a2_core", "dx_a345_expand_sparse", "dx_a4_sparse_add",
                                   "dx_a12_proj_core"};
  if (stage >= 0 && stage < 6) return names[stage];
  if (stage >= 6 && stage < 10) {
    if (stage == 6 && h && h->tr && h->tr->use_core) return dx_names[4];
    return dx_names[stage - 6];
  }
  return "";
}

int32_t lrs_conv_bwd_launches(const lrs_conv_bwd* h, int32_t* data_launches, int32_t* combined_launches) {
  if (!h) return 0;
  const int32_t d = lrs_conv_launches_per_forward(h->tr);
  // recompute GEMMs + the weight-gradient launch(es) (solo, CTA pairs) + the reduction
  const int32_t w = (h->svd ? 2 : 4) + (h->wg_ctas_l[0] > 0 ? 1 : 0) + (h->wg_ctas_l[1] > 0 ? 1 : 0) + 1 +
                    (h->cp ? 1 : 0);
  const bool reuse = h->svd ? (!h->tr->pw_ft && h->tr->r1p == h->r1p) : (h->tr->r2p == h->r1p);
  if (data_launches) *data_launches = d;
  if (combined_launches) *combined_launches = d + w - (reuse ? 1 : 0);
  return w;
}

}  // extern "C"
