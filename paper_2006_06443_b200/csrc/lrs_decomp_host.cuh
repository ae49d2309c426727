// lrs_decomp_host.cuh -- host side of the low-rank + sparse decomposition (include/lrs_conv.h
// "Decomposition").  Included at the end of lrs_conv.cu.

struct lrs_decomp {
  int device = 0;
  int sms = 148;
  lrs_decomp_params prm{};
  long long numel = 0;
  int q = 1;            // I2 * I3
  int rp = 2;           // rank rounded up to even (Jacobi pairing)
  long long nnz = 0;    // round(cardinality * numel)
  // workspace (device)
  double* t = nullptr;      // T = W - S  [numel]
  double* rsd = nullptr;    // W - L      [numel]
  double* part = nullptr;   // MTTKRP partial sums
  size_t part_n = 0;
  double* m = nullptr;      // MTTKRP result [max dim][R]
  double* gram[4] = {nullptr, nullptr, nullptr, nullptr};
  double* ja = nullptr;     // Jacobi workspaces [rp][rp]
  double* jv = nullptr;
  double* pinv = nullptr;   // [R][R]
  double* qt[4] = {nullptr, nullptr, nullptr, nullptr};  // per mode: last eigenvectors (warm start)
  int* sweeps = nullptr;
  unsigned long long* st = nullptr;  // radix-select state [4]
  unsigned int* hist = nullptr;      // [256]
  unsigned int *gt = nullptr, *eq = nullptr, *eq_pre = nullptr, *sel = nullptr, *sel_pre = nullptr;
  unsigned int *sums_a = nullptr, *sums_b = nullptr;
  double* eps_part = nullptr;
  double* scal = nullptr;   // [0] ||W||^2 partial target, [1] residual mass
  int chunks01[2] = {1, 1}; // MTTKRP chunking per mode (0, 1)
  int chunks23 = 1;
  long long chunk23 = 1;
  size_t pinv_smem = 0;     // dynamic shared memory of the pseudo-inverse (A resident), 0 = global
  bool force_eigen = false; // LRS_DECOMP_EIGEN at create: always the Jacobi eigen path
  // stage timing
  bool timing = false;
  TimingRing ring[4];       // mttkrp, pinv, residual, select
};

namespace {

lrs_status dc_alloc(void** p, size_t bytes) {
  if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess)
    return fail(LRS_ERR_OUT_OF_MEMORY, "decomposition workspace allocation failed");
  return LRS_OK;
}

struct DcTimer {
  lrs_decomp* h;
  cudaStream_t s;
  cudaEvent_t e1 = nullptr;
  lrs_status begin(int si) {
    if (!h->timing) return LRS_OK;
    TimingRing& r = h->ring[si];
    if (r.used + 2 > static_cast<int>(r.ev.size())) {
      const size_t old = r.ev.size();
      r.ev.resize(old + 256);
      for (size_t i = old; i < r.ev.size(); ++i) LRS_CUDA(cudaEventCreate(&r.ev[i]));
    }
    e1 = r.ev[r.used + 1];
    LRS_CUDA(cudaEventRecord(r.ev[r.used], s));
    r.used += 2;
    return LRS_OK;
  }
  lrs_status end() {
    if (e1) LRS_CUDA(cudaEventRecord(e1, s));
    e1 = nullptr;
    return LRS_OK;
  }
};

// T = W (S_0 = 0) and *wn2 = ||W||^2 (synchronises the stream)
lrs_status dc_begin(lrs_decomp* h, const double* w, cudaStream_t s, double* wn2_out) {
  const long long numel = h->numel;
  // ||W||^2 (T = W on entry: S_0 = 0)
  LRS_CUDA(cudaMemcpyAsync(h->t, w, numel * 8, cudaMemcpyDeviceToDevice, s));
  const unsigned nb_fin = static_cast<unsigned>((numel + kDThreads - 1) / kDThreads);
  {
    // residual mass of "no selection" on W itself: sum W^2 through the finish kernel's
    // reduction with an all-false selection (st = max key, nothing taken)
    const unsigned long long init[4] = {~0ull, ~0ull, 0ull, 0ull};
    LRS_CUDA(cudaMemcpyAsync(h->st, init, sizeof(init), cudaMemcpyHostToDevice, s));
    lrs_select_flags_kernel<<<nb_fin, kDThreads, 0, s>>>(w, numel, h->st, h->gt, h->eq);
    lrs_decomp_finish_kernel<<<nb_fin, kDThreads, 0, s>>>(w, w, numel, h->st, h->gt, h->eq, h->eq_pre, h->sums_a,
                                                           h->sel, h->rsd, h->eps_part);
    // (rsd scratch receives W here; overwritten by the first residual)
    LRS_CUDA(cudaGetLastError());
    lrs_decomp_eps_kernel<<<1, kDThreads, 0, s>>>(h->eps_part, static_cast<int>(nb_fin), h->scal);
  }
  double wn2 = 0.0;
  LRS_CUDA(cudaMemcpyAsync(&wn2, h->scal, 8, cudaMemcpyDeviceToHost, s));
  LRS_CUDA(cudaStreamSynchronize(s));
  *wn2_out = wn2;
  return LRS_OK;
}

// S = P_c(Rsd) (exact radix select + ordered compaction into s_idx / s_val), T = W - S, and the
// residual mass sum (W - L - S)^2 into scal[1] -- PAPER.md:144-146 (h->rsd holds W - L)
lrs_status dc_project(lrs_decomp* h, const double* w, long long nnz, int64_t* s_idx, double* s_val, cudaStream_t s) {
  const long long numel = h->numel;
  const unsigned nb_fin = static_cast<unsigned>((numel + kDThreads - 1) / kDThreads);
  const unsigned nb_scan = static_cast<unsigned>((numel + kScanBlock - 1) / kScanBlock);
  {
    unsigned long long init[4] = {0ull, 0ull, static_cast<unsigned long long>(nnz), 0ull};
    if (nnz == 0) init[0] = init[1] = ~0ull;  // nothing above the maximal key, no ties taken
    LRS_CUDA(cudaMemcpyAsync(h->st, init, sizeof(init), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
      LRS_CUDA(cudaMemsetAsync(h->hist, 0, 256 * 4, s));
      const unsigned gb = static_cast<unsigned>(std::min<long long>((numel + kDThreads - 1) / kDThreads, 8LL * h->sms));
      for (int shift = 56; shift >= 0; shift -= 8) {
        lrs_radix_hist_kernel<<<gb, kDThreads, 0, s>>>(h->rsd, numel, h->st, shift, h->hist);
        lrs_radix_pick_kernel<<<1, 1, 0, s>>>(h->st, shift, h->hist);
      }
    }
    lrs_select_flags_kernel<<<nb_fin, kDThreads, 0, s>>>(h->rsd, numel, h->st, h->gt, h->eq);
    lrs_scan_block_kernel<<<nb_scan, 256, 0, s>>>(h->eq, numel, h->eq_pre, h->sums_a);
    lrs_scan_sums_kernel<<<1, 32, 0, s>>>(h->sums_a, static_cast<int>(nb_scan));
    lrs_decomp_finish_kernel<<<nb_fin, kDThreads, 0, s>>>(w, h->rsd, numel, h->st, h->gt, h->eq, h->eq_pre,
                                                           h->sums_a, h->sel, h->t, h->eps_part);
    lrs_decomp_eps_kernel<<<1, kDThreads, 0, s>>>(h->eps_part, static_cast<int>(nb_fin), h->scal + 1);
    if (nnz > 0) {
      lrs_scan_block_kernel<<<nb_scan, 256, 0, s>>>(h->sel, numel, h->sel_pre, h->sums_b);
      lrs_scan_sums_kernel<<<1, 32, 0, s>>>(h->sums_b, static_cast<int>(nb_scan));
      lrs_decomp_compact_kernel<<<nb_fin, kDThreads, 0, s>>>(h->rsd, numel, h->sel, h->sel_pre, h->sums_b,
                                                              reinterpret_cast<long long*>(s_idx), s_val);
    }
    LRS_CUDA(cudaGetLastError());
  }
  return LRS_OK;
}

}  // namespace

extern "C" {

lrs_status lrs_decomp_destroy(lrs_decomp* h) {
  if (!h) return LRS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  void* bufs[] = {h->t, h->rsd, h->part, h->m, h->gram[0], h->gram[1], h->gram[2], h->gram[3], h->ja, h->jv,
                  h->qt[0], h->qt[1], h->qt[2], h->qt[3],
                  h->pinv, h->sweeps, h->st, h->hist, h->gt, h->eq, h->eq_pre, h->sel, h->sel_pre, h->sums_a,
                  h->sums_b, h->eps_part, h->scal};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto& r : h->ring)
    for (auto e : r.ev) cudaEventDestroy(e);
  cudaSetDevice(prev);
  delete h;
  return LRS_OK;
}

lrs_status lrs_decomp_create(const lrs_decomp_params* p, int device, lrs_decomp** out) {
  if (!out || !p) return fail(LRS_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  for (int i = 0; i < 4; ++i)
    if (p->dims[i] <= 0) return fail(LRS_ERR_INVALID_ARGUMENT, "dims must be > 0");
  if (p->rank < 1) return fail(LRS_ERR_INVALID_ARGUMENT, "rank < 1");
  if (!(p->cardinality >= 0.0 && p->cardinality < 1.0))
    return fail(LRS_ERR_INVALID_ARGUMENT, "cardinality must be in [0, 1)");
  if (p->max_iters < 1) return fail(LRS_ERR_INVALID_ARGUMENT, "max_iters < 1");
  if (!(p->rcond >= 0.0)) return fail(LRS_ERR_INVALID_ARGUMENT, "rcond < 0");
  if (p->rank > 256) return fail(LRS_ERR_UNSUPPORTED, "rank > 256");
  if (p->dims[2] > 8 || p->dims[3] > 8) return fail(LRS_ERR_UNSUPPORTED, "dims[2], dims[3] > 8 (kernel taps)");
  const long long numel = static_cast<long long>(p->dims[0]) * p->dims[1] * p->dims[2] * p->dims[3];
  if (numel >= (1ll << 31)) return fail(LRS_ERR_UNSUPPORTED, "tensor of 2^31 entries or more");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRS_ERR_CUDA, "no CUDA device available (there is no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(LRS_ERR_INVALID_ARGUMENT, "device %d out of range", device);
  DeviceGuard dg;
  LRS_CUDA(dg.enter(device));
  cudaDeviceProp prop;
  LRS_CUDA(cudaGetDeviceProperties(&prop, device));
  lrs_decomp* h = new lrs_decomp();
  auto cleanup_fail = [&](lrs_status s) {
    lrs_decomp_destroy(h);
    return s;
  };
  h->device = device;
  h->sms = prop.multiProcessorCount;
  h->prm = *p;
  h->numel = numel;
  h->q = p->dims[2] * p->dims[3];
  h->rp = (p->rank + 1) & ~1;
  h->nnz = static_cast<long long>(std::nearbyint(p->cardinality * static_cast<double>(numel)));  // half to even
  h->force_eigen = getenv("LRS_DECOMP_EIGEN") != nullptr;
  const int r = p->rank;
  // MTTKRP chunking: ~4 blocks per SM over the output rows x chunks x r slices
  const int rs = (r + 63) / 64;
  const int rs01 = (h->q == 9 || h->q == 1) ? 1 : rs;  // the register-blocked forms cover every rank
  for (int m = 0; m < 2; ++m) {
    const int rows = p->dims[m], other = p->dims[1 - m];
    int nc = std::max(1, (4 * h->sms) / std::max(1, rows * rs01));
    if (rs01 == 1) nc = std::max(nc, (other * h->q * 8 + 96 * 1024 - 1) / (96 * 1024));  // staged rows <= 96 KB
    nc = std::min(nc, other);
    h->chunks01[m] = nc;
  }
  {
    const long long pairs = static_cast<long long>(p->dims[0]) * p->dims[1];
    long long nc = std::max<long long>(1, (4LL * h->sms) / rs);
    nc = std::max<long long>(nc, (pairs * h->q * 8 + 48 * 1024 - 1) / (48 * 1024));  // staged rows <= 48 KB
    nc = std::min<long long>(nc, pairs);
    h->chunk23 = (pairs + nc - 1) / nc;
    h->chunks23 = static_cast<int>((pairs + h->chunk23 - 1) / h->chunk23);
  }
  size_t part_n = 0;
  for (int m = 0; m < 2; ++m) part_n = std::max(part_n, static_cast<size_t>(h->chunks01[m]) * p->dims[m] * r);
  part_n = std::max(part_n, static_cast<size_t>(h->chunks23) * std::max(p->dims[2], p->dims[3]) * r);
  h->part_n = part_n;
  const int dmax = std::max(std::max(p->dims[0], p->dims[1]), std::max(p->dims[2], p->dims[3]));
  const long long nb_scan = (numel + kScanBlock - 1) / kScanBlock;
  const long long nb_fin = (numel + kDThreads - 1) / kDThreads;
  lrs_status st;
#define DC_ALLOC(ptr, bytes)                                                          \
  if ((st = dc_alloc(reinterpret_cast<void**>(&(ptr)), (bytes))) != LRS_OK) return cleanup_fail(st)
  DC_ALLOC(h->t, numel * 8);
  DC_ALLOC(h->rsd, numel * 8);
  DC_ALLOC(h->part, part_n * 8);
  DC_ALLOC(h->m, static_cast<size_t>(dmax) * r * 8);
  for (int i = 0; i < 4; ++i) DC_ALLOC(h->gram[i], static_cast<size_t>(r) * r * 8);
  DC_ALLOC(h->ja, static_cast<size_t>(h->rp) * h->rp * 8);
  DC_ALLOC(h->jv, static_cast<size_t>(h->rp) * h->rp * 8);
  DC_ALLOC(h->pinv, static_cast<size_t>(r) * r * 8);
  for (int i = 0; i < 4; ++i) DC_ALLOC(h->qt[i], static_cast<size_t>(h->rp) * h->rp * 8);
  DC_ALLOC(h->sweeps, 16);
  DC_ALLOC(h->st, 4 * 8);
  DC_ALLOC(h->hist, 256 * 4);
  DC_ALLOC(h->gt, numel * 4);
  DC_ALLOC(h->eq, numel * 4);
  DC_ALLOC(h->eq_pre, numel * 4);
  DC_ALLOC(h->sel, numel * 4);
  DC_ALLOC(h->sel_pre, numel * 4);
  DC_ALLOC(h->sums_a, nb_scan * 4);
  DC_ALLOC(h->sums_b, nb_scan * 4);
  DC_ALLOC(h->eps_part, nb_fin * 8);
  DC_ALLOC(h->scal, 4 * 8);
#undef DC_ALLOC
  // the Jacobi matrix A in dynamic shared memory when it fits
  const size_t a_bytes = static_cast<size_t>(h->rp) * h->rp * 8;
  h->pinv_smem = a_bytes <= 200 * 1024 ? a_bytes : 0;
  if (h->pinv_smem) {
    cudaError_t e2 = cudaFuncSetAttribute(reinterpret_cast<const void*>(&lrs_sym_pinv_kernel),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h->pinv_smem));
    if (e2 != cudaSuccess) return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e2)));
  }
  for (const void* fn : {reinterpret_cast<const void*>(&lrs_mttkrp01q_kernel<9>),
                         reinterpret_cast<const void*>(&lrs_mttkrp01q_kernel<1>),
                         reinterpret_cast<const void*>(&lrs_mttkrp23_kernel)}) {
    cudaError_t e3 = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024 + 1024);
    if (e3 != cudaSuccess) return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e3)));
  }
  const size_t res_smem = static_cast<size_t>(r + h->q * r) * 8;
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&lrs_cp_residual_kernel),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(res_smem));
  if (e != cudaSuccess) return cleanup_fail(fail(LRS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)));
  *out = h;
  return LRS_OK;
}

lrs_status lrs_decomp_run(lrs_decomp* h, const double* w, double* f0, double* f1, double* f2, double* f3,
                          int64_t* s_idx, double* s_val, int64_t* s_count, double* eps_hist, int32_t* iters_done,
                          void* stream_) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (!w || !f0 || !f1 || !f2 || !f3 || !eps_hist || !iters_done || !s_count)
    return fail(LRS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (h->nnz > 0 && (!s_idx || !s_val)) return fail(LRS_ERR_INVALID_ARGUMENT, "s_idx / s_val is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  DeviceGuard dg;
  LRS_CUDA(dg.enter(h->device));
  const lrs_decomp_params& p = h->prm;
  const int r = p.rank;
  const long long numel = h->numel;
  double* f[4] = {f0, f1, f2, f3};
  DcTimer tm{h, s};
  lrs_status st;
  double wn2 = 0.0;
  if ((st = dc_begin(h, w, s, &wn2)) != LRS_OK) return st;
  if (wn2 == 0.0) {
    // a zero W gives zero factors, an empty S and eps 0
    for (int m = 0; m < 4; ++m) LRS_CUDA(cudaMemsetAsync(f[m], 0, static_cast<size_t>(p.dims[m]) * r * 8, s));
    eps_hist[0] = 0.0;
    *iters_done = 1;
    *s_count = 0;
    LRS_CUDA(cudaStreamSynchronize(s));
    return LRS_OK;
  }
  const long long nnz = static_cast<long long>(std::nearbyint(p.cardinality * static_cast<double>(numel)));
  for (int m = 0; m < 4; ++m) lrs_gram_kernel<<<r, 256, 0, s>>>(f[m], p.dims[m], r, h->gram[m]);
  LRS_CUDA(cudaGetLastError());
  int it = 0;
  for (; it < p.max_iters; ++it) {
    // ---------------------------------------------------------- 1. ALS sweep on T = W - S
    for (int mode = 0; mode < 4; ++mode) {
      if ((st = tm.begin(0)) != LRS_OK) return st;
      MttkrpParams mp{};
      mp.t = h->t;
      for (int i = 0; i < 4; ++i) mp.f[i] = f[i];
      mp.part = h->part;
      for (int i = 0; i < 4; ++i) mp.dims[i] = p.dims[i];
      mp.q = h->q;
      mp.r = r;
      mp.mode = mode;
      const unsigned rs = static_cast<unsigned>((r + 63) / 64);
      int nchunk;
      if (mode < 2) {
        nchunk = h->chunks01[mode];
        const int other = p.dims[1 - mode];
        mp.nchunk = nchunk;
        mp.chunk = (other + nchunk - 1) / nchunk;
        const size_t tsm = static_cast<size_t>(mp.chunk) * h->q * 8;  // the staged rows of T
        if (h->q == 9)
          lrs_mttkrp01q_kernel<9><<<dim3(static_cast<unsigned>(p.dims[mode]), static_cast<unsigned>(nchunk)), kDThreads,
                                    tsm, s>>>(mp);
        else if (h->q == 1)
          lrs_mttkrp01q_kernel<1><<<dim3(static_cast<unsigned>(p.dims[mode]), static_cast<unsigned>(nchunk)), kDThreads,
                                    tsm, s>>>(mp);
        else
          lrs_mttkrp01_kernel<<<dim3(static_cast<unsigned>(p.dims[mode]), static_cast<unsigned>(nchunk), rs), kDThreads,
                                0, s>>>(mp);
      } else {
        nchunk = h->chunks23;
        mp.nchunk = nchunk;
        mp.chunk = static_cast<int>(h->chunk23);
        lrs_mttkrp23_kernel<<<dim3(static_cast<unsigned>(nchunk), 1, rs), kDThreads,
                              static_cast<size_t>(mp.chunk) * h->q * 8, s>>>(mp);
      }
      const long long cnt = static_cast<long long>(p.dims[mode]) * r;
      lrs_part_sum_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(h->part, nchunk, cnt, h->m);
      LRS_CUDA(cudaGetLastError());
      if ((st = tm.end()) != LRS_OK) return st;
      if ((st = tm.begin(1)) != LRS_OK) return st;
      PinvParams pp{};
      for (int i = 0; i < 4; ++i) pp.g[i] = h->gram[i];
      pp.mode = mode;
      pp.r = r;
      pp.rp = h->rp;
      pp.rcond = p.rcond;
      pp.a = h->ja;
      pp.v = h->jv;
      pp.p = h->pinv;
      pp.sweeps = h->sweeps;
      pp.a_smem = h->pinv_smem ? 1 : 0;
      pp.qt = h->qt[mode];
      pp.warm = (it > 0 && h->pinv_smem) ? 1 : 0;  // from the second sweep on (needs A in shared memory)
      pp.force_eigen = h->force_eigen ? 1 : 0;
      lrs_sym_pinv_kernel<<<1, kJThreads, h->pinv_smem, s>>>(pp);
      lrs_cp_update_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(h->m, h->pinv, p.dims[mode], r,
                                                                                     f[mode]);
      lrs_gram_kernel<<<r, 256, 0, s>>>(f[mode], p.dims[mode], r, h->gram[mode]);
      LRS_CUDA(cudaGetLastError());
      if ((st = tm.end()) != LRS_OK) return st;
    }
    // ---------------------------------------------------------- 2. Rsd = W - L
    if ((st = tm.begin(2)) != LRS_OK) return st;
    {
      const long long row = static_cast<long long>(p.dims[1]) * h->q;
      const unsigned gy = static_cast<unsigned>(std::min<long long>((row + kDThreads - 1) / kDThreads,
                                                                    std::max(1, 4 * h->sms / p.dims[0])));
      lrs_cp_residual_kernel<<<dim3(static_cast<unsigned>(p.dims[0]), std::max(1u, gy)), kDThreads,
                               static_cast<size_t>(r + h->q * r) * 8, s>>>(w, f0, f1, f2, f3, p.dims[1], p.dims[3],
                                                                           h->q, r, h->rsd);
      LRS_CUDA(cudaGetLastError());
    }
    if ((st = tm.end()) != LRS_OK) return st;
    // ---------------------------------------------------------- 3. S = P_c(Rsd), 4. T, eps
    if ((st = tm.begin(3)) != LRS_OK) return st;
    if ((st = dc_project(h, w, nnz, s_idx, s_val, s)) != LRS_OK) return st;
    if ((st = tm.end()) != LRS_OK) return st;
    double rem = 0.0;
    LRS_CUDA(cudaMemcpyAsync(&rem, h->scal + 1, 8, cudaMemcpyDeviceToHost, s));
    LRS_CUDA(cudaStreamSynchronize(s));  // the stopping rule runs on the host
    eps_hist[it] = std::sqrt(rem / wn2);
    if (it > 0 && (eps_hist[it - 1] - eps_hist[it]) < p.tol) {
      ++it;
      break;
    }
  }
  *iters_done = it;
  *s_count = nnz;
  return LRS_OK;
}

int64_t lrs_decomp_nnz(const lrs_decomp* h) { return h ? h->nnz : -1; }

int32_t lrs_decomp_launches_per_iteration(const lrs_decomp* h) {
  // 4 modes x (MTTKRP, partial sums, pseudo-inverse, update, Gram) + residual + flags, scan x 2,
  // finish, eps; with S: 8 radix passes x (histogram, pick) + scan x 2 + compaction
  if (!h) return 0;
  return 4 * 5 + 1 + 5 + (h->nnz > 0 ? 16 + 3 : 0);
}

lrs_status lrs_decomp_set_timing(lrs_decomp* h, int32_t enable) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->timing = enable != 0;
  return LRS_OK;
}

lrs_status lrs_decomp_stage_times(lrs_decomp* h, float* ms, int64_t* counts, int32_t max_stages, int32_t* n_stages,
                                  int32_t reset) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  for (int si = 0; si < 4; ++si) {
    TimingRing& r = h->ring[si];
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
  for (int si = 0; si < 4 && si < max_stages; ++si) {
    if (ms) ms[si] = static_cast<float>(h->ring[si].ms);
    if (counts) counts[si] = h->ring[si].count;
  }
  if (reset)
    for (auto& r : h->ring) {
      r.ms = 0.0;
      r.count = 0;
    }
  return LRS_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------ Tucker-2
// include/lrs_conv.h "Tucker-2 decomposition"; oracle/lrs_decomp.py decompose_lrs_tucker2.
struct lrs_tucker2 {
  lrs_decomp* d = nullptr;  // W's shape: T, Rsd, the projection and the Jacobi workspaces
  lrs_tucker2_params prm{};
  double *z1 = nullptr, *z2 = nullptr, *x = nullptr, *y = nullptr, *c = nullptr, *p = nullptr, *hh = nullptr;
};

namespace {

void t2_gemm(const double* a, const double* b, double* c, const double* sub, int m, int n, int k, int batch,
             long long sam, long long sak, long long sab, long long sbk, long long sbn, long long sbb, long long scm,
             long long scn, long long scb, cudaStream_t s) {
  DgemmParams g{a, b, c, sub, m, n, k, sam, sak, sab, sbk, sbn, sbb, scm, scn, scb};
  lrs_dgemm_kernel<<<dim3(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((m + 63) / 64),
                          static_cast<unsigned>(batch)),
                     256, 0, s>>>(g);
}

// U <- orth(Z Z^T U) `inner` times: Z [rows][cols] row-major, U [rows][r] (in place);
// orth(Y) = Y L^-T (Cholesky-QR) or, for a rank-deficient Y, Y (Y^T Y)^-1/2 (the eigen path)
// -- both in the one-CTA pseudo-inverse kernel
lrs_status t2_subspace(lrs_tucker2* h, const double* z, int rows, int cols, double* u, int r, double* qt, bool warm,
                       cudaStream_t s) {
  lrs_decomp* d = h->d;
  for (int i = 0; i < h->prm.inner; ++i) {
    // X = Z^T U [cols][r];  Y = Z X [rows][r]
    t2_gemm(z, u, h->x, nullptr, cols, r, rows, 1, 1, cols, 0, r, 1, 0, r, 1, 0, s);
    t2_gemm(z, h->x, h->y, nullptr, rows, r, cols, 1, cols, 1, 0, r, 1, 0, r, 1, 0, s);
    lrs_gram_kernel<<<r, 256, 0, s>>>(h->y, rows, r, h->c);
    PinvParams pp{};
    pp.single = h->c;
    pp.inv_sqrt = 1;
    pp.chol_qr = 1;
    pp.r = r;
    pp.rp = (r + 1) & ~1;
    pp.rcond = h->prm.rcond;
    pp.a = d->ja;
    pp.v = d->jv;
    pp.p = h->p;
    pp.sweeps = d->sweeps;
    pp.a_smem = d->pinv_smem ? 1 : 0;
    pp.qt = qt;
    pp.warm = (warm || i > 0) && d->pinv_smem ? 1 : 0;
    lrs_sym_pinv_kernel<<<1, kJThreads, d->pinv_smem, s>>>(pp);
    lrs_cp_update_kernel<<<static_cast<unsigned>((static_cast<long long>(rows) * r + 255) / 256), 256, 0, s>>>(
        h->y, h->p, rows, r, u);
    LRS_CUDA(cudaGetLastError());
  }
  return LRS_OK;
}

}  // namespace

extern "C" {

lrs_status lrs_tucker2_destroy(lrs_tucker2* h) {
  if (!h) return LRS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (h->d) cudaSetDevice(h->d->device);
  for (double* b : {h->z1, h->z2, h->x, h->y, h->c, h->p, h->hh})
    if (b) cudaFree(b);
  lrs_decomp_destroy(h->d);
  cudaSetDevice(prev);
  delete h;
  return LRS_OK;
}

lrs_status lrs_tucker2_create(const lrs_tucker2_params* p, int device, lrs_tucker2** out) {
  if (!out || !p) return fail(LRS_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (p->r1 < 1 || p->r2 < 1) return fail(LRS_ERR_INVALID_ARGUMENT, "r1, r2 must be >= 1");
  if (p->inner < 1) return fail(LRS_ERR_INVALID_ARGUMENT, "inner < 1");
  for (int i = 0; i < 4; ++i)
    if (p->dims[i] <= 0) return fail(LRS_ERR_INVALID_ARGUMENT, "dims must be > 0");
  if (p->r1 > p->dims[0] || p->r2 > p->dims[1]) return fail(LRS_ERR_INVALID_ARGUMENT, "r1 > dims[0] or r2 > dims[1]");
  lrs_decomp_params dp{};
  for (int i = 0; i < 4; ++i) dp.dims[i] = p->dims[i];
  dp.rank = std::max(p->r1, p->r2);
  dp.cardinality = p->cardinality;
  dp.max_iters = p->max_iters;
  dp.tol = p->tol;
  dp.rcond = p->rcond;
  lrs_decomp* d = nullptr;
  lrs_status st = lrs_decomp_create(&dp, device, &d);  // validates the rest (rank <= 256, sizes, device)
  if (st != LRS_OK) return st;
  DeviceGuard dg;
  LRS_CUDA(dg.enter(device));
  lrs_tucker2* h = new lrs_tucker2();
  h->d = d;
  h->prm = *p;
  const long long q = d->q, cin = p->dims[0], cout = p->dims[1], rm = dp.rank;
  const long long zc = std::max(p->r2 * q, p->r1 * q);
  const size_t sizes[7] = {static_cast<size_t>(cin * p->r2 * q), static_cast<size_t>(cout * p->r1 * q),
                           static_cast<size_t>(zc * rm), static_cast<size_t>(std::max(cin, cout) * rm),
                           static_cast<size_t>(rm * rm), static_cast<size_t>(rm * rm),
                           static_cast<size_t>(p->r1 * cout * q)};
  double** bufs[7] = {&h->z1, &h->z2, &h->x, &h->y, &h->c, &h->p, &h->hh};
  for (int i = 0; i < 7; ++i)
    if ((st = dc_alloc(reinterpret_cast<void**>(bufs[i]), sizes[i] * 8)) != LRS_OK) {
      lrs_tucker2_destroy(h);
      return st;
    }
  *out = h;
  return LRS_OK;
}

lrs_status lrs_tucker2_run(lrs_tucker2* h, const double* w, double* u_in, double* u_out, double* core,
                           int64_t* s_idx, double* s_val, int64_t* s_count, double* eps_hist, int32_t* iters_done,
                           void* stream_) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (!w || !u_in || !u_out || !core || !eps_hist || !iters_done || !s_count)
    return fail(LRS_ERR_INVALID_ARGUMENT, "NULL argument");
  lrs_decomp* d = h->d;
  if (d->nnz > 0 && (!s_idx || !s_val)) return fail(LRS_ERR_INVALID_ARGUMENT, "s_idx / s_val is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  DeviceGuard dg;
  LRS_CUDA(dg.enter(d->device));
  const lrs_tucker2_params& p = h->prm;
  const int cin = p.dims[0], cout = p.dims[1], r1 = p.r1, r2 = p.r2, q = d->q;
  const long long nnz = d->nnz;
  DcTimer tm{d, s};
  lrs_status st;
  double wn2 = 0.0;
  if ((st = dc_begin(d, w, s, &wn2)) != LRS_OK) return st;
  if (wn2 == 0.0) {
    LRS_CUDA(cudaMemsetAsync(u_in, 0, static_cast<size_t>(cin) * r1 * 8, s));
    LRS_CUDA(cudaMemsetAsync(u_out, 0, static_cast<size_t>(cout) * r2 * 8, s));
    LRS_CUDA(cudaMemsetAsync(core, 0, static_cast<size_t>(r1) * r2 * q * 8, s));
    eps_hist[0] = 0.0;
    *iters_done = 1;
    *s_count = 0;
    LRS_CUDA(cudaStreamSynchronize(s));
    return LRS_OK;
  }
  const long long jq = static_cast<long long>(cout) * q;  // T's row stride (input channel)
  int it = 0;
  for (; it < p.max_iters; ++it) {
    // ------------------------------------------------ 1. HOOI sweep on T = W - S (stage 0: products, 1: orth)
    if ((st = tm.begin(0)) != LRS_OK) return st;
    // Z1[c][b][t] = sum_j T[c][j][t] U_out[j][b]   (batch t)
    t2_gemm(d->t, u_out, h->z1, nullptr, cin, r2, cout, q, jq, q, 1, r2, 1, 0, static_cast<long long>(r2) * q, q, 1, s);
    if ((st = tm.end()) != LRS_OK) return st;
    if ((st = tm.begin(1)) != LRS_OK) return st;
    if ((st = t2_subspace(h, h->z1, cin, r2 * q, u_in, r1, d->qt[0], it > 0, s)) != LRS_OK) return st;
    if ((st = tm.end()) != LRS_OK) return st;
    if ((st = tm.begin(0)) != LRS_OK) return st;
    // Z2[j][a][t] = sum_c T[c][j][t] U_in[c][a]   (batch t)
    t2_gemm(d->t, u_in, h->z2, nullptr, cout, r1, cin, q, q, jq, 1, r1, 1, 0, static_cast<long long>(r1) * q, q, 1, s);
    if ((st = tm.end()) != LRS_OK) return st;
    if ((st = tm.begin(1)) != LRS_OK) return st;
    if ((st = t2_subspace(h, h->z2, cout, r1 * q, u_out, r2, d->qt[1], it > 0, s)) != LRS_OK) return st;
    if ((st = tm.end()) != LRS_OK) return st;
    if ((st = tm.begin(0)) != LRS_OK) return st;
    // G[a][b][t] = sum_j Z2[j][a][t] U_out[j][b]   (batch t)
    t2_gemm(h->z2, u_out, core, nullptr, r1, r2, cout, q, q, static_cast<long long>(r1) * q, 1, r2, 1, 0,
            static_cast<long long>(r2) * q, q, 1, s);
    if ((st = tm.end()) != LRS_OK) return st;
    // ------------------------------------------------ 2. Rsd = W - L,  L = U_in (G x_out U_out)
    if ((st = tm.begin(2)) != LRS_OK) return st;
    // H[a][j][t] = sum_b G[a][b][t] U_out[j][b]   (batch t)
    t2_gemm(core, u_out, h->hh, nullptr, r1, cout, r2, q, static_cast<long long>(r2) * q, q, 1, 1, r2, 0, jq, q, 1, s);
    // Rsd[c][(j, t)] = W[c][(j, t)] - sum_a U_in[c][a] H[a][(j, t)]
    t2_gemm(u_in, h->hh, d->rsd, w, cin, static_cast<int>(jq), r1, 1, r1, 1, 0, jq, 1, 0, jq, 1, 0, s);
    LRS_CUDA(cudaGetLastError());
    if ((st = tm.end()) != LRS_OK) return st;
    // ------------------------------------------------ 3. S = P_c(Rsd), T = W - S, eps
    if ((st = tm.begin(3)) != LRS_OK) return st;
    if ((st = dc_project(d, w, nnz, s_idx, s_val, s)) != LRS_OK) return st;
    if ((st = tm.end()) != LRS_OK) return st;
    double rem = 0.0;
    LRS_CUDA(cudaMemcpyAsync(&rem, d->scal + 1, 8, cudaMemcpyDeviceToHost, s));
    LRS_CUDA(cudaStreamSynchronize(s));
    eps_hist[it] = std::sqrt(rem / wn2);
    if (it > 0 && (eps_hist[it - 1] - eps_hist[it]) < p.tol) {
      ++it;
      break;
    }
  }
  *iters_done = it;
  *s_count = nnz;
  return LRS_OK;
}

int64_t lrs_tucker2_nnz(const lrs_tucker2* h) { return h ? h->d->nnz : -1; }

lrs_status lrs_tucker2_set_timing(lrs_tucker2* h, int32_t enable) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  return lrs_decomp_set_timing(h->d, enable);
}

lrs_status lrs_tucker2_stage_times(lrs_tucker2* h, float* ms, int64_t* counts, int32_t max_stages, int32_t* n_stages,
                                   int32_t reset) {
  if (!h) return fail(LRS_ERR_INVALID_ARGUMENT, "handle is NULL");
  return lrs_decomp_stage_times(h->d, ms, counts, max_stages, n_stages, reset);
}

}  // extern "C"
