/*
 * lrs_conv.h -- C-ABI of the B200 (sm_100a) compressed convolution whose
 * weight is approximated as W ~ L + S (arXiv 2006.06443, the thesis in
 * /root/reference/PAPER.md; BASELINE.json north star).
 *
 *   Y = conv(X, L) + conv(X, S)
 *
 *   L  Tucker-2 chain  T1 = X U_in          (1x1 projection,   PAPER.md:162)
 *                      T2 = conv(T1, G)     (k x k core,       PAPER.md:165-166, :409)
 *                      Y_L = T2 U_out       (1x1 expansion,    PAPER.md:168)
 *      or the paper's CP chain (core_kind = LRS_CORE_CP):
 *                      T1 = X A, T2 = depthwise k x 1 (B) then 1 x k (C) over
 *                      the R rank channels, Y_L = T2 D^T
 *      or, for a 1x1 layer, an SVD pair  Y_L = (X U) V          (core == NULL)
 *   S  direct sparse convolution, CSR by output channel        PAPER.md:171-191 §3.4
 *   Y  = Y_L + Y_S, written to device memory once.
 *
 * Conventions (readings #2, #3, #6):
 *   - activations are NHWC (the paper's X_{smt}, batched);
 *   - cross-correlation, zero padding; out_h = (in_h + 2 pad_h - kernel_h)/stride_h + 1;
 *   - core is indexed [rank_in][rank_out][kernel_h][kernel_w] (the paper's
 *     (in, out, kx, ky) order), u_in [c_in][rank_in], u_out [rank_out][c_out];
 *   - CSR row j = output channel j; col = (c * kernel_h + ky) * kernel_w + kx,
 *     strictly increasing within a row (the OIHW flattening).
 * No bias: the paper's layer has none.
 *
 * No function aborts.  Every function returns an lrs_status;
 * lrs_conv_last_error() gives the text of the last non-OK status of the
 * calling thread.  There is no CPU fallback: a missing GPU is LRS_ERR_CUDA.
 * Nothing is printed unless LRS_VERBOSE is set (plan lines on stderr).  A
 * kernel whose pipeline wait exceeds ~9 s (a protocol bug, never expected)
 * traps: the launch fails with a CUDA error instead of hanging the device.
 *
 * Environment (read at create): LRS_VERBOSE; plan / engine overrides used by
 * the tests to cover every path -- LRS_NO_AUTOTUNE, LRS_NO_CORE, LRS_NO_TINY,
 * LRS_F32_FUSED, LRS_NO_PW, LRS_NO_SPTC, LRS_NO_EARLY, LRS_PW_{MPC,BP,FT,CPI,EPIBUF},
 * LRS_CORE_{IPT,TH,GRID,GSTREAM,T1_NOSWZ,SPLIT_RING}, LRS_TINY_CB,
 * LRS_WCONV_{TH,CB,CPW,NS,BPI,IPW,REUSE,NWB1,ERING,GATHER,PAIR,DENSE_LAST}, LRS_DECOMP_EIGEN, LRS_WGRAD_PAIR -- each selects another plan
 * that computes the same Y (up to the fp32 summation order where an engine changes).  Knobs that skip work (timing bisection) exist
 * only in -DLRS_EXPERIMENTS builds; bench.py refuses to time with any LRS_*
 * variable set.
 *
 * Threads: a handle keeps host-side per-call state (tensor-map caches, launch
 * parameters), so calls on ONE handle must not run concurrently from several
 * host threads; use one handle per thread (distinct handles are independent).
 */
#ifndef LRS_CONV_H_
#define LRS_CONV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LRS_OK = 0,
  LRS_ERR_INVALID_ARGUMENT = 1, /* malformed descriptor / pointer / size            */
  LRS_ERR_UNSUPPORTED = 2,      /* legal but not implemented (see lrs_conv_create) */
  LRS_ERR_OUT_OF_MEMORY = 3,    /* device or host allocation failed                */
  LRS_ERR_CUDA = 4              /* CUDA runtime / driver error (launch, no device) */
} lrs_status;

typedef enum {
  LRS_DTYPE_F32 = 0,  /* X, Y, factors fp32; chain on tensor cores as 3xTF32 split */
  LRS_DTYPE_BF16 = 1  /* X, Y, factors bf16; fp32 accumulation everywhere          */
} lrs_dtype;

typedef enum {
  LRS_CORE_TUCKER2 = 0, /* core = dense G [rank_in][rank_out][kernel_h][kernel_w]        */
  LRS_CORE_CP = 1       /* core = B [kernel_h][R] then C [kernel_w][R], R = rank_in = rank_out:
                           L[c,j,y,x] = sum_r u_in[c,r] B[y,r] C[x,r] u_out[r,j]
                           (A = u_in, D^T = u_out); stages 2-3 run as the
                           paper's two depthwise convolutions         */
} lrs_core_kind;

typedef struct lrs_conv lrs_conv; /* opaque; its weights are immutable after create */

typedef struct lrs_conv_desc {
  int32_t batch_max;              /* largest n accepted by forward (> 0)            */
  int32_t in_h, in_w, c_in, c_out;
  int32_t kernel_h, kernel_w;     /* 1..7                                           */
  int32_t stride_h, stride_w;     /* >= 1                                           */
  int32_t pad_h, pad_w;           /* >= 0                                           */
  int32_t rank_in, rank_out;      /* Tucker-2 (R1, R2); SVD pair: rank_in == rank_out */
  lrs_dtype dtype;                /* element type of X, Y, u_in, core, u_out        */
  const void *u_in;               /* host [c_in][rank_in], row-major, dtype         */
  const void *core;               /* host [rank_in][rank_out][kernel_h][kernel_w]   */
                                  /* or NULL: SVD pair (requires 1x1, stride 1, pad 0) */
  const void *u_out;              /* host [rank_out][c_out], row-major, dtype       */
  int64_t nnz;                    /* >= 0                                           */
  const int64_t *row_ptr;         /* host [c_out + 1]; 0, non-decreasing, nnz at end */
  const int32_t *col_idx;         /* host [nnz]; < c_in*kernel_h*kernel_w            */
  const float *values;            /* host [nnz]; fp32; bf16 layers round them to bf16 (RNE)
                                     at create (reading #12)               */
  lrs_core_kind core_kind;        /* LRS_CORE_TUCKER2 (0, the zero-initialised default)
                                     or LRS_CORE_CP; ignored when core == NULL        */
  /* Optional fused output epilogue (e.g. an inference BatchNorm + ReLU
     that follows the layer in a network): Y[..., j] = act(s_j * conv_j + b_j), applied
     in fp32 to the accumulator before the single store of Y.  All zero = identity.   */
  const float *out_scale;         /* host [c_out] or NULL (s = 1)                    */
  const float *out_bias;          /* host [c_out] or NULL (b = 0)                    */
  int32_t out_relu;               /* 1: act = max(., 0); 0: act = identity           */
} lrs_conv_desc;

/*
 * Create a layer on CUDA device `device`.  All desc arrays are host memory,
 * deep-copied and repacked (rank padding, K-major weight tiles, per-tile
 * sparse code streams); the caller may free them on return.  The handle
 * owns its device buffers (weights + scratch sized for batch_max).
 * INVALID_ARGUMENT: any extent <= 0, stride < 1, pad < 0, output extent < 1,
 *   malformed CSR (row_ptr not monotone / wrong ends, col out of range,
 *   unsorted or duplicate columns), core == NULL with a non-1x1 / strided /
 *   padded kernel or rank_in != rank_out, NULL required pointer.
 * UNSUPPORTED: kernel > 7, rank > 256, c_in or c_out not a multiple of 8
 *   (bf16) / 4 (fp32) (16-byte TMA rows), output width > 256; output width > 128
 *   unless the layer is bf16 with c_in % 64 == 0 and its core runs in the fused core
 *   kernel (stride 1, window <= 256 columns and fitting shared memory), is the CP form or
 *   an SVD pair (the GEMM core convolution tiles whole rows of <= 128 outputs).
 * bf16 layers with c_in % 64 == 0 run the fused expansion + sparse term on
 * the 2:4 sparse tensor cores (lrs_conv_sparse_engine() == 1); S is split at
 * create into exact 2:4 main and residual blocks (PAPER.md:171-191 evaluated
 * exactly).
 * bf16 stride-1 layers run a1 + a2 (or a1 + the CP depthwise pair) in one
 * kernel whose tile plan is chosen at create by timing a few candidate plans
 * on the device (back-to-back forwards on zero-filled scratch of batch_max
 * images; ~ms; synchronous on a private stream); so are the windowed fused
 * kernel's band height (jointly with that core plan) and the 1x1 pointwise
 * kernel's plan.  Every plan computes the same bits.  LRS_NO_AUTOTUNE=1 in the environment keeps the cost model's plan, and
 * so does a scratch allocation that runs out of memory (any other CUDA error
 * during tuning is LRS_ERR_CUDA).
 * OUT_OF_MEMORY / CUDA: allocation or driver failure (no handle is returned).
 */
lrs_status lrs_conv_create(const lrs_conv_desc *desc, int device, lrs_conv **out);

/*
 * Y = conv(X, L + S) for n images, enqueued on `stream` (a cudaStream_t;
 * NULL = legacy default stream).  x: device [n][in_h][in_w][c_in], y: device
 * [n][out_h][out_w][c_out], both dtype, contiguous, 16-byte aligned, on the
 * handle's device, not aliased.  y is overwritten.  No host sync and no
 * allocation: the call is CUDA-graph capturable.  The handle's scratch is
 * shared by all calls, so at most one forward may be in flight per handle.
 * n == 0 is a no-op.  INVALID_ARGUMENT: n < 0, n > batch_max, NULL or
 * misaligned pointer.  CUDA: launch failure (asynchronous faults surface at
 * the caller's next synchronisation).
 * Kernels are launched with programmatic dependent launch: each waits
 * (griddepcontrol.wait) before touching what the kernel before it may still
 * write.  Layers whose projection + core kernel feeds the fused kernel (bf16,
 * stride 1, not an SVD pair) keep two T2 buffers, and 1x1 SVD pairs on the pointwise
 * kernel two T1 buffers, and let that first kernel start computing before the
 * previous kernel on the stream has finished, unless x
 * overlaps the output of the library's previous forward on that stream (then it
 * waits first, as every other kernel does); the library assumes that kernels the
 * caller enqueues between forwards do not trigger their dependents early
 * (griddepcontrol.launch_dependents) before they finish writing.  Same results
 * either way.  LRS_NO_EARLY=1 in the environment at create disables it.
 */
lrs_status lrs_conv_forward(const lrs_conv *h, const void *x, void *y, int32_t n, void *stream);

/*
 * End-to-end variant with HOST buffers: copies x_host -> device, runs
 * lrs_conv_forward, copies the result -> y_host.  The batch is pipelined in up
 * to 4 chunks of >= 8 images on two handle-owned copy streams (chunk i+1 in,
 * chunk i computed, chunk i-1 out); the copies start after the caller's prior
 * work on `stream`, and `stream` is made to wait for the last copy out, so the
 * call behaves as if everything ran on `stream` (pinned host memory makes the
 * copies asynchronous).  The device staging buffers, streams and events are
 * created by the first call (so this call is not graph capturable) and owned
 * by the handle.  The caller synchronises `stream` before reading y_host.
 */
lrs_status lrs_conv_forward_host(lrs_conv *h, const void *x_host, void *y_host, int32_t n,
                                 void *stream);

/* NULL-safe.  Requires that no forward is in flight on the handle. */
lrs_status lrs_conv_destroy(lrs_conv *h);

/* Thread-local text of the last non-OK status ("" if none). Never NULL. */
const char *lrs_conv_last_error(void);

/* Output spatial extent of the layer. */
lrs_status lrs_conv_output_shape(const lrs_conv *h, int32_t *out_h, int32_t *out_w);

/* Number of kernels one lrs_conv_forward launches (n > 0). */
int32_t lrs_conv_launches_per_forward(const lrs_conv *h);

/*
 * Stage timing for measurement (bench.py roofline): when enabled, forward
 * records a CUDA event pair around every kernel it launches on the caller's
 * stream.  lrs_conv_stage_times sums, over all forwards since the last
 * reset, each stage's event-timed duration (ms) into ms[i] and the launch
 * count into counts[i], for i < min(max_stages, stage count); it
 * synchronises the recorded events.  Stage names: lrs_conv_stage_name.
 * Enabling adds an event record per launch; it is off by default.
 */
lrs_status lrs_conv_set_timing(lrs_conv *h, int32_t enable);
lrs_status lrs_conv_stage_times(lrs_conv *h, float *ms, int64_t *counts, int32_t max_stages,
                                int32_t *n_stages, int32_t reset);
const char *lrs_conv_stage_name(const lrs_conv *h, int32_t stage);

/*
 * Test hook: device pointer of an intermediate of the last forward,
 * which = 0: T1 [n*in_h*in_w][ld] ; 1: T2 [n*out_h*out_w][ld] (NULL for the SVD
 * pair).  *ld receives the padded row length (elements, dtype).
 */
lrs_status lrs_conv_debug_buffer(const lrs_conv *h, int32_t which, const void **ptr, int32_t *ld);

/*
 * Which engine evaluates the sparse term S of this layer (returns -1 for NULL):
 *   0  SIMT CSR gather fused into the epilogue of the expansion GEMM
 *      (fp32 layers and shapes the tensor-core path does not cover);
 *   1  2:4 sparse tensor cores (tcgen05.mma.sp): every group of 4 consecutive
 *      input channels of a (output channel, tap) is split exactly into a main
 *      2:4 block and, where the group holds 3-4 nonzeros, a residual 2:4 block;
 *      fused with the expansion GEMM (bf16 layers with c_in % 64 == 0);
 *   2  fp32 layers with out_w <= 64: one SIMT kernel computes the expansion
 *      (register-blocked fp32 GEMM over a shared-memory tile of T2) and the
 *      sparse term (CSR gather over shared-memory windows of 4 images) and
 *      writes Y once (set LRS_F32_FUSED=1 at create to select engine 0);
 *   3  small fp32 Tucker-2 or CP layers (weights + one tile's window fit in
 *      shared memory, grid <= 2 waves, e.g. batch 1): the whole layer --
 *      projection, core (dense k x k, or the CP form's two depthwise stages in
 *      the paper's order), expansion and sparse term -- in ONE SIMT kernel, a
 *      CTA per image x row band x column band (LRS_NO_TINY=1 at create
 *      disables it).
 * For engine 1, *main_blocks / *residual_blocks (may be NULL) receive the
 * number of 128-row compressed blocks of each kind.
 */
int32_t lrs_conv_sparse_engine(const lrs_conv *h, int32_t *main_blocks, int32_t *residual_blocks);

/*
 * The paper's sparse storage (§3.4) -> the CSR this
 * ABI takes.  Per input channel i (a "slice"), entries slice_ptr[i] .. slice_ptr[i+1]-1
 * of packed[] / values[] (host arrays) hold one nonzero each:
 *   packed = j * (kernel_h * kernel_w) + ky * kernel_w + kx    (output channel j, tap ky, kx)
 * as uint16 (packed_bytes = 2; requires c_out * kernel_h * kernel_w <= 65536, the
 * paper's "one int16 number") or uint32 (packed_bytes = 4).  Slices may hold any
 * number of entries in any order.  Writes row_ptr [c_out + 1], and col_idx / values_out
 * [slice_ptr[c_in]] sorted by (row, col) with col = (i * kernel_h + ky) * kernel_w + kx.
 * Host-only (no device needed).  INVALID_ARGUMENT: bad extents, packed_bytes not 2/4,
 * slice_ptr not starting at 0 / not monotone, an index decoding to j >= c_out, a
 * duplicate (j, col), or uint16 packing where c_out * taps > 65536.
 */
lrs_status lrs_sparse_from_slices(int32_t c_in, int32_t c_out, int32_t kernel_h, int32_t kernel_w,
                                  const int64_t *slice_ptr, const void *packed, int32_t packed_bytes,
                                  const float *values, int64_t *row_ptr, int32_t *col_idx, float *values_out);

/*
 * Which kernel evaluates the expansion a3 + sparse term a4 + the single store a5
 * (-1 for NULL):
 *   0  a GEMM / SIMT kernel (fp32 layers, shapes the tensor-core kernels do not cover);
 *   1  the windowed fused tensor-core kernel (lrs_wconv.cuh: k x k layers, any stride);
 *   2  the channel-stationary pointwise kernel (lrs_pw.cuh): 1x1 SVD-pair bf16 layers
 *      with c_in % 64 == 0 and c_in <= 512 -- each CTA keeps the V^T blocks and the 2:4
 *      blocks of a fixed group of 128-channel M-tiles resident (metadata in TMEM) and
 *      streams X and T1 position tiles through it (C4; PAPER.md:168, :171-191 at k = 1).
 *      LRS_NO_PW=1 at create selects kernel 1 instead; LRS_PW_MPC / LRS_PW_BP override
 *      the M-tiles per CTA / positions per tile; LRS_PW_FT=1 fuses the projection a1 into
 *      the same kernel (lrs_pwf.cuh: one launch, T1 never in HBM; measured slower at C4,
 *      so not the default) -- every choice computes the same bits.
 */
int32_t lrs_conv_expand_kernel(const lrs_conv *h);

/*
 * How the windowed tensor-core kernel (expand kernel 1) evaluates the entries of S
 * that an exact 2:4 main block cannot hold (the 3rd / 4th nonzero of a group of 4
 * input channels, PAPER.md:171-191 evaluated exactly):
 *   0   residual 2:4 blocks (lrs_conv_sparse_engine's residual_blocks), one per
 *       (M-tile, 64-channel chunk, tap) that has any such entry -- each costs a
 *       full sparse MMA pass over the tile's positions;
 *   g>0 g "overflow gather" chunks per 128-channel M-tile: the M-tile's distinct
 *       (input channel, tap) pairs of those entries become g * 64 (or g * R2 when
 *       R2 < 64) extra dense K columns G[pos][slot] = X[pos + tap][channel],
 *       gathered per tile by the kernel's epilogue warps into a device scratch of
 *       batch_max * out_h * out_w * n_mt * g * 64 bf16 and multiplied on the dense
 *       tensor cores by the entries' values (residual_blocks is then 0).
 * Chosen at create by cost (residual MMA steps vs gather chunks); LRS_WCONV_GATHER=0/1
 * in the environment at create forces it.  -1 for NULL; 0 for the other kernels.
 */
int32_t lrs_conv_overflow_chunks(const lrs_conv *h);

/*
 * 1 if the windowed tensor-core kernel runs in its CTA-pair form: clusters of two CTAs on
 * the two SMs of a TPC own two 128-channel M-tiles of the same positions, and one of them
 * issues tcgen05.mma.cta_group::2 (M = 256) for both, each SM holding half of the activation
 * window along N -- the 2:4 MMAs then run at the tensor rate instead of the shared-memory
 * bound of one SM.  Needs an even number of M-tiles, no residual 2:4 blocks
 * (the overflow gather takes their entries, with the union of the pair's slots) and MMA
 * units of one width.  Opt-in: LRS_WCONV_PAIR=1 in the environment at create takes it
 * wherever feasible (exact, tested against the oracle; measured slower than the one-CTA form
 * at C3).  0 otherwise, -1 for NULL.
 */
int32_t lrs_conv_cta_pairs(const lrs_conv *h);

/*
 * 1 if the projection a1 and the core convolution a2 of this layer run as one
 * kernel (bf16 Tucker-2 layers with stride 1 and c_in % 64 == 0: T1 is computed
 * on each tile's input window and kept in shared memory, never written to HBM;
 * PAPER.md:162-166), 0 if they run as two kernels with T1 in HBM, -1 for NULL.
 * With the fused kernel lrs_conv_debug_buffer(h, 0, ...) returns stale data.
 */
int32_t lrs_conv_core_fused(const lrs_conv *h);

/*
 * Debug hook: when dev_buf (device, >= 1005 uint64) is non-NULL, CTA 0 of the
 * fused tensor-core kernel stores %globaltimer stamps of its pipeline events
 * there (NULL disables).  Not for production use.
 */
lrs_status lrs_conv_debug_trace(lrs_conv *h, void *dev_buf);

/* ------------------------------------------------------------------------------------------
 * Backward pass: the gradients that fine-tuning the decomposed layer by
 * "ordinary back-propagation with respect to the original loss" needs (PAPER.md:194-195
 * §3.5; §5.5 fine-tunes each decomposed layer with SGD).  The trainable
 * parameters are the factors of L and the VALUES of S at its fixed support (the support is
 * chosen by the projection P_c).  Given dY = dLoss/dY:
 *
 *   dX                      the adjoint convolution of dY with W = L + S
 *                           (dX[n, ho*s+y-p, wo*s+x-p, c] += sum_j dY[n,ho,wo,j] W[c,j,y,x])
 *   dU_in [c_in][rank_in]   = X^T dT1          dT1 = adjoint of conv(., G) at dT2
 *   dG [rank_in][rank_out][kernel_h][kernel_w] = weight gradient of conv(T1, G) at dT2
 *   dU_out [rank_out][c_out] = T2^T dY         dT2 = dY U_out^T
 *   dvalues [nnz]           dvalues[e] = sum over output positions of dY[., j_e] X[shift_e(.), c_e]
 *   (SVD pair: dU = X^T (dY V^T), dV = (X U)^T dY.)
 * oracle/lrs_backward.py writes both formulations out.
 *
 * Engines:
 *   - dX is the FORWARD of the transposed layer (u_in' = U_out^T, core'[b][a][y][x] =
 *     G[a][b][kh-1-y][kw-1-x], u_out' = U_in^T, S' = S by input channel with flipped
 *     taps, pad' = kernel-1-pad, stride 1; on the zero-inserted dY at stride > 1), created inside the backward handle through
 *     lrs_conv_create: the same fused tensor-core kernels (2:4 sparse term included).
 *   - T1, T2 (recomputed from X), dT2 and dT1 run on the library's tcgen05 GEMM engine.
 *   - the four weight-gradient reductions over positions run as ONE grouped tcgen05
 *     launch with MN-major operands (lrs_wgrad.cuh); S's value gradient is the dense
 *     weight gradient of the taps at S's support (every 128 x 256 output tile holds
 *     nonzeros at 1-5 % uniform density, so skipping tiles saves nothing), summed over
 *     the K splits in a fixed order (deterministic: the same inputs give the same bits).
 *   Intermediates T1, T2, dT2, dT1 are bf16 (like the forward's); accumulation is fp32.
 *
 * Stride s > 1: the two adjoint convolutions (dX, dT1) run on zero-inserted gradients
 * (dY_up[n][ho*s][wo*s] = dY[n][ho][wo], extent (out-1) s + 1 + ((in + 2p - k) mod s)) through
 * the same stride-1 transposed layer; the shifted weight-gradient operands are TMA boxes
 * sampled every s positions.
 * The paper's CP core kind runs as its Tucker-2 embedding (diagonal core G[a][a][y][x] =
 * B[y][a] C[x][a], bf16) and folds dG into the CP factor gradients: d_core = [dB (kernel_h x R);
 * dC (kernel_w x R)] (the core array's layout), d_u_in = dA, d_u_out = dD^T.
 * Requirements: dtype BF16, stride <= 4, no
 * fused output epilogue (out_scale / out_bias / out_relu: back-propagate through them in
 * the caller), every forward requirement of the layer and of its transposed layer, and
 * rows of at most 128 positions (in_w <= 128); else LRS_ERR_UNSUPPORTED.
 */
typedef struct lrs_conv_bwd lrs_conv_bwd; /* opaque */

/* Parameter gradients, device fp32, overwritten (not accumulated).  Any pointer may be
   NULL to skip that output (its reduction is still computed when another needs it).    */
typedef struct lrs_conv_grads {
  float *d_u_in;   /* [c_in][rank_in]                                      */
  float *d_core;   /* [rank_in][rank_out][kernel_h][kernel_w] (CP kind: [kernel_h + kernel_w][R];
                      NULL for an SVD pair)                                                    */
  float *d_u_out;  /* [rank_out][c_out]                                    */
  float *d_values; /* [nnz], in the order of the descriptor's CSR entries  */
} lrs_conv_grads;

/* Create the backward state of a layer from the SAME descriptor as its forward (host
   arrays, deep-copied).  Owns the transposed layer, the recompute scratch (T1, T2, dT2,
   dT1 for batch_max images) and the K-split partial-sum slabs.  Errors as lrs_conv_create. */
lrs_status lrs_conv_bwd_create(const lrs_conv_desc *desc, int device, lrs_conv_bwd **out);

/* dX for n images: dy device [n][out_h][out_w][c_out] bf16 -> dx device
   [n][in_h][in_w][c_in] bf16 (overwritten).  Enqueued on `stream`; graph-capturable;
   no host sync.  n == 0: no-op.  n > batch_max, NULL or misaligned pointers:
   INVALID_ARGUMENT. */
lrs_status lrs_conv_backward_data(lrs_conv_bwd *h, const void *dy, void *dx, int32_t n, void *stream);

/* Parameter gradients for n images: x device [n][in_h][in_w][c_in] (the forward's input),
   dy as above, g->* device fp32 (overwritten).  Enqueued on `stream`; graph-capturable.
   The handle's scratch holds one call at a time: calls on one handle are stream-ordered. */
lrs_status lrs_conv_backward_weights(lrs_conv_bwd *h, const void *x, const void *dy, int32_t n,
                                     const lrs_conv_grads *g, void *stream);

/* Both at once: dX, then the parameter gradients with dT1 taken from the transposed layer's
   forward (its intermediate) instead of recomputed, and the recompute GEMMs (T1, T2, dT2) on
   the handle's internal side stream concurrently with that forward (fork / join events on
   `stream`: graph-capturable) -- one GEMM launch fewer than the two calls above (an SVD pair: when that forward keeps T1 in device memory); dX is identical,
   the gradients equal up to the fp32 summation order of dT1. */
lrs_status lrs_conv_backward(lrs_conv_bwd *h, const void *x, const void *dy, void *dx, int32_t n,
                             const lrs_conv_grads *g, void *stream);

/* Kernel launches of one backward_weights call (the recompute GEMMs, the grouped weight
   gradient, the split reduction); of backward_data (lrs_conv_launches_per_forward of the
   transposed layer) and of one lrs_conv_backward call, if the pointers are non-NULL. */
int32_t lrs_conv_bwd_launches(const lrs_conv_bwd *h, int32_t *data_launches, int32_t *combined_launches);

/* Stage timing of the backward (as lrs_conv_set_timing / lrs_conv_stage_times): stages
   0-5 bwd_t1, bwd_t2, bwd_dt2, bwd_dt1, wgrad, wgrad_reduce (backward_weights), 6-9 the
   transposed layer's forward stages (backward_data, names prefixed "dx_"). */
lrs_status lrs_conv_bwd_set_timing(lrs_conv_bwd *h, int32_t enable);
lrs_status lrs_conv_bwd_stage_times(lrs_conv_bwd *h, float *ms, int64_t *counts, int32_t max_stages,
                                    int32_t *n_stages, int32_t reset);
const char *lrs_conv_bwd_stage_name(const lrs_conv_bwd *h, int32_t stage);

lrs_status lrs_conv_bwd_destroy(lrs_conv_bwd *h); /* NULL-safe; no call may be in flight */

/* ------------------------------------------------------------------------------------------
 * Decomposition: the offline side of the method, W ~ L + S with L of CP rank
 * r (L_ijkt = A_ir B_jr C_kr D_tr) and S of fixed cardinality c, by the paper's
 * two-step iteration:  L_i = update(L_{i-1}, W - S_{i-1});  S_i = P_c(W - L_i)
 * with update = one alternating-least-squares sweep over the four factors (SPEC.md:151-158:
 * F_n = mttkrp(W - S, F, n) (*_{m != n} F_m^T F_m)^+, pseudo-inverse with a relative eigenvalue
 * cutoff rcond) and P_c = the n = round(c * numel) entries of largest |value|, ties to the
 * smaller linear index.  eps_i = ||W - L_i - S_i||_F / ||W||_F; the run stops
 * when eps improves by less than tol (after the first iteration) or after max_iters.
 * oracle/lrs_decomp.py writes the same algorithm out step by step.
 *
 * W: device fp64 [dims[0]][dims[1]][dims[2]][dims[3]] row-major (a conv weight (in, out, kh, kw):
 * F0 = u_in, F1 = u_out^T, F2 / F3 = the CP core kind's B / C, see LRS_CORE_CP).  Every step
 * runs in fp64 CUDA kernels (lrs_decomp.cuh): MTTKRP as split reductions added in a fixed order,
 * the R x R pseudo-inverse by a one-CTA parallel-ordering Jacobi eigensolver, the projection
 * by an exact radix select over the fp64 bit patterns of |W - L| plus an index-ordered
 * compaction -- deterministic: the same inputs give the same bits.
 * Requirements: dims > 0, dims[2], dims[3] <= 8, numel < 2^31, 1 <= rank <= 256,
 * 0 <= cardinality < 1, max_iters >= 1, rcond >= 0.
 */
typedef struct lrs_decomp_params {
  int32_t dims[4];     /* I0..I3 of W                                            */
  int32_t rank;        /* CP rank r                                              */
  double cardinality;  /* c: S keeps round(c * numel) entries (half to even)     */
  int32_t max_iters;   /* >= 1                                                   */
  double tol;          /* stop when eps_{i-1} - eps_i < tol (i >= 1)             */
  double rcond;        /* pseudo-inverse cutoff relative to the largest eigenvalue (SPEC: 1e-10) */
} lrs_decomp_params;

typedef struct lrs_decomp lrs_decomp; /* opaque: fp64 workspace for one W shape */

lrs_status lrs_decomp_create(const lrs_decomp_params *p, int device, lrs_decomp **out);

/* Run the iteration from the initial factors f0..f3 (device fp64 [dims[m]][rank], e.g. the
   leading singular vectors of the mode unfoldings, or random), which are
   overwritten with the result.  S: s_idx (device int64, linear indices ascending) and
   s_val (device fp64), capacity round(c * numel) (lrs_decomp_nnz); *s_count = entries
   written.  eps_hist: host [max_iters]; *iters_done = iterations run.  Enqueued on `stream`
   and synchronised once per iteration (the stopping rule runs on the host): NOT
   graph-capturable.  A zero W gives zero factors, an empty S and eps 0. */
lrs_status lrs_decomp_run(lrs_decomp *h, const double *w, double *f0, double *f1, double *f2, double *f3,
                          int64_t *s_idx, double *s_val, int64_t *s_count, double *eps_hist,
                          int32_t *iters_done, void *stream);
int64_t lrs_decomp_nnz(const lrs_decomp *h); /* round(c * numel) */
int32_t lrs_decomp_launches_per_iteration(const lrs_decomp *h); /* kernel launches per iteration */
/* stage timing: 0 MTTKRP (+ partial sums), 1 pseudo-inverse + factor update + Gram,
   2 residual W - L, 3 projection P_c + T = W - S + eps */
lrs_status lrs_decomp_set_timing(lrs_decomp *h, int32_t enable);
lrs_status lrs_decomp_stage_times(lrs_decomp *h, float *ms, int64_t *counts, int32_t max_stages,
                                  int32_t *n_stages, int32_t reset);
lrs_status lrs_decomp_destroy(lrs_decomp *h); /* NULL-safe */

/* ------------------------------------------------------------------------------------------
 * Tucker-2 decomposition (SURVEY §8(f) f4 "Alternating Tucker-2/CP-ALS on W - S"): the same
 * two-step iteration with L in the forward's primary form, Tucker-2 over the
 * channel modes -- L[c][j][y][x] = sum_{a,b} U_in[c][a] G[a][b][y][x] U_out[j][b] (PAPER.md:409,
 * §7: Tucker decomposition "might be extended to low rank and sparse form"; the north star's L is
 * this Tucker-2 form, SURVEY.md §1 note 2).  update = one higher-order orthogonal
 * iteration (HOOI) sweep on T = W - S: U_in <- `inner` subspace-iteration steps
 * orth(Z1 Z1^T U_in) on Z1 = T x_out U_out^T unfolded [Cin][R2 kh kw], then U_out likewise on
 * Z2 = T x_in U_in^T, then G = T x_in U_in^T x_out U_out^T; orth(Y) = Cholesky-QR Y L^-T
 * (Y^T Y = L L^T) while every pivot exceeds rcond * max_i (Y^T Y)_ii, else Y (Y^T Y)^-1/2 (Loewdin,
 * eigenvalues under rcond * the largest dropped).  P_c, eps and the stopping rule as
 * lrs_decomp_run.  oracle/lrs_decomp.py decompose_lrs_tucker2 writes the algorithm out; every step
 * runs in fp64 CUDA kernels (a strided batched fp64 GEMM for the mode products, the one-CTA
 * blocked Cholesky (Jacobi for the fallback), the radix-select projection), deterministic.
 * Requirements: as lrs_decomp_params with rank = max(r1, r2); 1 <= r1 <= dims[0], 1 <= r2 <= dims[1],
 * inner >= 1.
 */
typedef struct lrs_tucker2_params {
  int32_t dims[4];     /* Cin, Cout, kh, kw of W[c][j][y][x]                     */
  int32_t r1, r2;      /* channel ranks (U_in [Cin][r1], U_out [Cout][r2])       */
  double cardinality;  /* c: S keeps round(c * numel) entries (half to even)     */
  int32_t max_iters;   /* >= 1                                                   */
  double tol;          /* stop when eps_{i-1} - eps_i < tol (i >= 1)             */
  double rcond;        /* orth: Cholesky pivot floor / Loewdin eigenvalue cutoff (relative) */
  int32_t inner;       /* subspace-iteration steps per factor per sweep (>= 1)   */
} lrs_tucker2_params;

typedef struct lrs_tucker2 lrs_tucker2; /* opaque: fp64 workspace for one W shape */

lrs_status lrs_tucker2_create(const lrs_tucker2_params *p, int device, lrs_tucker2 **out);

/* Run from the initial factors u_in (device fp64 [Cin][r1]) and u_out (device fp64 [Cout][r2]:
   COLUMNS are the basis, i.e. the layer's u_out transposed), overwritten with the orthonormal
   result; core: device fp64 [r1][r2][kh][kw] (out).  S, eps_hist, iters_done, stream: as
   lrs_decomp_run (synchronised once per iteration, not graph-capturable).  A zero W gives zero
   factors and core, an empty S and eps 0. */
lrs_status lrs_tucker2_run(lrs_tucker2 *h, const double *w, double *u_in, double *u_out, double *core,
                           int64_t *s_idx, double *s_val, int64_t *s_count, double *eps_hist,
                           int32_t *iters_done, void *stream);
int64_t lrs_tucker2_nnz(const lrs_tucker2 *h); /* round(c * numel) */
/* stage timing: 0 mode products (Z1, Z2, G), 1 subspace steps + orth, 2 residual W - L,
   3 projection P_c + T = W - S + eps */
lrs_status lrs_tucker2_set_timing(lrs_tucker2 *h, int32_t enable);
lrs_status lrs_tucker2_stage_times(lrs_tucker2 *h, float *ms, int64_t *counts, int32_t max_stages,
                                   int32_t *n_stages, int32_t reset);
lrs_status lrs_tucker2_destroy(lrs_tucker2 *h); /* NULL-safe */

#ifdef __cplusplus
}
#endif
#endif /* LRS_CONV_H_ */
