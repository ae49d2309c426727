"""Thin ctypes binding of the C-ABI in include/lrs_conv.h.

Argument marshalling only: every step of the compressed convolution runs in
the CUDA kernels of liblrs_conv.so.  PyTorch is used for device memory and
streams.  There is no CPU fallback: if the shared library is missing or the
device is not an sm_100 GPU, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liblrs_conv.so")

LRS_OK, LRS_ERR_INVALID_ARGUMENT, LRS_ERR_UNSUPPORTED, LRS_ERR_OUT_OF_MEMORY, LRS_ERR_CUDA = range(5)
LRS_DTYPE_F32, LRS_DTYPE_BF16 = 0, 1
LRS_CORE_TUCKER2, LRS_CORE_CP = 0, 1
STATUS_NAMES = {0: "LRS_OK", 1: "LRS_ERR_INVALID_ARGUMENT", 2: "LRS_ERR_UNSUPPORTED",
                3: "LRS_ERR_OUT_OF_MEMORY", 4: "LRS_ERR_CUDA"}

#: every symbol include/lrs_conv.h declares
EXPORTED = ("lrs_conv_create", "lrs_conv_forward", "lrs_conv_forward_host", "lrs_conv_destroy",
            "lrs_conv_last_error", "lrs_conv_output_shape", "lrs_conv_launches_per_forward",
            "lrs_conv_set_timing", "lrs_conv_stage_times", "lrs_conv_stage_name",
            "lrs_conv_debug_buffer", "lrs_conv_debug_trace", "lrs_conv_sparse_engine", "lrs_conv_core_fused",
            "lrs_conv_expand_kernel",
            "lrs_conv_overflow_chunks",
            "lrs_conv_cta_pairs",
            "lrs_sparse_from_slices",
            "lrs_conv_bwd_create", "lrs_conv_backward_data", "lrs_conv_backward_weights", "lrs_conv_backward",
            "lrs_conv_bwd_launches", "lrs_conv_bwd_destroy", "lrs_conv_bwd_set_timing",
            "lrs_conv_bwd_stage_times", "lrs_conv_bwd_stage_name",
            "lrs_decomp_create", "lrs_decomp_run", "lrs_decomp_nnz", "lrs_decomp_launches_per_iteration", "lrs_decomp_set_timing",
            "lrs_decomp_stage_times", "lrs_decomp_destroy",
            "lrs_tucker2_create", "lrs_tucker2_run", "lrs_tucker2_nnz", "lrs_tucker2_set_timing",
            "lrs_tucker2_stage_times", "lrs_tucker2_destroy")


class LrsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class lrs_conv_desc(ctypes.Structure):
    _fields_ = [
        ("batch_max", ctypes.c_int32), ("in_h", ctypes.c_int32), ("in_w", ctypes.c_int32),
        ("c_in", ctypes.c_int32), ("c_out", ctypes.c_int32),
        ("kernel_h", ctypes.c_int32), ("kernel_w", ctypes.c_int32),
        ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32),
        ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
        ("rank_in", ctypes.c_int32), ("rank_out", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("u_in", ctypes.c_void_p), ("core", ctypes.c_void_p), ("u_out", ctypes.c_void_p),
        ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.POINTER(ctypes.c_int64)),
        ("col_idx", ctypes.POINTER(ctypes.c_int32)),
        ("values", ctypes.POINTER(ctypes.c_float)),
        ("core_kind", ctypes.c_int32),
        ("out_scale", ctypes.POINTER(ctypes.c_float)),
        ("out_bias", ctypes.POINTER(ctypes.c_float)),
        ("out_relu", ctypes.c_int32),
    ]


class lrs_decomp_params(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int32 * 4), ("rank", ctypes.c_int32), ("cardinality", ctypes.c_double),
                ("max_iters", ctypes.c_int32), ("tol", ctypes.c_double), ("rcond", ctypes.c_double)]


class lrs_tucker2_params(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int32 * 4), ("r1", ctypes.c_int32), ("r2", ctypes.c_int32),
                ("cardinality", ctypes.c_double), ("max_iters", ctypes.c_int32), ("tol", ctypes.c_double),
                ("rcond", ctypes.c_double), ("inner", ctypes.c_int32)]


class lrs_conv_grads(ctypes.Structure):
    _fields_ = [("d_u_in", ctypes.c_void_p), ("d_core", ctypes.c_void_p), ("d_u_out", ctypes.c_void_p),
                ("d_values", ctypes.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load liblrs_conv.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_2006_06443_b200._build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.lrs_conv_create.argtypes = [ctypes.POINTER(lrs_conv_desc), ctypes.c_int, ctypes.POINTER(P)]
    lib.lrs_conv_forward.argtypes = [P, P, P, ctypes.c_int32, P]
    lib.lrs_conv_forward_host.argtypes = [P, P, P, ctypes.c_int32, P]
    lib.lrs_conv_destroy.argtypes = [P]
    lib.lrs_conv_last_error.restype = ctypes.c_char_p
    lib.lrs_conv_output_shape.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    lib.lrs_conv_launches_per_forward.argtypes = [P]
    lib.lrs_conv_launches_per_forward.restype = ctypes.c_int32
    lib.lrs_conv_set_timing.argtypes = [P, ctypes.c_int32]
    lib.lrs_conv_stage_times.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64),
                                         ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]
    lib.lrs_conv_stage_name.argtypes = [P, ctypes.c_int32]
    lib.lrs_conv_stage_name.restype = ctypes.c_char_p
    lib.lrs_conv_debug_buffer.argtypes = [P, ctypes.c_int32, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_int32)]
    lib.lrs_conv_debug_trace.argtypes = [P, P]
    lib.lrs_conv_sparse_engine.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    lib.lrs_conv_sparse_engine.restype = ctypes.c_int32
    lib.lrs_conv_core_fused.argtypes = [P]
    lib.lrs_conv_core_fused.restype = ctypes.c_int32
    lib.lrs_conv_expand_kernel.argtypes = [P]
    lib.lrs_conv_expand_kernel.restype = ctypes.c_int32
    lib.lrs_conv_overflow_chunks.argtypes = [P]
    lib.lrs_conv_overflow_chunks.restype = ctypes.c_int32
    lib.lrs_conv_cta_pairs.argtypes = [P]
    lib.lrs_conv_cta_pairs.restype = ctypes.c_int32
    lib.lrs_sparse_from_slices.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.POINTER(ctypes.c_int64), P, ctypes.c_int32,
                                           ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64),
                                           ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float)]
    lib.lrs_sparse_from_slices.restype = ctypes.c_int
    lib.lrs_conv_bwd_create.argtypes = [ctypes.POINTER(lrs_conv_desc), ctypes.c_int, ctypes.POINTER(P)]
    lib.lrs_conv_backward_data.argtypes = [P, P, P, ctypes.c_int32, P]
    lib.lrs_conv_backward_weights.argtypes = [P, P, P, ctypes.c_int32, ctypes.POINTER(lrs_conv_grads), P]
    lib.lrs_conv_backward.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.POINTER(lrs_conv_grads), P]
    lib.lrs_conv_bwd_launches.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    lib.lrs_conv_bwd_launches.restype = ctypes.c_int32
    lib.lrs_conv_bwd_destroy.argtypes = [P]
    lib.lrs_conv_bwd_set_timing.argtypes = [P, ctypes.c_int32]
    lib.lrs_conv_bwd_stage_times.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64),
                                             ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]
    lib.lrs_conv_bwd_stage_name.argtypes = [P, ctypes.c_int32]
    lib.lrs_conv_bwd_stage_name.restype = ctypes.c_char_p
    for name in ("lrs_conv_bwd_create", "lrs_conv_backward_data", "lrs_conv_backward_weights", "lrs_conv_backward",
                 "lrs_conv_bwd_destroy", "lrs_conv_bwd_set_timing", "lrs_conv_bwd_stage_times"):
        getattr(lib, name).restype = ctypes.c_int
    lib.lrs_decomp_create.argtypes = [ctypes.POINTER(lrs_decomp_params), ctypes.c_int, ctypes.POINTER(P)]
    lib.lrs_decomp_run.argtypes = [P, P, P, P, P, P, P, P, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), P]
    lib.lrs_decomp_nnz.argtypes = [P]
    lib.lrs_decomp_nnz.restype = ctypes.c_int64
    lib.lrs_decomp_launches_per_iteration.argtypes = [P]
    lib.lrs_decomp_launches_per_iteration.restype = ctypes.c_int32
    lib.lrs_decomp_set_timing.argtypes = [P, ctypes.c_int32]
    lib.lrs_decomp_stage_times.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64),
                                           ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]
    lib.lrs_decomp_destroy.argtypes = [P]
    for name in ("lrs_decomp_create", "lrs_decomp_run", "lrs_decomp_set_timing", "lrs_decomp_stage_times",
                 "lrs_decomp_destroy"):
        getattr(lib, name).restype = ctypes.c_int
    lib.lrs_tucker2_create.argtypes = [ctypes.POINTER(lrs_tucker2_params), ctypes.c_int, ctypes.POINTER(P)]
    lib.lrs_tucker2_run.argtypes = [P, P, P, P, P, P, P, ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), P]
    lib.lrs_tucker2_nnz.argtypes = [P]
    lib.lrs_tucker2_nnz.restype = ctypes.c_int64
    lib.lrs_tucker2_set_timing.argtypes = [P, ctypes.c_int32]
    lib.lrs_tucker2_stage_times.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64),
                                            ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]
    lib.lrs_tucker2_destroy.argtypes = [P]
    for name in ("lrs_tucker2_create", "lrs_tucker2_run", "lrs_tucker2_set_timing", "lrs_tucker2_stage_times",
                 "lrs_tucker2_destroy"):
        getattr(lib, name).restype = ctypes.c_int
    for name in ("lrs_conv_debug_trace", "lrs_conv_create", "lrs_conv_forward", "lrs_conv_forward_host", "lrs_conv_destroy",
                 "lrs_conv_output_shape", "lrs_conv_set_timing", "lrs_conv_stage_times",
                 "lrs_conv_debug_buffer", "lrs_conv_debug_trace", "lrs_conv_sparse_engine"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(st: int):
    if st != LRS_OK:
        raise LrsError(st, load_library().lrs_conv_last_error().decode())


# ---------------------------------------------------------------- C-ABI names
def lrs_conv_create(desc: lrs_conv_desc, device: int = 0) -> int:
    h = ctypes.c_void_p()
    _check(load_library().lrs_conv_create(ctypes.byref(desc), device, ctypes.byref(h)))
    return h.value


def lrs_conv_forward(handle: int, x_ptr: int, y_ptr: int, n: int, stream: int = 0) -> None:
    _check(load_library().lrs_conv_forward(handle, x_ptr, y_ptr, n, stream))


def lrs_conv_forward_host(handle: int, x_ptr: int, y_ptr: int, n: int, stream: int = 0) -> None:
    _check(load_library().lrs_conv_forward_host(handle, x_ptr, y_ptr, n, stream))


def lrs_conv_destroy(handle: int) -> None:
    _check(load_library().lrs_conv_destroy(handle))


def lrs_conv_last_error() -> str:
    return load_library().lrs_conv_last_error().decode()


def bf16_bits_rne(a) -> np.ndarray:
    """uint16 bf16 bit patterns of float32 values, round-to-nearest-even
    (ties to the even mantissa); NaN stays a quiet NaN.  Exact for values
    that are already bf16-representable."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(a)
    if nan.any():
        r[nan] = 0x7FC0
    return np.ascontiguousarray(r)


def make_desc(batch_max: int, in_h: int, in_w: int, c_in: int, c_out: int, kernel: int,
              stride: int, pad: int, rank_in: int, rank_out: int, dtype: str,
              u_in: np.ndarray, core: Optional[np.ndarray], u_out: np.ndarray,
              row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, core_kind: int = LRS_CORE_TUCKER2,
              out_scale: Optional[np.ndarray] = None, out_bias: Optional[np.ndarray] = None, out_relu: bool = False):
    """Build an lrs_conv_desc from host arrays.  Factor arrays are float32; for
    bf16 layers they are rounded to bf16 round-to-nearest-even (bf16_bits_rne)
    and those bits are passed.  S values are passed as fp32 (the ABI's
    contract; a bf16 layer's engine rounds them itself).
    Returns (desc, keepalive) -- keep `keepalive` until lrs_conv_create returns."""
    def as_dtype(a):
        a = np.ascontiguousarray(a, np.float32)
        if dtype == "bf16":
            return bf16_bits_rne(a)
        return a
    keep = []

    def ptr(a):
        keep.append(a)
        return a.ctypes.data_as(ctypes.c_void_p)
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int32)
    va = np.ascontiguousarray(values, np.float32)
    keep += [rp, ci, va]
    d = lrs_conv_desc(
        batch_max=batch_max, in_h=in_h, in_w=in_w, c_in=c_in, c_out=c_out,
        kernel_h=kernel, kernel_w=kernel, stride_h=stride, stride_w=stride, pad_h=pad, pad_w=pad,
        rank_in=rank_in, rank_out=rank_out,
        dtype=LRS_DTYPE_BF16 if dtype == "bf16" else LRS_DTYPE_F32,
        u_in=ptr(as_dtype(u_in)), core=None if core is None else ptr(as_dtype(core)),
        u_out=ptr(as_dtype(u_out)), nnz=len(va),
        row_ptr=rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        col_idx=ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        values=va.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), core_kind=core_kind, out_relu=1 if out_relu else 0)
    for name, arr in (("out_scale", out_scale), ("out_bias", out_bias)):
        if arr is not None:
            a = np.ascontiguousarray(arr, np.float32)
            keep.append(a)
            setattr(d, name, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    return d, keep


def sparse_from_slices(c_in: int, c_out: int, kernel_h: int, kernel_w: int, vals, packed):
    """The paper's per-input-channel (values, packed index) slices -> CSR, through
    the C-ABI's host converter lrs_sparse_from_slices (include/lrs_conv.h).
    vals/packed: lists of c_in arrays (packed uint16 or uint32).  Returns
    (row_ptr int64 [c_out+1], col_idx int32 [nnz], values float32 [nnz])."""
    lib = load_library()
    lens = [len(v) for v in vals]
    sp = np.zeros(c_in + 1, np.int64)
    sp[1:] = np.cumsum(lens)
    nnz = int(sp[-1])
    width = 4 if any(np.asarray(p).dtype.itemsize == 4 for p in packed) else 2
    pk = np.ascontiguousarray(np.concatenate([np.asarray(p) for p in packed]) if nnz else np.zeros(1),
                              np.uint32 if width == 4 else np.uint16)
    va = np.ascontiguousarray(np.concatenate([np.asarray(v, np.float32) for v in vals]) if nnz else np.zeros(1),
                              np.float32)
    rp = np.zeros(c_out + 1, np.int64)
    ci = np.zeros(max(nnz, 1), np.int32)
    vo = np.zeros(max(nnz, 1), np.float32)
    _check(lib.lrs_sparse_from_slices(c_in, c_out, kernel_h, kernel_w,
                                      sp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                      pk.ctypes.data_as(ctypes.c_void_p), width,
                                      va.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                      rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                      ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                      vo.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
    return rp, ci[:nnz], vo[:nnz]


class LrsConv:
    """One compressed conv layer on one device: `LrsConv(...)(x) -> y`
    with x, y NHWC torch tensors (contiguous [n, H, W, C], or channels_last
    NCHW views of NHWC storage; checked by forward_into)."""

    def __init__(self, batch_max, in_h, in_w, c_in, c_out, kernel, stride, pad, rank_in, rank_out,
                 dtype, u_in, core, u_out, row_ptr, col_idx, values, device: int = 0,
                 core_kind: int = LRS_CORE_TUCKER2, out_scale=None, out_bias=None, out_relu: bool = False):
        import torch
        self.torch = torch
        self.dtype = dtype
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.device = device
        self.c_out = c_out
        desc, keep = make_desc(batch_max, in_h, in_w, c_in, c_out, kernel, stride, pad, rank_in,
                               rank_out, dtype, u_in, core, u_out, row_ptr, col_idx, values, core_kind,
                               out_scale, out_bias, out_relu)
        self.handle = lrs_conv_create(desc, device)
        del keep
        oh, ow = ctypes.c_int32(), ctypes.c_int32()
        _check(load_library().lrs_conv_output_shape(self.handle, ctypes.byref(oh), ctypes.byref(ow)))
        self.out_h, self.out_w = oh.value, ow.value
        self.batch_max, self.in_h, self.in_w, self.c_in = batch_max, in_h, in_w, c_in

    @classmethod
    def from_inputs(cls, inp, batch_max: Optional[int] = None, device: int = 0, out_scale=None, out_bias=None,
                    out_relu: bool = False) -> "LrsConv":
        c = inp.cfg
        return cls(batch_max or (inp.x.shape[0] if inp.x is not None else c.batch), c.in_h, c.in_w, c.c_in, c.c_out,
                   c.k, c.stride, c.pad, c.rank_in, c.rank_out, c.dtype, inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                   inp.col_idx, inp.values, device, out_scale=out_scale, out_bias=out_bias, out_relu=out_relu)

    @classmethod
    def from_cp(cls, batch_max: int, in_h: int, in_w: int, kernel: int, stride: int, pad: int, dtype: str,
                a, b, c, d, row_ptr, col_idx, values, device: int = 0) -> "LrsConv":
        """The paper's CP form L = A_ir B_kr C_pr D_jr: a [c_in][R],
        b [k][R] (taps along H), c [k][R] (taps along W), d [c_out][R]."""
        a, b, c, d = (np.asarray(t, np.float32) for t in (a, b, c, d))
        r = a.shape[1]
        core = np.concatenate([b, c], axis=0)  # [2k][R]: B then C
        return cls(batch_max, in_h, in_w, a.shape[0], d.shape[0], kernel, stride, pad, r, r, dtype,
                   a, core, np.ascontiguousarray(d.T), row_ptr, col_idx, values, device, core_kind=LRS_CORE_CP)

    @property
    def launches_per_forward(self) -> int:
        return load_library().lrs_conv_launches_per_forward(self.handle)

    @property
    def sparse_engine(self):
        """(engine, main_blocks, residual_blocks): engine 1 = 2:4 sparse tensor
        cores, 0 = SIMT CSR epilogue (see include/lrs_conv.h)."""
        m, r = ctypes.c_int32(), ctypes.c_int32()
        e = load_library().lrs_conv_sparse_engine(self.handle, ctypes.byref(m), ctypes.byref(r))
        return int(e), int(m.value), int(r.value)

    @property
    def expand_kernel(self) -> int:
        """0 GEMM / SIMT, 1 windowed tensor-core kernel, 2 channel-stationary 1x1 kernel
        (lrs_conv_expand_kernel, include/lrs_conv.h)."""
        return int(load_library().lrs_conv_expand_kernel(self.handle))

    @property
    def cta_pairs(self) -> bool:
        """True if the windowed kernel runs in its CTA-pair (cta_group::2) form
        (lrs_conv_cta_pairs, include/lrs_conv.h)."""
        return load_library().lrs_conv_cta_pairs(self.handle) == 1

    @property
    def overflow_chunks(self) -> int:
        """Overflow-gather chunks per M-tile of the windowed kernel, 0 if it uses residual
        2:4 blocks (lrs_conv_overflow_chunks, include/lrs_conv.h)."""
        return int(load_library().lrs_conv_overflow_chunks(self.handle))

    @property
    def core_fused(self) -> bool:
        """True if a1 + a2 run as one kernel with T1 kept on chip (include/lrs_conv.h)."""
        return load_library().lrs_conv_core_fused(self.handle) == 1

    def _check_act(self, t, name: str, h: int, w: int, c: int) -> None:
        """t must be this layer's dtype, on its device, with NHWC storage: either a
        contiguous [n, h, w, c] tensor or a channels_last [n, c, h, w] view."""
        torch = self.torch
        if t.dtype != self.tdtype:
            raise ValueError(f"{name}: dtype {t.dtype}, layer expects {self.tdtype}")
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{name}: must live on cuda:{self.device}, got {t.device}")
        if t.dim() != 4:
            raise ValueError(f"{name}: expected a 4-D tensor, got shape {tuple(t.shape)}")
        if tuple(t.shape[1:]) == (h, w, c) and t.is_contiguous():
            return
        if tuple(t.shape[1:]) == (c, h, w) and t.is_contiguous(memory_format=torch.channels_last):
            return
        raise ValueError(f"{name}: expected contiguous NHWC [n, {h}, {w}, {c}] or channels_last NCHW "
                         f"[n, {c}, {h}, {w}], got shape {tuple(t.shape)} strides {t.stride()}")

    def forward_into(self, x, y, stream=None) -> None:
        """y = layer(x) on `stream`; x / y are NHWC [n, H, W, C] contiguous tensors
        or channels_last NCHW views of the same storage (validated here)."""
        torch = self.torch
        self._check_act(x, "x", self.in_h, self.in_w, self.c_in)
        self._check_act(y, "y", self.out_h, self.out_w, self.c_out)
        n = x.shape[0]
        if y.shape[0] != n:
            raise ValueError(f"x has {n} images but y has {y.shape[0]}")
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        lrs_conv_forward(self.handle, x.data_ptr(), y.data_ptr(), n, s.cuda_stream)

    def __call__(self, x):
        """y = layer(x): x NHWC [n, H, W, C] (contiguous) -> new NHWC y; a
        channels_last NCHW x gives a channels_last NCHW y."""
        torch = self.torch
        self._check_act(x, "x", self.in_h, self.in_w, self.c_in)
        n = x.shape[0]
        if tuple(x.shape[1:]) == (self.in_h, self.in_w, self.c_in) and x.is_contiguous():
            y = torch.empty((n, self.out_h, self.out_w, self.c_out), dtype=self.tdtype, device=x.device)
        else:
            y = torch.empty((n, self.c_out, self.out_h, self.out_w), dtype=self.tdtype, device=x.device,
                            memory_format=torch.channels_last)
        self.forward_into(x, y)
        return y

    def forward_host(self, x_host, y_host, stream=None) -> None:
        """x_host / y_host: pinned CPU tensors; enqueued on `stream`."""
        torch = self.torch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        lrs_conv_forward_host(self.handle, x_host.data_ptr(), y_host.data_ptr(), x_host.shape[0], s.cuda_stream)

    def set_timing(self, on: bool) -> None:
        _check(load_library().lrs_conv_set_timing(self.handle, 1 if on else 0))

    def stage_times(self, reset: bool = True):
        """{stage name: (total ms, launches)} of event-timed kernels since the last reset."""
        ms = (ctypes.c_float * 8)()
        cnt = (ctypes.c_int64 * 8)()
        ns = ctypes.c_int32()
        lib = load_library()
        _check(lib.lrs_conv_stage_times(self.handle, ms, cnt, 8, ctypes.byref(ns), 1 if reset else 0))
        return {lib.lrs_conv_stage_name(self.handle, i).decode(): (ms[i], cnt[i]) for i in range(ns.value)}

    def debug_buffer(self, which: int, rows: int):
        """Intermediate T1 (which=0) / T2 (which=1) of the last forward as a torch tensor view copy."""
        torch = self.torch
        p = ctypes.c_void_p()
        ld = ctypes.c_int32()
        _check(load_library().lrs_conv_debug_buffer(self.handle, which, ctypes.byref(p), ctypes.byref(ld)))
        esz = 2 if self.dtype == "bf16" else 4
        nbytes = rows * ld.value * esz
        buf = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        torch.cuda.synchronize(self.device)
        cudart_memcpy(buf.data_ptr(), p.value, nbytes)
        return buf.view(self.tdtype).view(rows, ld.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            lrs_conv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lrs_conv_bwd_create(desc: lrs_conv_desc, device: int = 0) -> int:
    h = ctypes.c_void_p()
    _check(load_library().lrs_conv_bwd_create(ctypes.byref(desc), device, ctypes.byref(h)))
    return h.value


def lrs_conv_backward_data(handle: int, dy_ptr: int, dx_ptr: int, n: int, stream: int = 0) -> None:
    _check(load_library().lrs_conv_backward_data(handle, dy_ptr, dx_ptr, n, stream))


def lrs_conv_backward_weights(handle: int, x_ptr: int, dy_ptr: int, n: int, grads: lrs_conv_grads,
                              stream: int = 0) -> None:
    _check(load_library().lrs_conv_backward_weights(handle, x_ptr, dy_ptr, n, ctypes.byref(grads), stream))


def lrs_conv_backward(handle: int, x_ptr: int, dy_ptr: int, dx_ptr: int, n: int, grads: lrs_conv_grads,
                      stream: int = 0) -> None:
    _check(load_library().lrs_conv_backward(handle, x_ptr, dy_ptr, dx_ptr, n, ctypes.byref(grads), stream))


def lrs_conv_bwd_destroy(handle: int) -> None:
    _check(load_library().lrs_conv_bwd_destroy(handle))


class LrsConvBackward:
    """The backward pass of one compressed layer (include/lrs_conv.h "Backward pass";
    PAPER.md:194-195 fine-tuning by back-propagation): built from the same arguments as
    LrsConv.  `backward_data(dy) -> dx` and `backward_weights(x, dy) -> dict` of fp32
    gradients {d_u_in, d_core, d_u_out, d_values}; tensors NHWC bf16 on the device."""

    def __init__(self, batch_max, in_h, in_w, c_in, c_out, kernel, stride, pad, rank_in, rank_out,
                 dtype, u_in, core, u_out, row_ptr, col_idx, values, device: int = 0,
                 core_kind: int = LRS_CORE_TUCKER2):
        import torch
        self.torch = torch
        self.device = device
        self.svd = core is None
        self.cp = core is not None and core_kind == LRS_CORE_CP
        self.in_h, self.in_w, self.c_in, self.c_out = in_h, in_w, c_in, c_out
        self.out_h = (in_h + 2 * pad - kernel) // stride + 1
        self.out_w = (in_w + 2 * pad - kernel) // stride + 1
        self.kernel, self.rank_in = kernel, rank_in
        self.rank_out = rank_in if core is None else rank_out
        self.nnz = len(values)
        desc, keep = make_desc(batch_max, in_h, in_w, c_in, c_out, kernel, stride, pad, rank_in, rank_out,
                               dtype, u_in, core, u_out, row_ptr, col_idx, values, core_kind)
        self.handle = lrs_conv_bwd_create(desc, device)
        del keep

    @classmethod
    def from_cp(cls, batch_max: int, in_h: int, in_w: int, kernel: int, stride: int, pad: int, dtype: str,
                a, b, c, d, row_ptr, col_idx, values, device: int = 0) -> "LrsConvBackward":
        """The backward of the paper's CP layer (LrsConv.from_cp's arguments):
        d_u_in = dA [c_in][R], d_u_out = dD^T [R][c_out], d_core = [dB (k x R); dC (k x R)]."""
        a, b, c, d = (np.asarray(t, np.float32) for t in (a, b, c, d))
        r = a.shape[1]
        core = np.concatenate([b, c], axis=0)
        return cls(batch_max, in_h, in_w, a.shape[0], d.shape[0], kernel, stride, pad, r, r, dtype,
                   a, core, np.ascontiguousarray(d.T), row_ptr, col_idx, values, device, core_kind=LRS_CORE_CP)

    @classmethod
    def from_inputs(cls, inp, batch_max: Optional[int] = None, device: int = 0) -> "LrsConvBackward":
        c = inp.cfg
        return cls(batch_max or c.batch, c.in_h, c.in_w, c.c_in, c.c_out, c.k, c.stride, c.pad, c.rank_in,
                   c.rank_out, c.dtype, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values,
                   device)

    def _check(self, t, name, h, w, c):
        if t.dtype != self.torch.bfloat16 or not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{name}: expected a bf16 tensor on cuda:{self.device}")
        if t.dim() != 4 or tuple(t.shape[1:]) != (h, w, c) or not t.is_contiguous():
            raise ValueError(f"{name}: expected contiguous NHWC [n, {h}, {w}, {c}], got {tuple(t.shape)}")

    def alloc_grads(self):
        torch = self.torch
        dev = f"cuda:{self.device}"
        g = {"d_u_in": torch.empty((self.c_in, self.rank_in), dtype=torch.float32, device=dev),
             "d_core": None if self.svd else (
                 torch.empty((2 * self.kernel, self.rank_in), dtype=torch.float32, device=dev) if self.cp else
                 torch.empty((self.rank_in, self.rank_out, self.kernel, self.kernel), dtype=torch.float32, device=dev)),
             "d_u_out": torch.empty((self.rank_out, self.c_out), dtype=torch.float32, device=dev),
             "d_values": torch.empty((max(self.nnz, 1),), dtype=torch.float32, device=dev)[:self.nnz]}
        return g

    def backward_data_into(self, dy, dx, stream=None) -> None:
        self._check(dy, "dy", self.out_h, self.out_w, self.c_out)
        self._check(dx, "dx", self.in_h, self.in_w, self.c_in)
        if dx.shape[0] != dy.shape[0]:
            raise ValueError("dx / dy image counts differ")
        s = self.torch.cuda.current_stream(self.device) if stream is None else stream
        lrs_conv_backward_data(self.handle, dy.data_ptr(), dx.data_ptr(), dy.shape[0], s.cuda_stream)

    def backward_data(self, dy):
        dx = self.torch.empty((dy.shape[0], self.in_h, self.in_w, self.c_in), dtype=self.torch.bfloat16,
                              device=dy.device)
        self.backward_data_into(dy, dx)
        return dx

    def _grads_struct(self, grads: dict):
        sizes = {"d_u_in": self.c_in * self.rank_in, "d_u_out": self.rank_out * self.c_out,
                 "d_core": 0 if self.svd else (2 * self.kernel * self.rank_in if self.cp else
                                               self.rank_in * self.rank_out * self.kernel ** 2),
                 "d_values": self.nnz}
        ptrs = {}
        for k, numel in sizes.items():
            t = grads.get(k)
            if t is None or numel == 0:
                ptrs[k] = None
                continue
            if t.dtype != self.torch.float32 or not t.is_contiguous() or t.numel() != numel or not t.is_cuda:
                raise ValueError(f"{k}: expected a contiguous fp32 CUDA tensor of {numel} elements")
            ptrs[k] = t.data_ptr()
        return lrs_conv_grads(**ptrs)

    def backward_weights_into(self, x, dy, grads: dict, stream=None) -> None:
        self._check(x, "x", self.in_h, self.in_w, self.c_in)
        self._check(dy, "dy", self.out_h, self.out_w, self.c_out)
        if x.shape[0] != dy.shape[0]:
            raise ValueError("x / dy image counts differ")
        g = self._grads_struct(grads)
        s = self.torch.cuda.current_stream(self.device) if stream is None else stream
        lrs_conv_backward_weights(self.handle, x.data_ptr(), dy.data_ptr(), x.shape[0], g, s.cuda_stream)

    def backward_into(self, x, dy, dx, grads: dict, stream=None) -> None:
        """dX and the parameter gradients in one call (lrs_conv_backward: dT1 reused from
        the transposed layer's forward)."""
        self._check(x, "x", self.in_h, self.in_w, self.c_in)
        self._check(dy, "dy", self.out_h, self.out_w, self.c_out)
        self._check(dx, "dx", self.in_h, self.in_w, self.c_in)
        if not (x.shape[0] == dy.shape[0] == dx.shape[0]):
            raise ValueError("x / dy / dx image counts differ")
        g = self._grads_struct(grads)
        s = self.torch.cuda.current_stream(self.device) if stream is None else stream
        lrs_conv_backward(self.handle, x.data_ptr(), dy.data_ptr(), dx.data_ptr(), x.shape[0], g, s.cuda_stream)

    def backward(self, x, dy):
        """(dx, gradients) of one batch."""
        dx = self.torch.empty_like(x)
        g = self.alloc_grads()
        self.backward_into(x, dy, dx, g)
        return dx, g

    def backward_weights(self, x, dy) -> dict:
        g = self.alloc_grads()
        self.backward_weights_into(x, dy, g)
        return g

    def set_timing(self, on: bool) -> None:
        _check(load_library().lrs_conv_bwd_set_timing(self.handle, 1 if on else 0))

    def stage_times(self, reset: bool = True):
        """{stage name: (total ms, launches)} of event-timed backward kernels since the last reset."""
        ms = (ctypes.c_float * 10)()
        cnt = (ctypes.c_int64 * 10)()
        ns = ctypes.c_int32()
        lib = load_library()
        _check(lib.lrs_conv_bwd_stage_times(self.handle, ms, cnt, 10, ctypes.byref(ns), 1 if reset else 0))
        return {lib.lrs_conv_bwd_stage_name(self.handle, i).decode(): (ms[i], cnt[i]) for i in range(ns.value)
                if cnt[i]}

    @property
    def launches(self):
        """(backward_weights launches, backward_data launches, backward (combined) launches)"""
        d, c = ctypes.c_int32(), ctypes.c_int32()
        w = load_library().lrs_conv_bwd_launches(self.handle, ctypes.byref(d), ctypes.byref(c))
        return int(w), int(d.value), int(c.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            lrs_conv_bwd_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LrsDecomp:
    """The low-rank + sparse decomposition W ~ L + S on the GPU (include/lrs_conv.h
    "Decomposition"): CP rank `rank`, S of cardinality c, by the paper's
    two-step iteration.  run(w, factors) takes W as a device fp64 tensor [I0, I1, I2, I3] and
    the initial factors (device fp64 [I_m, rank]; overwritten with the result) and returns
    (s_idx int64, s_val fp64 device tensors, eps history list)."""

    STAGES = ("mttkrp", "pinv_update", "residual", "project")

    def __init__(self, dims, rank: int, cardinality: float, max_iters: int = 100, tol: float = 1e-6,
                 rcond: float = 1e-10, device: int = 0):
        import torch
        self.torch = torch
        self.dims = tuple(int(d) for d in dims)
        self.rank, self.max_iters, self.device = int(rank), int(max_iters), device
        prm = lrs_decomp_params(dims=(ctypes.c_int32 * 4)(*self.dims), rank=self.rank, cardinality=float(cardinality),
                                max_iters=self.max_iters, tol=float(tol), rcond=float(rcond))
        h = ctypes.c_void_p()
        _check(load_library().lrs_decomp_create(ctypes.byref(prm), device, ctypes.byref(h)))
        self.handle = h.value
        self.nnz = int(load_library().lrs_decomp_nnz(self.handle))
        self.launches_per_iteration = int(load_library().lrs_decomp_launches_per_iteration(self.handle))

    def run(self, w, factors, stream=None):
        torch = self.torch
        if w.dtype != torch.float64 or not w.is_cuda or tuple(w.shape) != self.dims or not w.is_contiguous():
            raise ValueError(f"w: expected a contiguous fp64 CUDA tensor of shape {self.dims}")
        for m, f in enumerate(factors):
            if f.dtype != torch.float64 or not f.is_cuda or tuple(f.shape) != (self.dims[m], self.rank) or \
                    not f.is_contiguous():
                raise ValueError(f"factor {m}: expected a contiguous fp64 CUDA tensor [{self.dims[m]}, {self.rank}]")
        dev = w.device
        idx = torch.empty(max(self.nnz, 1), dtype=torch.int64, device=dev)
        val = torch.empty(max(self.nnz, 1), dtype=torch.float64, device=dev)
        eps = (ctypes.c_double * self.max_iters)()
        cnt = ctypes.c_int64()
        its = ctypes.c_int32()
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        _check(load_library().lrs_decomp_run(self.handle, w.data_ptr(), *(f.data_ptr() for f in factors),
                                             idx.data_ptr(), val.data_ptr(), ctypes.byref(cnt), eps, ctypes.byref(its),
                                             s.cuda_stream))
        return idx[:cnt.value], val[:cnt.value], [eps[i] for i in range(its.value)]

    def set_timing(self, on: bool) -> None:
        _check(load_library().lrs_decomp_set_timing(self.handle, 1 if on else 0))

    def stage_times(self, reset: bool = True):
        ms = (ctypes.c_float * 4)()
        cnt = (ctypes.c_int64 * 4)()
        ns = ctypes.c_int32()
        _check(load_library().lrs_decomp_stage_times(self.handle, ms, cnt, 4, ctypes.byref(ns), 1 if reset else 0))
        return {self.STAGES[i]: (ms[i], cnt[i]) for i in range(ns.value)}

    def close(self) -> None:
        if getattr(self, "handle", None):
            _check(load_library().lrs_decomp_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LrsTucker2Decomp:
    """The low-rank + sparse decomposition with L in Tucker-2 form on the GPU (include/lrs_conv.h
    "Tucker-2 decomposition"): run(w, u_in, u_out) takes W (device fp64 [Cin, Cout, kh, kw]) and
    the initial channel bases (device fp64 [Cin, r1] / [Cout, r2]; overwritten with the
    orthonormal result) and returns (core [r1, r2, kh, kw], s_idx, s_val, eps history).  The
    layer's u_out is the returned u_out transposed."""

    STAGES = ("mode_products", "subspace_orth", "residual", "project")

    def __init__(self, dims, r1: int, r2: int, cardinality: float, max_iters: int = 100, tol: float = 1e-6,
                 rcond: float = 1e-10, inner: int = 1, device: int = 0):
        import torch
        self.torch = torch
        self.dims = tuple(int(d) for d in dims)
        self.r1, self.r2, self.max_iters, self.device = int(r1), int(r2), int(max_iters), device
        prm = lrs_tucker2_params(dims=(ctypes.c_int32 * 4)(*self.dims), r1=self.r1, r2=self.r2,
                                 cardinality=float(cardinality), max_iters=self.max_iters, tol=float(tol),
                                 rcond=float(rcond), inner=int(inner))
        h = ctypes.c_void_p()
        _check(load_library().lrs_tucker2_create(ctypes.byref(prm), device, ctypes.byref(h)))
        self.handle = h.value
        self.nnz = int(load_library().lrs_tucker2_nnz(self.handle))

    def run(self, w, u_in, u_out, stream=None):
        torch = self.torch

        def check(t, shape, name):
            if t.dtype != torch.float64 or not t.is_cuda or tuple(t.shape) != shape or not t.is_contiguous():
                raise ValueError(f"{name}: expected a contiguous fp64 CUDA tensor of shape {shape}")
        check(w, self.dims, "w")
        check(u_in, (self.dims[0], self.r1), "u_in")
        check(u_out, (self.dims[1], self.r2), "u_out")
        dev = w.device
        core = torch.empty((self.r1, self.r2) + self.dims[2:], dtype=torch.float64, device=dev)
        idx = torch.empty(max(self.nnz, 1), dtype=torch.int64, device=dev)
        val = torch.empty(max(self.nnz, 1), dtype=torch.float64, device=dev)
        eps = (ctypes.c_double * self.max_iters)()
        cnt = ctypes.c_int64()
        its = ctypes.c_int32()
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        _check(load_library().lrs_tucker2_run(self.handle, w.data_ptr(), u_in.data_ptr(), u_out.data_ptr(),
                                              core.data_ptr(), idx.data_ptr(), val.data_ptr(), ctypes.byref(cnt), eps,
                                              ctypes.byref(its), s.cuda_stream))
        return core, idx[:cnt.value], val[:cnt.value], [eps[i] for i in range(its.value)]

    def set_timing(self, on: bool) -> None:
        _check(load_library().lrs_tucker2_set_timing(self.handle, 1 if on else 0))

    def stage_times(self, reset: bool = True):
        ms = (ctypes.c_float * 4)()
        cnt = (ctypes.c_int64 * 4)()
        ns = ctypes.c_int32()
        _check(load_library().lrs_tucker2_stage_times(self.handle, ms, cnt, 4, ctypes.byref(ns), 1 if reset else 0))
        return {self.STAGES[i]: (ms[i], cnt[i]) for i in range(ns.value)}

    def close(self) -> None:
        if getattr(self, "handle", None):
            _check(load_library().lrs_tucker2_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cudart_memcpy(dst: int, src: int, nbytes: int) -> None:
    """device->device copy through torch (used only by the debug hook)."""
    import torch
    s = torch.cuda.current_stream()
    _cudart = ctypes.CDLL("libcudart.so.12") if not hasattr(cudart_memcpy, "_lib") else cudart_memcpy._lib
    cudart_memcpy._lib = _cudart
    _cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    r = _cudart.cudaMemcpyAsync(dst, src, nbytes, 3, s.cuda_stream)
    if r != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed {r}")
    torch.cuda.synchronize()
