"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/lrs_conv.h declares, and create() rejects malformed or
unsupported descriptors with the documented status (validation runs before
any device call), while a well-formed descriptor on a GPU-less host fails
loudly with LRS_ERR_CUDA (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2006_06443_b200 as P
from paper_2006_06443_b200 import lrs_conv as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "lrs_conv.h")).read()
    return sorted(set(re.findall(r"^\s*(?:lrs_status|const char \*|int32_t|int64_t)\s*\**\s*(lrs_(?:conv|sparse|decomp|tucker2)_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = P.load_library()
    names = header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(B.EXPORTED)


def base_desc_args(**over):
    rng = np.random.default_rng(0)
    a = dict(batch_max=2, in_h=8, in_w=8, c_in=16, c_out=16, kernel=3, stride=1, pad=1,
             rank_in=4, rank_out=4, dtype="bf16",
             u_in=rng.standard_normal((16, 4)).astype(np.float32),
             core=rng.standard_normal((4, 4, 3, 3)).astype(np.float32),
             u_out=rng.standard_normal((4, 16)).astype(np.float32),
             row_ptr=np.r_[0, np.full(16, 1).cumsum()].astype(np.int64),
             col_idx=np.arange(16, dtype=np.int32) * 9 + 4, values=np.ones(16, np.float32))
    a.update(over)
    return a


def create_status(**over):
    a = base_desc_args(**over)
    d, keep = B.make_desc(**a)
    for k, v in over.pop("_patch", {}).items() if "_patch" in over else []:
        setattr(d, k, v)
    lib = P.load_library()
    h = ctypes.c_void_p()
    st = lib.lrs_conv_create(ctypes.byref(d), 0, ctypes.byref(h))
    if st == 0:
        lib.lrs_conv_destroy(h)
    return st, lib.lrs_conv_last_error().decode()


def patched_status(**fields):
    d, keep = B.make_desc(**base_desc_args())
    for k, v in fields.items():
        setattr(d, k, v)
    lib = P.load_library()
    h = ctypes.c_void_p()
    st = lib.lrs_conv_create(ctypes.byref(d), 0, ctypes.byref(h))
    return st, lib.lrs_conv_last_error().decode()


@pytest.mark.parametrize("fields", [
    dict(batch_max=0), dict(in_h=0), dict(c_out=-1), dict(rank_in=0),
    dict(stride_h=0), dict(pad_w=-1), dict(kernel_h=20),  # output extent < 1
    dict(dtype=7), dict(nnz=-1), dict(core_kind=5),
])
def test_invalid_descriptors(fields):
    st, msg = patched_status(**fields)
    assert st == B.LRS_ERR_INVALID_ARGUMENT, (st, msg)
    assert msg


def test_invalid_csr():
    rp = np.r_[0, np.full(16, 1).cumsum()].astype(np.int64)
    st, _ = create_status(row_ptr=rp[::-1].copy())
    assert st == B.LRS_ERR_INVALID_ARGUMENT
    st, _ = create_status(col_idx=np.full(16, 16 * 9, np.int32))  # col out of range
    assert st == B.LRS_ERR_INVALID_ARGUMENT
    rp2 = np.zeros(17, np.int64)
    rp2[1:] = 16
    st, msg = create_status(row_ptr=rp2, col_idx=np.r_[np.arange(15, dtype=np.int32), 3])  # unsorted/dup
    assert st == B.LRS_ERR_INVALID_ARGUMENT and "increasing" in msg


def test_svd_pair_requires_1x1():
    st, msg = create_status(core=None)
    assert st == B.LRS_ERR_INVALID_ARGUMENT and "SVD" in msg
    st, msg = create_status(core=None, kernel=1, pad=0, rank_out=5,
                            col_idx=np.arange(16, dtype=np.int32))
    assert st == B.LRS_ERR_INVALID_ARGUMENT and "rank_in == rank_out" in msg


@pytest.mark.parametrize("over,needle", [
    (dict(c_in=12, u_in=np.zeros((12, 4), np.float32), col_idx=np.arange(16, dtype=np.int32)), "multiples"),
    (dict(rank_in=300, u_in=np.zeros((16, 300), np.float32), core=np.zeros((300, 4, 3, 3), np.float32)), "rank"),
])
def test_unsupported_descriptors(over, needle):
    st, msg = create_status(**over)
    assert st == B.LRS_ERR_UNSUPPORTED and needle in msg


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, msg = create_status()
    assert st == B.LRS_ERR_CUDA and "no CUDA device" in msg


def test_product_package_does_not_import_oracle():
    """The CUDA path and the oracle share no code (only workloads/ feeds both)."""
    pkg = os.path.join(ROOT, "paper_2006_06443_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2006_06443_b200" not in src and "from paper_2006_06443_b200" not in src, f


def test_cp_core_requires_core_and_equal_ranks():
    """LRS_CORE_CP (include/lrs_conv.h): R = rank_in = rank_out and a core array."""
    st, msg = patched_status(core_kind=1, rank_out=3)
    assert st == B.LRS_ERR_INVALID_ARGUMENT and "CP" in msg
    st, msg = patched_status(core_kind=1, core=None)
    assert st == B.LRS_ERR_INVALID_ARGUMENT and "CP" in msg


def test_binding_rounds_factors_to_nearest_even():
    """make_desc's fp32 -> bf16 conversion is round-to-nearest-even (ties to even),
    matching torch's own fp32 -> bf16 cast bit for bit, including ties, subnormals,
    infinities and values that round up into the next binade; NaN stays NaN."""
    import torch
    rng = np.random.default_rng(5)
    a = (rng.standard_normal(100000) * np.exp(rng.uniform(-60, 60, 100000))).astype(np.float32)
    ties = (np.arange(0, 65536, dtype=np.uint32) << 16 | 0x8000).view(np.float32)  # exact halfway points
    special = np.array([0.0, -0.0, 1e-40, -1e-40, np.inf, -np.inf, 3.3895314e38, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9],
                       np.float32)
    v = np.concatenate([a, ties[np.isfinite(ties)], special])
    got = B.bf16_bits_rne(v)
    want = torch.from_numpy(v).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, want)
    nan = B.bf16_bits_rne(np.array([np.nan], np.float32))[0]
    assert (nan & 0x7F80) == 0x7F80 and (nan & 0x7F) != 0
    # and it is what make_desc hands to the ABI for a bf16 layer
    args = base_desc_args()
    args["u_in"] = args["u_in"] + np.float32(1e-3)
    d, keep = B.make_desc(**args)
    u = np.ctypeslib.as_array(ctypes.cast(d.u_in, ctypes.POINTER(ctypes.c_uint16)), shape=(16 * 4,))
    assert np.array_equal(u, B.bf16_bits_rne(args["u_in"]).ravel())


def test_wide_rows_need_a_bf16_tensor_core_layer():
    """Output rows wider than 128 are refused before any device call for fp32 layers and
    for c_in % 64 != 0 (their engines tile whole rows of <= 128 outputs); > 256 always."""
    for over in (dict(dtype="f32", in_w=200), dict(in_w=200), dict(in_w=300, c_in=64)):
        args = base_desc_args(**{k: v for k, v in over.items() if k in ("dtype", "in_w")})
        if "c_in" in over:
            rng = np.random.default_rng(1)
            args["c_in"] = 64
            args["u_in"] = rng.standard_normal((64, 4)).astype(np.float32)
            args["col_idx"] = np.zeros(16, np.int32)
        d, keep = B.make_desc(**args)
        h = ctypes.c_void_p()
        st = P.load_library().lrs_conv_create(ctypes.byref(d), 0, ctypes.byref(h))
        assert st == B.LRS_ERR_UNSUPPORTED, (over, st)


def bwd_status(**over):
    d, keep = B.make_desc(**base_desc_args(**over))
    lib = P.load_library()
    h = ctypes.c_void_p()
    st = lib.lrs_conv_bwd_create(ctypes.byref(d), 0, ctypes.byref(h))
    if st == 0:
        lib.lrs_conv_bwd_destroy(h)
    return st, lib.lrs_conv_last_error().decode()


def test_backward_create_validation_before_any_device_call():
    """The backward's documented refusals (include/lrs_conv.h "Backward pass") come before
    any device call; a well-formed layer on this GPU-less host is LRS_ERR_CUDA."""
    assert bwd_status(stride=5)[0] == B.LRS_ERR_UNSUPPORTED
    assert bwd_status(dtype="f32", u_in=base_desc_args()["u_in"])[0] == B.LRS_ERR_UNSUPPORTED
    assert bwd_status(batch_max=0)[0] == B.LRS_ERR_INVALID_ARGUMENT
    st, msg = bwd_status()
    assert st == B.LRS_ERR_CUDA and "no CPU fallback" in msg


def test_decomp_create_validation_before_any_device_call():
    lib = P.load_library()

    def status(**kw):
        a = dict(dims=(8, 8, 3, 3), rank=4, cardinality=0.01, max_iters=5, tol=1e-6, rcond=1e-10)
        a.update(kw)
        prm = B.lrs_decomp_params(dims=(ctypes.c_int32 * 4)(*a["dims"]), rank=a["rank"], cardinality=a["cardinality"],
                                  max_iters=a["max_iters"], tol=a["tol"], rcond=a["rcond"])
        h = ctypes.c_void_p()
        return lib.lrs_decomp_create(ctypes.byref(prm), 0, ctypes.byref(h))

    assert status(rank=0) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(dims=(8, 0, 3, 3)) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(cardinality=1.0) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(max_iters=0) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(rank=257) == B.LRS_ERR_UNSUPPORTED
    assert status(dims=(8, 8, 9, 3)) == B.LRS_ERR_UNSUPPORTED
    assert status() == B.LRS_ERR_CUDA


def test_tucker2_create_validation_before_any_device_call():
    lib = P.load_library()

    def status(**kw):
        a = dict(dims=(8, 8, 3, 3), r1=4, r2=3, cardinality=0.01, max_iters=5, tol=1e-6, rcond=1e-10, inner=1)
        a.update(kw)
        prm = B.lrs_tucker2_params(dims=(ctypes.c_int32 * 4)(*a["dims"]), r1=a["r1"], r2=a["r2"],
                                   cardinality=a["cardinality"], max_iters=a["max_iters"], tol=a["tol"],
                                   rcond=a["rcond"], inner=a["inner"])
        h = ctypes.c_void_p()
        return lib.lrs_tucker2_create(ctypes.byref(prm), 0, ctypes.byref(h))

    assert status(r1=0) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(r2=9) == B.LRS_ERR_INVALID_ARGUMENT  # r2 > Cout
    assert status(inner=0) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(cardinality=-0.1) == B.LRS_ERR_INVALID_ARGUMENT
    assert status(dims=(300, 300, 3, 3), r1=257, r2=4) == B.LRS_ERR_UNSUPPORTED
    assert status() == B.LRS_ERR_CUDA
    assert lib.lrs_tucker2_destroy(None) == B.LRS_OK
