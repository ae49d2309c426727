"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the
same seeded inputs (workloads/), element by element.

Tolerances (BASELINE.json north star): fp32 path relL2 <= 1e-5 and
max-abs <= 1e-4; bf16 path relL2 <= 2e-2.  Exactness checks (bitwise) where
the arithmetic fixes the result: single-nonzero sparse term, power-of-two
scaling, determinism, empty terms.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O
import parity

pytestmark = pytest.mark.gpu


def lrs():
    from paper_2006_06443_b200 import LrsConv
    return LrsConv


def tdt(dtype):
    return torch.bfloat16 if dtype == "bf16" else torch.float32


def run(inp, x=None, batch_max=None):
    layer = lrs().from_inputs(inp, batch_max=batch_max)
    xx = torch.from_numpy(inp.x if x is None else x).to(tdt(inp.cfg.dtype)).cuda()
    y = layer(xx)
    torch.cuda.synchronize()
    return layer, xx, y


def oracle(inp, x=None):
    c = inp.cfg
    return O.forward_factored((inp.x if x is None else x).astype(np.float64), inp.u_in, inp.core, inp.u_out,
                              inp.row_ptr, inp.col_idx, inp.values, c.stride, c.pad)


def check(y_gpu, y_ref, dtype):
    """whole tensor + per image / 128-channel block / border row (tests/parity.py)"""
    return parity.check(y_gpu, y_ref, dtype)


# small batches that still span several 128-pixel tiles and a ragged tail
SMALL = [("c1", 1), ("c2_f32", 3), ("c2_bf16", 3), ("c3", 5), ("c4", 3)]


@pytest.mark.parametrize("name,batch", SMALL)
def test_config_small_batch_vs_oracle(name, batch):
    inp = workloads.generate(workloads.CONFIGS[name], batch=batch)
    _, _, y = run(inp)
    check(y, oracle(inp), inp.cfg.dtype)


@pytest.mark.parametrize("name", ["c1", "c2_f32", "c2_bf16", "c3", "c4"])
def test_config_full_size_vs_oracle(name):
    """BASELINE.json full sizes, in the launch configuration bench.py times."""
    inp = workloads.generate(workloads.CONFIGS[name])
    _, _, y = run(inp)
    check(y, oracle(inp), inp.cfg.dtype)


GEOMS = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density, dtype, svd)
    (2, 14, 14, 32, 48, 3, 2, 1, 12, 20, 0.05, "bf16", False),   # stride 2, ragged ranks
    (3, 9, 11, 16, 72, 3, 1, 1, 8, 8, 0.03, "bf16", False),      # Cout not a multiple of BN
    (2, 10, 10, 24, 40, 3, 1, 0, 16, 16, 0.04, "f32", False),    # pad 0
    (1, 28, 28, 32, 32, 3, 2, 1, 8, 8, 0.02, "f32", False),      # stride 2 fp32
    (5, 6, 6, 64, 64, 1, 1, 0, 32, 32, 0.02, "bf16", True),      # SVD, tiles spanning images
    (2, 12, 12, 16, 16, 5, 1, 2, 16, 16, 0.05, "bf16", False),   # 5x5
    (300, 7, 7, 16, 16, 3, 1, 1, 16, 16, 0.05, "bf16", False),   # many images per tile
    (2, 14, 14, 64, 64, 3, 2, 1, 48, 32, 0.03, "bf16", False),   # stride 2 (two kernels), R1 = 48: K chunks per tap
    (2, 10, 10, 16, 32, 3, 1, 1, 40, 24, 0.03, "f32", False),    # fp32, R1 = 40 -> 48 (192 B per tap)
]


@pytest.mark.parametrize("geom", GEOMS)
def test_geometries_vs_oracle(geom):
    n, h, w, cin, cout, k, s, p, r1, r2, dens, dtype, svd = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r1, r1 if svd else r2, dens, dtype, svd, seed=7)
    inp = workloads.generate(cfg)
    _, _, y = run(inp)
    check(y, oracle(inp), dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_empty_sparse_and_zero_lowrank(dtype):
    """S = {} -> Y equals the L path; U_out = 0 -> Y equals the S path
    (SPEC.md:292-293), each against the oracle of that single term."""
    cfg = workloads.CONFIGS["c2_f32" if dtype == "f32" else "c2_bf16"]
    inp = workloads.generate(cfg, batch=2)
    inp_l = workloads.LayerInputs(cfg, inp.x, inp.u_in, inp.core, inp.u_out,
                                  np.zeros(cfg.c_out + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    _, _, y = run(inp_l)
    check(y, oracle(inp_l), dtype)
    inp_s = workloads.LayerInputs(cfg, inp.x, inp.u_in, inp.core, np.zeros_like(inp.u_out),
                                  inp.row_ptr, inp.col_idx, inp.values)
    _, _, y = run(inp_s)
    check(y, oracle(inp_s), dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_single_nonzero_is_bitwise(dtype):
    """One sparse entry (j, c, y, x, v), U_out = 0: Y[..., j] = fl(v * X[shifted, c])
    exactly (one rounding), all other channels exactly 0."""
    n, h, w, cin, cout, k = 2, 9, 9, 16, 16, 3
    rng = np.random.default_rng(3)
    x = workloads.bf16_round(np.maximum(rng.standard_normal((n, h, w, cin)), 0).astype(np.float32))
    j, c, ty, tx, v = 5, 7, 0, 2, np.float32(0.3)
    rp = np.zeros(cout + 1, np.int64)
    rp[j + 1:] = 1
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, 1, 1, 16, 16, 0.0, dtype)
    inp = workloads.LayerInputs(cfg, x, np.ones((cin, 16), np.float32), np.ones((16, 16, k, k), np.float32),
                                np.zeros((16, cout), np.float32), rp, np.array([(c * k + ty) * k + tx], np.int32),
                                np.array([v], np.float32))
    _, _, y = run(inp)
    yg = y.float().cpu().numpy()
    xp = np.zeros((n, h + 2, w + 2, cin), np.float32)
    xp[:, 1:-1, 1:-1] = x
    ref = np.zeros((n, h, w, cout), np.float32)
    ref[..., j] = v * xp[:, ty:ty + h, tx:tx + w, c]
    if dtype == "bf16":
        ref = workloads.bf16_round(ref)
    assert np.array_equal(yg, ref)


@pytest.mark.parametrize("name", ["c2_f32", "c3"])
def test_power_of_two_scaling_and_determinism(name):
    inp = workloads.generate(workloads.CONFIGS[name], batch=3)
    layer, x, y1 = run(inp)
    y2 = layer(x)
    y3 = layer(2 * x)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(y3, 2 * y1)


def test_identity_chain_is_exact():
    """U_in = I, centre-tap identity core, U_out = I, S = {} -> Y = X bitwise."""
    for dtype in ("bf16", "f32"):
        c = 32
        rng = np.random.default_rng(4)
        x = workloads.bf16_round(rng.standard_normal((2, 8, 8, c)).astype(np.float32))
        core = np.zeros((c, c, 3, 3), np.float32)
        core[np.arange(c), np.arange(c), 1, 1] = 1
        cfg = workloads.LayerConfig("t", 2, 8, 8, c, c, 3, 1, 1, c, c, 0.0, dtype)
        inp = workloads.LayerInputs(cfg, x, np.eye(c, dtype=np.float32), core, np.eye(c, dtype=np.float32),
                                    np.zeros(c + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
        _, _, y = run(inp)
        assert np.array_equal(y.float().cpu().numpy(), x), dtype


def test_partial_batch_and_noop():
    """n < batch_max uses the first n images; n = 0 is a no-op."""
    inp = workloads.generate(workloads.CONFIGS["c2_bf16"], batch=4)
    layer = lrs().from_inputs(inp, batch_max=8)
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    y = layer(x)
    torch.cuda.synchronize()
    check(y, oracle(inp), "bf16")
    from paper_2006_06443_b200 import lrs_conv_forward
    lrs_conv_forward(layer.handle, x.data_ptr(), y.data_ptr(), 0, 0)
    from paper_2006_06443_b200 import LrsError
    with pytest.raises(LrsError):
        lrs_conv_forward(layer.handle, x.data_ptr(), y.data_ptr(), 9, 0)


def test_host_io_and_graph_capture():
    inp = workloads.generate(workloads.CONFIGS["c4"], batch=8)
    layer, x, y = run(inp)
    xh = x.cpu().pin_memory()
    yh = torch.empty(y.shape, dtype=y.dtype).pin_memory()
    layer.forward_host(xh, yh)
    torch.cuda.synchronize()
    assert torch.equal(yh, y.cpu())
    y2 = torch.empty_like(y)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        layer.forward_into(x, y2, stream=s)  # warm
        torch.cuda.synchronize()
        y2.zero_()
        with torch.cuda.graph(g, stream=s):
            layer.forward_into(x, y2, stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y2, y)


@pytest.mark.parametrize("name,batch", [("c2_bf16", 64), ("c2_bf16", 37), ("c2_f32", 20), ("c3", 24)])
def test_host_io_pipelined_chunks_bitwise(name, batch):
    """lrs_conv_forward_host splits the batch into up to 4 chunks of >= 8 images
    (copy in / compute / copy out overlapped on two handle streams); the result is
    bitwise the device forward's, on a non-default caller stream, twice in a row."""
    inp = workloads.generate(workloads.CONFIGS[name], batch=batch)
    layer, x, y = run(inp)
    xh = x.cpu().pin_memory()
    s = torch.cuda.Stream()
    for _ in range(2):
        yh = torch.full(y.shape, -7.0, dtype=y.dtype).pin_memory()
        with torch.cuda.stream(s):
            layer.forward_host(xh, yh, stream=s)
        s.synchronize()
        assert torch.equal(yh, y.cpu())


EDGE = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density, dtype)  -- the ABI's limits
    (2, 16, 16, 64, 64, 7, 1, 3, 32, 32, 0.02, "bf16"),     # largest kernel (7x7)
    (2, 9, 9, 64, 64, 7, 2, 3, 16, 16, 0.03, "f32"),        # 7x7, stride 2, fp32
    (3, 7, 7, 256, 256, 3, 1, 1, 256, 256, 0.02, "bf16"),   # largest ranks (256)
    (2, 5, 128, 64, 64, 3, 1, 1, 16, 16, 0.02, "bf16"),     # 128-wide rows (the GEMM core convolution's limit)
    (2, 4, 168, 64, 64, 3, 1, 1, 16, 16, 0.02, "bf16"),     # 168-wide rows (ResNet-50 layer1 at 3x input): fused core
    (1, 3, 200, 64, 128, 3, 1, 1, 32, 32, 0.03, "bf16"),    # 200-wide rows: the fused core kernel's X slots near their limit
    (1, 4, 4, 8, 8, 3, 1, 1, 4, 4, 0.5, "bf16"),            # smallest channels (8), dense-ish S
]


@pytest.mark.parametrize("geom", EDGE)
def test_edge_geometries_vs_oracle(geom):
    n, h, w, cin, cout, k, s, p, r1, r2, dens, dtype = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r1, r2, dens, dtype, seed=31)
    inp = workloads.generate(cfg)
    _, _, y = run(inp)
    check(y, oracle(inp), dtype)


def test_wide_rows_cp_and_svd_and_refusal():
    """Output rows wider than 128 (Table 4's 3x input):
    the paper's CP form (fused projection + depthwise stages) and the 1x1 SVD pair run them;
    a strided Tucker-2 layer, which needs the GEMM core convolution (whole rows of <= 128
    outputs), is refused with LRS_ERR_UNSUPPORTED -- never computed wrongly."""
    from paper_2006_06443_b200 import LrsConv, LrsError
    cfg = workloads.LayerConfig("cpw", 2, 4, 168, 64, 64, 3, 1, 1, 16, 16, 0.02, "bf16", seed=41)
    inp = workloads.generate_cp(cfg)
    layer = LrsConv.from_cp(2, 4, 168, 3, 1, 1, "bf16", inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx,
                            inp.values)
    y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    ref = O.forward_cp(inp.x.astype(np.float64), inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx, inp.values, 1, 1)
    check(y, ref, "bf16")
    svd = workloads.generate(workloads.LayerConfig("svdw", 2, 3, 168, 64, 256, 1, 1, 0, 32, 32, 0.02, "bf16",
                                                   svd=True, seed=42))
    _, _, y = run(svd)
    check(y, oracle(svd), "bf16")
    s2 = workloads.generate(workloads.LayerConfig("s2w", 1, 4, 338, 64, 64, 3, 2, 1, 16, 16, 0.02, "bf16", seed=43))
    with pytest.raises(LrsError) as e:
        run(s2)
    assert e.value.status == 2  # LRS_ERR_UNSUPPORTED
