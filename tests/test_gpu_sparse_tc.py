"""GPU parity of the 2:4 sparse tensor-core engine (lrs_wconv.cuh): the fused
a3 + a4 + a5 kernel that runs bf16 layers with c_in % 64 == 0, against the
fp64 oracle (PAPER.md:160 direct convolution of W = L + S, :189 sparse term).

The engine splits every group of 4 consecutive input channels of S into an
exact main 2:4 block plus a residual 2:4 block, builds im2col operands from a
shared-memory window whose core matrices are 8 images of one position, and
merges output rows into wide MMA units; each case below pins one of those
mechanisms (bf16 tolerance relL2 <= 2e-2, BASELINE.json north star; exact
cases bitwise).
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O
import parity

pytestmark = pytest.mark.gpu


def layer_of(inp, batch_max=None):
    from paper_2006_06443_b200 import LrsConv
    return LrsConv.from_inputs(inp, batch_max=batch_max)


def run(inp):
    layer = layer_of(inp)
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    y = layer(x)
    torch.cuda.synchronize()
    return layer, y.float().cpu().numpy().astype(np.float64)


def oracle(inp):
    c = inp.cfg
    return O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, c.stride, c.pad)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", ["c2_bf16", "c3", "c4"])
def test_configs_use_the_tensor_core_engine(name):
    inp = workloads.generate(workloads.CONFIGS[name], batch=2)
    layer = layer_of(inp)
    eng, main, res = layer.sparse_engine
    assert eng == 1 and main > 0


GEOMS = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density, svd)  -- all bf16, cin % 64 == 0
    (9, 14, 14, 64, 128, 3, 2, 1, 16, 32, 0.03, False),     # stride 2, ragged batch (9), R2 = 32 (SW64 T window)
    (10, 7, 7, 64, 200, 3, 1, 1, 32, 48, 0.05, False),      # Cout not a multiple of 128, R2 48 -> 64
    (3, 9, 9, 128, 192, 1, 1, 0, 16, 16, 0.02, True),       # SVD pair, R = 16 (SW32 T window)
    (8, 12, 12, 64, 64, 5, 1, 2, 64, 64, 0.05, False),      # 5x5: 25 taps
    (2, 40, 40, 64, 64, 3, 1, 1, 16, 16, 0.02, False),      # Wo = 40 > 32: split rows
    (8, 10, 10, 64, 128, 3, 1, 0, 32, 32, 0.02, False),     # pad 0
    (4, 28, 28, 128, 128, 3, 2, 1, 32, 32, 0.02, False),    # stride 2, 28 -> 14
    (3, 7, 7, 128, 128, 3, 1, 1, 32, 32, 0.30, False),      # dense-ish S: most groups need a residual block
    (4, 14, 14, 64, 128, 3, 1, 1, 32, 32, 0.0, False),      # empty S: no X windows, the dense MMAs start the sum
    (3, 9, 9, 128, 192, 1, 1, 0, 16, 16, 0.0, True),        # empty S, SVD pair
]


@pytest.mark.parametrize("geom", GEOMS)
def test_tensor_core_geometries_vs_oracle(geom):
    n, h, w, cin, cout, k, s, p, r1, r2, dens, svd = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r1, r1 if svd else r2, dens, "bf16", svd, seed=11)
    inp = workloads.generate(cfg)
    layer, y = run(inp)
    assert layer.sparse_engine[0] == 1
    parity.check(y, oracle(inp), "bf16")


def test_full_groups_need_residual_and_stay_exact():
    """Rows whose groups of 4 channels are completely nonzero (4 of 4) are
    split into main + residual 2:4 blocks; with U_out = 0 and a small S the
    result is the sparse conv alone, compared with the oracle (fp64)."""
    n, h, w, cin, cout, k = 8, 6, 6, 64, 128, 3
    rng = np.random.default_rng(5)
    x = workloads.bf16_round(np.maximum(rng.standard_normal((n, h, w, cin)), 0).astype(np.float32))
    rows, cols, vals = [], [], []
    for j in range(cout):
        for g in range(0, 8, 2):          # groups 0,2,4,6 of channels: full 4/4, tap depends on j
            tap = (j + g) % (k * k)
            ty, tx = divmod(tap, k)
            for c in range(4 * g, 4 * g + 4):
                rows.append(j)
                cols.append((c * k + ty) * k + tx)
                vals.append(rng.standard_normal() * 0.3)
    order = np.lexsort((cols, rows))
    rows, cols = np.array(rows)[order], np.array(cols, np.int32)[order]
    vals = workloads.bf16_round(np.array(vals, np.float32)[order])
    rp = np.zeros(cout + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, 1, 1, 16, 16, 0.0, "bf16")
    u_in = workloads.bf16_round(rng.standard_normal((cin, 16)).astype(np.float32) / 8)
    core = workloads.bf16_round(rng.standard_normal((16, 16, k, k)).astype(np.float32) / 12)
    inp = workloads.LayerInputs(cfg, x, u_in, core, np.zeros((16, cout), np.float32), rp, cols, vals)
    layer, y = run(inp)
    eng, main, res = layer.sparse_engine
    assert eng == 1 and (res > 0 or layer.overflow_chunks > 0)
    parity.check(y, oracle(inp), "bf16")


def test_single_nonzero_bitwise_tensor_core():
    """One entry (j, c, y, x, v) with v bf16-exact and U_out = 0: the tensor
    core computes v * X exactly in fp32 (one product, no other term), then one
    bf16 rounding -> bitwise equal to bf16(v * X[shifted])."""
    n, h, w, cin, cout, k = 8, 9, 9, 64, 128, 3
    rng = np.random.default_rng(3)
    x = workloads.bf16_round(np.maximum(rng.standard_normal((n, h, w, cin)), 0).astype(np.float32))
    j, c, ty, tx, v = 77, 45, 2, 0, np.float32(0.375)
    rp = np.zeros(cout + 1, np.int64)
    rp[j + 1:] = 1
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, 1, 1, 16, 16, 0.0, "bf16")
    inp = workloads.LayerInputs(cfg, x, np.ones((cin, 16), np.float32), np.ones((16, 16, k, k), np.float32),
                                np.zeros((16, cout), np.float32), rp, np.array([(c * k + ty) * k + tx], np.int32),
                                np.array([v], np.float32))
    layer, y = run(inp)
    assert layer.sparse_engine[0] == 1
    xp = np.zeros((n, h + 2, w + 2, cin), np.float32)
    xp[:, 1:-1, 1:-1] = x
    ref = np.zeros((n, h, w, cout), np.float32)
    ref[..., j] = workloads.bf16_round(v * xp[:, ty:ty + h, tx:tx + w, c])
    assert np.array_equal(y.astype(np.float32), ref)


IPW_CASES = [  # (n, h, w, cin, cout, k, p, r1, r2, density) -- stride 1 (4-image windows need it)
    (13, 7, 7, 512, 512, 3, 1, 128, 128, 0.05),   # C3 shape, ragged image groups (13 = 3 x 4 + 1)
    (6, 14, 14, 256, 256, 3, 1, 64, 64, 0.02),    # C2 shape
    (5, 12, 12, 64, 200, 5, 2, 32, 48, 0.05),     # 5x5, Cout not /128
    (9, 6, 6, 128, 128, 1, 0, 64, 64, 0.30),      # 1x1 Tucker-2 (G 1x1), dense S: residual blocks
]


@pytest.mark.parametrize("geom", IPW_CASES)
def test_four_image_windows_bitwise_equal_eight(geom):
    """The windowed kernel with 4 images per window (a core matrix = 2 positions x 4 images,
    tap offsets of 512 B) accumulates every output in the same order as with 8: bitwise
    equal, and against the oracle."""
    import os
    n, h, w, cin, cout, k, p, r1, r2, dens = geom
    cfg = workloads.LayerConfig("ipw", n, h, w, cin, cout, k, 1, p, r1, r2, dens, "bf16", seed=23)
    inp = workloads.generate(cfg)
    ys = {}
    for ipw in ("8", "4"):
        os.environ["LRS_WCONV_IPW"] = ipw
        try:
            layer = layer_of(inp)
        finally:
            os.environ.pop("LRS_WCONV_IPW", None)
        assert layer.expand_kernel == 1
        y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
        torch.cuda.synchronize()
        ys[ipw] = y
    assert torch.equal(ys["8"], ys["4"])
    parity.check(ys["4"], oracle(inp), "bf16")


GATHER_CASES = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density, ipw)
    (13, 7, 7, 512, 512, 3, 1, 1, 128, 128, 0.05, "8"),   # C3 shape, ragged image group
    (9, 14, 14, 64, 128, 3, 2, 1, 16, 32, 0.08, "8"),     # stride 2, R2 = 32 (32-slot chunks)
    (10, 7, 7, 128, 200, 3, 1, 1, 32, 48, 0.08, "8"),     # Cout not a multiple of 128 (last M-tile partial)
    (2, 40, 40, 64, 64, 3, 1, 1, 16, 16, 0.08, "8"),      # split rows (Wo 40 > 32), R2 = 16
    (5, 12, 12, 64, 200, 5, 1, 2, 32, 48, 0.06, "4"),     # 4-image windows, 5x5, padding 2
    (6, 10, 10, 128, 128, 3, 1, 0, 64, 64, 0.06, "8"),    # pad 0
]


@pytest.mark.parametrize("geom", GATHER_CASES)
def test_overflow_gather_vs_residual_blocks(geom):
    """The overflow-gather form (LRS_WCONV_GATHER=1: a group's 3rd/4th nonzero becomes a dense
    K column G[pos][slot] = X[pos + tap][c] gathered by the epilogue warps) against the
    residual-block form (=0) and the fp64 oracle, with a partial batch (n < batch_max) and a
    fused output epilogue; both forms hold every entry of S exactly, they only sum in another
    order."""
    import os
    from paper_2006_06443_b200 import LrsConv
    n, h, w, cin, cout, k, s, p, r1, r2, dens, ipw = geom
    cfg = workloads.LayerConfig("g", n, h, w, cin, cout, k, s, p, r1, r2, dens, "bf16", seed=31)
    inp = workloads.generate(cfg)
    rng = np.random.default_rng(6)
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    bias = rng.standard_normal(cout).astype(np.float32) * 0.1
    ref = O.output_epilogue(oracle(inp), scale, bias, relu=True)
    for mode in ("0", "1"):
        os.environ.update({"LRS_WCONV_GATHER": mode, "LRS_WCONV_IPW": ipw})
        try:
            layer = LrsConv.from_inputs(inp, batch_max=n + 5, out_scale=scale, out_bias=bias, out_relu=True)
        finally:
            os.environ.pop("LRS_WCONV_GATHER", None)
            os.environ.pop("LRS_WCONV_IPW", None)
        assert layer.expand_kernel == 1
        _, _, res = layer.sparse_engine
        if mode == "1":
            assert layer.overflow_chunks > 0 and res == 0
        else:
            assert layer.overflow_chunks == 0 and res > 0
        y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
        torch.cuda.synchronize()
        parity.check(y, ref, "bf16")
        # a second forward on other images: the gather scratch is rewritten, not stale
        x2 = workloads.generate_x(cfg, n, seed=77)
        y2 = layer(torch.from_numpy(x2).to(torch.bfloat16).cuda())
        torch.cuda.synchronize()
        c = inp.cfg
        ref2 = O.output_epilogue(O.forward_factored(x2.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                                                    inp.col_idx, inp.values, c.stride, c.pad), scale, bias, relu=True)
        parity.check(y2, ref2, "bf16")


def test_c3_takes_the_overflow_gather():
    """At C3 (5 % uniform S over 512 x 4608) 63 % of the (M-tile, chunk, tap) blocks have a
    group of 4 with 3+ nonzeros: the cost rule replaces those residual blocks by gather chunks."""
    inp = workloads.generate(workloads.CONFIGS["c3"], batch=2)
    layer = layer_of(inp)
    assert layer.overflow_chunks > 0 and layer.sparse_engine[2] == 0
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    y = layer(x)
    torch.cuda.synchronize()
    parity.check(y, oracle(inp), "bf16")


@pytest.mark.parametrize("name", ["c2_bf16", "c4", "c3"])
def test_simt_csr_engine_matches_oracle(name):
    """LRS_NO_SPTC=1: the same bf16 layer on engine 0 (tensor-core a3 GEMM with the SIMT CSR
    sparse term in its epilogue, no 2:4 blocks) -- the head-to-head arm of DESIGN §5 --
    against the fp64 oracle, and against the 2:4 engine within the bf16 bar."""
    import os
    from paper_2006_06443_b200 import LrsConv
    inp = workloads.generate(workloads.CONFIGS[name], batch=8)
    os.environ["LRS_NO_SPTC"] = "1"
    try:
        simt = LrsConv.from_inputs(inp, batch_max=8)
    finally:
        os.environ.pop("LRS_NO_SPTC", None)
    assert simt.sparse_engine[0] == 0 and simt.expand_kernel == 0
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    y = simt(x)
    torch.cuda.synchronize()
    parity.check(y, oracle(inp), "bf16")


PAIR_CASES = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density)
    (13, 7, 7, 512, 512, 3, 1, 1, 128, 128, 0.05),   # C3 shape: pairs of M-tiles + the pair-union gather
    (9, 14, 14, 256, 256, 3, 1, 1, 64, 64, 0.02),    # C2 shape, ragged image group
    (6, 12, 12, 128, 256, 5, 1, 2, 32, 48, 0.06),    # 5x5, padding 2, R2 48 -> 64
    (5, 9, 9, 64, 512, 3, 1, 0, 32, 32, 0.03),       # pad 0, 4 M-tiles (2 pairs)
]


def _make_env(inp, env, batch_max=None, **kw):
    import os
    from paper_2006_06443_b200 import LrsConv
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return LrsConv.from_inputs(inp, batch_max=batch_max, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("geom", PAIR_CASES)
def test_cta_pair_form_vs_oracle(geom):
    """The CTA-pair form (LRS_WCONV_PAIR=1: clusters of 2 CTAs, tcgen05.mma.cta_group::2 with
    M = 256, each SM holding half of every window along N) against the fp64 oracle, with a
    fused output epilogue, a partial batch and a second forward on other images."""
    n, h, w, cin, cout, k, s, p, r1, r2, dens = geom
    cfg = workloads.LayerConfig("pair", n, h, w, cin, cout, k, s, p, r1, r2, dens, "bf16", seed=37)
    inp = workloads.generate(cfg)
    rng = np.random.default_rng(8)
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    bias = rng.standard_normal(cout).astype(np.float32) * 0.1
    layer = _make_env(inp, {"LRS_WCONV_PAIR": "1"}, batch_max=n + 3, out_scale=scale, out_bias=bias, out_relu=True)
    assert layer.expand_kernel == 1 and layer.cta_pairs
    assert layer.sparse_engine[2] == 0  # no residual blocks in the pair form
    c = inp.cfg
    for seed in (None, 91):
        x = inp.x if seed is None else workloads.generate_x(cfg, n, seed=seed)
        y = layer(torch.from_numpy(x).to(torch.bfloat16).cuda())
        torch.cuda.synchronize()
        ref = O.output_epilogue(O.forward_factored(x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                                                   inp.col_idx, inp.values, c.stride, c.pad), scale, bias, relu=True)
        parity.check(y, ref, "bf16")


def test_cta_pair_bitwise_equal_single_without_overflow():
    """Without overflow entries (an S with <= 2 nonzeros per group of 4) both forms
    issue the same MMAs in the same K order -- the pair form only splits B between the two
    SMs: bitwise equal to the one-CTA form (LRS_WCONV_PAIR=0)."""
    cfg = workloads.LayerConfig("pair1", 10, 7, 7, 512, 512, 3, 1, 1, 128, 128, 0.02, "bf16", seed=3)
    g = workloads.generate(cfg)
    # keep at most 2 nonzeros per (row, group of 4 channels, tap): an exact 2:4 S
    taps = cfg.k * cfg.k
    rows, cols, vals = [], [], []
    for j in range(cfg.c_out):
        seen = {}
        for e in range(g.row_ptr[j], g.row_ptr[j + 1]):
            col = int(g.col_idx[e])
            key = ((col // taps) // 4, col % taps)
            if seen.get(key, 0) < 2:
                seen[key] = seen.get(key, 0) + 1
                rows.append(j)
                cols.append(col)
                vals.append(g.values[e])
    rp = np.zeros(cfg.c_out + 1, np.int64)
    np.add.at(rp, np.array(rows) + 1, 1)
    inp = workloads.LayerInputs(cfg, g.x, g.u_in, g.core, g.u_out, np.cumsum(rp), np.array(cols, np.int32),
                                np.array(vals, np.float32))
    a = _make_env(inp, {"LRS_WCONV_PAIR": "1"})
    b = _make_env(inp, {"LRS_WCONV_PAIR": "0", "LRS_WCONV_IPW": "4"})
    assert a.cta_pairs and not b.cta_pairs
    assert a.sparse_engine[2] == 0 and a.overflow_chunks == 0
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    ya, yb = a(x), b(x)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
    parity.check(ya, oracle(inp), "bf16")


@pytest.mark.parametrize("th", ["1", "2", "4"])
def test_band_heights_bitwise_equal(th):
    """autotune_w picks the windowed kernel's band height by timing; every height accumulates
    each output in the same K order (sparse blocks by chunk and tap, then T, then the overflow
    gather): bitwise equal to the tallest band (one tile per image group), and to the oracle."""
    cfg = workloads.LayerConfig("th", 16, 7, 7, 512, 512, 3, 1, 1, 128, 128, 0.05, "bf16", seed=43)
    inp = workloads.generate(cfg)
    a = _make_env(inp, {"LRS_WCONV_TH": th})
    b = _make_env(inp, {"LRS_WCONV_TH": "7"})
    assert a.expand_kernel == 1 and b.expand_kernel == 1
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    ya, yb = a(x), b(x)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
    parity.check(ya, oracle(inp), "bf16")


def test_autotuned_band_height_at_the_two_gpu_shard():
    """C3 with 128 images (its 2-GPU shard): the cost model's band height and the tallest one
    are both timed at create; whichever wins, Y matches the fp64 oracle on sampled images."""
    cfg = workloads.CONFIGS["c3"]
    inp = workloads.generate(cfg, batch=1)
    from paper_2006_06443_b200 import LrsConv
    layer = LrsConv.from_inputs(inp, batch_max=128)
    x_np = workloads.generate_x(cfg, 128, seed=5)
    y = layer(torch.from_numpy(x_np).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    idx = np.array([0, 63, 127])
    c = inp.cfg
    ref = O.forward_factored(x_np[idx].astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                             inp.values, c.stride, c.pad)
    parity.check(y[idx], ref, "bf16")
