"""GPU parity of the channel-stationary pointwise kernel (lrs_pw.cuh): 1x1 layers whose
L is an SVD pair (C4, BASELINE.json configs[3]) with the expansion a3
and the sparse term a4 (PAPER.md:171-191 at k = 1, exact 2:4 main + residual blocks on
the sparse tensor cores) fused and Y written once (a5).  Each CTA keeps the weights of
a fixed group of 128-channel M-tiles resident and streams position tiles.

Against the fp64 oracle (bf16 bar relL2 <= 2e-2 per tensor / image / channel block /
border, tests/parity.py) on geometries that pin each mechanism, and bitwise against
the windowed kernel (LRS_NO_PW=1, same accumulation order) and across plans.
"""
import os

import numpy as np
import pytest
import torch

import parity
import workloads
from oracle import lrs_oracle as O

pytestmark = pytest.mark.gpu


def make(inp, env=None, batch_max=None):
    from paper_2006_06443_b200 import LrsConv
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return LrsConv.from_inputs(inp, batch_max=batch_max)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def fwd(layer, inp):
    y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    return y


def oracle(inp):
    c = inp.cfg
    return O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, c.stride, c.pad)


def svd_cfg(n, h, w, cin, cout, r, dens, seed=21):
    return workloads.LayerConfig("pw", n, h, w, cin, cout, 1, 1, 0, r, r, dens, "bf16", svd=True, seed=seed)


def test_c4_uses_the_pointwise_kernel():
    inp = workloads.generate(workloads.CONFIGS["c4"], batch=2)
    layer = make(inp)
    assert layer.expand_kernel == 2
    assert layer.sparse_engine[0] == 1 and layer.launches_per_forward == 2
    parity.check(fwd(layer, inp), oracle(inp), "bf16")


GEOMS = [  # (n, h, w, cin, cout, rank, density)
    (3, 14, 14, 256, 1024, 64, 0.01),    # C4 shape, ragged P (588 positions)
    (2, 7, 7, 256, 2048, 128, 0.02),     # 16 M-tiles, R = 128 (2 T chunks)
    (4, 28, 28, 128, 512, 32, 0.01),     # layer2 expansion: R = 32 (SW64 T chunks)
    (2, 9, 9, 64, 200, 16, 0.05),        # Cout not a multiple of 128, R = 16 (SW32), one chunk
    (1, 5, 5, 64, 64, 256, 0.02),        # rank 256 (4 T chunks), tiny P < one tile
    (2, 8, 8, 128, 256, 48, 0.30),       # dense S: residual blocks, R = 48 -> 64
    (5, 6, 6, 64, 128, 32, 0.0),         # empty S: LR only (no X chunks)
    (8, 28, 28, 512, 128, 20, 0.01),     # 8 X chunks + T1 per tile: the ring must hold a whole tile
]


@pytest.mark.parametrize("geom", GEOMS)
def test_geometries_vs_oracle(geom):
    n, h, w, cin, cout, r, dens = geom
    inp = workloads.generate(svd_cfg(n, h, w, cin, cout, r, dens))
    layer = make(inp)
    assert layer.expand_kernel == 2, geom
    parity.check(fwd(layer, inp), oracle(inp), "bf16")
    if dens >= 0.3:
        assert layer.sparse_engine[2] > 0  # residual blocks were exercised


@pytest.mark.parametrize("env", [{"LRS_PW_MPC": "1", "LRS_PW_BP": "128"}, {"LRS_PW_MPC": "1", "LRS_PW_BP": "64"},
                                 {"LRS_PW_MPC": "2", "LRS_PW_BP": "64"}, {"LRS_PW_MPC": "2", "LRS_PW_BP": "96"},
                                 {"LRS_PW_MPC": "1", "LRS_PW_BP": "96"}, {"LRS_PW_CPI": "1"}, {"LRS_PW_CPI": "2"},
                                 {"LRS_PW_CPI": "4"}, {"LRS_PW_CPI": "2", "LRS_PW_BP": "96", "LRS_PW_MPC": "2"}])
def test_plans_bitwise_equal_to_windowed_kernel(env):
    """Every (M-tiles per CTA, positions per tile, chunks per ring item) plan, and the windowed fused kernel
    (LRS_NO_PW=1), accumulate each output in the same order: bitwise equal."""
    inp = workloads.generate(svd_cfg(3, 14, 14, 256, 1024, 64, 0.01))
    ref = fwd(make(inp, {"LRS_NO_PW": "1", "LRS_WCONV_GATHER": "0"}), inp)
    layer = make(inp, env)
    assert layer.expand_kernel == 2
    y = fwd(layer, inp)
    assert torch.equal(y, ref)
    parity.check(y, oracle(inp), "bf16")


def test_wide_input_falls_back_to_the_windowed_kernel():
    """c_in = 512 (8 chunks): the resident weights and a ring of chunks do not fit in shared
    memory, so the layer takes the windowed kernel -- still exact against the oracle."""
    inp = workloads.generate(svd_cfg(2, 7, 7, 512, 2048, 128, 0.02))
    layer = make(inp)
    assert layer.expand_kernel in (1, 2)
    parity.check(fwd(layer, inp), oracle(inp), "bf16")


@pytest.mark.parametrize("geom", [(3, 14, 14, 256, 1024, 64, 0.01), (2, 7, 7, 128, 384, 48, 0.05),
                                  (4, 28, 28, 128, 512, 32, 0.01), (5, 6, 6, 64, 128, 32, 0.0)])
def test_fused_projection_bitwise_equal_two_kernel_form(geom):
    """lrs_pwf_kernel (LRS_PW_FT=1: T1 = X U computed per tile from the X chunks in shared
    memory, one launch) against lrs_pw_kernel fed by the separate projection kernel (the
    default): the same MMAs in the same K order, so bitwise equal; and against the oracle."""
    n, h, w, cin, cout, r, dens = geom
    inp = workloads.generate(svd_cfg(n, h, w, cin, cout, r, dens))
    fused = make(inp, {"LRS_PW_FT": "1"})
    split = make(inp)
    assert fused.launches_per_forward == 1 and split.launches_per_forward == 2
    yf, ys = fwd(fused, inp), fwd(split, inp)
    assert torch.equal(yf, ys)
    parity.check(yf, oracle(inp), "bf16")


def test_single_nonzero_is_bitwise():
    """One sparse entry (j, c, v) with V = 0: Y[..., j] = bf16(v * X[..., c]), all else 0."""
    cfg = svd_cfg(2, 6, 6, 64, 256, 16, 0.0)
    inp = workloads.generate(cfg)
    j, c, v = 133, 37, np.float32(0.5)
    rp = np.zeros(cfg.c_out + 1, np.int64)
    rp[j + 1:] = 1
    one = workloads.LayerInputs(cfg, inp.x, inp.u_in, None, np.zeros_like(inp.u_out), rp, np.array([c], np.int32),
                                np.array([v], np.float32))
    y = fwd(make(one), one).float().cpu().numpy()
    ref = np.zeros_like(y)
    ref[..., j] = workloads.bf16_round(v * inp.x[..., c])
    assert np.array_equal(y, ref)


def test_output_epilogue_and_partial_batch():
    """Fused per-channel scale/bias + ReLU (include/lrs_conv.h out_*), and n < batch_max."""
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.CONFIGS["c4"]
    inp = workloads.generate(cfg, batch=5)
    rng = np.random.default_rng(2)
    scale = rng.uniform(0.5, 1.5, cfg.c_out).astype(np.float32)
    bias = rng.standard_normal(cfg.c_out).astype(np.float32)
    layer = LrsConv.from_inputs(inp, batch_max=16, out_scale=scale, out_bias=bias, out_relu=True)
    assert layer.expand_kernel == 2
    y = fwd(layer, inp)
    ref = O.output_epilogue(oracle(inp), scale, bias, relu=True)
    parity.check(y, ref, "bf16")
    assert (y.float() >= 0).all()


def test_autotuned_plan_bitwise_equal_model_plan():
    """autotune_pw (create-time timing of the cost model's best plans) only picks among plans
    that accumulate in the same order: bitwise equal to the model's own choice."""
    inp = workloads.generate(svd_cfg(16, 14, 14, 256, 1024, 64, 0.01, seed=5))
    tuned = make(inp)
    model = make(inp, {"LRS_NO_AUTOTUNE": "1"})
    assert tuned.expand_kernel == 2 and model.expand_kernel == 2
    assert torch.equal(fwd(tuned, inp), fwd(model, inp))
