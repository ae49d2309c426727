"""GPU parity of the fused projection + core kernel (lrs_core.cuh): a1 and a2 in
one kernel with T1 computed per input window and kept in shared memory
(PAPER.md:162-166).  Checked against the fp64 oracle (bf16 bar relL2 <= 2e-2,
BASELINE.json north star) and against the two-kernel path (LRS_NO_CORE=1),
which rounds the same fp32 T1 to bf16 and sums the same products in the same
order, so the two must agree bit for bit.
"""
import os

import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O
import parity

pytestmark = pytest.mark.gpu


def make(inp, env=None):
    from paper_2006_06443_b200 import LrsConv
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return LrsConv.from_inputs(inp)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def fwd(layer, inp):
    y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


def oracle(inp):
    c = inp.cfg
    return O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, c.stride, c.pad)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", ["c2_bf16", "c3"])
def test_bf16_tucker_configs_fuse_a1_a2(name):
    layer = make(workloads.generate(workloads.CONFIGS[name], batch=1))
    assert layer.core_fused
    assert layer.launches_per_forward == 2


GEOMS = [  # (n, h, w, cin, cout, k, pad, r1, r2, density)  bf16, stride 1, cin % 64 == 0
    (5, 14, 14, 64, 128, 3, 1, 64, 64, 0.02),     # C2-like, ragged batch
    (3, 7, 7, 128, 128, 3, 1, 128, 128, 0.05),    # C3-like ranks (T1 window 2 K chunks of 64)
    (2, 56, 56, 64, 64, 3, 1, 16, 16, 0.02),      # ResNet layer1 shape: wide rows, R = 16 (SW32 G chunks)
    (3, 28, 28, 128, 128, 3, 1, 32, 32, 0.02),    # layer2 shape: R = 32 (SW64 G chunks)
    (4, 12, 12, 64, 64, 5, 2, 48, 32, 0.03),      # 5x5 taps, R1 = 48 (3 G chunks of 16)
    (3, 10, 10, 64, 64, 3, 0, 32, 64, 0.02),      # pad 0 (window fully inside the image)
    (9, 9, 9, 64, 192, 3, 1, 64, 32, 0.02),       # odd size, R2 < R1
]


@pytest.mark.parametrize("geom", GEOMS)
def test_fused_core_vs_oracle_and_two_kernel_path(geom):
    n, h, w, cin, cout, k, p, r1, r2, dens = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, 1, p, r1, r2, dens, "bf16", seed=21)
    inp = workloads.generate(cfg)
    fused = make(inp)
    split = make(inp, {"LRS_NO_CORE": "1"})
    assert fused.core_fused and not split.core_fused
    yf, ys = fwd(fused, inp), fwd(split, inp)
    parity.check(yf, oracle(inp), "bf16")
    assert np.array_equal(yf, ys)


def test_stride_two_keeps_two_kernels():
    cfg = workloads.LayerConfig("t", 2, 14, 14, 64, 64, 3, 2, 1, 16, 16, 0.02, "bf16", seed=3)
    inp = workloads.generate(cfg)
    layer = make(inp)
    assert not layer.core_fused
    parity.check(fwd(layer, inp), oracle(inp), "bf16")


PLAN_GEOMS = {  # ragged batches at the C2 / C3 layer shapes
    "c2": (9, 14, 14, 256, 256, 3, 1, 64, 64, 0.02),
    "c3": (10, 7, 7, 512, 512, 3, 1, 128, 128, 0.05),
}
PLANS = [  # planner overrides (read at create): tile shape, persistent grid, T1 window layout
    ("c2", {"LRS_CORE_IPT": "2", "LRS_CORE_TH": "7"}),
    ("c2", {"LRS_CORE_IPT": "1", "LRS_CORE_TH": "7", "LRS_CORE_GRID": "5"}),   # several tiles per CTA
    ("c2", {"LRS_CORE_IPT": "4", "LRS_CORE_TH": "2", "LRS_CORE_GRID": "3"}),
    ("c2", {"LRS_CORE_T1_NOSWZ": "1"}),                                     # SWIZZLE_NONE T1 window
    ("c2", {"LRS_CORE_IPT": "2", "LRS_CORE_TH": "7", "LRS_CORE_GRID": "4", "LRS_CORE_GSTREAM": "1"}),  # G streamed
    ("c3", {"LRS_CORE_GRID": "5", "LRS_CORE_GSTREAM": "1"}),
    ("c3", {"LRS_CORE_GRID": "7"}),
    ("c3", {"LRS_CORE_IPT": "2", "LRS_CORE_TH": "3", "LRS_CORE_GRID": "4"}),
    ("c3", {"LRS_CORE_IPT": "1", "LRS_CORE_TH": "7", "LRS_CORE_T1_NOSWZ": "1"}),
]


@pytest.mark.parametrize("geom,env", PLANS)
def test_core_plans_bitwise_equal_to_two_kernel_path(geom, env):
    """Every tile shape / grid / window layout the planner can pick computes the same
    bits as the two-kernel path (same bf16 T1, same products, same order)."""
    n, h, w, cin, cout, k, p, r1, r2, dens = PLAN_GEOMS[geom]
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, 1, p, r1, r2, dens, "bf16", seed=8)
    inp = workloads.generate(cfg)
    fused = make(inp, env)
    split = make(inp, {"LRS_NO_CORE": "1"})
    assert fused.core_fused
    yf, ys = fwd(fused, inp), fwd(split, inp)
    assert np.array_equal(yf, ys)
    parity.check(yf, oracle(inp), "bf16")
