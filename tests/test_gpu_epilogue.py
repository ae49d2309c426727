"""GPU parity of the fused output epilogue (include/lrs_conv.h out_scale / out_bias /
out_relu): Y = act(s * conv(X, L + S) + b) on every engine that writes
Y -- the 2:4 tensor-core kernel (bf16), the SIMT expansion + sparse kernel (fp32), the
one-kernel small fp32 path, the fused SIMT epilogue of the generic GEMM (bf16 layers with
c_in % 64 != 0) and the CP path -- against oracle.output_epilogue(forward) at the north
star's tolerances."""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O
import parity

pytestmark = pytest.mark.gpu

CASES = [  # (name, cfg, expected engine)
    ("wconv", workloads.LayerConfig("t", 5, 14, 14, 64, 128, 3, 1, 1, 32, 32, 0.02, "bf16", seed=4), 1),
    ("spadd", workloads.LayerConfig("t", 6, 14, 14, 64, 72, 3, 1, 1, 16, 32, 0.03, "f32", seed=4), 2),
    ("tiny", workloads.LayerConfig("t", 1, 20, 20, 32, 48, 3, 1, 1, 8, 8, 0.03, "f32", seed=4), 3),
    ("simt_epilogue", workloads.LayerConfig("t", 3, 12, 12, 32, 40, 3, 1, 1, 16, 16, 0.04, "bf16", seed=4), 0),
    ("svd", workloads.LayerConfig("t", 8, 9, 9, 128, 192, 1, 1, 0, 32, 32, 0.02, "bf16", svd=True, seed=4), 1),
]


@pytest.mark.parametrize("name,cfg,eng", CASES, ids=[c[0] for c in CASES])
def test_fused_output_epilogue_vs_oracle(name, cfg, eng):
    import os
    from paper_2006_06443_b200 import LrsConv
    inp = workloads.generate(cfg)
    rng = np.random.default_rng(2)
    scale = (0.5 + rng.random(cfg.c_out)).astype(np.float32) * np.where(rng.random(cfg.c_out) < 0.2, -1, 1)
    bias = rng.standard_normal(cfg.c_out).astype(np.float32) * 0.3
    old = os.environ.get("LRS_NO_TINY")
    if eng == 2:
        os.environ["LRS_NO_TINY"] = "1"  # this small fp32 layer would otherwise take the one-kernel path
    else:
        os.environ.pop("LRS_NO_TINY", None)
    try:
        layer = LrsConv.from_inputs(inp, out_scale=scale, out_bias=bias, out_relu=True)
    finally:
        if old is None:
            os.environ.pop("LRS_NO_TINY", None)
        else:
            os.environ["LRS_NO_TINY"] = old
    assert layer.sparse_engine[0] == eng
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    y = layer(torch.from_numpy(inp.x).to(tdt).cuda()).float().cpu().numpy().astype(np.float64)
    ref = O.output_epilogue(O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                                               inp.col_idx, inp.values, cfg.stride, cfg.pad), scale, bias, relu=True)
    parity.check(y, ref, cfg.dtype)
    assert (y >= 0).all()  # the ReLU


def test_epilogue_identity_is_bitwise_noop():
    """out_scale = 1, out_bias = 0, no ReLU gives bitwise the plain layer."""
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.LayerConfig("t", 4, 14, 14, 64, 128, 3, 1, 1, 32, 32, 0.02, "bf16", seed=9)
    inp = workloads.generate(cfg)
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    ya = LrsConv.from_inputs(inp)(x)
    yb = LrsConv.from_inputs(inp, out_scale=np.ones(cfg.c_out, np.float32), out_bias=np.zeros(cfg.c_out, np.float32))(x)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
