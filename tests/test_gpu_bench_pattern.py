"""GPU parity of exactly what bench.py times: full-size layers (the create-time
autotuned plan at the bench's batch), several forwards captured back to back in
ONE CUDA graph on DIFFERENTLY seeded inputs, replayed twice.

At C2-bf16 the autotuner picks the co-resident schedule: the a1 + a2 kernel of
forward i+1 runs on the SMs the fused expansion + sparse kernel of forward i
leaves free, chained by programmatic dependent launch, and consecutive forwards
share the handle's T2 scratch -- a cross-forward race on T2 would show up here
as a wrong Y for one of the inputs (identical inputs would hide it).

Every Y is checked against the fp64 oracle on that input (PAPER.md:160,
Y = conv(X, L + S); bf16 relL2 <= 2e-2 on the whole tensor, per image, per
128-channel block and per border row -- tests/parity.py) and must be bitwise
equal to an eager single forward of the same input.
"""
import numpy as np
import pytest
import torch

import parity
import workloads
from oracle import lrs_oracle as O

pytestmark = pytest.mark.gpu

N_FWD = 4


def oracle_images(inp, x, idx):
    """fp64 oracle on the images `idx` of x (each image's output depends only on
    that image, so a subset is exact)."""
    c = inp.cfg
    return O.forward_factored(x[idx].astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, c.stride, c.pad)


def sample_images(n):
    """images the oracle checks: all of a small batch; for a large one the first and
    last 8-image group (the fused kernel's image groups) and two groups in between."""
    if n <= 64:
        return np.arange(n)
    return np.unique(np.concatenate([np.arange(0, 8), np.arange(n // 2 - 4, n // 2 + 4),
                                     np.arange(n - 40, n - 32), np.arange(n - 8, n)]))


@pytest.mark.parametrize("name", ["c2_bf16", "c3", "c4"])
def test_graph_of_forwards_on_distinct_inputs(name):
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.CONFIGS[name]
    inp = workloads.generate(cfg)
    n = cfg.batch
    layer = LrsConv.from_inputs(inp, batch_max=n)
    xs_np = [workloads.generate_x(cfg, n, seed=100 + i) for i in range(N_FWD)]
    xs = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs_np]
    ys = [torch.full((n, cfg.out_h, cfg.out_w, cfg.c_out), float("nan"), dtype=torch.bfloat16, device="cuda")
          for _ in range(N_FWD)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(N_FWD):  # warm (eager)
            layer.forward_into(xs[i], ys[i], stream=s)
    s.synchronize()
    for y in ys:
        y.fill_(float("nan"))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(N_FWD):
                layer.forward_into(xs[i], ys[i], stream=s)
    outs = []
    for rep in range(2):
        for y in ys:
            y.fill_(float("nan"))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        outs.append([y.clone() for y in ys])
    # eager single forwards, one at a time
    eager = []
    for i in range(N_FWD):
        y = torch.empty_like(ys[i])
        layer.forward_into(xs[i], y)
        torch.cuda.synchronize()
        eager.append(y)
    idx = sample_images(n)
    for i in range(N_FWD):
        assert torch.equal(outs[0][i], eager[i]), f"graph replay 0, forward {i} != eager"
        assert torch.equal(outs[1][i], eager[i]), f"graph replay 1, forward {i} != eager"
        ref = oracle_images(inp, xs_np[i], idx)
        parity.check(eager[i][torch.from_numpy(idx).cuda()], ref, "bf16")
    # the inputs differ, so must the outputs (guards against a test that checks one Y 4 times)
    assert not torch.equal(eager[0], eager[1])
    layer.close()


def test_fp32_sparse_values_reach_bf16_layers_unrounded():
    """The ABI takes fp32 S values (include/lrs_conv.h); a bf16 layer rounds them
    itself.  The generator keeps them fp32 (SURVEY §8(c) reading #12), so every bf16
    parity test already compares against the oracle on the caller's fp32 S; here the
    sparse term alone (U_out = 0) is checked, where that rounding is all the error."""
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.CONFIGS["c2_bf16"]
    inp = workloads.generate(cfg, batch=16)
    assert not np.array_equal(workloads.bf16_round(inp.values), inp.values)  # really fp32 values
    only_s = workloads.LayerInputs(cfg, inp.x, inp.u_in, inp.core, np.zeros_like(inp.u_out), inp.row_ptr,
                                   inp.col_idx, inp.values)
    layer = LrsConv.from_inputs(only_s)
    y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, np.zeros_like(inp.u_out), inp.row_ptr,
                             inp.col_idx, inp.values, cfg.stride, cfg.pad)
    err, _ = parity.check(y, ref, "bf16")
    assert err < 5e-3, err  # S rounding (2^-9) + Y rounding: ~3e-3, well inside the bar


def test_unrounded_fp32_factors_round_to_nearest_even():
    """make_desc rounds fp32 factors to bf16 RNE: a layer built from raw fp32 factors
    computes bitwise what a layer built from pre-rounded (RNE) factors computes."""
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.CONFIGS["c2_bf16"]
    inp = workloads.generate(cfg, batch=8)
    rng = np.random.default_rng(11)
    raw = [(t.astype(np.float64) + rng.standard_normal(t.shape) * 1e-3).astype(np.float32)
           for t in (inp.u_in, inp.core, inp.u_out)]
    assert not np.array_equal(workloads.bf16_round(raw[0]), raw[0])
    a = LrsConv.from_inputs(workloads.LayerInputs(cfg, inp.x, *raw, inp.row_ptr, inp.col_idx, inp.values))
    b = LrsConv.from_inputs(workloads.LayerInputs(cfg, inp.x, *[workloads.bf16_round(t) for t in raw], inp.row_ptr,
                                                  inp.col_idx, inp.values))
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    ya, yb = a(x), b(x)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
