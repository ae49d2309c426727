"""GPU checks of the early-start protocol (include/lrs_conv.h, lrs_conv_forward):
for core -> fused-kernel layers the projection + core kernel of forward f+1 starts before
forward f's fused kernel has finished (T2 and the overflow-gather scratch alternate between
two buffers), unless X is the output of the library's previous forward on the stream.

Each pattern below is enqueued without host synchronisation (eager and inside one CUDA
graph) and compared bitwise with the same forwards run one at a time with a device sync in
between (no overlap possible), and a sample with the fp64 oracle."""
import os

import numpy as np
import pytest
import torch

import parity
import workloads
from oracle import lrs_oracle as O

pytestmark = pytest.mark.gpu


def cfg_sq(n=16, seed=41, dens=0.05):
    # C3-like square layer (512 -> 512, 3x3, 7x7) so that Y of one forward can be X of the next
    return workloads.LayerConfig("sq", n, 7, 7, 512, 512, 3, 1, 1, 128, 128, dens, "bf16", seed=seed)


def make(inp, batch_max, env=None):
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


def one_at_a_time(layers, xs):
    outs = []
    for layer, x in zip(layers, xs):
        torch.cuda.synchronize()
        outs.append(layer(x).clone())
        torch.cuda.synchronize()
    return outs


def test_rotating_inputs_same_output_buffer():
    """forward(x_i, y) back to back on ONE y buffer (nothing else enqueued in between, so
    consecutive forwards overlap): the final Y is that of the last input, bitwise."""
    cfg = cfg_sq()
    inp = workloads.generate(cfg)
    layer = make(inp, cfg.batch)
    xs = [torch.from_numpy(workloads.generate_x(cfg, cfg.batch, seed=200 + i)).to(torch.bfloat16).cuda()
          for i in range(6)]
    ref = one_at_a_time([layer] * 6, xs)
    y = torch.empty_like(ref[0])
    s = torch.cuda.Stream()
    for rep in range(3):
        y.fill_(float("nan"))
        with torch.cuda.stream(s):
            for x in xs[rep:] + xs[:rep]:
                layer.forward_into(x, y, stream=s)
        s.synchronize()
        assert torch.equal(y, ref[(rep - 1) % 6])


def test_chained_layers_x_is_previous_output():
    """y1 = A(x), y2 = B(y1), y3 = A(y2), ... without syncs, eager and in a graph: each X
    is the previous forward's Y, so each forward must wait for the previous one (the
    hazard check) -- bitwise equal to one-at-a-time, and the first against the oracle."""
    ca, cb = cfg_sq(seed=41), cfg_sq(seed=42)
    ia, ib = workloads.generate(ca), workloads.generate(cb)
    a, b = make(ia, ca.batch), make(ib, cb.batch)
    x0 = torch.from_numpy(ia.x).to(torch.bfloat16).cuda()
    # reference: one at a time
    ref, x = [], x0
    for layer in (a, b, a, b):
        torch.cuda.synchronize()
        x = layer(x).clone()
        torch.cuda.synchronize()
        ref.append(x)
    c = ia.cfg
    y1 = O.forward_factored(ia.x.astype(np.float64), ia.u_in, ia.core, ia.u_out, ia.row_ptr, ia.col_idx, ia.values,
                            c.stride, c.pad)
    parity.check(ref[0], y1, "bf16")
    bufs = [torch.empty_like(ref[0]) for _ in range(4)]
    s = torch.cuda.Stream()

    def chain():
        src = x0
        for layer, dst in zip((a, b, a, b), bufs):
            layer.forward_into(src, dst, stream=s)
            src = dst

    with torch.cuda.stream(s):
        chain()
    s.synchronize()
    for got, r in zip(bufs, ref):
        assert torch.equal(got, r)
    for t in bufs:
        t.fill_(float("nan"))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            chain()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for got, r in zip(bufs, ref):
        assert torch.equal(got, r)


def test_same_layer_applied_to_its_own_output():
    """y = A(A(A(x))) through one handle and two ping-pong buffers."""
    cfg = cfg_sq(seed=43)
    inp = workloads.generate(cfg)
    layer = make(inp, cfg.batch)
    x0 = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    ref = x0
    for _ in range(3):
        torch.cuda.synchronize()
        ref = layer(ref).clone()
    torch.cuda.synchronize()
    p, q = torch.empty_like(x0), torch.empty_like(x0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        layer.forward_into(x0, p, stream=s)
        layer.forward_into(p, q, stream=s)
        layer.forward_into(q, p, stream=s)
    s.synchronize()
    assert torch.equal(p, ref)


@pytest.mark.parametrize("name", ["c3", "c2_bf16"])
def test_early_start_bitwise_equal_to_waiting(name):
    """The protocol changes when kernels start, not what they compute: LRS_NO_EARLY=1 gives
    the same bits on a graph of rotating inputs."""
    cfg = workloads.CONFIGS[name]
    inp = workloads.generate(cfg, batch=32)
    outs = {}
    xs = [torch.from_numpy(workloads.generate_x(cfg, 32, seed=300 + i)).to(torch.bfloat16).cuda() for i in range(5)]
    for mode, env in (("early", None), ("wait", {"LRS_NO_EARLY": "1"})):
        layer = make(inp, 32, env)
        ys = [torch.empty((32, cfg.out_h, cfg.out_w, cfg.c_out), dtype=torch.bfloat16, device="cuda") for _ in xs]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for x, y in zip(xs, ys):
                layer.forward_into(x, y, stream=s)
        s.synchronize()
        outs[mode] = ys
    for a, b in zip(outs["early"], outs["wait"]):
        assert torch.equal(a, b)


def test_pointwise_chain_early_start():
    """The same protocol on the 1x1 SVD-pair chain (projection GEMM -> pointwise kernel, T1
    double-buffered): rotating inputs into one output buffer, and a layer fed its own output,
    enqueued without syncs -- bitwise equal to one forward at a time."""
    cfg = workloads.LayerConfig("pw_chain", 32, 14, 14, 256, 256, 1, 1, 0, 64, 64, 0.01, "bf16", svd=True, seed=51)
    inp = workloads.generate(cfg)
    layer = make(inp, cfg.batch)
    assert layer.expand_kernel == 2
    xs = [torch.from_numpy(workloads.generate_x(cfg, cfg.batch, seed=400 + i)).to(torch.bfloat16).cuda()
          for i in range(5)]
    ref = one_at_a_time([layer] * 5, xs)
    y = torch.empty_like(ref[0])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for x in xs:
            layer.forward_into(x, y, stream=s)
    s.synchronize()
    assert torch.equal(y, ref[-1])
    # self-feeding: x -> p -> q -> p
    r = xs[0]
    for _ in range(3):
        torch.cuda.synchronize()
        r = layer(r).clone()
    torch.cuda.synchronize()
    p, q = torch.empty_like(xs[0]), torch.empty_like(xs[0])
    with torch.cuda.stream(s):
        layer.forward_into(xs[0], p, stream=s)
        layer.forward_into(p, q, stream=s)
        layer.forward_into(q, p, stream=s)
    s.synchronize()
    assert torch.equal(p, r)


def test_tiny_kernel_early_start():
    """The one-kernel fp32 path (lrs_tiny.cuh) computes a forward before the previous one has
    finished and waits only before storing Y: rotating inputs into one output buffer and a
    layer fed its own output, enqueued without syncs -- bitwise equal to one at a time."""
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.LayerConfig("tiny_chain", 1, 14, 14, 64, 64, 3, 1, 1, 16, 16, 0.02, "f32", seed=53)
    inp = workloads.generate(cfg)
    layer = LrsConv.from_inputs(inp, batch_max=1)
    assert layer.sparse_engine[0] == 3  # the tiny kernel
    xs = [torch.from_numpy(workloads.generate_x(cfg, 1, seed=500 + i)).cuda() for i in range(6)]
    ref = one_at_a_time([layer] * 6, xs)
    y = torch.empty_like(ref[0])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for x in xs:
            layer.forward_into(x, y, stream=s)
    s.synchronize()
    assert torch.equal(y, ref[-1])
    r = xs[0]
    for _ in range(3):
        torch.cuda.synchronize()
        r = layer(r).clone()
    torch.cuda.synchronize()
    p, q = torch.empty_like(xs[0]), torch.empty_like(xs[0])
    with torch.cuda.stream(s):
        layer.forward_into(xs[0], p, stream=s)
        layer.forward_into(p, q, stream=s)
        layer.forward_into(q, p, stream=s)
    s.synchronize()
    assert torch.equal(p, r)
