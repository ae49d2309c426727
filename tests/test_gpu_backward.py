"""GPU parity of the backward pass (§3.5 fine-tuning by
back-propagation) against the fp64 oracle (oracle/lrs_backward.py, pinned in
tests/test_backward_oracle.py), through the C-ABI (lrs_conv_bwd_create /
lrs_conv_backward_data / lrs_conv_backward_weights).

bf16 path, tolerance relL2 <= 2e-2 (BASELINE.json north star) on dX (whole tensor, per
image, per 128-channel block, border rows / columns: tests/parity.py) and on every
parameter gradient (dU_in, dG, dU_out, and S's value gradient); shapes span several
tiles, ragged image groups, padding 0 (the transposed layer then pads 2), stride 2 (even /
odd extents, a C5-like 28x28 layer), an SVD pair, an empty S, and the full-size C2 / C3 / C4
layers.
"""
import numpy as np
import pytest
import torch

import parity
import workloads
from oracle import lrs_backward as B

pytestmark = pytest.mark.gpu

CFG = workloads.LayerConfig
CASES = {
    "small_3x3": CFG("small_3x3", 6, 14, 14, 128, 192, 3, 1, 1, 64, 32, 0.02, "bf16"),
    "pad0": CFG("pad0", 3, 9, 9, 64, 128, 3, 1, 0, 32, 48, 0.03, "bf16"),
    "c2_b8": workloads.CONFIGS["c2_bf16"].replace(batch=8),
    "c3_b20": workloads.CONFIGS["c3"].replace(batch=20),
    "c4_b5": workloads.CONFIGS["c4"].replace(batch=5),
    "no_s": CFG("no_s", 4, 14, 14, 128, 128, 3, 1, 1, 32, 32, 0.0, "bf16"),
    "k5": CFG("k5", 2, 12, 12, 64, 64, 5, 1, 2, 32, 32, 0.02, "bf16"),
    # stride 2 (the adjoints run on zero-inserted gradients; the shifted weight-gradient
    # operands are TMA boxes sampled every 2 positions): even and odd input extents (r = 0 / 1)
    "s2_even": CFG("s2_even", 4, 14, 14, 64, 128, 3, 2, 1, 32, 32, 0.02, "bf16"),
    "s2_odd": CFG("s2_odd", 3, 15, 13, 128, 64, 3, 2, 1, 48, 16, 0.03, "bf16"),
    "s2_c5": workloads.CONFIGS["c2_bf16"].replace(name="s2_c5", batch=6, in_h=28, in_w=28, c_in=128, c_out=128,
                                                  stride=2, rank_in=32, rank_out=32),
    # channel counts and ranks off the 64 / 16 grids (padded boxes, odd R2 pitch), 7x7 kernel
    "odd": CFG("odd", 3, 10, 11, 32, 96, 3, 1, 1, 24, 40, 0.03, "bf16"),
    "k7": CFG("k7", 2, 9, 9, 64, 128, 7, 1, 3, 16, 48, 0.02, "bf16"),
}


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_gpu(inp, dy_np, batch_max=None):
    from paper_2006_06443_b200 import LrsConvBackward
    n = inp.x.shape[0]
    bw = LrsConvBackward.from_inputs(inp, batch_max=batch_max or n)
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    dy = torch.from_numpy(dy_np).to(torch.bfloat16).cuda()
    dx = bw.backward_data(dy)
    g = bw.backward_weights(x, dy)
    torch.cuda.synchronize()
    return bw, x, dy, dx, g


def check_grads(g, ref, svd):
    errs = {}
    for key in ("d_u_in", "d_u_out", "d_values") + (() if svd else ("d_core",)):
        got = g[key].cpu().numpy().astype(np.float64)
        want = ref[key]
        assert got.shape == want.shape, (key, got.shape, want.shape)
        assert np.isfinite(got).all(), key
        if want.size == 0:
            continue
        errs[key] = rel(got, want)
        assert errs[key] <= 2e-2, f"{key}: relL2 {errs[key]:.3e}"
    return errs


@pytest.mark.parametrize("name", list(CASES))
def test_backward_matches_oracle(name):
    cfg = CASES[name]
    inp = workloads.generate(cfg)
    dy_np = workloads.generate_dy(cfg, seed=11)
    bw, x, dy, dx, g = run_gpu(inp, dy_np)
    ref = B.backward_factored(inp.x, dy_np, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, cfg.stride, cfg.pad)
    parity.check(dx, ref["dx"], "bf16")
    check_grads(g, ref, cfg.svd)


@pytest.mark.parametrize("name", ["c3_b20", "small_3x3", "s2_odd"])
def test_backward_deterministic_and_graph_capturable(name):
    """Same inputs -> the same bits (fixed split-sum order), eagerly and replayed from a
    CUDA graph; a smaller n than batch_max on the same handle (ragged split ranges)."""
    cfg = CASES[name]
    inp = workloads.generate(cfg)
    dy_np = workloads.generate_dy(cfg, seed=12)
    bw, x, dy, dx, g = run_gpu(inp, dy_np, batch_max=cfg.batch + 5)
    g2 = bw.alloc_grads()
    dx2 = torch.empty_like(dx)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        bw.backward_data_into(dy, dx2, stream=s)
        bw.backward_weights_into(x, dy, g2, stream=s)
    s.synchronize()
    assert torch.equal(dx, dx2)
    for k in g:
        if g[k] is not None:
            assert torch.equal(g[k], g2[k]), k
    graph = torch.cuda.CUDAGraph()
    g3 = bw.alloc_grads()
    dx3 = torch.full_like(dx, float("nan"))
    with torch.cuda.graph(graph, stream=s):
        bw.backward_data_into(dy, dx3, stream=s)
        bw.backward_weights_into(x, dy, g3, stream=s)
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(dx, dx3)
    for k in g:
        if g[k] is not None:
            assert torch.equal(g[k], g3[k]), k


@pytest.mark.parametrize("name", ["c3_b20", "c4_b5", "small_3x3", "s2_even", "s2_odd"])
def test_combined_backward_matches_oracle_and_split_calls(name):
    """lrs_conv_backward (dT1 reused from the transposed layer's forward): the oracle's
    tolerance on every output, dX bitwise the backward_data result, the gradients within
    fp32-summation-order distance (1e-3) of the two-call form."""
    cfg = CASES[name]
    inp = workloads.generate(cfg)
    dy_np = workloads.generate_dy(cfg, seed=15)
    bw, x, dy, dx, g = run_gpu(inp, dy_np)
    dx2, g2 = bw.backward(x, dy)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2)
    ref = B.backward_factored(inp.x, dy_np, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, cfg.stride, cfg.pad)
    check_grads(g2, ref, cfg.svd)
    for k in g:
        if g[k] is not None and g[k].numel():
            assert rel(g2[k].cpu().double().numpy(), g[k].cpu().double().numpy()) < 1e-3, k


def test_backward_linearity_in_the_batch():
    """Weight gradients are sums over images: g(X, dY) = g(first half) + g(second half)
    (a property at any size; here through two calls of the same handle)."""
    cfg = workloads.CONFIGS["c2_bf16"].replace(batch=16)
    inp = workloads.generate(cfg)
    dy_np = workloads.generate_dy(cfg, seed=13)
    bw, x, dy, dx, g = run_gpu(inp, dy_np)
    ga = bw.backward_weights(x[:7].contiguous(), dy[:7].contiguous())
    gb = bw.backward_weights(x[7:].contiguous(), dy[7:].contiguous())
    torch.cuda.synchronize()
    for k in ("d_u_in", "d_core", "d_u_out", "d_values"):
        s = (ga[k] + gb[k]).cpu().double().numpy()
        assert rel(s, g[k].cpu().double().numpy()) < 1e-5, k


@pytest.mark.parametrize("name", ["c3", "c2_bf16", "c4"])
def test_backward_full_size(name):
    """The BASELINE layer at its full batch (the bench's configuration): dX on sampled
    images (each image's dX depends only on its own dY), every parameter gradient whole."""
    cfg = workloads.CONFIGS[name]
    inp = workloads.generate(cfg)
    dy_np = workloads.generate_dy(cfg, seed=14)
    bw, x, dy, dx, g = run_gpu(inp, dy_np)
    ref = B.backward_factored(inp.x, dy_np, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, cfg.stride, cfg.pad)
    check_grads(g, ref, cfg.svd)
    idx = np.unique(np.r_[0:4, cfg.batch // 2, cfg.batch - 3:cfg.batch])
    parity.check(dx[idx], ref["dx"][idx], "bf16")


def test_backward_n0_and_errors():
    from paper_2006_06443_b200 import LrsConvBackward, LrsError
    cfg = CASES["small_3x3"]
    inp = workloads.generate(cfg)
    bw = LrsConvBackward.from_inputs(inp, batch_max=cfg.batch)
    g = bw.alloc_grads()
    for t in g.values():
        if t is not None:
            t.fill_(float("nan"))
    x = torch.zeros((0, cfg.in_h, cfg.in_w, cfg.c_in), dtype=torch.bfloat16, device="cuda")
    dy = torch.zeros((0, cfg.out_h, cfg.out_w, cfg.c_out), dtype=torch.bfloat16, device="cuda")
    bw.backward_weights_into(x, dy, g)
    torch.cuda.synchronize()
    for t in g.values():
        if t is not None:
            assert torch.count_nonzero(t).item() == 0
    with pytest.raises(LrsError):
        big = torch.zeros((cfg.batch + 1, cfg.in_h, cfg.in_w, cfg.c_in), dtype=torch.bfloat16, device="cuda")
        bdy = torch.zeros((cfg.batch + 1, cfg.out_h, cfg.out_w, cfg.c_out), dtype=torch.bfloat16, device="cuda")
        bw.backward_weights_into(big, bdy, g)
    # fp32 and strides > 4 are refused (UNSUPPORTED), not silently wrong
    for bad in (cfg.replace(stride=5), cfg.replace(dtype="f32")):
        binp = workloads.generate(bad.replace(batch=1))
        with pytest.raises(LrsError, match="UNSUPPORTED"):
            LrsConvBackward.from_inputs(binp, batch_max=1)


@pytest.mark.parametrize("name", ["c3_b20", "c4_b5", "small_3x3"])
def test_pair_and_solo_weight_gradient_forms_agree(name, monkeypatch):
    """The weight-gradient kernel's one-CTA form (default) and its CTA-pair form
    (LRS_WGRAD_PAIR=1: cta_group::2, M = 256 items, B split across the pair, small problems
    padded) compute the same sums (up to the fp32 order of the K splits), both at the oracle's
    bar."""
    cfg = CASES[name]
    inp = workloads.generate(cfg)
    dy_np = workloads.generate_dy(cfg, seed=16)
    _, _, _, _, g_solo = run_gpu(inp, dy_np)
    monkeypatch.setenv("LRS_WGRAD_PAIR", "1")
    _, _, _, _, g_pair = run_gpu(inp, dy_np)
    ref = B.backward_factored(inp.x, dy_np, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, cfg.stride, cfg.pad)
    check_grads(g_pair, ref, cfg.svd)
    check_grads(g_solo, ref, cfg.svd)
    for k in g_pair:
        if g_pair[k] is not None and g_pair[k].numel():
            assert rel(g_pair[k].cpu().double().numpy(), g_solo[k].cpu().double().numpy()) < 1e-5, k


@pytest.mark.parametrize("name,batch", [("c2_cp", 6), ("c1_cp", 1)])
def test_cp_layer_backward_matches_oracle(name, batch):
    """The paper's own decomposed layer (CP) fine-tuned by back-propagation
    (§3.5): dX, dA, dB, dC, dD and the S value gradients against oracle/lrs_backward.backward_cp
    (pinned to torch autograd).  The GPU runs the CP layer's Tucker-2 embedding (diagonal core,
    bf16-rounded products) and folds dG into dB, dC."""
    from paper_2006_06443_b200 import LrsConvBackward
    cfg = workloads.CP_CONFIGS[name]
    if cfg.dtype != "bf16":
        cfg = cfg.replace(dtype="bf16")
    inp = workloads.generate_cp(cfg, batch=batch)
    dy_np = workloads.generate_dy(cfg, batch, seed=17)
    bw = LrsConvBackward.from_cp(batch, cfg.in_h, cfg.in_w, cfg.k, cfg.stride, cfg.pad, "bf16", inp.a, inp.b, inp.c,
                                 inp.d, inp.row_ptr, inp.col_idx, inp.values)
    x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    dy = torch.from_numpy(dy_np).to(torch.bfloat16).cuda()
    dx, g = bw.backward(x, dy)
    torch.cuda.synchronize()
    xr = x.float().cpu().numpy().astype(np.float64)
    ref = B.backward_cp(xr, dy_np, inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx, inp.values, cfg.stride,
                        cfg.pad)
    parity.check(dx, ref["dx"], "bf16")
    k = cfg.k
    got = {"d_a": g["d_u_in"], "d_d": g["d_u_out"].T, "d_b": g["d_core"][:k], "d_c": g["d_core"][k:],
           "d_values": g["d_values"]}
    for key, t in got.items():
        e = rel(t.cpu().double().numpy(), ref[key])
        assert e <= 2e-2, f"{key}: relL2 {e:.3e}"
