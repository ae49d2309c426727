"""GPU parity of the paper's CP form of L (LRS_CORE_CP, include/lrs_conv.h;
PAPER.md:158-168): T1 = X A on the tensor cores, the two depthwise stages
(lrs_cpdw.cuh: k x 1 with B along H, then 1 x k with C along W), then the
expansion by D fused with the sparse term, against the fp64 oracle
`forward_cp` (the paper's four stages + sparse scatter; dense reconstruction
at stride 2).  Tolerances of the BASELINE.json north star (fp32 relL2 <= 1e-5
and max-abs <= 1e-4; bf16 relL2 <= 2e-2).  Also: the sparse term given in the
paper's own per-input-channel packed format goes through
lrs_sparse_from_slices and yields the identical layer.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O
import parity

pytestmark = pytest.mark.gpu


def run(inp, batch_max=None, csr=None):
    from paper_2006_06443_b200 import LrsConv
    c = inp.cfg
    rp, ci, va = csr if csr is not None else (inp.row_ptr, inp.col_idx, inp.values)
    layer = LrsConv.from_cp(batch_max or inp.x.shape[0], c.in_h, c.in_w, c.k, c.stride, c.pad, c.dtype,
                            inp.a, inp.b, inp.c, inp.d, rp, ci, va)
    tdt = torch.bfloat16 if c.dtype == "bf16" else torch.float32
    y = layer(torch.from_numpy(inp.x).to(tdt).cuda())
    torch.cuda.synchronize()
    return layer, y.float().cpu().numpy().astype(np.float64)


def oracle(inp):
    c = inp.cfg
    return O.forward_cp(inp.x.astype(np.float64), inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx,
                        inp.values, c.stride, c.pad)


def check(y, ref, dtype):
    parity.check(y, ref, dtype)


@pytest.mark.parametrize("name,batch", [("c1_cp", 1), ("c2_cp", 5), ("c2_cp", 64)])
def test_cp_configs_vs_oracle(name, batch):
    inp = workloads.generate_cp(workloads.CP_CONFIGS[name], batch=batch)
    layer, y = run(inp)
    c = inp.cfg
    # bf16, stride 1, Cin % 64 == 0: a1 and the depthwise pair in one kernel (T1 on chip)
    assert layer.core_fused == (c.dtype == "bf16" and c.stride == 1 and c.c_in % 64 == 0)
    check(y, oracle(inp), inp.cfg.dtype)


GEOMS = [  # (n, h, w, cin, cout, k, s, p, R, density, dtype)
    (3, 14, 14, 64, 128, 3, 2, 1, 48, 0.03, "bf16"),    # stride 2, R = 48 (rank padding)
    (2, 12, 12, 16, 32, 5, 1, 2, 16, 0.05, "f32"),      # 5x5 taps
    (4, 9, 11, 64, 64, 3, 1, 0, 32, 0.02, "bf16"),      # pad 0, non-square
    (2, 10, 10, 32, 64, 3, 2, 1, 24, 0.04, "f32"),      # fp32 stride 2, R = 24
]


@pytest.mark.parametrize("geom", GEOMS)
def test_cp_geometries_vs_oracle(geom):
    n, h, w, cin, cout, k, s, p, r, dens, dt = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r, r, dens, dt, seed=5)
    inp = workloads.generate_cp(cfg)
    _, y = run(inp)
    check(y, oracle(inp), dt)


def test_packed_slices_give_the_same_layer():
    """The paper's storage -> lrs_sparse_from_slices -> CSR: the layer
    output is bitwise the one built from the original CSR."""
    from paper_2006_06443_b200 import sparse_from_slices
    inp = workloads.generate_cp(workloads.CP_CONFIGS["c2_cp"], batch=3)
    c = inp.cfg
    vals, packed = O.pack_sparse_slices(c.c_in, c.c_out, c.k, inp.row_ptr, inp.col_idx, inp.values)
    csr = sparse_from_slices(c.c_in, c.c_out, c.k, c.k, vals, packed)
    _, ya = run(inp)
    _, yb = run(inp, csr=csr)
    assert np.array_equal(ya, yb)


def test_cp_equals_tucker_embedding_on_gpu():
    """The CP form is the Tucker-2 special case G[a,b,y,x] = delta_ab B[y,a] C[x,a]
    (reading #1): both GPU paths agree with each other within the fp32 bar."""
    from paper_2006_06443_b200 import LrsConv
    cfg = workloads.LayerConfig("t", 2, 10, 10, 32, 32, 3, 1, 1, 8, 8, 0.03, "f32", seed=2)
    inp = workloads.generate_cp(cfg)
    _, y_cp = run(inp)
    g = np.zeros((8, 8, 3, 3), np.float32)
    for q in range(8):
        g[q, q] = np.outer(inp.b[:, q], inp.c[:, q])
    lt = LrsConv(2, 10, 10, 32, 32, 3, 1, 1, 8, 8, "f32", inp.a, g, np.ascontiguousarray(inp.d.T),
                 inp.row_ptr, inp.col_idx, inp.values)
    y_t = lt(torch.from_numpy(inp.x).cuda()).cpu().numpy().astype(np.float64)
    assert np.linalg.norm(y_cp - y_t) / np.linalg.norm(y_t) <= 1e-5


@pytest.mark.parametrize("geom", [g for g in GEOMS if g[-1] == "f32"])
@pytest.mark.parametrize("no_tiny", [False, True])
def test_cp_fp32_one_kernel_and_chain(geom, no_tiny, monkeypatch):
    """Small fp32 CP layers run the whole layer in the one-kernel path (the paper's two
    depthwise stages in its order, lrs_tiny.cuh); LRS_NO_TINY keeps the three-kernel chain.
    Both meet the fp32 bar against the oracle."""
    if no_tiny:
        monkeypatch.setenv("LRS_NO_TINY", "1")
    n, h, w, cin, cout, k, s, p, r, dens, dt = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r, r, dens, dt, seed=9)
    inp = workloads.generate_cp(cfg)
    layer, y = run(inp)
    assert (layer.sparse_engine[0] == 3) != no_tiny
    check(y, oracle(inp), dt)


@pytest.mark.parametrize("geom", [
    (9, 14, 14, 256, 256, 3, 1, 1, 64, 0.02, "bf16"),    # C2 CP shape, ragged batch
    (4, 9, 11, 64, 64, 3, 1, 0, 32, 0.02, "bf16"),       # pad 0, non-square, R = 32 (SWIZZLE_NONE window)
    (3, 12, 12, 128, 64, 5, 1, 2, 48, 0.03, "bf16"),     # 5x5, R = 48
])
def test_cp_fused_core_bitwise_equal_to_chain(geom, monkeypatch):
    """a1 + the two depthwise stages fused (lrs_core.cuh CPDW: T1 restaged on chip) compute
    the same bits as the three-kernel chain (a1 GEMM -> T1 in HBM -> lrs_cpdw.cuh): the same
    bf16 T1 and the same fp32 FMA order."""
    from paper_2006_06443_b200 import LrsConv
    n, h, w, cin, cout, k, s, p, r, dens, dt = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r, r, dens, dt, seed=31)
    inp = workloads.generate_cp(cfg)
    fused, yf = run(inp)
    assert fused.core_fused
    monkeypatch.setenv("LRS_NO_CORE", "1")
    chain, yc = run(inp)
    assert not chain.core_fused
    assert np.array_equal(yf, yc)
    check(yf, oracle(inp), dt)
