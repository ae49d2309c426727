"""GPU parity of the one-kernel fp32 path (lrs_tiny.cuh): a1, a2, a3 and the sparse
term of a small fp32 layer in a single SIMT kernel,
Y written once.  C1 (batch 1, the BASELINE fp32 config) takes it; the checks below
pin stride 2, 5x5, unequal ranks, Cout not a multiple of 8, pad 0, several images
and an empty S against the fp64 oracle at the fp32 bar (relL2 <= 1e-5, max-abs <=
1e-4), and a bitwise single-nonzero case."""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O
import parity

pytestmark = pytest.mark.gpu


def run(inp):
    from paper_2006_06443_b200 import LrsConv
    layer = LrsConv.from_inputs(inp)
    y = layer(torch.from_numpy(inp.x).float().cuda())
    torch.cuda.synchronize()
    return layer, y.cpu().numpy().astype(np.float64)


def oracle(inp):
    c = inp.cfg
    return O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                              inp.values, c.stride, c.pad)


def check(y, ref):
    parity.check(y, ref, "f32")


def test_c1_is_one_launch_and_matches_oracle():
    inp = workloads.generate(workloads.CONFIGS["c1"])
    layer, y = run(inp)
    assert layer.sparse_engine[0] == 3 and layer.launches_per_forward == 1
    check(y, oracle(inp))


GEOMS = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density)
    (1, 28, 28, 32, 64, 3, 2, 1, 16, 8, 0.02),     # stride 2, R2 < R1
    (2, 12, 12, 16, 36, 5, 1, 2, 8, 12, 0.05),     # 5x5, Cout 36
    (3, 10, 9, 24, 32, 3, 1, 0, 12, 16, 0.03),     # pad 0, odd width, ranks not multiples of 16
    (1, 56, 56, 64, 64, 3, 1, 1, 16, 16, 0.0),     # empty S
]


@pytest.mark.parametrize("geom", GEOMS)
def test_tiny_geometries_vs_oracle(geom):
    n, h, w, cin, cout, k, s, p, r1, r2, dens = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r1, r2, dens, "f32", seed=17)
    inp = workloads.generate(cfg)
    layer, y = run(inp)
    assert layer.sparse_engine[0] == 3
    check(y, oracle(inp))


def test_tiny_single_nonzero_is_bitwise():
    n, h, w, cin, cout, k = 1, 9, 9, 16, 16, 3
    rng = np.random.default_rng(4)
    x = np.maximum(rng.standard_normal((n, h, w, cin)), 0).astype(np.float32)
    j, c, ty, tx, v = 3, 9, 2, 0, np.float32(-0.7)
    rp = np.zeros(cout + 1, np.int64)
    rp[j + 1:] = 1
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, 1, 1, 8, 8, 0.0, "f32")
    inp = workloads.LayerInputs(cfg, x, np.ones((cin, 8), np.float32), np.ones((8, 8, k, k), np.float32),
                                np.zeros((8, cout), np.float32), rp, np.array([(c * k + ty) * k + tx], np.int32),
                                np.array([v], np.float32))
    layer, y = run(inp)
    assert layer.sparse_engine[0] == 3
    xp = np.zeros((n, h + 2, w + 2, cin), np.float32)
    xp[:, 1:-1, 1:-1] = x
    ref = np.zeros((n, h, w, cout), np.float32)
    ref[..., j] = v * xp[:, ty:ty + h, tx:tx + w, c]
    assert np.array_equal(y.astype(np.float32), ref)


@pytest.mark.parametrize("geom,cb", [
    ((1, 56, 56, 64, 64, 3, 1, 1, 16, 16, 0.01), 3),   # C1 shape, 3 column bands of 19/19/18
    ((3, 10, 9, 24, 32, 3, 1, 0, 12, 16, 0.03), 2),    # pad 0, 7 output columns -> bands of 4 + 3
    ((1, 28, 28, 32, 64, 3, 2, 1, 16, 8, 0.02), 4),    # stride 2, 14 output columns -> 4 bands
])
def test_tiny_column_bands_vs_oracle(geom, cb, monkeypatch):
    """CTA = image x row band x column band (the window's halo columns recomputed)."""
    monkeypatch.setenv("LRS_TINY_CB", str(cb))
    n, h, w, cin, cout, k, s, p, r1, r2, dens = geom
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r1, r2, dens, "f32", seed=23)
    inp = workloads.generate(cfg)
    layer, y = run(inp)
    assert layer.sparse_engine[0] == 3
    check(y, oracle(inp))
