"""Out-of-bounds write checks (compute-sanitizer is closed on this GPU pool, so the
library's own guard bands stand in for memcheck): every engine writes Y into the middle
of a larger device buffer whose guard bands hold a byte pattern; after the forward the
guards must be bitwise untouched and the output finite and correct against the oracle.
Ragged batches / widths / channel counts put partial tiles at every edge."""
import numpy as np
import pytest
import torch

import parity
import workloads
from oracle import lrs_oracle as O

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side


CASES = [  # (n, h, w, cin, cout, k, s, p, r1, r2, density, dtype, svd)
    (1, 56, 56, 64, 64, 3, 1, 1, 16, 16, 0.01, "f32", False),      # one-kernel SIMT (tiny)
    (3, 14, 14, 256, 256, 3, 1, 1, 64, 64, 0.02, "f32", False),    # SIMT expansion + sparse (spadd)
    (5, 14, 14, 256, 256, 3, 1, 1, 64, 64, 0.02, "bf16", False),   # core + windowed tensor-core kernel
    (3, 7, 7, 512, 512, 3, 1, 1, 128, 128, 0.05, "bf16", False),   # C3 shape, residual blocks
    (3, 14, 14, 256, 1000, 1, 1, 0, 64, 64, 0.01, "bf16", True),   # pointwise kernel, Cout not /128
    (2, 15, 13, 64, 72, 3, 2, 1, 16, 24, 0.03, "bf16", False),     # stride 2: three kernels, ragged
    (2, 9, 9, 24, 40, 3, 1, 1, 8, 8, 0.05, "bf16", False),         # c_in % 64 != 0: GEMM + SIMT epilogue
]


@pytest.mark.parametrize("case", CASES)
def test_output_guard_bands_untouched(case):
    from paper_2006_06443_b200 import LrsConv
    n, h, w, cin, cout, k, s, p, r1, r2, dens, dtype, svd = case
    cfg = workloads.LayerConfig("g", n, h, w, cin, cout, k, s, p, r1, r1 if svd else r2, dens, dtype, svd, seed=17)
    inp = workloads.generate(cfg)
    layer = LrsConv.from_inputs(inp)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    ny = n * cfg.out_h * cfg.out_w * cout
    buf = torch.empty(GUARD + ny + GUARD, dtype=tdt, device="cuda")
    buf.view(torch.int16 if dtype == "bf16" else torch.int32).fill_(0x5A5A)
    guard_lo, guard_hi = buf[:GUARD].clone(), buf[GUARD + ny:].clone()
    y = buf[GUARD:GUARD + ny].view(n, cfg.out_h, cfg.out_w, cout)
    # the input sits inside a larger buffer too (reads past it would pick up the pattern)
    nx = n * h * w * cin
    xbuf = torch.full((GUARD + nx + GUARD,), float("nan"), dtype=tdt, device="cuda")
    x = xbuf[GUARD:GUARD + nx].view(n, h, w, cin)
    x.copy_(torch.from_numpy(inp.x).to(tdt))
    layer.forward_into(x, y)
    torch.cuda.synchronize()
    assert torch.equal(buf[:GUARD], guard_lo), "write before Y"
    assert torch.equal(buf[GUARD + ny:], guard_hi), "write past Y"
    assert torch.isfinite(y.float()).all(), "non-finite output (an out-of-bounds read of X's NaN guard?)"
    ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                             inp.values, cfg.stride, cfg.pad)
    parity.check(y, ref, dtype)
