"""Pins of the fp64 backward oracle (oracle/lrs_backward.py) against things other
than itself (CPU only): torch.autograd in fp64 (a library's reverse mode through
torch.nn.functional.conv2d, and through the factor chain with the S values as
leaf tensors), the adjoint identity <conv(X, W), dY> = <X, conv^T(dY, W)>,
central finite differences, and the agreement of the two formulations
(definition vs back-propagation through the method's stages).  A dropped term,
a flipped tap, a transposed factor or a wrong stride/pad offset in either
formulation fails at least one of them.  PAPER.md:194-195 (§3.5, fine-tuning by
ordinary back-propagation), :125 (W = L + S), :160 (the convolution).
"""
import numpy as np
import pytest
import torch

from oracle import lrs_oracle as O
from oracle import lrs_backward as B
from test_oracle_pins import rand_layer, rel_l2

CASES = [  # (n, h, w, cin, cout, k, s, p, r1, r2, nnz, svd)
    (2, 7, 6, 5, 6, 3, 1, 1, 3, 4, 20, False),
    (2, 9, 8, 5, 6, 3, 2, 1, 3, 2, 25, False),
    (1, 8, 7, 4, 3, 5, 1, 2, 2, 3, 30, False),
    (2, 6, 5, 4, 7, 1, 1, 0, 3, 3, 6, True),
    (1, 6, 6, 3, 4, 3, 1, 0, 2, 2, 9, False),  # pad 0: output smaller than input
]


def torch_autograd(x, dy, u_in, core, u_out, row_ptr, col_idx, values, s, p):
    """Library pin: torch reverse mode in fp64 through the factor chain, with W
    assembled from leaf tensors (U_in, G, U_out, S values) exactly as PAPER.md:125
    states W = L + S, and Y = conv2d(X, W)."""
    k = 1 if core is None else core.shape[2]
    cin, cout = u_in.shape[0], u_out.shape[1]
    t = lambda a: torch.tensor(np.asarray(a, np.float64), requires_grad=True)
    xt, ui, uo, vt = t(x), t(u_in), t(u_out), t(values)
    gt = None if core is None else t(core)
    wl = (ui @ uo)[:, :, None, None] if core is None else torch.einsum("ca,abyx,bj->cjyx", ui, gt, uo)
    rows = np.repeat(np.arange(cout), np.diff(row_ptr))
    c, rem = np.divmod(col_idx.astype(np.int64), k * k)
    yy, xx = np.divmod(rem, k)
    ws = torch.zeros((cin, cout, k, k), dtype=torch.float64).index_put(
        (torch.from_numpy(c), torch.from_numpy(rows), torch.from_numpy(yy), torch.from_numpy(xx)), vt,
        accumulate=True)
    w = wl + ws
    y = torch.nn.functional.conv2d(xt.permute(0, 3, 1, 2), w.permute(1, 0, 2, 3), stride=s, padding=p)
    y.permute(0, 2, 3, 1).backward(torch.from_numpy(np.asarray(dy, np.float64)))
    return {"dx": xt.grad.numpy(), "d_u_in": ui.grad.numpy(), "d_core": None if gt is None else gt.grad.numpy(),
            "d_u_out": uo.grad.numpy(), "d_values": vt.grad.numpy()}


def case_arrays(case, seed=0):
    n, h, w, cin, cout, k, s, p, r1, r2, nnz, svd = case
    rng = np.random.default_rng(seed)
    x, u_in, core, u_out, row_ptr, col_idx, vals = rand_layer(rng, n, h, w, cin, cout, k, r1, r2, nnz, svd)
    ho, wo = O.out_size(h, k, s, p), O.out_size(w, k, s, p)
    dy = rng.standard_normal((n, ho, wo, cout))
    return x, dy, u_in, core, u_out, row_ptr, col_idx, vals, s, p


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("form", ["dense", "factored"])
def test_backward_matches_torch_autograd(case, form):
    x, dy, u_in, core, u_out, rp, ci, va, s, p = case_arrays(case)
    fn = B.backward_dense if form == "dense" else B.backward_factored
    got = fn(x, dy, u_in, core, u_out, rp, ci, va, s, p)
    ref = torch_autograd(x, dy, u_in, core, u_out, rp, ci, va, s, p)
    for key in ("dx", "d_u_in", "d_core", "d_u_out", "d_values"):
        if ref[key] is None:
            assert got[key] is None
            continue
        assert got[key].shape == ref[key].shape, key
        assert rel_l2(got[key], ref[key]) < 1e-12, key


@pytest.mark.parametrize("case", CASES)
def test_adjoint_identity(case):
    """<conv(X, W), dY> = <X, conv^T(dY, W)>: conv_adjoint_input is the adjoint
    of the oracle's forward (an exact identity of linear maps)."""
    x, dy, u_in, core, u_out, rp, ci, va, s, p = case_arrays(case, seed=3)
    y = O.forward_dense(x, u_in, core, u_out, rp, ci, va, s, p)
    dx = B.backward_dense(x, dy, u_in, core, u_out, rp, ci, va, s, p)["dx"]
    lhs, rhs = float(np.sum(y * dy)), float(np.sum(x * dx))
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs))


def test_finite_differences():
    """Central differences of L = <Y(theta), dY> in a few coordinates of every
    parameter and of X (exact up to O(h^2) = 0: L is linear in each one)."""
    case = CASES[0]
    x, dy, u_in, core, u_out, rp, ci, va, s, p = case_arrays(case, seed=5)
    g = B.backward_factored(x, dy, u_in, core, u_out, rp, ci, va, s, p)

    def loss(xx=x, ui=u_in, gg=core, uo=u_out, vv=va):
        return float(np.sum(O.forward_factored(xx, ui, gg, uo, rp, ci, vv, s, p) * dy))

    h = 1e-3
    rng = np.random.default_rng(1)
    for name, arr, key in (("xx", x, "dx"), ("ui", u_in, "d_u_in"), ("gg", core, "d_core"),
                           ("uo", u_out, "d_u_out"), ("vv", va, "d_values")):
        for _ in range(3):
            idx = tuple(int(rng.integers(0, d)) for d in arr.shape)
            a1, a2 = arr.copy(), arr.copy()
            a1[idx] += h
            a2[idx] -= h
            fd = (loss(**{name: a1}) - loss(**{name: a2})) / (2 * h)
            assert abs(fd - g[key][idx]) <= 1e-7 * max(1.0, abs(fd)), (key, idx)


@pytest.mark.parametrize("case", CASES)
def test_dense_equals_factored_and_values_are_dw_at_support(case):
    x, dy, u_in, core, u_out, rp, ci, va, s, p = case_arrays(case, seed=7)
    a = B.backward_dense(x, dy, u_in, core, u_out, rp, ci, va, s, p)
    b = B.backward_factored(x, dy, u_in, core, u_out, rp, ci, va, s, p)
    for key in ("dx", "d_u_in", "d_u_out", "d_values"):
        assert rel_l2(a[key], b[key]) < 1e-12, key
    if core is not None:
        assert rel_l2(a["d_core"], b["d_core"]) < 1e-12
    # the full weight gradient with torch's conv2d weight-gradient routine (library pin)
    k = a["dw"].shape[2]
    xt = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 3, 1, 2)))
    gt = torch.from_numpy(np.ascontiguousarray(dy.transpose(0, 3, 1, 2)))
    dw_t = torch.nn.grad.conv2d_weight(xt, (dy.shape[3], x.shape[3], k, k), gt, stride=case[6], padding=case[7])
    assert rel_l2(a["dw"], dw_t.numpy().transpose(1, 0, 2, 3)) < 1e-12


@pytest.mark.parametrize("case", [c for c in CASES if c[6] == 1])
def test_transposed_layer_forward_is_dx(case):
    """At stride 1, the forward of the transposed layer (U_out^T, flipped G^T,
    U_in^T, S by input channel, pad k-1-p) on dY is dX -- the construction the
    GPU path uses for its input gradient."""
    x, dy, u_in, core, u_out, rp, ci, va, s, p = case_arrays(case, seed=9)
    dx = B.backward_dense(x, dy, u_in, core, u_out, rp, ci, va, s, p)["dx"]
    ui, g, uo, rp2, ci2, va2, p2 = B.transposed_layer(u_in, core, u_out, rp, ci, va, x.shape[3], p)
    y = O.forward_factored(dy, ui, g, uo, rp2, ci2, va2, 1, p2)
    assert y.shape == dx.shape
    assert rel_l2(y, dx) < 1e-12


@pytest.mark.parametrize("case", [c for c in CASES if c[5] > 1])
def test_cp_backward_matches_torch_autograd(case):
    """The CP layer's gradients (PAPER.md:137 L = A o B o C o D, fine-tuned per §3.5) against
    torch reverse mode in fp64 through the CP reconstruction and conv2d."""
    n, h, w, cin, cout, k, s, p, r1, r2, nnz, svd = case
    rng = np.random.default_rng(11)
    x, _, _, _, row_ptr, col_idx, vals = rand_layer(rng, n, h, w, cin, cout, k, r1, r2, nnz)
    r = 3
    a, b, c, d = (rng.standard_normal(sh) for sh in ((cin, r), (k, r), (k, r), (cout, r)))
    ho, wo = O.out_size(h, k, s, p), O.out_size(w, k, s, p)
    dy = rng.standard_normal((n, ho, wo, cout))
    got = B.backward_cp(x, dy, a, b, c, d, row_ptr, col_idx, vals, s, p)
    t = lambda v: torch.tensor(v, requires_grad=True)
    xt, at, bt, ct, dt, vt = t(x), t(a), t(b), t(c), t(d), t(vals)
    wl = torch.einsum("ir,kr,pr,jr->ijkp", at, bt, ct, dt)
    rows = np.repeat(np.arange(cout), np.diff(row_ptr))
    cc, rem = np.divmod(col_idx.astype(np.int64), k * k)
    yy, xx = np.divmod(rem, k)
    ws = torch.zeros((cin, cout, k, k), dtype=torch.float64).index_put(
        (torch.from_numpy(cc), torch.from_numpy(rows), torch.from_numpy(yy), torch.from_numpy(xx)), vt, accumulate=True)
    y = torch.nn.functional.conv2d(xt.permute(0, 3, 1, 2), (wl + ws).permute(1, 0, 2, 3), stride=s, padding=p)
    y.permute(0, 2, 3, 1).backward(torch.from_numpy(dy))
    for key, tt in (("dx", xt), ("d_a", at), ("d_b", bt), ("d_c", ct), ("d_d", dt), ("d_values", vt)):
        assert rel_l2(got[key], tt.grad.numpy()) < 1e-12, key
