"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a library routine
(torch.nn.functional.conv2d in fp64), an independent brute-force loop, a
closed form or value printed in PAPER.md / SPEC.md, or an exact algebraic
invariant.  A plausible slip in the oracle (dropped term, wrong sign of a tap
displacement, transposed factor, off-by-one in stride/pad) fails at least one.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_oracle as O


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def torch_conv_nhwc(x, w_cjyx, stride, pad):
    """Library pin: torch conv2d (fp64, CPU) with W in (in,out,ky,kx) -> OIHW."""
    xt = torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float64).transpose(0, 3, 1, 2)))
    wt = torch.from_numpy(np.ascontiguousarray(np.asarray(w_cjyx, np.float64).transpose(1, 0, 2, 3)))
    y = torch.nn.functional.conv2d(xt, wt, stride=stride, padding=pad)
    return y.numpy().transpose(0, 2, 3, 1)


def rand_layer(rng, n, h, w, cin, cout, k, r1, r2, nnz, svd=False):
    x = rng.standard_normal((n, h, w, cin))
    u_in = rng.standard_normal((cin, r1))
    core = None if svd else rng.standard_normal((r1, r2, k, k))
    u_out = rng.standard_normal((r1 if svd else r2, cout))
    numel = cout * cin * k * k
    pos = np.sort(rng.choice(numel, size=nnz, replace=False))
    rows, cols = pos // (cin * k * k), pos % (cin * k * k)
    row_ptr = np.zeros(cout + 1, np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    vals = rng.standard_normal(nnz)
    return x, u_in, core, u_out, row_ptr, cols.astype(np.int32), vals


CONV_CASES = [  # (n, h, w, cin, cout, k, s, p)
    (2, 9, 7, 5, 6, 3, 1, 1),
    (2, 9, 8, 5, 6, 3, 2, 1),
    (1, 6, 6, 4, 3, 1, 1, 0),
    (1, 11, 10, 3, 4, 5, 1, 2),
    (2, 8, 9, 3, 2, 3, 1, 0),
    (1, 13, 12, 3, 4, 7, 2, 3),
    (1, 5, 5, 2, 2, 1, 2, 0),
]


@pytest.mark.parametrize("n,h,w,cin,cout,k,s,p", CONV_CASES)
def test_conv_direct_matches_torch_conv2d(n, h, w, cin, cout, k, s, p):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, h, w, cin))
    wt = rng.standard_normal((cin, cout, k, k))
    assert rel_l2(O.conv_direct(x, wt, s, p), torch_conv_nhwc(x, wt, s, p)) < 1e-13


@pytest.mark.parametrize("s,p", [(1, 1), (2, 1), (1, 0), (2, 0)])
def test_conv_direct_matches_brute_force_loop(s, p):
    """a second, independently written quintuple loop."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 5, 6, 3))
    wt = rng.standard_normal((3, 4, 3, 3))
    assert rel_l2(O.conv_direct(x, wt, s, p), O.brute_force_conv(x, wt, s, p)) < 1e-13


@pytest.mark.parametrize("n,h,w,cin,cout,k,s,p", [c for c in CONV_CASES])
def test_factored_equals_dense_and_torch(n, h, w, cin, cout, k, s, p):
    """O2 (the method) == O1 (W = L + S densely) == torch conv2d on W."""
    rng = np.random.default_rng(3)
    svd = (k == 1 and p == 0 and s == 1)
    r1 = 3
    nnz = max(1, (cout * cin * k * k) // 10)
    x, u_in, core, u_out, rp, ci, v = rand_layer(rng, n, h, w, cin, cout, k, r1, 2, nnz, svd)
    y2 = O.forward_factored(x, u_in, core, u_out, rp, ci, v, s, p)
    y1 = O.forward_dense(x, u_in, core, u_out, rp, ci, v, s, p)
    assert rel_l2(y2, y1) < 1e-12
    wfull = O.reconstruct_tucker2(u_in, core, u_out) + O.densify_sparse(cin, cout, k, rp, ci, v)
    assert rel_l2(y2, torch_conv_nhwc(x, wfull, s, p)) < 1e-12


def test_tucker2_reconstruction_matches_explicit_sum():
    """W_L[c,j,y,x] = sum_ab U_in[c,a] G[a,b,y,x] U_out[b,j], element by element."""
    rng = np.random.default_rng(4)
    u_in, g, u_out = rng.standard_normal((3, 2)), rng.standard_normal((2, 4, 3, 3)), rng.standard_normal((4, 5))
    wl = O.reconstruct_tucker2(u_in, g, u_out)
    c, j, y, x = 2, 3, 0, 2
    ref = sum(u_in[c, a] * g[a, b, y, x] * u_out[b, j] for a in range(2) for b in range(4))
    assert abs(wl[c, j, y, x] - ref) < 1e-13


def test_tucker_with_identity_factors_is_dense_conv():
    """U_in = I (R1 = Cin), U_out = I (R2 = Cout): the chain reduces to a dense
    k x k convolution with the core as its weight."""
    rng = np.random.default_rng(5)
    cin, cout, k = 4, 5, 3
    x = rng.standard_normal((2, 7, 6, cin))
    g = rng.standard_normal((cin, cout, k, k))
    y = O.forward_factored(x, np.eye(cin), g, np.eye(cout), np.zeros(cout + 1, np.int64),
                           np.zeros(0, np.int32), np.zeros(0), 1, 1)
    assert rel_l2(y, torch_conv_nhwc(x, g, 1, 1)) < 1e-13


def test_linearity_in_terms_and_scaling():
    """conv(X, L+S) = conv(X, L) + conv(X, S) (BASELINE north
    star); scaling X by 2 scales Y by exactly 2 (power-of-two, no rounding)."""
    rng = np.random.default_rng(6)
    x, u_in, core, u_out, rp, ci, v = rand_layer(rng, 2, 8, 8, 6, 7, 3, 3, 4, 30)
    y = O.forward_factored(x, u_in, core, u_out, rp, ci, v, 1, 1)
    y_l = O.forward_factored(x, u_in, core, u_out, np.zeros(8, np.int64), np.zeros(0, np.int32), np.zeros(0), 1, 1)
    y_s = O.forward_factored(x, u_in, core, np.zeros_like(u_out), rp, ci, v, 1, 1)
    assert rel_l2(y, y_l + y_s) < 1e-14
    y2 = O.forward_factored(2 * x, u_in, core, u_out, rp, ci, v, 1, 1)
    assert np.array_equal(y2, 2 * y)
    x2 = rng.standard_normal(x.shape)
    ya = O.forward_factored(3 * x + x2, u_in, core, u_out, rp, ci, v, 1, 1)
    yb = 3 * y + O.forward_factored(x2, u_in, core, u_out, rp, ci, v, 1, 1)
    assert rel_l2(ya, yb) < 1e-13


def test_identity_and_zero_kernels():
    """identity 1x1 kernel -> Y = X; zero kernel -> Y = 0."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((1, 5, 4, 3))
    assert np.array_equal(O.conv_direct(x, np.eye(3)[:, :, None, None]), x)
    assert not O.conv_direct(x, np.zeros((3, 2, 3, 3)), 1, 1).any()
    # SVD pair with U = I, V = I and no S is the identity too
    y = O.forward_factored(x, np.eye(3), None, np.eye(3), np.zeros(4, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert np.array_equal(y, x)


def test_sparse_single_centre_tap_copies_channel():
    """one centre entry of value 1, i = j = 0 -> Y[...,0] = X[...,0]."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((2, 6, 5, 3))
    k = 3
    col = (0 * k + 1) * k + 1
    y = O.sparse_conv_scatter(x, 2, k, np.array([0, 1, 1]), np.array([col], np.int32), np.array([1.0]), 1, 1)
    assert np.array_equal(y[..., 0], x[..., 0])
    assert not y[..., 1].any()


@pytest.mark.parametrize("dy,dx", [(1, 1), (-1, 1), (1, 0), (0, -1)])
def test_paper_displacement_rule(dy, dx):
    """an entry at kernel position (1, 1) relative to the centre
    displaces its contribution by (-1, -1)."""
    x = np.zeros((1, 7, 7, 1))
    h0, w0 = 3, 4
    x[0, h0, w0, 0] = 1.0
    k = 3
    col = (0 * k + (dy + 1)) * k + (dx + 1)
    y = O.sparse_conv_scatter(x, 1, k, np.array([0, 1]), np.array([col], np.int32), np.array([2.5]), 1, 1)
    nz = np.argwhere(y[0, :, :, 0] != 0)
    assert nz.tolist() == [[h0 - dy, w0 - dx]]
    assert y[0, h0 - dy, w0 - dx, 0] == 2.5


def test_cp_rank1_all_ones_hand_value():
    """rank-1 all-ones CP factors, all-ones input, 1x1 kernel ->
    constant output equal to the number of input channels I."""
    i_ch = 3
    x = np.ones((1, 4, 4, i_ch))
    y = O.cp_conv(x, np.ones((i_ch, 1)), np.ones((1, 1)), np.ones((1, 1)), np.ones((1, 1)))
    assert np.array_equal(y, np.full((1, 4, 4, 1), float(i_ch)))


def test_cp_chain_equals_dense_and_tucker_embedding():
    """the 4-stage CP chain equals the dense conv with the
    reconstructed CP kernel, and the CP form is the Tucker-2
    special case G[a,b,y,x] = delta_ab B[y,a] C[x,a] (reading #1)."""
    rng = np.random.default_rng(9)
    i_ch, j_ch, k, r = 5, 4, 3, 3
    a, b, c, d = (rng.standard_normal(s) for s in ((i_ch, r), (k, r), (k, r), (j_ch, r)))
    x = rng.standard_normal((2, 6, 7, i_ch))
    y_cp = O.cp_conv(x, a, b, c, d)
    y_dense = O.conv_direct(x, O.reconstruct_cp(a, b, c, d), 1, 1)
    assert rel_l2(y_cp, y_dense) < 1e-13
    g = np.zeros((r, r, k, k))
    for q in range(r):
        g[q, q] = np.outer(b[:, q], c[:, q])
    y_t = O.forward_factored(x, a, g, d.T, np.zeros(j_ch + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), 1, 1)
    assert rel_l2(y_t, y_cp) < 1e-13


def test_rank_permutation_invariance():
    rng = np.random.default_rng(10)
    x, u_in, core, u_out, rp, ci, v = rand_layer(rng, 1, 6, 6, 4, 5, 3, 4, 3, 10)
    perm = rng.permutation(4)
    y0 = O.forward_factored(x, u_in, core, u_out, rp, ci, v, 1, 1)
    y1 = O.forward_factored(x, u_in[:, perm], core[perm], u_out, rp, ci, v, 1, 1)
    assert rel_l2(y0, y1) < 1e-13


def test_interior_translation_equivariance():
    """shifting X by one pixel shifts Y identically away from borders."""
    rng = np.random.default_rng(11)
    x, u_in, core, u_out, rp, ci, v = rand_layer(rng, 1, 10, 10, 3, 4, 3, 2, 2, 12)
    xs = np.zeros_like(x)
    xs[:, 1:, :, :] = x[:, :-1, :, :]
    y0 = O.forward_factored(x, u_in, core, u_out, rp, ci, v, 1, 1)
    y1 = O.forward_factored(xs, u_in, core, u_out, rp, ci, v, 1, 1)
    assert rel_l2(y1[:, 2:-1], y0[:, 1:-2]) < 1e-13


def test_param_counts_closed_forms():
    """P(W) = IJKT and P(L) = r(I+J+K+T) for the CP form, checked
    against counting the entries of the factor arrays; Tucker-2 counts of the
    four configs."""
    i_ch, j_ch, k, r = 64, 128, 3, 7
    a, b, c, d = np.ones((i_ch, r)), np.ones((k, r)), np.ones((k, r)), np.ones((j_ch, r))
    assert O.cp_param_count(i_ch, j_ch, k, k, r) == a.size + b.size + c.size + d.size
    assert O.param_counts(i_ch, j_ch, k, 4, 4, 0)["P_W"] == O.reconstruct_cp(a, b, c, d).size
    expect = {"c1": (36864, 4352), "c2_bf16": (589824, 69632), "c3": (2359296, 278528), "c4": (262144, 81920)}
    for name, (pw, pl) in expect.items():
        cfg = workloads.CONFIGS[name]
        got = O.param_counts(cfg.c_in, cfg.c_out, cfg.k, cfg.rank_in, cfg.rank_out, cfg.nnz, cfg.svd)
        assert (got["P_W"], got["P_L"]) == (pw, pl)
        inp = workloads.generate(cfg.replace(batch=1) if name != "c3" else cfg.replace(batch=1))
        n_l = inp.u_in.size + (0 if inp.core is None else inp.core.size) + inp.u_out.size
        assert n_l == pl


def test_table2_total_params_and_strides():
    """the conv kernels of ResNet-50 hold 23,454,912 parameters;
    Table 2 has 53 layers; the 16 3x3 layers, three of them
    stride 2 (input size of the next layer halves)."""
    rows = workloads.resnet50_table2()
    assert len(rows) == 53
    assert sum(cout * cin * k * k for _, cin, _, _, cout, k in rows) == 23454912
    three = [r for r in rows if r[5] == 3]
    assert [r[0] for r in three] == sorted(workloads.RESNET50_COMPRESSED_3X3)
    by_idx = {r[0]: r for r in rows}
    for idx, s in workloads.RESNET50_COMPRESSED_3X3.items():
        h_in = by_idx[idx][2]
        h_next = by_idx[idx + 1][2]
        assert h_next == O.out_size(h_in, 3, s, 1)


def test_pack_sparse_slices_spec_examples():
    """empty -> empty slices; (i=2, j=5, kx=1, ky=2) in a 3x3
    kernel -> packed 50 in slice 2; J=2048 3x3 still fits u16; round trip."""
    k = 3
    vals, packed = O.pack_sparse_slices(3, 8, k, np.zeros(9, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert all(len(v) == 0 for v in vals)
    col = (2 * k + 1) * k + 2
    rp = np.zeros(9, np.int64)
    rp[6:] = 1
    vals, packed = O.pack_sparse_slices(3, 8, k, rp, np.array([col], np.int32), np.array([0.5]))
    assert packed[2].tolist() == [50] and packed[2].dtype == np.uint16
    _, p2 = O.pack_sparse_slices(1, 2048, k, np.r_[np.zeros(2048, np.int64), 1], np.array([8], np.int32), np.array([1.0]))
    assert p2[0].dtype == np.uint16 and int(p2[0][0]) == 2047 * 9 + 8
    rng = np.random.default_rng(12)
    *_, rp, ci, v = rand_layer(rng, 1, 3, 3, 6, 9, 3, 1, 1, 40)
    rp2, ci2, v2 = O.unpack_sparse_slices(6, 9, 3, *O.pack_sparse_slices(6, 9, 3, rp, ci, v))
    assert np.array_equal(rp2, rp) and np.array_equal(ci2, ci)
    assert np.array_equal(v2, np.asarray(v, np.float32))


@pytest.mark.parametrize("s,p,k", [(1, 1, 3), (2, 1, 3), (1, 0, 1)])
def test_sparse_mac_count_matches_ones_convolution(s, p, k):
    """Closed-form in-bounds MAC count == sum of Y_S with X = 1 and v = 1."""
    rng = np.random.default_rng(13)
    n, h, w, cin, cout = 2, 9, 7, 3, 4
    *_, rp, ci, _ = rand_layer(rng, n, h, w, cin, cout, k, 1, 1, min(20, cout * cin * k * k // 2))
    y = O.sparse_conv_scatter(np.ones((n, h, w, cin)), cout, k, rp, ci, np.ones(len(ci)), s, p)
    assert int(round(y.sum())) == O.sparse_mac_count(n, h, w, k, s, p, ci)


def test_workload_generator_contract():
    """nnz per config (369 of 36864 etc.), CSR well-formed, deterministic,
    bf16 rounding equals torch's own float32 -> bfloat16 conversion."""
    expect = {"c1": 369, "c2_f32": 11796, "c2_bf16": 11796, "c3": 117965, "c4": 2621}
    for name, nnz in expect.items():
        cfg = workloads.CONFIGS[name]
        assert cfg.nnz == nnz
        inp = workloads.generate(cfg, batch=1)
        assert inp.row_ptr[0] == 0 and inp.row_ptr[-1] == nnz and len(inp.col_idx) == nnz
        assert np.all(np.diff(inp.row_ptr) >= 0)
        for j in range(0, cfg.c_out, max(1, cfg.c_out // 16)):
            c = inp.col_idx[inp.row_ptr[j]:inp.row_ptr[j + 1]]
            assert np.all(np.diff(c) > 0) and (c.size == 0 or c.max() < cfg.c_in * cfg.k ** 2)
        assert (inp.x >= 0).all()
    a = workloads.generate(workloads.CONFIGS["c1"])
    b = workloads.generate(workloads.CONFIGS["c1"])
    assert np.array_equal(a.x, b.x) and np.array_equal(a.values, b.values)
    r = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 7
    ref = torch.from_numpy(r).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(workloads.bf16_round(r), ref)


def test_c5_reference_network_pinned_to_dense_conv2d():
    """C5 oracle (§5.5): the ResNet-50 whose 16 3x3 convs are
    evaluated by forward_factored (and its other convs by conv_direct) equals
    the same network with each conv2 weight set to the dense W = L + S and
    every conv run by torch's own fp64 conv2d (an independent library route;
    strides of layer{2,3,4}.0.conv2 included).  32x32 images keep torch's fp64
    CPU convs fast; both routes are size-agnostic."""
    import workloads
    from oracle import resnet_oracle as R
    img = workloads.resnet50_images(1, seed=3)[:, :, :32, :32].copy()
    a = R.reference_logits(img)
    b = R.reference_logits(img, dense_conv2=True, torch_convs=True)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-10
    layers = workloads.resnet50_compressed_layers()
    assert len(layers) == 16
    assert sum(c.stride == 2 for _, _, c in layers) == 3
    assert {n for _, n, c in layers if c.stride == 2} == {"layer2.0.conv2", "layer3.0.conv2", "layer4.0.conv2"}


@pytest.mark.parametrize("stride,pad", [(1, 1), (2, 1), (1, 0)])
def test_forward_cp_against_brute_force(stride, pad):
    """O.forward_cp (the CP layer the GPU CP path is compared with) against the
    independent quintuple loop on the densified kernel, tiny input: the CP
    kernel L = A_ir B_kr C_pr D_jr written out with loops here,
    plus the sparse entries placed by hand."""
    rng = np.random.default_rng(21)
    i_ch, j_ch, k, r = 3, 4, 3, 2
    a, b, c, d = (rng.standard_normal(s) for s in ((i_ch, r), (k, r), (k, r), (j_ch, r)))
    x = rng.standard_normal((1, 5, 6, i_ch))
    w = np.zeros((i_ch, j_ch, k, k))
    for ii in range(i_ch):
        for jj in range(j_ch):
            for y in range(k):
                for xx in range(k):
                    w[ii, jj, y, xx] = sum(a[ii, q] * b[y, q] * c[xx, q] * d[jj, q] for q in range(r))
    row_ptr = np.array([0, 1, 1, 3, 3], np.int64)
    col_idx = np.array([4, 0, 26], np.int32)        # (c*k + y)*k + x
    values = np.array([0.5, -1.0, 2.0])
    w[0, 0, 1, 1] += 0.5
    w[0, 2, 0, 0] += -1.0
    w[2, 2, 2, 2] += 2.0
    ref = O.brute_force_conv(x, w, stride, pad)
    got = O.forward_cp(x, a, b, c, d, row_ptr, col_idx, values, stride, pad)
    assert rel_l2(got, ref) < 1e-13


def test_output_epilogue_hand_values():
    """The fused output epilogue (BatchNorm-style affine + ReLU per output channel) on
    a hand-computed case: channel 0 -> 2*y - 1, channel 1 -> -y + 0.5, then ReLU."""
    y = np.array([[[[1.0, 1.0], [0.25, -2.0]]]])
    got = O.output_epilogue(y, [2.0, -1.0], [-1.0, 0.5], relu=True)
    assert np.array_equal(got, np.array([[[[1.0, 0.0], [0.0, 2.5]]]]))
    assert np.array_equal(O.output_epilogue(y), y)
    assert np.array_equal(O.output_epilogue(y, bias=[1.0, 0.0]), y + np.array([1.0, 0.0]))
