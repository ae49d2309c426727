"""GPU parity of the low-rank + sparse decomposition
against the fp64 oracle (oracle/lrs_decomp.py, pinned in tests/test_decomp_oracle.py),
through the C-ABI (lrs_decomp_create / lrs_decomp_run).

Both sides compute in fp64; the projection P_c is integer / index work and must select
exactly the oracle's entries (ties to the smaller index) -- bit-exact when both sides see
the same tensor (zero initial factors make L = 0, so P_c acts on W itself), and identical
supports along short runs where the residuals agree to ~1e-13.  Factors and eps histories
within 1e-8 relative (fp64, different summation orders).
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import lrs_decomp as D

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_gpu(w, f0, card, iters, tol=0.0, rcond=1e-10):
    from paper_2006_06443_b200 import LrsDecomp
    dc = LrsDecomp(w.shape, f0[0].shape[1], card, max_iters=iters, tol=tol, rcond=rcond)
    wd = torch.from_numpy(np.ascontiguousarray(w, np.float64)).cuda()
    fs = [torch.from_numpy(np.ascontiguousarray(f, np.float64)).cuda() for f in f0]
    idx, val, eps = dc.run(wd, fs)
    torch.cuda.synchronize()
    return [f.cpu().numpy() for f in fs], idx.cpu().numpy(), val.cpu().numpy(), eps


def test_projection_exact_with_ties():
    """Zero initial factors keep L = 0 (V = 0 has an empty pseudo-inverse), so S = P_c(W):
    the GPU's radix select + ordered compaction must pick exactly the oracle's entries,
    including runs of equal |value| decided by the index."""
    rng = np.random.default_rng(0)
    dims = (64, 48, 3, 3)
    w = np.round(rng.standard_normal(dims) * 4) / 4  # many exact ties in |w|
    f0 = [np.zeros((d, 4)) for d in dims]
    for card in (0.0, 0.001, 0.01, 0.05, 0.3):
        f, idx, val, eps = run_gpu(w, f0, card, 1)
        ridx, rval = D.project_sparse(w, card)
        assert np.array_equal(idx, ridx), card
        assert np.array_equal(val, rval), card
        assert all(not np.any(x) for x in f)


@pytest.mark.parametrize("rank", [8, 33])
def test_one_iteration_matches_oracle(rank):
    rng = np.random.default_rng(1)
    dims = (40, 36, 3, 3)
    w = rng.standard_normal(dims)
    f0 = [rng.standard_normal((d, rank)) for d in dims]
    f, idx, val, eps = run_gpu(w, f0, 0.02, 1)
    rf, (ridx, rval), reps = D.decompose_lrs(w, f0, 0.02, max_iters=1, tol=0.0)
    for m in range(4):
        assert rel(f[m], rf[m]) < 1e-8, m
    assert np.array_equal(idx, ridx)
    assert rel(val, rval) < 1e-8
    assert abs(eps[0] - reps[0]) < 1e-9


def test_iterations_match_oracle_on_a_planted_tensor():
    cfg = workloads.DecompConfig("t", (48, 40, 3, 3), 6, 8, 0.01)
    w, f0 = workloads.generate_decomp(cfg)
    f, idx, val, eps = run_gpu(w, f0, cfg.cardinality, 12)
    rf, (ridx, rval), reps = D.decompose_lrs(w, f0, cfg.cardinality, max_iters=12, tol=0.0)
    assert len(eps) == len(reps) == 12
    assert np.allclose(eps, reps, rtol=1e-7, atol=1e-12)
    assert np.array_equal(idx, ridx)
    l_gpu = D.cp_reconstruct(f)
    assert rel(l_gpu, D.cp_reconstruct(rf)) < 1e-7


def test_planted_spikes_recovered_on_gpu():
    """SPEC.md:167 (as in tests/test_decomp_oracle.py): rank 2 + 1 % spikes of magnitude 10."""
    rng = np.random.default_rng(7)
    dims = (10, 10, 3, 3)
    low = D.cp_reconstruct([rng.standard_normal((d, 2)) for d in dims])
    n = int(round(0.01 * low.size))
    spikes = np.sort(rng.choice(low.size, n, replace=False))
    w = low.copy()
    w.flat[spikes] += 10.0 * np.sign(rng.standard_normal(n))
    f, idx, val, eps = run_gpu(w, D.svd_init(w, 2), 0.01, 300, tol=0.0)
    assert eps[-1] < 1e-3
    assert np.array_equal(idx, spikes)


def test_stopping_rule_determinism_and_zero_w():
    cfg = workloads.DecompConfig("t", (32, 24, 3, 3), 4, 6, 0.02, seed=3)
    w, f0 = workloads.generate_decomp(cfg)
    a = run_gpu(w, f0, cfg.cardinality, 200, tol=1e-4)
    b = run_gpu(w, f0, cfg.cardinality, 200, tol=1e-4)
    _, _, reps = D.decompose_lrs(w, f0, cfg.cardinality, max_iters=200, tol=1e-4)
    assert len(a[3]) == len(reps) < 200  # the same stopping iteration as the oracle
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(x, y)  # bitwise reproducible
    assert np.array_equal(a[1], b[1]) and a[3] == b[3]
    z = np.zeros((8, 8, 3, 3))
    f, idx, val, eps = run_gpu(z, [np.ones((d, 3)) for d in z.shape], 0.05, 10)
    assert idx.size == 0 and eps == [0.0] and all(not np.any(x) for x in f)


def test_full_size_c3_weight():
    """The C3 layer's weight shape (512 x 512 x 3 x 3), rank 128, c = 1 %: three iterations
    against the oracle (eps history, factors, S support)."""
    cfg = workloads.DECOMP_CONFIGS["c3_decomp"]
    w, f0 = workloads.generate_decomp(cfg)
    f, idx, val, eps = run_gpu(w, f0, cfg.cardinality, 3)
    rf, (ridx, rval), reps = D.decompose_lrs(w, f0, cfg.cardinality, max_iters=3, tol=0.0)
    assert np.allclose(eps, reps, rtol=1e-7)
    assert np.array_equal(idx, ridx)
    for m in range(4):
        assert rel(f[m], rf[m]) < 1e-6, m


def test_eigen_path_equals_cholesky_path(monkeypatch):
    """The pseudo-inverse's two paths (include/lrs_conv.h: the certified Cholesky inverse, and
    the Jacobi eigensolver with the rcond cutoff, forced by LRS_DECOMP_EIGEN) give the same
    iterations up to fp64 rounding, both against the oracle."""
    cfg = workloads.DecompConfig("t", (64, 56, 3, 3), 8, 12, 0.01, seed=5)
    w, f0 = workloads.generate_decomp(cfg)
    a = run_gpu(w, f0, cfg.cardinality, 6)
    monkeypatch.setenv("LRS_DECOMP_EIGEN", "1")
    b = run_gpu(w, f0, cfg.cardinality, 6)
    _, (ridx, _), reps = D.decompose_lrs(w, f0, cfg.cardinality, max_iters=6, tol=0.0)
    assert np.allclose(a[3], b[3], rtol=1e-9) and np.allclose(a[3], reps, rtol=1e-8)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[1], ridx)
    for x, y in zip(a[0], b[0]):
        assert rel(x, y) < 1e-8


def test_decomposed_weight_runs_as_a_cp_layer():
    """The paper's pipeline end to end on the GPU: decompose a conv weight W[c][j][y][x] into
    CP factors + S (f4), load them as a CP layer (F0 = A = u_in, F1 = D,
    F2 = B, F3 = C; S's linear indices -> CSR by output channel) and run
    its forward: Y = conv(X, L + S) of the decomposed weight (the fp64 oracle on the same
    factors), and ||W - L - S|| / ||W|| equal to the decomposition's last eps."""
    from paper_2006_06443_b200 import LrsConv
    from oracle import lrs_oracle as O
    cin, cout, k, r = 64, 128, 3, 16
    cfg = workloads.DecompConfig("pipe", (cin, cout, k, k), 12, r, 0.02, seed=9)
    w, f0 = workloads.generate_decomp(cfg)
    f, idx, val, eps = run_gpu(w, f0, cfg.cardinality, 20)
    a, d, b, c = f  # mode order (in, out, ky, kx)
    l = D.cp_reconstruct(f)
    s_dense = D.sparse_dense(w.shape, idx, val)
    assert abs(np.linalg.norm(w - l - s_dense) / np.linalg.norm(w) - eps[-1]) < 1e-9
    # S -> CSR by output channel j, col (c*k + y)*k + x, columns increasing
    cc, rem = np.divmod(idx, cout * k * k)
    j, rem = np.divmod(rem, k * k)
    y, xx = np.divmod(rem, k)
    col = (cc * k + y) * k + xx
    order = np.lexsort((col, j))
    row_ptr = np.zeros(cout + 1, np.int64)
    np.add.at(row_ptr, j + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    col_idx = col[order].astype(np.int32)
    values = val[order].astype(np.float32)
    # the layer in fp32 (the decomposition's fp64 factors rounded to fp32 only)
    n, hh = 2, 10
    layer = LrsConv.from_cp(n, hh, hh, k, 1, 1, "f32", a, b, c, d, row_ptr, col_idx, values)
    x = np.maximum(np.random.default_rng(3).standard_normal((n, hh, hh, cin)), 0).astype(np.float32)
    yg = layer(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    ref = O.conv_direct(x.astype(np.float64), l + s_dense, 1, 1)
    e = rel(yg.cpu().numpy(), ref)
    assert e < 1e-5, e


# ------------------------------------------------------------------ Tucker-2 form (lrs_tucker2_*)

def run_t2(w, u_in0, u_out0, card, iters, tol=0.0, inner=1):
    from paper_2006_06443_b200 import LrsTucker2Decomp
    dc = LrsTucker2Decomp(w.shape, u_in0.shape[1], u_out0.shape[1], card, max_iters=iters, tol=tol, inner=inner)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    wd, ui, uo = dev(w), dev(u_in0), dev(u_out0)
    core, idx, val, eps = dc.run(wd, ui, uo)
    torch.cuda.synchronize()
    return ui.cpu().numpy(), uo.cpu().numpy(), core.cpu().numpy(), idx.cpu().numpy(), val.cpu().numpy(), eps


@pytest.mark.parametrize("inner", [1, 2])
@pytest.mark.parametrize("planted,r1,r2", [(8, 8, 8), (6, 8, 10)])
def test_tucker2_iterations_match_oracle(inner, planted, r1, r2):
    """At the planted ranks (a wide spectral gap) the factors themselves match; over-ranked, the
    extra directions lie in the noise spectrum (tiny gaps amplify rounding), so the unique
    quantities are compared: eps, S and L = U_in G U_out^T."""
    cfg = workloads.DecompConfig("t2", (48, 40, 3, 3), planted, 0, 0.01, seed=4)
    w, ui0, uo0 = workloads.generate_decomp_tucker2(cfg, r1, r2)
    ui, uo, g, idx, val, eps = run_t2(w, ui0, uo0, cfg.cardinality, 6, inner=inner)
    (rui, ruo, rg), (ridx, rval), reps = D.decompose_lrs_tucker2(w, ui0, uo0, cfg.cardinality, max_iters=6, tol=0.0,
                                                                inner=inner)
    assert len(eps) == len(reps) == 6
    assert np.allclose(eps, reps, rtol=1e-8, atol=1e-13)
    assert np.array_equal(idx, ridx)
    assert rel(val, rval) < 1e-9
    assert rel(D.tucker2_reconstruct(ui, g, uo), D.tucker2_reconstruct(rui, rg, ruo)) < 1e-8
    if planted == r1 == r2:
        assert rel(ui, rui) < 1e-8 and rel(uo, ruo) < 1e-8 and rel(g, rg) < 1e-8
    # orthonormal bases (Loewdin through the Gram: the error grows with its condition number; the
    # over-ranked noise directions leave ~1e-8, the oracle's own level)
    assert np.allclose(ui.T @ ui, np.eye(r1), atol=1e-6) and np.allclose(uo.T @ uo, np.eye(r2), atol=1e-6)


def test_tucker2_ragged_shapes_and_1x1():
    """Shapes off every GEMM tile (Cin 70, Cout 33, ranks 5 / 17, a 1 x 1 and a 5 x 5 kernel)."""
    for dims, r1, r2 in (((70, 33, 1, 1), 5, 17), ((21, 19, 5, 5), 7, 3)):
        cfg = workloads.DecompConfig("t2r", dims, 4, 0, 0.02, seed=6)
        w, ui0, uo0 = workloads.generate_decomp_tucker2(cfg, r1, r2)
        ui, uo, g, idx, val, eps = run_t2(w, ui0, uo0, cfg.cardinality, 4)
        (rui, ruo, rg), (ridx, _), reps = D.decompose_lrs_tucker2(w, ui0, uo0, cfg.cardinality, max_iters=4, tol=0.0)
        assert np.allclose(eps, reps, rtol=1e-8, atol=1e-13), dims
        assert np.array_equal(idx, ridx), dims
        assert rel(D.tucker2_reconstruct(ui, g, uo), D.tucker2_reconstruct(rui, rg, ruo)) < 1e-8, dims


def test_tucker2_full_size_c3_weight():
    """The C3 weight shape (512 x 512 x 3 x 3) at the north star's Tucker ranks 128 / 128, c = 1 %:
    three sweeps against the oracle."""
    cfg = workloads.DECOMP_CONFIGS["c3_decomp"]
    w, ui0, uo0 = workloads.generate_decomp_tucker2(cfg, 128, 128)
    ui, uo, g, idx, val, eps = run_t2(w, ui0, uo0, cfg.cardinality, 3)
    (rui, ruo, rg), (ridx, _), reps = D.decompose_lrs_tucker2(w, ui0, uo0, cfg.cardinality, max_iters=3, tol=0.0)
    assert np.allclose(eps, reps, rtol=1e-8)
    assert np.array_equal(idx, ridx)
    assert rel(D.tucker2_reconstruct(ui, g, uo), D.tucker2_reconstruct(rui, rg, ruo)) < 1e-8


def test_tucker2_determinism_stopping_and_zero_w():
    cfg = workloads.DecompConfig("t2d", (32, 24, 3, 3), 4, 0, 0.02, seed=3)
    w, ui0, uo0 = workloads.generate_decomp_tucker2(cfg, 6, 6)
    a = run_t2(w, ui0, uo0, cfg.cardinality, 100, tol=1e-6)
    b = run_t2(w, ui0, uo0, cfg.cardinality, 100, tol=1e-6)
    _, _, reps = D.decompose_lrs_tucker2(w, ui0, uo0, cfg.cardinality, max_iters=100, tol=1e-6)
    assert len(a[5]) == len(reps) < 100
    for x, y in zip(a[:5], b[:5]):
        assert np.array_equal(x, y)  # bitwise reproducible
    z = np.zeros((8, 8, 3, 3))
    ui, uo, g, idx, val, eps = run_t2(z, np.ones((8, 2)), np.ones((8, 3)), 0.05, 10)
    assert idx.size == 0 and eps == [0.0] and not np.any(ui) and not np.any(uo) and not np.any(g)


def test_tucker2_decomposed_weight_runs_as_the_layer():
    """Decompose W into Tucker-2 + S on the GPU and run it as the forward's Tucker-2 layer
    (u_in, core, u_out = U_out^T; S -> CSR by output channel): Y = conv(X, L + S)."""
    from paper_2006_06443_b200 import LrsConv
    from oracle import lrs_oracle as O
    cin, cout, k, r1, r2 = 64, 96, 3, 16, 24
    cfg = workloads.DecompConfig("t2pipe", (cin, cout, k, k), 10, 0, 0.02, seed=8)
    w, ui0, uo0 = workloads.generate_decomp_tucker2(cfg, r1, r2)
    ui, uo, g, idx, val, eps = run_t2(w, ui0, uo0, cfg.cardinality, 15)
    l = D.tucker2_reconstruct(ui, g, uo)
    s_dense = D.sparse_dense(w.shape, idx, val)
    assert abs(np.linalg.norm(w - l - s_dense) / np.linalg.norm(w) - eps[-1]) < 1e-9
    cc, rem = np.divmod(idx, cout * k * k)
    j, rem = np.divmod(rem, k * k)
    y, xx = np.divmod(rem, k)
    col = (cc * k + y) * k + xx
    order = np.lexsort((col, j))
    row_ptr = np.cumsum(np.concatenate([[0], np.bincount(j, minlength=cout)])).astype(np.int64)
    n, hh = 2, 10
    layer = LrsConv(n, hh, hh, cin, cout, k, 1, 1, r1, r2, "f32", ui.astype(np.float32), g.astype(np.float32),
                    np.ascontiguousarray(uo.T).astype(np.float32), row_ptr, col[order].astype(np.int32),
                    val[order].astype(np.float32))
    x = np.maximum(np.random.default_rng(3).standard_normal((n, hh, hh, cin)), 0).astype(np.float32)
    yg = layer(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    ref = O.conv_direct(x.astype(np.float64), l + s_dense, 1, 1)
    assert rel(yg.cpu().numpy(), ref) < 1e-5
