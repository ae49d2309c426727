"""Pins of the fp64 decomposition oracle (oracle/lrs_decomp.py) against
things other than itself (CPU only): a full Python sort for P_c, brute-force loops for the
MTTKRP, numpy's least-squares solver on the explicitly unfolded system for one ALS mode
update, and SPEC.md's own examples: cardinality 0,
an already-feasible tensor, a fixed point, a monotone residual, planted-rank recovery and
planted-spike recovery.  PAPER.md:124-146 §3.2.
"""
import itertools

import numpy as np
import pytest

from oracle import lrs_decomp as D


def rand_factors(rng, dims, r):
    return [rng.standard_normal((d, r)) for d in dims]


def test_project_sparse_matches_a_full_sort_with_index_ties():
    rng = np.random.default_rng(0)
    t = rng.standard_normal((4, 4, 3, 3))
    t.flat[[5, 9, 17, 60]] = 2.5  # four-way tie in |v|
    t.flat[[11, 40]] = -2.5
    for c in (0.01, 0.05, 0.1, 0.37):
        n = int(round(c * t.size))
        ranked = sorted(range(t.size), key=lambda i: (-abs(t.flat[i]), i))  # SPEC: smaller index wins ties
        want = sorted(ranked[:n])
        idx, vals = D.project_sparse(t, c)
        assert list(idx) == want
        assert np.array_equal(vals, t.flat[want])


def test_project_sparse_spec_examples():
    t = np.zeros((2, 3, 3, 3))
    assert D.project_sparse(np.ones((2, 3, 3, 3)), 0.0)[0].size == 0  # SPEC.md:147 cardinality 0
    t.flat[[3, 7]] = [1.0, -2.0]
    idx, vals = D.project_sparse(t, 0.1)  # n = 5 >= 2 nonzeros: both kept, zero ties by index
    assert set([3, 7]) <= set(idx.tolist()) and len(idx) == 5
    assert np.array_equal(vals[np.isin(idx, [3, 7])], [1.0, -2.0])


def test_mttkrp_brute_force():
    rng = np.random.default_rng(1)
    dims, r = (3, 4, 2, 3), 2
    t = rng.standard_normal(dims)
    f = rand_factors(rng, dims, r)
    for mode in range(4):
        m = np.zeros((dims[mode], r))
        for idx in itertools.product(*(range(d) for d in dims)):
            for q in range(r):
                p = t[idx]
                for o in range(4):
                    if o != mode:
                        p *= f[o][idx[o], q]
                m[idx[mode], q] += p
        assert np.allclose(D.mttkrp(t, f, mode), m, rtol=1e-13, atol=1e-13)


def test_one_mode_update_is_the_least_squares_solution():
    """F_0 <- argmin ||T_(0) - F_0 KR^T||: numpy lstsq on the explicitly formed Khatri-Rao."""
    rng = np.random.default_rng(2)
    dims, r = (5, 4, 3, 3), 3
    t = rng.standard_normal(dims)
    f = rand_factors(rng, dims, r)
    kr = np.einsum("br,cr,dr->bcdr", f[1], f[2], f[3]).reshape(-1, r)
    want = np.linalg.lstsq(kr, t.reshape(dims[0], -1).T, rcond=None)[0].T
    got = D.mttkrp(t, f, 0) @ D.sym_pinv(D.gram_hadamard(f, 0))
    assert np.allclose(got, want, rtol=1e-9, atol=1e-10)


def test_sym_pinv_cutoff():
    q, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((4, 4)))
    v = (q * np.array([5.0, 1.0, 1e-12, 0.0])) @ q.T
    p = D.sym_pinv(v)
    assert np.allclose(p, (q[:, :2] * np.array([0.2, 1.0])) @ q[:, :2].T, atol=1e-10)


def test_als_fixed_point_and_monotone_residual():
    rng = np.random.default_rng(4)
    dims, r = (6, 5, 3, 3), 3
    f = rand_factors(rng, dims, r)
    target = D.cp_reconstruct(f)
    f2 = D.cp_als_step(f, target)
    assert np.linalg.norm(D.cp_reconstruct(f2) - target) <= 1e-9 * np.linalg.norm(target)
    t = rng.standard_normal(dims)
    g = rand_factors(rng, dims, 2)
    prev = np.inf
    for _ in range(50):  # non-increasing over 50 sweeps
        g = D.cp_als_step(g, t)
        res = np.linalg.norm(t - D.cp_reconstruct(g))
        assert res <= prev + 1e-6
        prev = res


def test_als_recovers_a_planted_rank():
    rng = np.random.default_rng(5)
    dims = (8, 7, 3, 3)
    target = D.cp_reconstruct(rand_factors(rng, dims, 2))
    g = rand_factors(rng, dims, 2)
    for _ in range(200):
        g = D.cp_als_step(g, target)
    assert np.linalg.norm(target - D.cp_reconstruct(g)) / np.linalg.norm(target) < 1e-4


def test_decompose_recovers_planted_spikes():
    """rank-2 + 1 % large spikes (magnitude 10 x the N(0,1) factor scale), rank 2,
    cardinality 0.01 -> eps < 1e-3 and the spike positions are S's support.  (CP-ALS is
    non-convex: some draws stall in a local minimum -- e.g. seed 6 at eps 0.09;
    this seed's draw is recovered to round-off, which a slip in any step would prevent.)"""
    rng = np.random.default_rng(7)
    dims = (10, 10, 3, 3)
    low = D.cp_reconstruct(rand_factors(rng, dims, 2))
    n = int(round(0.01 * low.size))
    spikes = np.sort(rng.choice(low.size, n, replace=False))
    w = low.copy()
    w.flat[spikes] += 10.0 * np.sign(rng.standard_normal(n))
    f, (idx, vals), hist = D.decompose_lrs(w, D.svd_init(w, 2), 0.01, max_iters=300, tol=0.0)
    assert hist[-1] < 1e-3
    assert np.array_equal(idx, spikes)
    # the S-step is an exact projection and the L-step a descent sweep: non-increasing
    assert all(b <= a + 1e-6 for a, b in zip(hist, hist[1:]))


def test_decompose_degenerate_cases():
    rng = np.random.default_rng(7)
    dims = (6, 5, 3, 3)
    w = D.cp_reconstruct(rand_factors(rng, dims, 1))
    f, (idx, _), hist = D.decompose_lrs(w, D.svd_init(w, 1), 0.0, max_iters=100, tol=0.0)
    assert idx.size == 0 and hist[-1] < 1e-4
    z = np.zeros(dims)
    f, (idx, _), hist = D.decompose_lrs(z, D.svd_init(z + 1.0, 2), 0.01)  # SPEC.md:163 zero W
    assert idx.size == 0 and hist == [0.0] and all(not np.any(x) for x in f)


def rand_tucker2(rng, dims, r1, r2):
    u = np.linalg.qr(rng.standard_normal((dims[0], r1)))[0]
    v = np.linalg.qr(rng.standard_normal((dims[1], r2)))[0]
    g = rng.standard_normal((r1, r2) + dims[2:])
    return u, v, g


def test_lowdin_is_the_closest_orthonormal_basis():
    """orth_lowdin(Y) = U V^T of the SVD Y = U s V^T (numpy's SVD: the polar factor)."""
    y = np.random.default_rng(20).standard_normal((9, 4))
    u, _, vt = np.linalg.svd(y, full_matrices=False)
    q = D.orth_lowdin(y)
    assert np.allclose(q, u @ vt, atol=1e-12)
    assert np.allclose(q.T @ q, np.eye(4), atol=1e-12)


def test_cholqr_is_numpy_qr_with_a_positive_r_diagonal():
    """orth_cholqr(Y) = the Q of numpy's thin QR with column signs making diag(R) > 0 (library
    pin); a rank-deficient Y (a repeated column) takes the Loewdin fallback: an orthonormal basis
    of span(Y) of dimension rank(Y), the dropped direction a zero column."""
    y = np.random.default_rng(23).standard_normal((11, 5))
    q, r = np.linalg.qr(y)
    sg = np.sign(np.diag(r))
    assert np.allclose(D.orth_cholqr(y), q * sg, atol=1e-12)
    yd = np.concatenate([y[:, :3], y[:, :1]], axis=1)
    qd = D.orth_cholqr(yd)
    assert np.allclose(qd, D.orth_lowdin(yd))
    assert np.linalg.matrix_rank(qd, tol=1e-8) == 3
    assert np.allclose(qd @ qd.T @ yd, yd, atol=1e-10)  # spans span(Y)


def test_hooi_recovers_a_planted_tucker2_tensor():
    """An exact Tucker-2 tensor of ranks (3, 2) is reproduced to round-off (cardinality 0),
    and the factors span the same subspaces as numpy's SVD of the unfoldings (library pin)."""
    rng = np.random.default_rng(21)
    dims = (12, 10, 3, 3)
    u, v, g = rand_tucker2(rng, dims, 3, 2)
    w = D.tucker2_reconstruct(u, g, v)
    (ui, uo, gg), (idx, _), hist = D.decompose_lrs_tucker2(w, rng.standard_normal((12, 3)),
                                                          rng.standard_normal((10, 2)), 0.0, max_iters=30, tol=-1)
    assert hist[-1] < 1e-10 and idx.size == 0
    su = np.linalg.svd(w.reshape(12, -1), full_matrices=False)[0][:, :3]
    sv = np.linalg.svd(np.moveaxis(w, 1, 0).reshape(10, -1), full_matrices=False)[0][:, :2]
    assert np.allclose(ui @ ui.T, su @ su.T, atol=1e-8)
    assert np.allclose(uo @ uo.T, sv @ sv.T, atol=1e-8)


def test_tucker2_decompose_monotone_and_spikes():
    """W = Tucker-2 (4, 4) + 1 % spikes of magnitude 10: eps non-increasing and the spikes
    recovered as S's support."""
    rng = np.random.default_rng(22)
    dims = (16, 14, 3, 3)
    u, v, g = rand_tucker2(rng, dims, 4, 4)
    low = D.tucker2_reconstruct(u, g * 3.0, v)
    n = int(round(0.01 * low.size))
    spikes = np.sort(rng.choice(low.size, n, replace=False))
    w = low.copy()
    w.flat[spikes] += 10.0 * np.sign(rng.standard_normal(n))
    (ui, uo, gg), (idx, _), hist = D.decompose_lrs_tucker2(w, rng.standard_normal((16, 4)),
                                                          rng.standard_normal((14, 4)), 0.01, max_iters=60, tol=-1)
    assert all(b <= a + 1e-9 for a, b in zip(hist, hist[1:]))
    assert hist[-1] < 1e-6
    assert np.array_equal(idx, spikes)
