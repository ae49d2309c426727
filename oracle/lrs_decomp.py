"""fp64 CPU oracle for the low-rank + sparse DECOMPOSITION W ~ L + S.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and bench.py's
`cpu_baseline` / `--impl reference` leg may import this module.  The product path never
imports it and shares no code with it.

PAPER.md:124-146 (§3.2): min ||W - L - S|| subject to rank(L) = r (the CP rank,
L_ijkt = A_ir B_jr C_kr D_tr) and card(S) = c; "Any iterative approach can be
easily extended to low rank and sparse version.  On each step i:
  1. L_i = update(L_{i-1}, W - S_{i-1})
  2. S_i = P_c(W - L_i)
Here P_c(A) is projection of some matrix A on the space of matrices with a fixed cardinality
c.  The nonzero elements a choised by the maximum absolute value."  SPEC.md:142-184 fixes
the pieces this oracle writes out step by step, in that order and notation:
  * project_sparse: keep exactly n = round(c * numel) entries of largest
    |value|, ties to the smaller linear index (SPEC design decision), values unmodified;
  * cp_als_step: one sweep of alternating least squares over A, B, C, D,
    each "solved from the mode-n unfolding against the Khatri-Rao of the other three":
    F_n = T_(n) KR(others) (Hadamard of the other Gram matrices)^+, pseudo-inverse with a
    1e-10 singular-value cutoff (relative to the largest; reading #19);
  * decompose_lrs: S_0 = 0; per iteration an ALS sweep on W - S, then
    S = P_c(W - L); eps = ||W - L - S||_F / ||W||_F; stop when the fit 1 - eps improves by
    less than tol, or after max_iters.
Mode order: a tensor T[i0][i1][i2][i3] with factors F0 [I0][R] .. F3 [I3][R],
T ~ sum_r F0[i0,r] F1[i1,r] F2[i2,r] F3[i3,r].  For a conv weight W[c][j][y][x] (in, out,
ky, kx) F0 = A (U_in), F1 = D (U_out^T), F2 = B, F3 = C of the forward's CP core kind.
Pins: tests/test_decomp_oracle.py (full sort, brute-force MTTKRP loops, numpy lstsq of the
unfolded system, SPEC's planted-rank / planted-spike / fixed-point / monotonicity examples).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = ["cp_reconstruct", "mttkrp", "gram_hadamard", "sym_pinv", "cp_als_step", "project_sparse",
           "sparse_dense", "decompose_lrs", "rel_residual", "orth_lowdin", "orth_cholqr", "tucker2_reconstruct",
           "tucker2_hooi_step", "decompose_lrs_tucker2"]


def cp_reconstruct(f: Sequence[np.ndarray]) -> np.ndarray:
    """L[i0,i1,i2,i3] = sum_r F0[i0,r] F1[i1,r] F2[i2,r] F3[i3,r]."""
    return np.einsum("ar,br,cr,dr->abcd", *(np.asarray(x, np.float64) for x in f), optimize=True)


def mttkrp(t: np.ndarray, f: Sequence[np.ndarray], mode: int) -> np.ndarray:
    """M[i,r] = sum over the other three indices of T times the product of the other three
    factors' r-th columns: the mode-n unfolding of T times the Khatri-Rao product of the
    other factors."""
    t = np.asarray(t, np.float64)
    letters = "abcd"
    others = [m for m in range(4) if m != mode]
    spec = "abcd," + ",".join(letters[m] + "r" for m in others) + "->" + letters[mode] + "r"
    return np.einsum(spec, t, *(np.asarray(f[m], np.float64) for m in others), optimize=True)


def gram_hadamard(f: Sequence[np.ndarray], mode: int) -> np.ndarray:
    """V = Hadamard product of F_m^T F_m over the other three modes: the normal-equation
    matrix of the mode-n least-squares problem (KR^T KR = *_m F_m^T F_m)."""
    v = None
    for m in range(4):
        if m == mode:
            continue
        g = np.asarray(f[m], np.float64).T @ np.asarray(f[m], np.float64)
        v = g if v is None else v * g
    return v


def sym_pinv(v: np.ndarray, rcond: float = 1e-10) -> np.ndarray:
    """Pseudo-inverse of a symmetric PSD matrix: eigenvalues below rcond * the largest are
    dropped ("pseudo-inverse with 1e-10 singular-value cutoff")."""
    lam, q = np.linalg.eigh(np.asarray(v, np.float64))
    lmax = float(np.max(np.abs(lam))) if lam.size else 0.0
    keep = np.abs(lam) > rcond * lmax
    inv = np.zeros_like(lam)
    inv[keep] = 1.0 / lam[keep]
    return (q * inv) @ q.T


def cp_als_step(f: Sequence[np.ndarray], target: np.ndarray, rcond: float = 1e-10) -> List[np.ndarray]:
    """One ALS sweep over the four factors in order: for mode n,
    F_n = mttkrp(target, F, n) @ pinv(gram_hadamard(F, n)), using the factors already
    updated earlier in the sweep."""
    f = [np.array(x, np.float64) for x in f]
    for mode in range(4):
        f[mode] = mttkrp(target, f, mode) @ sym_pinv(gram_hadamard(f, mode), rcond)
    return f


def project_sparse(t: np.ndarray, cardinality: float) -> Tuple[np.ndarray, np.ndarray]:
    """P_c: the n = round(c * numel) entries of largest
    |value| (ties: smaller linear index first).  Returns (linear indices ascending, values)."""
    flat = np.asarray(t, np.float64).reshape(-1)
    n = int(round(cardinality * flat.size))
    if n <= 0:
        return np.zeros(0, np.int64), np.zeros(0, np.float64)
    order = np.lexsort((np.arange(flat.size), -np.abs(flat)))  # last key primary: -|v|, then index
    keep = np.sort(order[:n])
    return keep.astype(np.int64), flat[keep]


def sparse_dense(shape, idx, vals) -> np.ndarray:
    s = np.zeros(int(np.prod(shape)), np.float64)
    s[np.asarray(idx, np.int64)] = vals
    return s.reshape(shape)


def rel_residual(w, l, s_dense) -> float:
    w = np.asarray(w, np.float64)
    nw = np.linalg.norm(w)
    return 0.0 if nw == 0.0 else float(np.linalg.norm(w - l - s_dense) / nw)


def decompose_lrs(w: np.ndarray, f0: Sequence[np.ndarray], cardinality: float, max_iters: int = 100,
                  tol: float = 1e-6, rcond: float = 1e-10):
    """The two-step iteration of PAPER.md:142-144 from S_0 = 0:
      F_i = cp_als_step(F_{i-1}, W - S_{i-1})        (L_i = update(L_{i-1}, W - S_{i-1}))
      S_i = project_sparse(W - L_i, c)                (S_i = P_c(W - L_i))
      eps_i = ||W - L_i - S_i|| / ||W||
    stopping when (1 - eps_i) - (1 - eps_{i-1}) < tol (after the first iteration) or after
    max_iters.  Returns (factors, (S indices, S values), eps history)."""
    w = np.asarray(w, np.float64)
    if not np.any(w):
        r = np.asarray(f0[0]).shape[1]
        return [np.zeros((d, r)) for d in w.shape], (np.zeros(0, np.int64), np.zeros(0)), [0.0]
    f = [np.array(x, np.float64) for x in f0]
    s_dense = np.zeros_like(w)
    idx, vals = np.zeros(0, np.int64), np.zeros(0)
    hist: List[float] = []
    for it in range(max_iters):
        f = cp_als_step(f, w - s_dense, rcond)
        l = cp_reconstruct(f)
        idx, vals = project_sparse(w - l, cardinality)
        s_dense = sparse_dense(w.shape, idx, vals)
        hist.append(rel_residual(w, l, s_dense))
        if it > 0 and (hist[-2] - hist[-1]) < tol:
            break
    return f, (idx, vals), hist


def svd_init(w: np.ndarray, rank: int, seed: int = 0) -> List[np.ndarray]:
    """SPEC.md:195 initialisation (a design decision of the SPEC, recorded in DESIGN.md):
    the leading `rank` left singular vectors of each mode unfolding, sign fixed so the
    largest-magnitude entry of each column is positive; a mode with fewer rows than `rank`
    takes its singular vectors plus N(0,1) columns from PCG64(seed)."""
    w = np.asarray(w, np.float64)
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for mode in range(4):
        unf = np.moveaxis(w, mode, 0).reshape(w.shape[mode], -1)
        u, _, _ = np.linalg.svd(unf, full_matrices=False)
        u = u[:, :rank]
        if u.shape[1] < rank:
            u = np.concatenate([u, rng.standard_normal((w.shape[mode], rank - u.shape[1]))], axis=1)
        sgn = np.sign(u[np.argmax(np.abs(u), axis=0), np.arange(u.shape[1])])
        sgn[sgn == 0] = 1.0
        out.append(u * sgn)
    return out


# --------------------------------------------------------------------------
# Tucker-2 form (BASELINE's primary L; SURVEY §8(f) f4 "Alternating Tucker-2/CP-ALS"
# §7 names Tucker decomposition "extended to low rank and sparse form" as the next step)
# --------------------------------------------------------------------------
# W[c][j][y][x] ~ L = sum_{a,b} U_in[c,a] G[a,b,y,x] U_out[j,b] with orthonormal U_in [Cin][R1],
# U_out [Cout][R2] (the layer's u_out = U_out^T), the kernel modes uncompressed.  `update`
# = one higher-order orthogonal iteration (HOOI) sweep on T = W - S: each channel
# factor becomes the dominant R-dimensional left singular subspace of T contracted with the
# other factor, computed by `inner` steps of subspace iteration U <- orth(Z Z^T U), then
# G = T x U_in^T x U_out^T.  orth = Cholesky-QR (Y = Q R, R upper triangular with a positive
# diagonal: the Gram-Schmidt basis) while the Gram Y^T Y has every Cholesky pivot above
# rcond * its largest diagonal entry, else the symmetric (Loewdin) Y (Y^T Y)^(-1/2) with the rcond
# eigenvalue cutoff (a rank-deficient Y; reading #22).  L = U_in G U_out^T depends on the
# subspaces only, so the choice of basis changes U and G, not eps or S.

def orth_lowdin(y: np.ndarray, rcond: float = 1e-10) -> np.ndarray:
    """Y (Y^T Y)^(-1/2) through the eigendecomposition of the Gram matrix (eigenvalues under
    rcond * the largest dropped): the orthonormal basis of span(Y) closest to Y."""
    y = np.asarray(y, np.float64)
    lam, q = np.linalg.eigh(y.T @ y)
    lmax = float(np.max(np.abs(lam))) if lam.size else 0.0
    keep = np.abs(lam) > rcond * lmax
    inv = np.zeros_like(lam)
    inv[keep] = 1.0 / np.sqrt(np.abs(lam[keep]))
    return y @ ((q * inv) @ q.T)


def orth_cholqr(y: np.ndarray, rcond: float = 1e-10) -> np.ndarray:
    """Q = Y L^-T with C = Y^T Y = L L^T (the textbook Cholesky loop, written out); a pivot at or
    under rcond * max_i C_ii -> orth_lowdin(Y) instead."""
    y = np.asarray(y, np.float64)
    c = y.T @ y
    r = c.shape[0]
    thr = rcond * (float(np.max(np.diag(c))) if r else 0.0)
    l = np.zeros_like(c)
    for k in range(r):
        d = c[k, k] - float(np.dot(l[k, :k], l[k, :k]))
        if not d > thr:
            return orth_lowdin(y, rcond)
        l[k, k] = np.sqrt(d)
        for i in range(k + 1, r):
            l[i, k] = (c[i, k] - float(np.dot(l[i, :k], l[k, :k]))) / l[k, k]
    return np.linalg.solve(l, y.T).T  # Y L^-T


def tucker2_reconstruct(u_in, g, u_out) -> np.ndarray:
    """L[c,j,y,x] = sum_{a,b} U_in[c,a] G[a,b,y,x] U_out[j,b]."""
    return np.einsum("ca,abyx,jb->cjyx", np.asarray(u_in, np.float64), np.asarray(g, np.float64),
                     np.asarray(u_out, np.float64), optimize=True)


def tucker2_hooi_step(u_in, u_out, target, inner: int = 1, rcond: float = 1e-10):
    """One HOOI sweep on `target` [Cin][Cout][kh][kw] (see the section comment)."""
    t = np.asarray(target, np.float64)
    cin, cout = t.shape[0], t.shape[1]
    u_in = np.array(u_in, np.float64)
    u_out = np.array(u_out, np.float64)
    z1 = np.einsum("cjyx,jb->cbyx", t, u_out, optimize=True).reshape(cin, -1)  # T x_out U_out^T
    for _ in range(inner):
        u_in = orth_cholqr(z1 @ (z1.T @ u_in), rcond)
    z2 = np.einsum("cjyx,ca->jayx", t, u_in, optimize=True).reshape(cout, -1)  # T x_in U_in^T
    for _ in range(inner):
        u_out = orth_cholqr(z2 @ (z2.T @ u_out), rcond)
    g = np.einsum("cjyx,ca,jb->abyx", t, u_in, u_out, optimize=True)
    return u_in, u_out, g


def decompose_lrs_tucker2(w, u_in0, u_out0, cardinality: float, max_iters: int = 100, tol: float = 1e-6,
                          inner: int = 1, rcond: float = 1e-10):
    """PAPER.md:142-144 with the Tucker-2 update: from S_0 = 0,
      (U_in, U_out, G)_i = tucker2_hooi_step(.., W - S_{i-1});  S_i = P_c(W - L_i);
      eps_i = ||W - L_i - S_i|| / ||W||, stopping as decompose_lrs.  Returns
    ((U_in, U_out, G), (S indices, values), eps history)."""
    w = np.asarray(w, np.float64)
    if not np.any(w):  # as decompose_lrs: zero factors and core, empty S, eps 0
        r1, r2 = np.asarray(u_in0).shape[1], np.asarray(u_out0).shape[1]
        return ((np.zeros((w.shape[0], r1)), np.zeros((w.shape[1], r2)), np.zeros((r1, r2) + w.shape[2:])),
                (np.zeros(0, np.int64), np.zeros(0)), [0.0])
    u_in, u_out = np.array(u_in0, np.float64), np.array(u_out0, np.float64)
    s_dense = np.zeros_like(w)
    idx, vals = np.zeros(0, np.int64), np.zeros(0)
    hist: List[float] = []
    g = None
    for it in range(max_iters):
        u_in, u_out, g = tucker2_hooi_step(u_in, u_out, w - s_dense, inner, rcond)
        l = tucker2_reconstruct(u_in, g, u_out)
        idx, vals = project_sparse(w - l, cardinality)
        s_dense = sparse_dense(w.shape, idx, vals)
        hist.append(rel_residual(w, l, s_dense))
        if it > 0 and (hist[-2] - hist[-1]) < tol:
            break
    return (u_in, u_out, g), (idx, vals), hist
