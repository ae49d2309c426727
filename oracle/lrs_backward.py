"""fp64 CPU oracle for the backward pass of the compressed convolution
Y = conv(X, L + S) -- the gradients fine-tuning needs.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
bench.py's `cpu_baseline` / `--impl reference` leg may import this module.
The product path never imports it and shares no code with it.

PAPER.md:194-195 (§3.5): "the decomposed layer should be fine-tuned using
ordinary back-propagation with respect to the original loss"; PAPER.md:383
(§5.5): fine-tuning of each decomposed layer with SGD.  The trainable
parameters of the decomposed layer are the factors of L (U_in, G, U_out, or
U, V of the SVD pair) and the VALUES of S at its fixed support (the support is
chosen by the projection P_c, and is not a parameter).  Given
the upstream gradient dY = dLoss/dY this module computes

  dX        = dLoss/dX         (the layer's input gradient, fed to the layer below)
  dU_in, dG, dU_out, dvalues   (the parameter gradients)

Two independent formulations:
  * `backward_dense` -- the definition: Y = conv(X, W) is linear in X and in W,
    so dX is the adjoint convolution with the densified W = W_L + W_S
     written tap by tap as a scatter, and dW is the full
    weight gradient dW[c,j,y,x] = sum_{n,ho,wo} X[n, ho*s+y-p, wo*s+x-p, c] dY[n,ho,wo,j];
    the parameter gradients follow by the chain rule through W_L = U_in G U_out
    (contractions of dW with the other two factors) and dvalues[e] = dW at e.
  * `backward_factored` -- back-propagation through the method's own order of
    operations (T1 = X U_in, T2 = conv(T1, G), Y = T2 U_out + sparse conv,
    PAPER.md:162-168, :189), stage by stage in reverse.
Pins (tests/test_backward_oracle.py): torch.autograd in fp64 through
torch.nn.functional.conv2d of the densified weight and through the factor
chain with the S values as leaf tensors; the adjoint identity
<conv(X, W), dY> = <X, dX>; central finite differences; dense == factored.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from .lrs_oracle import (conv_1x1, conv_direct, densify_sparse, out_size, reconstruct_cp, reconstruct_tucker2)

__all__ = ["conv_adjoint_input", "weight_grad_dense", "backward_dense", "backward_factored",
           "sparse_values_grad", "transposed_layer", "backward_cp"]


def conv_adjoint_input(dy: np.ndarray, w: np.ndarray, in_h: int, in_w: int, stride: int = 1,
                       pad: int = 0) -> np.ndarray:
    """dX[n, ho*s+y-p, wo*s+x-p, c] += sum_j dY[n,ho,wo,j] W[c,j,y,x]: the adjoint of
    conv_direct (PAPER.md:160's Einstein sum read with X as the unknown), tap by
    tap; contributions that land in the zero padding are dropped."""
    dy = np.asarray(dy, np.float64)
    w = np.asarray(w, np.float64)
    n, ho, wo, j = dy.shape
    c, j2, kh, kw = w.shape
    assert j == j2
    assert out_size(in_h, kh, stride, pad) == ho and out_size(in_w, kw, stride, pad) == wo
    hp, wp = in_h + 2 * pad + stride, in_w + 2 * pad + stride
    dxp = np.zeros((n, hp, wp, c), dtype=np.float64)
    for ty in range(kh):
        for tx in range(kw):
            dxp[:, ty:ty + stride * (ho - 1) + 1:stride, tx:tx + stride * (wo - 1) + 1:stride, :] += \
                dy @ w[:, :, ty, tx].T
    return dxp[:, pad:pad + in_h, pad:pad + in_w, :]


def weight_grad_dense(x: np.ndarray, dy: np.ndarray, k: int, stride: int = 1, pad: int = 0) -> np.ndarray:
    """dW[c,j,y,x] = sum_{n,ho,wo} X[n, ho*s+y-p, wo*s+x-p, c] dY[n,ho,wo,j]
    (the derivative of PAPER.md:160 with respect to W_ijkp), one fp64 matmul per tap
    over all output positions."""
    x = np.asarray(x, np.float64)
    dy = np.asarray(dy, np.float64)
    n, h, wd, c = x.shape
    _, ho, wo, j = dy.shape
    xp = np.zeros((n, h + 2 * pad, wd + 2 * pad, c), dtype=np.float64)
    xp[:, pad:pad + h, pad:pad + wd, :] = x
    dw = np.zeros((c, j, k, k), dtype=np.float64)
    for ty in range(k):
        for tx in range(k):
            win = xp[:, ty:ty + stride * (ho - 1) + 1:stride, tx:tx + stride * (wo - 1) + 1:stride, :]
            dw[:, :, ty, tx] = win.reshape(-1, c).T @ dy.reshape(-1, j)
    return dw


def sparse_values_grad(dw: np.ndarray, row_ptr, col_idx) -> np.ndarray:
    """dvalues[e] = dW[c_e, j, y_e, x_e] for CSR entry e of row j with
    col_e = (c*k + y)*k + x: S's values enter W only at their own index
    (W = L + S), so each value's gradient is dW there."""
    k = dw.shape[2]
    row_ptr = np.asarray(row_ptr)
    out = np.zeros(int(row_ptr[-1]), dtype=np.float64)
    for j in range(dw.shape[1]):
        for e in range(int(row_ptr[j]), int(row_ptr[j + 1])):
            c, rem = divmod(int(col_idx[e]), k * k)
            y, x = divmod(rem, k)
            out[e] = dw[c, j, y, x]
    return out


def backward_dense(x, dy, u_in, core, u_out, row_ptr, col_idx, values, stride=1, pad=0) -> dict:
    """The definition (see module docstring).  Chain rule through
    W_L[c,j,y,x] = sum_{a,b} U_in[c,a] G[a,b,y,x] U_out[b,j]:
      dU_in[c,a]    = sum_{j,y,x,b} dW[c,j,y,x] G[a,b,y,x] U_out[b,j]
      dG[a,b,y,x]   = sum_{c,j} U_in[c,a] dW[c,j,y,x] U_out[b,j]
      dU_out[b,j]   = sum_{c,a,y,x} U_in[c,a] G[a,b,y,x] dW[c,j,y,x]
    (SVD pair: W_L[c,j] = sum_a U[c,a] V[a,j], dU = dW V^T, dV = U^T dW)."""
    x = np.asarray(x, np.float64)
    u_in = np.asarray(u_in, np.float64)
    u_out = np.asarray(u_out, np.float64)
    c_in, c_out = u_in.shape[0], u_out.shape[1]
    k = 1 if core is None else np.asarray(core).shape[2]
    w = reconstruct_tucker2(u_in, core, u_out) + densify_sparse(c_in, c_out, k, row_ptr, col_idx, values)
    dx = conv_adjoint_input(dy, w, x.shape[1], x.shape[2], stride, pad)
    dw = weight_grad_dense(x, dy, k, stride, pad)
    if core is None:
        d_u_in = dw[:, :, 0, 0] @ u_out.T
        d_core = None
        d_u_out = u_in.T @ dw[:, :, 0, 0]
    else:
        g = np.asarray(core, np.float64)
        d_u_in = np.einsum("cjyx,abyx,bj->ca", dw, g, u_out, optimize=True)
        d_core = np.einsum("ca,cjyx,bj->abyx", u_in, dw, u_out, optimize=True)
        d_u_out = np.einsum("ca,abyx,cjyx->bj", u_in, g, dw, optimize=True)
    return {"dx": dx, "d_u_in": d_u_in, "d_core": d_core, "d_u_out": d_u_out,
            "d_values": sparse_values_grad(dw, row_ptr, col_idx), "dw": dw}


def backward_factored(x, dy, u_in, core, u_out, row_ptr, col_idx, values, stride=1, pad=0,
                      return_intermediates: bool = False) -> dict:
    """Back-propagation through the method's forward (PAPER.md:162-168 chain,
    :189 sparse term), stage by stage in reverse:
      forward   T1 = X U_in;  T2 = conv(T1, G; s, p);  Y = T2 U_out + conv(X, S)
      dT2    = dY U_out^T                                   (adjoint of the expansion)
      dU_out = T2^T dY          (sum over all output positions)
      dG     = weight gradient of conv(T1, G) at dT2       (adjoint in G)
      dT1    = adjoint of conv(., G) applied to dT2        (adjoint in T1)
      dU_in  = X^T dT1          (sum over all input positions)
      dX     = dT1 U_in^T + adjoint of the sparse conv applied to dY
      dvalues[e] = sum over output positions of dY[., j_e] X[shift_e(.), c_e]
    SVD pair (core=None): T1 = X U, Y = T1 V + S; dT1 = dY V^T, dV = T1^T dY,
    dU = X^T dT1, dX = dT1 U^T + S-adjoint."""
    x = np.asarray(x, np.float64)
    dy = np.asarray(dy, np.float64)
    u_in = np.asarray(u_in, np.float64)
    u_out = np.asarray(u_out, np.float64)
    n, h, wd, c_in = x.shape
    c_out = u_out.shape[1]
    k = 1 if core is None else np.asarray(core).shape[2]
    ws = densify_sparse(c_in, c_out, k, row_ptr, col_idx, values)
    t1 = conv_1x1(x, u_in)
    out = {}
    if core is None:
        dt1 = conv_1x1(dy, u_out.T)
        d_u_out = t1.reshape(-1, t1.shape[-1]).T @ dy.reshape(-1, c_out)
        d_core = None
        inter = {"t1": t1, "dt1": dt1}
    else:
        g = np.asarray(core, np.float64)
        t2 = conv_direct(t1, g, stride, pad)
        dt2 = conv_1x1(dy, u_out.T)
        d_u_out = t2.reshape(-1, t2.shape[-1]).T @ dy.reshape(-1, c_out)
        d_core = weight_grad_dense(t1, dt2, k, stride, pad)
        dt1 = conv_adjoint_input(dt2, g, h, wd, stride, pad)
        inter = {"t1": t1, "t2": t2, "dt2": dt2, "dt1": dt1}
    d_u_in = x.reshape(-1, c_in).T @ dt1.reshape(-1, dt1.shape[-1])
    dx = conv_1x1(dt1, u_in.T) + conv_adjoint_input(dy, ws, h, wd, stride, pad)
    # dvalues, entry by entry from the definition of the sparse term
    xp = np.zeros((n, h + 2 * pad, wd + 2 * pad, c_in), dtype=np.float64)
    xp[:, pad:pad + h, pad:pad + wd, :] = x
    ho, wo = dy.shape[1], dy.shape[2]
    row_ptr = np.asarray(row_ptr)
    d_values = np.zeros(int(row_ptr[-1]), dtype=np.float64)
    for j in range(c_out):
        for e in range(int(row_ptr[j]), int(row_ptr[j + 1])):
            c, rem = divmod(int(col_idx[e]), k * k)
            ty, tx = divmod(rem, k)
            win = xp[:, ty:ty + stride * (ho - 1) + 1:stride, tx:tx + stride * (wo - 1) + 1:stride, c]
            d_values[e] = float(np.sum(win * dy[:, :, :, j]))
    out.update({"dx": dx, "d_u_in": d_u_in, "d_core": d_core, "d_u_out": d_u_out, "d_values": d_values})
    if return_intermediates:
        out.update(inter)
    return out


def transposed_layer(u_in, core, u_out, row_ptr, col_idx, values, c_in: int, pad: int):
    """The layer whose forward is dX at stride 1: conv_adjoint_input(dY, W) =
    conv(dY, W') with W'[j,c,y,x] = W[c,j,k-1-y,k-1-x] and padding k-1-p
    (a test helper for the GPU path's construction; the factors of W' are
    U_out^T, G'[b,a,y,x] = G[a,b,k-1-y,k-1-x], U_in^T, and S' by input channel).
    Returns (u_in', core', u_out', row_ptr', col_idx', values', pad')."""
    u_in = np.asarray(u_in, np.float64)
    u_out = np.asarray(u_out, np.float64)
    c_out = u_out.shape[1]
    k = 1 if core is None else np.asarray(core).shape[2]
    core_t = None if core is None else np.ascontiguousarray(
        np.asarray(core, np.float64).transpose(1, 0, 2, 3)[:, :, ::-1, ::-1])
    ents = [[] for _ in range(c_in)]
    row_ptr = np.asarray(row_ptr)
    for j in range(c_out):
        for e in range(int(row_ptr[j]), int(row_ptr[j + 1])):
            c, rem = divmod(int(col_idx[e]), k * k)
            y, x = divmod(rem, k)
            ents[c].append(((j * k + (k - 1 - y)) * k + (k - 1 - x), float(values[e])))
    rp, ci, va = [0], [], []
    for c in range(c_in):
        for col, v in sorted(ents[c]):
            ci.append(col)
            va.append(v)
        rp.append(len(ci))
    return (u_out.T.copy(), core_t, u_in.T.copy(), np.asarray(rp, np.int64), np.asarray(ci, np.int32),
            np.asarray(va, np.float64), k - 1 - pad)


def backward_cp(x, dy, a, b, c, d, row_ptr, col_idx, values, stride=1, pad=0) -> dict:
    """The gradients of a layer whose L is in the paper's CP form, L_ijkp = A_ir B_kr C_pr D_jr
    (A [Cin][R], B [k][R] (taps along H), C [k][R] (along W), D [Cout][R]),
    the paper's own decomposed layer that §3.5 fine-tunes: dX as the adjoint
    convolution with W = L + S, dW the full weight gradient, and the chain rule through the
    four factors
      dA[i,r] = sum dW[i,j,k,p] B[k,r] C[p,r] D[j,r]      dB[k,r] = sum dW A[i,r] C[p,r] D[j,r]
      dC[p,r] = sum dW A[i,r] B[k,r] D[j,r]               dD[j,r] = sum dW A[i,r] B[k,r] C[p,r]
    and dvalues = dW at S's support."""
    x = np.asarray(x, np.float64)
    a, b, c, d = (np.asarray(t, np.float64) for t in (a, b, c, d))
    k = b.shape[0]
    w = reconstruct_cp(a, b, c, d) + densify_sparse(a.shape[0], d.shape[0], k, row_ptr, col_idx, values)
    dx = conv_adjoint_input(dy, w, x.shape[1], x.shape[2], stride, pad)
    dw = weight_grad_dense(x, dy, k, stride, pad)
    return {"dx": dx,
            "d_a": np.einsum("ijkp,kr,pr,jr->ir", dw, b, c, d, optimize=True),
            "d_b": np.einsum("ijkp,ir,pr,jr->kr", dw, a, c, d, optimize=True),
            "d_c": np.einsum("ijkp,ir,kr,jr->pr", dw, a, b, d, optimize=True),
            "d_d": np.einsum("ijkp,ir,kr,pr->jr", dw, a, b, c, optimize=True),
            "d_values": sparse_values_grad(dw, row_ptr, col_idx), "dw": dw}
