"""fp64 CPU oracle for the compressed convolution Y = conv(X, L + S).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
bench.py's `cpu_baseline` / `--impl reference` leg may import this module.
The product path (`paper_2006_06443_b200`) never imports it and shares no
code with it; the two meet only through the seeded arrays of `workloads/`.

Plain, slow, obviously correct.  Every function cites the passage of
/root/reference/PAPER.md (the thesis, arXiv 2006.06443) or SPEC.md it writes
out.  Notation follows PAPER.md §3.3: X_{s m t} is (x, y, channel) i.e. HWC
(here batched NHWC), the conv weight W_{i j k p} is indexed (in, out, kx, ky)
with the centre tap at k = p = 0.  Reading #3: the convolution is
a cross-correlation with zero padding, output size floor((H + 2p - k)/s) + 1.

Pins (tests/test_oracle_pins.py): torch.nn.functional.conv2d in fp64 on the
densified weight, a pure-Python quintuple loop on tiny inputs, the identity
O1 == O2, linearity, the paper's displacement rule, SPEC's
hand values, the paper's closed-form parameter counts and the
Table-2 parameter total.  No function here is parity-unpinned.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

__all__ = [
    "out_size", "conv_direct", "reconstruct_tucker2", "reconstruct_cp",
    "densify_sparse", "forward_dense", "conv_1x1", "sparse_conv_scatter",
    "forward_factored", "cp_conv", "forward_cp", "brute_force_conv", "param_counts", "cp_param_count",
    "output_epilogue",
    "pack_sparse_slices", "unpack_sparse_slices", "sparse_mac_count",
]


def out_size(n: int, k: int, s: int, p: int) -> int:
    """Output extent of a k-tap conv with stride s and zero padding p
    (PyTorch convention; equals PAPER.md:160's centred form at s=1, p=k//2)."""
    return (n + 2 * p - k) // s + 1


# --------------------------------------------------------------------------
# O1: dense definition (PAPER.md:58 §1.1, :160 §3.3)
# --------------------------------------------------------------------------

def conv_direct(x: np.ndarray, w: np.ndarray, stride: int = 1, pad: int = 0) -> np.ndarray:
    """Y[n,ho,wo,j] = sum_{y,x,c} X[n, ho*s+y-p, wo*s+x-p, c] * W[c,j,y,x].

    The Einstein sum of PAPER.md:160 (Y_smj = X_(s+k)(m+p)i W_ijkp) written
    out tap by tap; terms outside the image are omitted (zero padding).
    x: [N,H,W,C] ; w: [C, J, k, k] in the paper's (in, out, kx, ky) order.
    Each tap is a plain fp64 matmul over the input channel index i.
    """
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    n, h, wd, c = x.shape
    c2, j, kh, kw = w.shape
    assert c == c2, "input channels of X and W differ"
    ho, wo = out_size(h, kh, stride, pad), out_size(wd, kw, stride, pad)
    assert ho >= 1 and wo >= 1
    xp = np.zeros((n, h + 2 * pad, wd + 2 * pad, c), dtype=np.float64)
    xp[:, pad:pad + h, pad:pad + wd, :] = x
    y = np.zeros((n, ho, wo, j), dtype=np.float64)
    for ty in range(kh):
        for tx in range(kw):
            win = xp[:, ty:ty + stride * (ho - 1) + 1:stride, tx:tx + stride * (wo - 1) + 1:stride, :]
            y += win @ w[:, :, ty, tx]
    return y


def reconstruct_tucker2(u_in: np.ndarray, core: Optional[np.ndarray], u_out: np.ndarray) -> np.ndarray:
    """W_L[c,j,y,x] = sum_a sum_b U_in[c,a] G[a,b,y,x] U_out[b,j].

    The Tucker-2 form of the low-rank term that BASELINE.json's north star
    names (1x1 projection -> k x k core -> 1x1 expansion); §7.3
    names Tucker as the follow-up of the CP form of PAPER.md:158.  With
    core=None (SVD pair for 1x1 layers) W_L[c,j,0,0] = sum_a U[c,a] V[a,j].
    """
    u_in = np.asarray(u_in, np.float64)
    u_out = np.asarray(u_out, np.float64)
    if core is None:
        return (u_in @ u_out)[:, :, None, None]
    core = np.asarray(core, np.float64)
    return np.einsum("ca,abyx,bj->cjyx", u_in, core, u_out, optimize=True)


def reconstruct_cp(a: np.ndarray, b: np.ndarray, c: np.ndarray, d: np.ndarray) -> np.ndarray:
    """L_{ijkp} = A_ir B_kr C_pr D_jr (§3.3).
    a: [I, r] input channels, b: [K, r] kx taps, c: [P, r] ky taps,
    d: [J, r] output channels.  Returns L[i, j, k, p]."""
    return np.einsum("ir,kr,pr,jr->ijkp", *(np.asarray(t, np.float64) for t in (a, b, c, d)))


def densify_sparse(c_in: int, c_out: int, k: int, row_ptr, col_idx, values) -> np.ndarray:
    """W_S[c,j,y,x] = v_e for each CSR entry e of row j with col_e = (c*k+y)*k+x
    (the OIHW flattening of the ABI, reading #6)."""
    ws = np.zeros((c_in, c_out, k, k), dtype=np.float64)
    row_ptr = np.asarray(row_ptr)
    for j in range(c_out):
        for e in range(int(row_ptr[j]), int(row_ptr[j + 1])):
            col = int(col_idx[e])
            c, rem = divmod(col, k * k)
            y, x = divmod(rem, k)
            ws[c, j, y, x] += float(values[e])
    return ws


def forward_dense(x, u_in, core, u_out, row_ptr, col_idx, values, stride=1, pad=0) -> np.ndarray:
    """O1: W = W_L + W_S reconstructed densely, then one direct convolution
    (PAPER.md:125 W = L + S; :160 the convolution)."""
    c_in = np.asarray(u_in).shape[0]
    c_out = np.asarray(u_out).shape[1]
    k = 1 if core is None else np.asarray(core).shape[2]
    w = reconstruct_tucker2(u_in, core, u_out) + densify_sparse(c_in, c_out, k, row_ptr, col_idx, values)
    return conv_direct(x, w, stride, pad)


# --------------------------------------------------------------------------
# O2: factored evaluation, the method's own order of operations
# --------------------------------------------------------------------------

def conv_1x1(x: np.ndarray, m: np.ndarray) -> np.ndarray:
    """Y^A_{smr} = X_{smi} A_{ir}: a 1x1 convolution = matmul
    over the channel index."""
    return np.asarray(x, np.float64) @ np.asarray(m, np.float64)


def sparse_conv_scatter(x: np.ndarray, c_out: int, k: int, row_ptr, col_idx, values,
                        stride: int = 1, pad: int = 0) -> np.ndarray:
    """Direct sparse convolution, §3.4.

    "For each input channel i ... iterate through these arrays, multiply each
    element in the input by value and add the result to the corresponding
    channel of output with the spatial displacement related to the position
    of the element in kernel."  Entries are first regrouped per input channel
    (the paper's per-slice storage), then each entry (j, y, x, v) adds
    v * X[:, ho*s+y-p, wo*s+x-p, i] into Y[..., j]; the displacement of a
    tap at (dy, dx) from the centre is (-dy, -dx) (the paper's "(1,1) ->
    displaced by -1,-1").  Positions outside the input contribute nothing.
    """
    x = np.asarray(x, np.float64)
    n, h, w, c_in = x.shape
    ho, wo = out_size(h, k, stride, pad), out_size(w, k, stride, pad)
    y = np.zeros((n, ho, wo, c_out), dtype=np.float64)
    xp = np.zeros((n, h + 2 * pad, w + 2 * pad, c_in), dtype=np.float64)
    xp[:, pad:pad + h, pad:pad + w, :] = x
    # per-input-channel slices: (value, out channel j, tap y, tap x)
    slices = [[] for _ in range(c_in)]
    row_ptr = np.asarray(row_ptr)
    for j in range(c_out):
        for e in range(int(row_ptr[j]), int(row_ptr[j + 1])):
            c, rem = divmod(int(col_idx[e]), k * k)
            ty, tx = divmod(rem, k)
            slices[c].append((float(values[e]), j, ty, tx))
    for i in range(c_in):
        plane = xp[:, :, :, i]
        for v, j, ty, tx in slices[i]:
            y[:, :, :, j] += v * plane[:, ty:ty + stride * (ho - 1) + 1:stride,
                                       tx:tx + stride * (wo - 1) + 1:stride]
    return y


def forward_factored(x, u_in, core, u_out, row_ptr, col_idx, values, stride=1, pad=0,
                     return_parts: bool = False):
    """O2: the method (BASELINE.json north star; §3.3 + §3.4):
    T1 = X U_in (1x1 projection), T2 = conv(T1, G; s, p)
    (k x k core; the Tucker-2 generalisation of PAPER.md:165-166),
    Y_L = T2 U_out (1x1 expansion), Y_S = sparse conv of X
    (PAPER.md:189), Y = Y_L + Y_S.  SVD pair: T1 = X U,
    Y_L = T1 V (core=None, 1x1)."""
    c_out = np.asarray(u_out).shape[1]
    if core is None:
        t1 = conv_1x1(x, u_in)
        y_l = conv_1x1(t1, u_out)
        k = 1
        assert stride == 1 and pad == 0, "SVD pair is a 1x1 layer"
    else:
        core = np.asarray(core, np.float64)
        k = core.shape[2]
        t1 = conv_1x1(x, u_in)
        t2 = conv_direct(t1, core, stride, pad)
        y_l = conv_1x1(t2, u_out)
    y_s = sparse_conv_scatter(x, c_out, k, row_ptr, col_idx, values, stride, pad)
    if return_parts:
        return y_l + y_s, y_l, y_s
    return y_l + y_s


def cp_conv(x, a, b, c, d, pad: Optional[int] = None) -> np.ndarray:
    """The paper's CP-decomposed convolution, four stages (PAPER.md:162-168,
    stride 1, centred taps):
      Y^A_{smr} = X_{smi} A_{ir}                     1x1
      Y^B_{smr} = Y^A_{(s+k)mr} B_{kr}               kx-tap depthwise (reading #5: the
                                                      paper writes C_kr here, a typo)
      Y^C_{smr} = Y^B_{s(m+p)r} C_{pr}               ky-tap depthwise
      Y_{smj}   = Y^C_{smr} D_{jr}                   1x1
    Axis s is the first spatial axis (H here), m the second (W)."""
    x = np.asarray(x, np.float64)
    a, b, c, d = (np.asarray(t, np.float64) for t in (a, b, c, d))
    kk = b.shape[0]
    p = kk // 2 if pad is None else pad
    n, h, w, _ = x.shape
    ya = x @ a
    r = ya.shape[-1]
    ypad = np.zeros((n, h + 2 * p, w, r))
    ypad[:, p:p + h] = ya
    yb = np.zeros((n, h + 2 * p - kk + 1, w, r))
    for t in range(kk):
        yb += ypad[:, t:t + yb.shape[1]] * b[t]
    h2 = yb.shape[1]
    ypad = np.zeros((n, h2, w + 2 * p, r))
    ypad[:, :, p:p + w] = yb
    yc = np.zeros((n, h2, w + 2 * p - kk + 1, r))
    for t in range(kk):
        yc += ypad[:, :, t:t + yc.shape[2]] * c[t]
    return yc @ d.T


def forward_cp(x, a, b, c, d, row_ptr, col_idx, values, stride: int = 1, pad: int = 0) -> np.ndarray:
    """A layer whose L is in the paper's CP form plus the sparse
    term: Y = conv(X, L) + conv(X, S).  At stride 1 with centred
    padding L runs as the paper's four stages (cp_conv); the
    paper has no strided form (reading #4), so other strides/paddings evaluate
    conv(X, L) on the reconstructed kernel (reconstruct_cp + conv_direct) --
    the plain definition the four stages equal.  The sparse term is
    sparse_conv_scatter."""
    x = np.asarray(x, np.float64)
    k = np.asarray(b).shape[0]
    if stride == 1 and pad == k // 2:
        y_l = cp_conv(x, a, b, c, d, pad)
    else:
        y_l = conv_direct(x, reconstruct_cp(a, b, c, d), stride, pad)
    d = np.asarray(d)
    return y_l + sparse_conv_scatter(x, d.shape[0], k, row_ptr, col_idx, values, stride, pad)


def output_epilogue(y, scale=None, bias=None, relu: bool = False) -> np.ndarray:
    """The library's optional fused output epilogue (include/lrs_conv.h; SURVEY §8(f) f3 --
    an inference BatchNorm y*s + b with its scale/shift per output channel, and a ReLU,
    as in ResNet's conv2 -> bn2 -> relu):  act(y[..., j] * scale[j] + bias[j])."""
    y = np.asarray(y, np.float64)
    if scale is not None:
        y = y * np.asarray(scale, np.float64)
    if bias is not None:
        y = y + np.asarray(bias, np.float64)
    return np.maximum(y, 0.0) if relu else y


def brute_force_conv(x, w, stride=1, pad=0) -> np.ndarray:
    """Independent quintuple loop over tiny inputs, pure
    Python: Y[n,o,q,j] = sum_{c,y,x} X[n, o*s+y-p, q*s+x-p, c] * W[c,j,y,x]."""
    n, h, wd, c = x.shape
    _, j, kh, kw = w.shape
    ho, wo = out_size(h, kh, stride, pad), out_size(wd, kw, stride, pad)
    out = np.zeros((n, ho, wo, j))
    for b in range(n):
        for o in range(ho):
            for q in range(wo):
                for jj in range(j):
                    acc = 0.0
                    for cc in range(c):
                        for yy in range(kh):
                            for xx in range(kw):
                                hi, wi = o * stride + yy - pad, q * stride + xx - pad
                                if 0 <= hi < h and 0 <= wi < wd:
                                    acc += float(x[b, hi, wi, cc]) * float(w[cc, jj, yy, xx])
                    out[b, o, q, jj] = acc
    return out


def param_counts(c_in: int, c_out: int, k: int, r1: int, r2: int, nnz: int, svd: bool = False) -> dict:
    """Parameter accounting, §3.2: P(W) = IJKT; the CP form has
    P(L) = r(I+J+K+T); the Tucker-2 form of the north star stores
    Cin*R1 + R1*R2*k*k + R2*Cout (SVD pair: Cin*R + R*Cout); the CSR sparse
    term stores nnz values + nnz column indices + (Cout+1) row pointers
    (reading #19: the paper's P(S) = alpha IJKT lacks the cardinality)."""
    p_w = c_in * c_out * k * k
    p_l = c_in * r1 + r1 * c_out if svd else c_in * r1 + r1 * r2 * k * k + r2 * c_out
    p_s = 2 * nnz + c_out + 1
    return {"P_W": p_w, "P_L": p_l, "P_S_csr": p_s, "compression": p_w / (p_l + p_s),
            "compression_L_only": p_w / p_l}


def cp_param_count(i: int, j: int, k: int, t: int, r: int) -> int:
    """P(L) = r(I + J + K + T) for the CP form."""
    return r * (i + j + k + t)


def pack_sparse_slices(c_in: int, c_out: int, k: int, row_ptr, col_idx, values):
    """The paper's sparse storage: per input
    channel i, a values array and a packed index array with
    packed = j*(k*k) + kx*k + ky (int16 when c_out*k*k <= 65536, else u32)."""
    wide = c_out * k * k > 65536
    vals = [[] for _ in range(c_in)]
    packed = [[] for _ in range(c_in)]
    row_ptr = np.asarray(row_ptr)
    for j in range(c_out):
        for e in range(int(row_ptr[j]), int(row_ptr[j + 1])):
            c, rem = divmod(int(col_idx[e]), k * k)
            kx, ky = divmod(rem, k)
            vals[c].append(float(values[e]))
            packed[c].append(j * k * k + kx * k + ky)
    dt = np.uint32 if wide else np.uint16
    return [np.array(v, np.float32) for v in vals], [np.array(p, dt) for p in packed]


def unpack_sparse_slices(c_in: int, c_out: int, k: int, vals, packed):
    """Inverse of pack_sparse_slices, back to CSR by output channel."""
    entries = []
    for i in range(c_in):
        for v, pk in zip(vals[i], packed[i]):
            j, rem = divmod(int(pk), k * k)
            entries.append((j, (i * k * k) + rem, float(v)))
    entries.sort()
    row_ptr = np.zeros(c_out + 1, np.int64)
    for j, _, _ in entries:
        row_ptr[j + 1] += 1
    row_ptr = np.cumsum(row_ptr)
    col = np.array([e[1] for e in entries], np.int32)
    val = np.array([e[2] for e in entries], np.float32)
    return row_ptr, col, val


def sparse_mac_count(n: int, h: int, w: int, k: int, stride: int, pad: int, col_idx) -> int:
    """In-bounds multiply-adds of the sparse term:
    N * sum_e V(y_e) V(x_e), V(t) = #{o in [0,Ho): 0 <= o*s + t - p < H}."""
    ho, wo = out_size(h, k, stride, pad), out_size(w, k, stride, pad)
    vh = [sum(1 for o in range(ho) if 0 <= o * stride + t - pad < h) for t in range(k)]
    vw = [sum(1 for o in range(wo) if 0 <= o * stride + t - pad < w) for t in range(k)]
    tot = 0
    for col in np.asarray(col_idx):
        rem = int(col) % (k * k)
        tot += vh[rem // k] * vw[rem % k]
    return n * tot
