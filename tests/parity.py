"""Shared parity check of a GPU output against the fp64 oracle.

Tolerances (BASELINE.json north star): fp32 path relL2 <= 1e-5 and
max-abs <= 1e-4; bf16 path relL2 <= 2e-2.  The relative L2 bound is applied to
the whole tensor AND to every image, every 128-output-channel block (the
fused kernel's M-tile) and the first / last output row and column (the
padded borders), so a defect confined to one image, one M-tile or one
border row cannot hide inside a whole-tensor norm.
"""
from __future__ import annotations

import numpy as np

TOL = {"f32": 1e-5, "bf16": 2e-2}


def _rel(a: np.ndarray, b: np.ndarray) -> float:
    nb = np.linalg.norm(b)
    na = np.linalg.norm(a - b)
    if nb == 0.0:
        return 0.0 if na == 0.0 else float("inf")
    return float(na / nb)


def slices(y_ref: np.ndarray):
    """(name, index) of every sub-tensor the bound is applied to; y is NHWC."""
    n, h, w, c = y_ref.shape
    out = [("all", np.s_[...])]
    out += [(f"image {i}", np.s_[i]) for i in range(n)]
    out += [(f"channels {j}:{j + 128}", np.s_[..., j:j + 128]) for j in range(0, c, 128)] if c > 128 else []
    out += [("row 0", np.s_[:, 0]), (f"row {h - 1}", np.s_[:, h - 1]),
            ("col 0", np.s_[:, :, 0]), (f"col {w - 1}", np.s_[:, :, w - 1])]
    return out


def check(y_gpu, y_ref: np.ndarray, dtype: str):
    """Assert parity; y_gpu a torch tensor (any dtype) or array, y_ref fp64 NHWC.
    Returns (whole-tensor relL2, max-abs)."""
    yg = y_gpu.float().cpu().numpy().astype(np.float64) if hasattr(y_gpu, "cpu") else np.asarray(y_gpu, np.float64)
    assert yg.shape == y_ref.shape, (yg.shape, y_ref.shape)
    assert np.isfinite(yg).all()
    tol = TOL[dtype]
    for name, ix in slices(y_ref):
        e = _rel(yg[ix], y_ref[ix])
        assert e <= tol, f"relL2 {e:.3e} > {tol:g} on {name}"
    err = _rel(yg, y_ref)
    mx = float(np.abs(yg - y_ref).max()) if yg.size else 0.0
    if dtype == "f32":
        assert mx <= 1e-4, f"max-abs {mx:.3e} > 1e-4"
    return err, mx
