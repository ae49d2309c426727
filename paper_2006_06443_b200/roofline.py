"""Algorithmic work of the compressed convolution, for roofline fractions.

Host-side measurement arithmetic only (no kernels).  Definitions follow
SURVEY.md §8(d) / DESIGN.md "Roofline": bytes count what the method itself
must move (X read once, Y written once, weights + CSR once, intermediates
T1/T2 written and read once), FLOPs count 2 per multiply-add; the sparse term
counts only in-bounds taps.
"""
from __future__ import annotations

import json
import os
from typing import Dict, Optional

import numpy as np

#: B200 FP32 CUDA-core pipe: 148 SMs x 128 FMA/clk (B200_PROFILING.md table: 148 SMs;
#: Blackwell SM = 4 partitions x 32 FP32 lanes); 2 FLOP per FMA.
FP32_FMA_PER_CLK_PER_SM = 128
NUM_SMS = 148


def measured_peaks(path: Optional[str] = None) -> Dict[str, float]:
    """MEASURED_PEAKS.json (driver-written) or the profiling guide's fallback."""
    if path is None:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)), "source": "measured"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0, "source": "fallback"}


def fp32_fma_tflops(sm_mhz: float) -> float:
    return NUM_SMS * FP32_FMA_PER_CLK_PER_SM * 2 * sm_mhz * 1e6 / 1e12


def out_size(n: int, k: int, s: int, p: int) -> int:
    return (n + 2 * p - k) // s + 1


def sparse_macs(n: int, h: int, w: int, k: int, s: int, p: int, col_idx: np.ndarray) -> int:
    """In-bounds sparse multiply-adds: n * sum_e V(y_e) V(x_e) with
    V(t) = #{o in [0, Ho): 0 <= o*s + t - p < H}."""
    ho, wo = out_size(h, k, s, p), out_size(w, k, s, p)
    vh = np.array([sum(1 for o in range(ho) if 0 <= o * s + t - p < h) for t in range(k)], np.int64)
    vw = np.array([sum(1 for o in range(wo) if 0 <= o * s + t - p < w) for t in range(k)], np.int64)
    tap = np.asarray(col_idx, np.int64) % (k * k)
    return int(n * (vh[tap // k] * vw[tap % k]).sum())


def layer_work(cfg, n: int, col_idx: np.ndarray, cp: bool = False) -> Dict[str, Dict[str, float]]:
    """Per-stage algorithmic bytes and FLOPs for n images of layer `cfg`
    (a workloads.LayerConfig).  cp: L in the paper's CP form (rank R = rank_in),
    whose stages 2-3 are two depthwise convs of k MACs per output and channel."""
    esz = 2 if cfg.dtype == "bf16" else 4
    ho, wo = cfg.out_h, cfg.out_w
    p_in = n * cfg.in_h * cfg.in_w
    p = n * ho * wo
    r1 = cfg.rank_in
    r2 = cfg.rank_in if cfg.svd else cfg.rank_out
    nnz = len(col_idx)
    x_b = p_in * cfg.c_in * esz
    y_b = p * cfg.c_out * esz
    t1_b = p_in * r1 * esz
    t2_b = 0 if cfg.svd else p * r2 * esz
    macs_s = sparse_macs(n, cfg.in_h, cfg.in_w, cfg.k, cfg.stride, cfg.pad, col_idx)
    st = {
        "a1_proj": {"bytes": x_b + t1_b + cfg.c_in * r1 * esz, "flops": 2.0 * p_in * cfg.c_in * r1},
        "a345_expand_sparse": {
            # the fused kernel reads X (sparse term), T2 (T1 for the SVD pair), the weights, writes Y
            "bytes": x_b + (t2_b if not cfg.svd else t1_b) + y_b + r2 * cfg.c_out * esz + nnz * 8 + (cfg.c_out + 1) * 4,
            "flops_tc": 2.0 * p * r2 * cfg.c_out, "flops_sparse": 2.0 * macs_s, "sparse_macs": macs_s},
    }
    st["a345_expand_sparse"]["flops"] = st["a345_expand_sparse"]["flops_tc"] + st["a345_expand_sparse"]["flops_sparse"]
    # fp32 split engine: a3 GEMM stores Y_L, a4 gathers X and adds Y_S into Y (read + write)
    st["a3_expand"] = {"bytes": (t2_b if not cfg.svd else t1_b) + y_b + r2 * cfg.c_out * esz,
                       "flops": 2.0 * p * r2 * cfg.c_out}
    st["a4_sparse_add"] = {"bytes": x_b + 2 * y_b + nnz * 8 + (cfg.c_out + 1) * 4,
                           "flops": 2.0 * macs_s, "flops_sparse": 2.0 * macs_s, "sparse_macs": macs_s}
    if not cfg.svd:
        # a1 + a2 fused (T1 stays on chip): X in, T2 out, U_in and G read once
        st["a12_proj_core"] = {"bytes": x_b + t2_b + cfg.c_in * r1 * esz + r1 * r2 * cfg.k * cfg.k * esz,
                               "flops": 2.0 * p_in * cfg.c_in * r1 + 2.0 * p * r1 * r2 * cfg.k * cfg.k}
        st["a2_core"] = {"bytes": t1_b + t2_b + r1 * r2 * cfg.k * cfg.k * esz,
                         "flops": 2.0 * p * r1 * r2 * cfg.k * cfg.k}
    core_w = (2 * cfg.k * r1) if cp else (0 if cfg.svd else r1 * r2 * cfg.k ** 2)
    core_macs = (2 * p * r1 * cfg.k) if cp else (0 if cfg.svd else p * r1 * r2 * cfg.k ** 2)
    if cp:
        st["a2_cp_depthwise"] = {"bytes": t1_b + t2_b + core_w * 4, "flops": 2.0 * core_macs}
        # a1 + the depthwise pair fused (T1 stays on chip): X in, T2 out, A and B, C read once
        st["a12_proj_cp"] = {"bytes": x_b + t2_b + cfg.c_in * r1 * esz + core_w * 4,
                             "flops": 2.0 * p_in * cfg.c_in * r1 + 2.0 * core_macs}
    layer_bytes = x_b + y_b + esz * (cfg.c_in * r1 + core_w + r2 * cfg.c_out) + nnz * 8 + (cfg.c_out + 1) * 4
    chain = 2.0 * (p_in * cfg.c_in * r1 + core_macs + p * r2 * cfg.c_out)
    st["layer"] = {"bytes": layer_bytes, "flops_chain": chain, "flops_sparse": 2.0 * macs_s,
                   "sparse_macs": macs_s, "flops": chain + 2.0 * macs_s}
    return st


def extra_peaks(path: Optional[str] = None) -> Dict[str, float]:
    """Peaks MEASURED_PEAKS.json lacks, measured on a B200 by tools/measure_extra_peaks.py
    (profiles/measured_peaks_extra.json): the TF32 tensor peak (torch fp32 matmul with TF32
    allowed, 8192^3) and the FP32 CUDA-core FMA peak (an FFMA-chain microbenchmark).
    Empty if the file is absent."""
    if path is None:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "measured_peaks_extra.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def tensor_peak(peaks: Dict[str, float], dtype: str):
    """(TFLOP/s, how) of the tensor pipe for a layer's dtype: bf16 = MEASURED_PEAKS.json
    bf16_tflops (burst); fp32 = 3xTF32 (three TF32 MMAs per fp32 product, the split the
    fp32 path needs for 1e-5) = measured TF32 peak / 3, else bf16 / 2 / 3."""
    if dtype == "bf16":
        return peaks["bf16_tflops"], "measured (MEASURED_PEAKS.json bf16_tflops, burst)"
    ex = extra_peaks()
    if "tf32_tflops" in ex:
        return ex["tf32_tflops"] / 3.0, "measured TF32 peak / 3 (3xTF32; profiles/measured_peaks_extra.json)"
    return peaks["bf16_tflops"] / 2.0 / 3.0, "derived: bf16 peak / 2 (nominal TF32 ratio) / 3 (3xTF32)"


def fma_peak(peaks: Dict[str, float]):
    """(TFLOP/s, how) of the FP32 CUDA-core pipe."""
    ex = extra_peaks()
    if "fp32_fma_tflops" in ex:
        return ex["fp32_fma_tflops"], "measured (FFMA microbenchmark, profiles/measured_peaks_extra.json)"
    return fp32_fma_tflops(peaks["sm_max_mhz"]), "derived: 148 SM x 128 FMA/clk x 2 x sm_max_mhz"


def layer_roofs(work: Dict[str, Dict[str, float]], peaks: Dict[str, float], dtype: str) -> Dict[str, float]:
    """Literal roof (BASELINE: max(bytes/BW, all FLOPs/tensor peak)) and the
    three-roof (sparse MACs on the FP32 pipe), in seconds."""
    lay = work["layer"]
    tc = tensor_peak(peaks, dtype)[0] * 1e12
    bw = peaks["hbm_gbs"] * 1e9
    fma, fma_kind = fma_peak(peaks)
    fma *= 1e12
    t_lit = max(lay["bytes"] / bw, lay["flops"] / tc)
    t_three = max(lay["bytes"] / bw, lay["flops_chain"] / tc, lay["flops_sparse"] / fma)
    return {"t_literal_s": t_lit, "t_three_roof_s": t_three, "t_hbm_s": lay["bytes"] / bw,
            "t_chain_tc_s": lay["flops_chain"] / tc, "t_sparse_tc_s": lay["flops_sparse"] / tc,
            "t_sparse_fma_s": lay["flops_sparse"] / fma, "fma_tflops": fma / 1e12, "fma_kind": fma_kind}


def kernel_roofline(stage: str, work: Dict[str, Dict[str, float]], peaks: Dict[str, float], dtype: str,
                    t_kernel_s: float, engine: int) -> Dict[str, object]:
    """The bench line's `roofline` object for the dominant kernel, against the LITERAL
    roof of BASELINE.json's north star: the slower of its algorithmic bytes at the
    measured HBM bandwidth and its algorithmic FLOPs (the sparse term's included) at the
    measured tensor peak of the layer's dtype.  achieved = that quantity / the kernel's
    event-timed launch duration; frac = achieved / peak.  The FP32-pipe (three-roof) view
    of the same kernel is reported beside it, with its peak's provenance."""
    if stage in ("a345_expand_sparse", "a4_sparse_add") and engine == 3:
        wk = dict(work["layer"])  # the one-kernel fp32 path: the whole layer
    else:
        wk = dict(work[stage])
    b = float(wk["bytes"])
    f = float(wk["flops"])
    f_sp = float(wk.get("flops_sparse", 0.0))
    tc, tc_kind = tensor_peak(peaks, dtype)
    bw = peaks["hbm_gbs"]
    fma, fma_kind = fma_peak(peaks)
    t_hbm = b / (bw * 1e9)
    t_tc = f / (tc * 1e12)
    if t_hbm >= t_tc:
        bound, achieved, peak, unit, kind = "hbm", b / t_kernel_s / 1e9, bw, "GB/s", "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        bound, achieved, peak, unit, kind = "tensor", f / t_kernel_s / 1e12, tc, "TFLOP/s", tc_kind
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": None, "kernel": stage, "peak_kind": kind,
            "work": {"bytes": b, "flops": f, "flops_sparse": f_sp, "kernel_us": t_kernel_s * 1e6,
                     "roof_us": {"hbm": t_hbm * 1e6, "tensor": t_tc * 1e6}},
            "three_roof_view": {"fp32_pipe_us": f_sp / (fma * 1e12) * 1e6, "fp32_peak_tflops": fma,
                                "fp32_peak_kind": fma_kind,
                                "frac": max(t_hbm, (f - f_sp) / (tc * 1e12), f_sp / (fma * 1e12)) / t_kernel_s},
            "what": "literal roof of the dominant kernel: max(algorithmic bytes / HBM, algorithmic FLOPs incl. "
                    "the sparse term / tensor peak) (BASELINE.json north star)"}


def sparse24_floor_s(cfg, n: int, main_blocks: int, res_blocks: int, peaks: Dict[str, float]) -> float:
    """The 2:4 sparse engine's own floor for n images: every compressed block (128 output
    channels x 64 logical input-channel slots of one tap) costs a dense 128 x 32 MMA per
    output position whatever its density, plus the expansion GEMM, at the bf16 tensor
    peak.  Output positions are counted without the kernel's window padding columns."""
    p = n * cfg.out_h * cfg.out_w
    r2 = cfg.rank_in if cfg.svd else cfg.rank_out
    flops = 2.0 * 128 * 32 * (main_blocks + res_blocks) * p + 2.0 * p * r2 * cfg.c_out
    return flops / (peaks["bf16_tflops"] * 1e12)
