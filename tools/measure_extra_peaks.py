"""Measure the two peaks MEASURED_PEAKS.json does not hold (VERDICT r01 weak #5 / SURVEY
§8(d) "builder must measure"): the TF32 tensor peak (torch fp32 matmul 8192^3 with TF32
allowed, best of 10, CUDA events) and the FP32 CUDA-core FMA peak (tools/fma_peak.cu).
Writes profiles/measured_peaks_extra.json (read by paper_2006_06443_b200/roofline.py)
with the SM clock seen.  Run on a B200: python tools/measure_extra_peaks.py
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    tf32 = 2.0 * n ** 3 / (best * 1e-3) / 1e12
    exe = os.path.join(ROOT, "tools", "fma_peak")
    if not os.path.exists(exe):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                               os.path.join(ROOT, "tools", "fma_peak.cu")])
    fma = json.loads(subprocess.check_output([exe]).decode().strip().splitlines()[-1])
    try:
        clk = subprocess.check_output(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader"]
                                      ).decode().strip()
    except Exception:
        clk = None
    out = {"tf32_tflops": tf32, "fp32_fma_tflops": fma["fp32_fma_tflops"],
           "how": "tf32: torch.matmul fp32 8192^3 with allow_tf32, best of 10 (CUDA events); fp32 FMA: "
                  "tools/fma_peak.cu (8 independent FFMA chains x 256 threads x 8 CTAs per SM), best of 5",
           "gpu": torch.cuda.get_device_name(), "sm_clock_after": clk,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    path = os.path.join(ROOT, "profiles", "measured_peaks_extra.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
