"""Planner sweep of the fused a1 + a2 kernel (lrs_core.cuh) at one config: for each
(images per tile, band height) the layer is re-created with LRS_CORE_IPT / LRS_CORE_TH
and the step is timed graph-replayed over rotating X/Y sets (L2 defeated), once with
the whole layer and once with the expansion + sparse kernel skipped (LRS_SKIP=4), which
leaves the core kernel alone.  Timing experiment only.

usage: python tools/core_sweep.py [config] [ipt,th[,grid[,wconv_th]] ...]  (grid 0 = all SMs)
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv, LrsError  # noqa: E402


def step_us(inp, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        layer = LrsConv.from_inputs(inp, device=0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if env.get("LRS_CORE_TH") and not layer.core_fused:
        layer.close()
        raise LrsError(-1, "planner: this (ipt, th) does not fit")
    cfg = inp.cfg
    n = inp.x.shape[0]
    x0 = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
    sets = max(2, math.ceil(2.1 * 126e6 / (2 * x0.numel() + 2 * n * cfg.out_h * cfg.out_w * cfg.c_out)))
    xs = [x0.clone() for _ in range(sets)]
    ys = [torch.empty((n, cfg.out_h, cfg.out_w, cfg.c_out), dtype=torch.bfloat16, device="cuda") for _ in range(sets)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(sets):
            layer.forward_into(xs[i], ys[i], stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(sets):
            layer.forward_into(xs[i], ys[i], stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, 400 // sets)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e3 / (reps * sets)
    layer.close()
    return t


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2_bf16"
    cfg = workloads.CONFIGS[name]
    inp = workloads.generate(cfg)
    combos = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]] or \
        [(i, t) for i in (1, 2, 4, 8) for t in range(1, cfg.out_h + 1)]
    print(f"{name}: default full {step_us(inp, {}):.2f} us, core only {step_us(inp, {'LRS_SKIP': 4}):.2f} us",
          flush=True)
    for combo in combos:
        ipt, th = combo[0], combo[1]
        env = {"LRS_CORE_IPT": ipt, "LRS_CORE_TH": th}
        if len(combo) > 2 and combo[2]:
            env["LRS_CORE_GRID"] = combo[2]
        if len(combo) > 3:
            env["LRS_WCONV_TH"] = combo[3]
        try:
            full = step_us(inp, env)
            core = step_us(inp, dict(env, LRS_SKIP=4))
        except LrsError as e:
            print(f"{combo}: {e}")
            continue
        print(f"ipt,th,grid={combo}: full {full:.2f} us  core-only {core:.2f} us", flush=True)


if __name__ == "__main__":
    main()
