"""Timing ablation of one layer config under experiment knobs (debug tool; needs the
LRS_EXPERIMENTS build: `LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force`).

usage: python tools/ablate.py <config> "<ENV=V ENV2=V>" ["<...>" ...]
Each argument after the config is one setting (space-separated env assignments, or
"base"; a CFG_<field>=<value> item changes the layer config, e.g. CFG_density=0.02); the layer is created under that environment, K forwards over rotating X/Y
sets are captured in a CUDA graph and replayed; prints us per forward (median of 5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv  # noqa: E402


def run(cfg, inp, env):
    saved = {}
    for kv in env:
        k, v = kv.split("=", 1)
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        layer = LrsConv.from_inputs(inp, batch_max=cfg.batch)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    n = cfg.batch
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    nsets = 8
    xs = [torch.from_numpy(workloads.generate_x(cfg, n, seed=i)).to(tdt).cuda() for i in range(nsets)]
    ys = [torch.empty((n, cfg.out_h, cfg.out_w, cfg.c_out), dtype=tdt, device="cuda") for _ in range(nsets)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(nsets):
            layer.forward_into(xs[i], ys[i], stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for r in range(4):
                for i in range(nsets):
                    layer.forward_into(xs[i], ys[i], stream=s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / (4 * nsets))
    layer.set_timing(True)
    layer.stage_times(reset=True)
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(2e7))
        for i in range(nsets):
            layer.forward_into(xs[i], ys[i], stream=s)
    torch.cuda.synchronize()
    st = {k: round(v[0] / v[1] * 1e3, 1) for k, v in layer.stage_times(reset=True).items() if v[1]}
    layer.set_timing(False)
    eng = layer.sparse_engine
    layer.close()
    return float(np.median(ts)), st, eng


def main():
    import dataclasses
    name = sys.argv[1]
    base = workloads.CONFIGS[name]
    for setting in sys.argv[2:]:
        env = [] if setting == "base" else setting.split()
        over = {kv[4:].split("=")[0]: kv.split("=", 1)[1] for kv in env if kv.startswith("CFG_")}
        env = [kv for kv in env if not kv.startswith("CFG_")]
        cfg = dataclasses.replace(base, **{k: type(getattr(base, k))(v) for k, v in over.items()})
        inp = workloads.generate(cfg, batch=1)
        us, st, eng = run(cfg, inp, env)
        print(f"{name} [{setting}] {us:.2f} us/forward  stages {st}  engine {eng}", flush=True)


if __name__ == "__main__":
    main()
