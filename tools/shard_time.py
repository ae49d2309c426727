"""Per-GPU forward time of a config at the shard sizes of strong scaling (global batch split
over 1/2/4/8 ranks), measured on ONE GPU: what each rank of `bench.py --gpus N` runs.
python tools/shard_time.py [config]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = workloads.CONFIGS[name]
tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
base = None
for world in (1, 2, 4, 8):
    n = math.ceil(cfg.batch / world)
    layer = LrsConv.from_inputs(workloads.generate(cfg, batch=1), batch_max=n)
    nsets = max(2, math.ceil(2.1 * 126e6 / (n * (cfg.in_h * cfg.in_w * cfg.c_in + cfg.out_h * cfg.out_w * cfg.c_out) * 2)))
    xs = [torch.from_numpy(workloads.generate_x(cfg, n, seed=i)).to(tdt).cuda() for i in range(nsets)]
    ys = [torch.empty((n, cfg.out_h, cfg.out_w, cfg.c_out), dtype=tdt, device="cuda") for _ in range(nsets)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(nsets):
            layer.forward_into(xs[i], ys[i], stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(nsets):
                layer.forward_into(xs[i], ys[i], stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (reps * nsets) * 1e3
    if base is None:
        base = us
    print(f"{name} world {world}: {n} images per GPU, {us:.1f} us per forward, projected strong-scaling "
          f"efficiency {base / (world * us):.2f}, whole-job {cfg.batch / (us * 1e-6) / 1e6:.2f} M img/s", flush=True)
    layer.close()
