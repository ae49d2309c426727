"""Backward step time of a config under plan overrides (env set by the caller), CUDA graph of
rotating sets, per-stage event times: python tools/bwd_time.py <config>"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConvBackward  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = cfg.batch
bw = LrsConvBackward.from_inputs(workloads.generate(cfg, batch=1), batch_max=n)
sets = 6
xs = [torch.from_numpy(workloads.generate_x(cfg, n, seed=i)).to(torch.bfloat16).cuda() for i in range(sets)]
dys = [torch.from_numpy(workloads.generate_dy(cfg, n, seed=50 + i)).to(torch.bfloat16).cuda() for i in range(sets)]
dxs = [torch.empty_like(x) for x in xs]
g = bw.alloc_grads()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(sets):
        bw.backward_into(xs[i], dys[i], dxs[i], g, stream=s)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(graph, stream=s):
        for i in range(sets):
            bw.backward_into(xs[i], dys[i], dxs[i], g, stream=s)
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(10):
        graph.replay()
    e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / (10 * sets) * 1e3
bw.set_timing(True)
bw.stage_times(reset=True)
with torch.cuda.stream(s):
    torch.cuda._sleep(int(2e7))
    for i in range(sets):
        bw.backward_into(xs[i], dys[i], dxs[i], g, stream=s)
torch.cuda.synchronize()
st = {k: round(v[0] / v[1] * 1e3, 1) for k, v in bw.stage_times().items()}
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("LRS_"))
print(f"{cfg.name} [{env or 'base'}]: {us:.1f} us per backward step; stages {st}", flush=True)
