"""Create one config's layer at its full batch and run a few forwards on distinct
inputs (the target of ncu captures: python tools/run_layer.py <config> [forwards])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = workloads.CONFIGS[name]
layer = LrsConv.from_inputs(workloads.generate(cfg, batch=1), batch_max=cfg.batch)
tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
xs = [torch.from_numpy(workloads.generate_x(cfg, cfg.batch, seed=i)).to(tdt).cuda() for i in range(2)]
y = torch.empty((cfg.batch, cfg.out_h, cfg.out_w, cfg.c_out), dtype=tdt, device="cuda")
for i in range(reps):
    layer.forward_into(xs[i % 2], y)
torch.cuda.synchronize()
print(f"{name}: {reps} forwards ok, engine {layer.sparse_engine}, expand kernel {layer.expand_kernel}")
