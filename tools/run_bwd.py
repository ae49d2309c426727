"""Create one config's backward state at its full batch and run a few backward passes
(dX + parameter gradients) on distinct inputs (the target of ncu captures:
python tools/run_bwd.py <config> [passes])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConvBackward  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = workloads.CONFIGS[name]
bw = LrsConvBackward.from_inputs(workloads.generate(cfg, batch=1), batch_max=cfg.batch)
xs = [torch.from_numpy(workloads.generate_x(cfg, cfg.batch, seed=i)).to(torch.bfloat16).cuda() for i in range(2)]
dys = [torch.from_numpy(workloads.generate_dy(cfg, cfg.batch, seed=10 + i)).to(torch.bfloat16).cuda()
       for i in range(2)]
dx = torch.empty_like(xs[0])
g = bw.alloc_grads()
for i in range(reps):
    bw.backward_into(xs[i % 2], dys[i % 2], dx, g)
torch.cuda.synchronize()
print(f"{name}: {reps} backward passes ok, launches {bw.launches}")
