"""Timeline of CTA 0 of the channel-stationary 1x1 kernel (lrs_pw.cuh; debug tool, needs
a LRS_WCONV_DEBUG=1 or LRS_EXPERIMENTS=1 build).  usage: python tools/ptrace.py [config]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv  # noqa: E402
from paper_2006_06443_b200.lrs_conv import load_library  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = workloads.CONFIGS[name]
layer = LrsConv.from_inputs(workloads.generate(cfg, batch=1), batch_max=cfg.batch)
x = torch.from_numpy(workloads.generate_x(cfg, cfg.batch)).to(torch.bfloat16).cuda()
y = torch.empty((cfg.batch, cfg.out_h, cfg.out_w, cfg.c_out), dtype=torch.bfloat16, device="cuda")
for _ in range(2000):
    layer.forward_into(x, y)
torch.cuda.synchronize()
tr = torch.zeros(4000, dtype=torch.int64, device="cuda")
load_library().lrs_conv_debug_trace(ctypes.c_void_p(layer.handle), ctypes.c_void_p(tr.data_ptr()))
for _ in range(2):
    layer.forward_into(x, y)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
t0 = t[0]
print(f"{name}: weights in after {t[1] - t0} ns")
for k in range(16):
    if t[100 + 4 * k] == 0:
        break
    a, b, c, d = (t[100 + 4 * k + i] - t0 if t[100 + 4 * k + i] else -1 for i in range(4))
    print(f"tile {k}: mma start {a} acc free {b} | epi woke {c} done {d}")
prod = [(t[1000 + 2 * i] - t0, t[1001 + 2 * i] - t[1000 + 2 * i]) for i in range(200) if t[1000 + 2 * i]]
mma = [(t[2000 + i] - t0) for i in range(200) if t[2000 + i]]
print("producer (slot acquired, issue ns):", prod[:60])
print("mma chunk arrived:     ", mma[:60])
