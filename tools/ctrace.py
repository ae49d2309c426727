"""Per-CTA timeline of the fused a1 + a2 kernel (lrs_core.cuh; debug tool, needs a
LRS_WCONV_DEBUG=1 build).  Stamps (ns from CTA 0's start): producer first X request,
MMA got first X chunk / a1 issued / T1 window restaged / a2 issued, epilogue woke on
T1 / restage done / woke on T2 / T2 stored -- per tile of CTA 0.
usage: python tools/ctrace.py <config> [batch]   (env LRS_CORE_IPT / LRS_CORE_TH apply)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv  # noqa: E402
from paper_2006_06443_b200.lrs_conv import load_library  # noqa: E402

name = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = workloads.CONFIGS[name]
inp = workloads.generate(cfg, batch=batch)
layer = LrsConv.from_inputs(inp)
x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
y = layer(x)
torch.cuda.synchronize()
for _ in range(3000):  # warm the clocks up first (an idle GPU runs the first forwards slowly)
    layer.forward_into(x, y)
torch.cuda.synchronize()
tr = torch.zeros(14000, dtype=torch.int64, device="cuda")
load_library().lrs_conv_debug_trace(ctypes.c_void_p(layer.handle), ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    layer.forward_into(x, y)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
nb = 0
while nb < 2048 and t[9000 + 2 * nb] != 0:
    nb += 1
st = np.array([t[9000 + 2 * b] for b in range(nb)])
en = np.array([t[9000 + 2 * b + 1] for b in range(nb)])
base = st.min()
print(f"{name} n={x.shape[0]}: core kernel {nb} CTAs; start spread {st.max() - base} ns; end max {en.max() - base} ns;"
      f" CTA dur min {(en - st).min()} med {np.median(en - st):.0f} max {(en - st).max()}")
w0 = t[2000] if t[2000] else 0
if w0:
    print(f"  fused kernel CTA 0 start at {w0 - base} ns after the core kernel's first CTA")
t0 = t[9000]
print(f"  CTA 0: pdl wait returned {t[8190] - t0} ns after start")
labels = ["-", "prod X req", "mma got X", "a1 issued", "epi T1 woke", "restaged", "mma T1s woke", "a2 issued",
          "epi T2 woke", "T2 stored"]
for k in range(4):
    if t[8200 + 10 * k + 2] == 0:
        break
    print(f"  tile {k}: " + ", ".join(f"{labels[i]} {t[8200 + 10 * k + i] - t0}" for i in range(1, 10)
                                    if t[8200 + 10 * k + i]))
