"""Debug: one small bf16 CP layer through the fused core kernel (CPDW) vs the chain."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads
from paper_2006_06443_b200 import LrsConv
a = [int(v) for v in sys.argv[1:]] or [2, 9, 11, 64, 64, 3, 0, 32]
n_, h_, w_, ci, co, k_, pd, r_ = a
cfg = workloads.LayerConfig("t", n_, h_, w_, ci, co, k_, 1, pd, r_, r_, 0.02, "bf16", seed=31)
inp = workloads.generate_cp(cfg)
c = cfg
layer = LrsConv.from_cp(n_, c.in_h, c.in_w, c.k, c.stride, c.pad, c.dtype, inp.a, inp.b, inp.c, inp.d,
                        inp.row_ptr, inp.col_idx, inp.values)
print("fused", layer.core_fused, flush=True)
y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
torch.cuda.synchronize()
print("ok", float(y.float().abs().sum()))
