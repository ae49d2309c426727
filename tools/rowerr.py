"""Per-output-row / per-channel-block error of one config vs the oracle (debug)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads
from oracle import lrs_oracle as O
from paper_2006_06443_b200 import LrsConv
name = sys.argv[1]; batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = workloads.CONFIGS[name]; inp = workloads.generate(cfg, batch=batch)
layer = LrsConv.from_inputs(inp)
x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
y = layer(x).float().cpu().numpy().astype(np.float64); torch.cuda.synchronize()
ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values, cfg.stride, cfg.pad)
e = np.abs(y - ref)
print("per ho row max err:", [f"{e[:, h].max():.2e}" for h in range(e.shape[1])])
print("per wo col max err:", [f"{e[:, :, w].max():.2e}" for w in range(e.shape[2])])
print("per image max err:", [f"{e[n].max():.2e}" for n in range(e.shape[0])])
print("per 32-ch block max err:", [f"{e[..., c:c+32].max():.2e}" for c in range(0, e.shape[3], 32)])
