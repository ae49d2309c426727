"""Debug: fp32 split-engine error pattern per geometry (images, channels, rows)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads
from oracle import lrs_oracle as O
from paper_2006_06443_b200 import LrsConv
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_spadd_f32 import GEOMS

for g in GEOMS:
    n, h, w, cin, cout, k, s, p, r1, r2, dens, svd, eng = g
    cfg = workloads.LayerConfig("t", n, h, w, cin, cout, k, s, p, r1, r1 if svd else r2, dens, "f32", svd, seed=13)
    inp = workloads.generate(cfg)
    layer = LrsConv.from_inputs(inp)
    y = layer(torch.from_numpy(inp.x).float().cuda()).cpu().numpy().astype(np.float64)
    ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                             inp.values, s, p)
    d = np.abs(y - ref)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    bad = d > 1e-4
    print(g, "engine", layer.sparse_engine[0], "relL2 %.3e" % err, "bad", int(bad.sum()), flush=True)
    if bad.any():
        print("  images", np.unique(np.nonzero(bad)[0])[:20], "rows", np.unique(np.nonzero(bad)[1])[:20],
              "cols", np.unique(np.nonzero(bad)[2])[:20], "chans", np.unique(np.nonzero(bad)[3])[:40])
    layer.close()
