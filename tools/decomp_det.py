"""Determinism / parity probe of the GPU decomposition (f4): two runs of k iterations on the
same inputs, factors compared bitwise and against the oracle, per k."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from oracle import lrs_decomp as D  # noqa: E402
from paper_2006_06443_b200 import LrsDecomp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_decomp"
cfg = workloads.DECOMP_CONFIGS[name]
w, f0 = workloads.generate_decomp(cfg)
wd = torch.from_numpy(w).cuda()
for k in (1, 2, 3):
    outs = []
    for rep in range(2):
        dc = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=k, tol=-float("inf"))
        fs = [torch.from_numpy(f).cuda() for f in f0]
        idx, val, eps = dc.run(wd, fs)
        torch.cuda.synchronize()
        outs.append(([f.cpu().numpy() for f in fs], idx.cpu().numpy(), eps))
    rf, (ridx, _), reps = D.decompose_lrs(w, f0, cfg.cardinality, max_iters=k, tol=-float("inf"))
    same = [bool(np.array_equal(a, b)) for a, b in zip(outs[0][0], outs[1][0])]
    rel = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(outs[0][0], rf)]
    print(f"k={k}: runs bitwise per factor {same}, S same {np.array_equal(outs[0][1], outs[1][1])}, "
          f"rel vs oracle {['%.2e' % x for x in rel]}, S = oracle {np.array_equal(outs[0][1], ridx)}, "
          f"eps {outs[0][2]} vs {reps}")

# concurrent handles, as bench.py --decompose creates them
never = -float("inf")
warm = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=3, tol=never)
fw = [torch.from_numpy(f).cuda() for f in f0]
warm.run(wd, fw)
dc = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=30, tol=never)
fs = [torch.from_numpy(f).cuda() for f in f0]
_, _, eps = dc.run(wd, fs)
chk = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=3, tol=never)
fc = [torch.from_numpy(f).cuda() for f in f0]
_, _, ce = chk.run(wd, fc)
print("concurrent handles: timed", eps[:3], "chk", ce)
