"""Small forwards of every engine for compute-sanitizer (racecheck / synccheck / memcheck):
python tools/sanitize_run.py.  One process, tiny batches, each output checked against the
fp64 oracle so a tool-perturbed run that computes garbage also fails."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from oracle import lrs_oracle as O  # noqa: E402
from paper_2006_06443_b200 import LrsConv  # noqa: E402

CASES = [("c1", 1), ("c2_bf16", 2), ("c2_f32", 2), ("c3", 2), ("c4", 2)]


def main():
    worst = 0.0
    for name, n in CASES:
        cfg = workloads.CONFIGS[name]
        inp = workloads.generate(cfg, batch=n)
        layer = LrsConv.from_inputs(inp)
        tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        y = layer(torch.from_numpy(inp.x).to(tdt).cuda())
        torch.cuda.synchronize()
        ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                                 inp.values, cfg.stride, cfg.pad)
        err = float(np.linalg.norm(y.float().cpu().numpy() - ref) / np.linalg.norm(ref))
        tol = 1e-5 if cfg.dtype == "f32" else 2e-2
        print(f"{name} n={n}: engine {layer.sparse_engine} expand {layer.expand_kernel} core_fused {layer.core_fused} "
              f"relL2 {err:.2e}", flush=True)
        assert err <= tol, (name, err)
        worst = max(worst, err / tol)
        layer.close()
    # a CP layer (fused a1 + depthwise) and a stride-2 layer (three kernels)
    cfg = workloads.CP_CONFIGS["c2_cp"]
    inp = workloads.generate_cp(cfg, batch=2)
    layer = LrsConv.from_cp(2, cfg.in_h, cfg.in_w, cfg.k, cfg.stride, cfg.pad, cfg.dtype, inp.a, inp.b, inp.c, inp.d,
                            inp.row_ptr, inp.col_idx, inp.values)
    y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    ref = O.forward_cp(inp.x.astype(np.float64), inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx, inp.values,
                       cfg.stride, cfg.pad)
    err = float(np.linalg.norm(y.float().cpu().numpy() - ref) / np.linalg.norm(ref))
    print(f"c2_cp n=2: relL2 {err:.2e}", flush=True)
    assert err <= 2e-2
    cfg = workloads.LayerConfig("s2", 2, 14, 14, 64, 64, 3, 2, 1, 16, 16, 0.03, "bf16", seed=3)
    inp = workloads.generate(cfg)
    layer = LrsConv.from_inputs(inp)
    y = layer(torch.from_numpy(inp.x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                             inp.values, cfg.stride, cfg.pad)
    err = float(np.linalg.norm(y.float().cpu().numpy() - ref) / np.linalg.norm(ref))
    print(f"stride-2 bf16 n=2: relL2 {err:.2e}", flush=True)
    assert err <= 2e-2
    print("sanitize_run: all cases ok")


if __name__ == "__main__":
    main()
