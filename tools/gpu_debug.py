"""Stage-by-stage GPU check of one config against numpy fp64 (debug tool).

usage: python tools/gpu_debug.py <config> [batch]
Prints relative L2 errors of T1, T2 and Y vs the oracle; exits non-zero on
failure.  Run each config in its own process (a device fault kills the context).
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads
from oracle import lrs_oracle as O
from paper_2006_06443_b200 import LrsConv


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    name = sys.argv[1]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
    cfg = workloads.CONFIGS[name]
    inp = workloads.generate(cfg, batch=batch)
    n = inp.x.shape[0]
    t0 = time.time()
    layer = LrsConv.from_inputs(inp)
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    x = torch.from_numpy(inp.x).to(tdt).cuda()
    y = layer(x)
    torch.cuda.synchronize()
    print(f"[{name}] n={n} forward ok ({time.time()-t0:.2f}s) launches={layer.launches_per_forward}", flush=True)
    X = inp.x.astype(np.float64)
    P_in = n * cfg.in_h * cfg.in_w
    t1 = layer.debug_buffer(0, P_in).float().cpu().numpy()[:, :cfg.rank_in]
    t1_ref = X.reshape(P_in, -1) @ inp.u_in.astype(np.float64)
    print(f"  T1 relL2 = {rel(t1, t1_ref):.3e}")
    if inp.core is not None:
        P = n * cfg.out_h * cfg.out_w
        t2 = layer.debug_buffer(1, P).float().cpu().numpy()[:, :cfg.rank_out]
        t2_ref = O.conv_direct(t1_ref.reshape(n, cfg.in_h, cfg.in_w, -1), inp.core, cfg.stride, cfg.pad).reshape(P, -1)
        print(f"  T2 relL2 = {rel(t2, t2_ref):.3e}   (vs T2 from GPU T1: {rel(t2, O.conv_direct(t1.reshape(n, cfg.in_h, cfg.in_w, -1).astype(np.float64), inp.core, cfg.stride, cfg.pad).reshape(P,-1)):.3e})")
    yref, yl, ys = O.forward_factored(X, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                                      inp.values, cfg.stride, cfg.pad, return_parts=True)
    yg = y.float().cpu().numpy().astype(np.float64)
    e = rel(yg, yref)
    print(f"  Y relL2 = {e:.3e}  maxabs = {np.abs(yg - yref).max():.3e}  |Y_L|={np.linalg.norm(yl):.3e} |Y_S|={np.linalg.norm(ys):.3e}")
    print(f"  Y - Y_L relL2 vs Y_S: {rel(yg - yl, ys):.3e};  Y - Y_S vs Y_L: {rel(yg - ys, yl):.3e}")
    tol = 1e-5 if cfg.dtype == "f32" else 2e-2
    # timing
    layer.set_timing(True)
    for _ in range(3):
        layer.forward_into(x, y)
    torch.cuda.synchronize()
    layer.stage_times(reset=True)
    iters = 20
    s, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        layer.forward_into(x, y)
    e2.record()
    torch.cuda.synchronize()
    st = layer.stage_times(reset=True)
    print(f"  forward {s.elapsed_time(e2)/iters*1e3:.1f} us/iter; stages: " +
          ", ".join(f"{k}={v[0]/max(v[1],1)*1e3:.1f}us" for k, v in st.items()))
    sys.exit(0 if e < tol else 1)


if __name__ == "__main__":
    main()
