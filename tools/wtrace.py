"""Pipeline trace of CTA 0 of the fused tensor-core kernel (debug tool).
usage: python tools/wtrace.py <config> [batch]"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads
from paper_2006_06443_b200 import LrsConv
from paper_2006_06443_b200.lrs_conv import load_library
name = sys.argv[1]; batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = workloads.CONFIGS[name]; inp = workloads.generate(cfg, batch=batch)
layer = LrsConv.from_inputs(inp)
x = torch.from_numpy(inp.x).to(torch.bfloat16).cuda()
y = layer(x); torch.cuda.synchronize()
tr = torch.zeros(12000, dtype=torch.int64, device="cuda")
load_library().lrs_conv_debug_trace(ctypes.c_void_p(layer.handle), ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    layer.forward_into(x, y)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
t0 = t[1004]
print(f"epilogue: woke {t[1001]-t0} staged {t[1005]-t0} barrier {t[1006]-t0} store-read {t[1007]-t0} end {t[1002]-t0}")
print(f"kernel start -> tmem ready {t[1003]-t0} ns; acc_full(mma done) {t[1000]-t0} ns; epi start {t[1001]-t0}; end {t[1002]-t0}")
idx = [i for i in range(500) if t[2*i] != 0]
w = [(t[2*i]-t0, t[2*i+1]-t0) for i in idx]
n = len(w)
print(f"{n} sparse items; first wait start {w[0][0]} done {w[0][1]}")
for i in range(0, n, max(1, n // 25)):
    print(f"item {i:4d}: wait start {w[i][0]:8d} ns, got {w[i][1]:8d} ns (waited {w[i][1]-w[i][0]:6d})")
gaps = np.diff([x[1] for x in w])
print(f"median item-to-item {np.median(gaps):.0f} ns, mean {gaps.mean():.0f} ns; total waiting {sum(x[1]-x[0] for x in w)} ns")

nb = 0
while nb < 2048 and t[2000 + 3 * nb] != 0: nb += 1
st = np.array([t[2000 + 3 * b] for b in range(nb)]); en = np.array([t[2000 + 3 * b + 2] for b in range(nb)])
sm = np.array([t[2000 + 3 * b + 1] for b in range(nb)]); ep = np.array([t[8200 + b] for b in range(nb)])
base = st.min()
print(f"{nb} CTAs: start spread {st.max()-base} ns; end min {en.min()-base} max {en.max()-base}; dur min {(en-st).min()} med {np.median(en-st):.0f} max {(en-st).max()}")
print(f"  mainloop (start->acc_full) med {np.median(ep-st):.0f} max {(ep-st).max()}; epilogue (acc_full->end) med {np.median(en-ep):.0f} max {(en-ep).max()}")
print(f"  distinct SMs {len(set(sm.tolist()))}")
