"""Per-CTA timeline of the fused tensor-core kernel (debug tool).
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
for _ in range(3000):  # warm the clocks up first (an idle GPU runs the first forwards slowly)
    layer.forward_into(x, y)
torch.cuda.synchronize()
tr = torch.zeros(12000, dtype=torch.int64, device="cuda")
load_library().lrs_conv_debug_trace(ctypes.c_void_p(layer.handle), ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    layer.forward_into(x, y)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
nb = 0
while nb < 2048 and t[2000 + 3 * nb] != 0: nb += 1
st = np.array([t[2000 + 3 * b] for b in range(nb)]); en = np.array([t[2000 + 3 * b + 2] for b in range(nb)])
base = st.min()
print(f"{name} n={x.shape[0]}: {nb} CTAs; start spread {st.max()-base} ns; end max {en.max()-base} ns; "
      f"CTA dur min {(en-st).min()} med {np.median(en-st):.0f} max {(en-st).max()}")
t0 = t[2000]
for k in range(16):
    if t[100 + 4 * k] == 0: break
    a, b, c, d = (t[100 + 4 * k + i] - t0 for i in range(4))
    ws = [(t[200 + 16 * k + 2 * w] - t0, t[200 + 16 * k + 2 * w + 1] - t0) for w in range(8) if t[200 + 16 * k + 2 * w]]
    print(f"tile {k}: mma start {a} end {b} | epi woke {c} done {d} | windows (wait, got): {ws}")
pi = [(t[3000 + 3 * i] - t0, t[3000 + 3 * i + 1] - t0, t[3000 + 3 * i + 2] - t0) for i in range(64) if t[3000 + 3 * i]]
mi = [(t[3300 + 3 * i] - t0, t[3300 + 3 * i + 1] - t0, t[3300 + 3 * i + 2] - t0) for i in range(64) if t[3300 + 3 * i]]
print("producer items (wait a_empty, got, issued):", pi[:14])
print("mma items (wait a_full, got, committed):", mi[:14])
wi = [t[3600 + i] - t0 for i in range(16) if t[3600 + i]]
print("producer window issue times:", wi)
pi = [(t[3000 + 3 * i] - t0, t[3000 + 3 * i + 1] - t0, t[3000 + 3 * i + 2] - t0) for i in range(64) if t[3000 + 3 * i]]
print("producer items (start, got slot, issued):", pi[:12])
