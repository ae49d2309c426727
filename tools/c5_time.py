"""Quick C5 timing (debug): full network forward at batch 256, CUDA graph."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_2006_06443_b200.resnet import build_compressed_resnet50
import torchvision
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
model, comp = build_compressed_resnet50(batch_max=n)
x = torch.from_numpy(workloads.resnet50_images(n)).to(torch.bfloat16).cuda().contiguous(memory_format=torch.channels_last)
def tg(m):
    s = torch.cuda.Stream()
    with torch.no_grad(), torch.cuda.stream(s):
        m(x); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            m(x)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [g.replay() for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10
t = tg(model)
print(f"compressed resnet50 n={n}: {t:.3f} ms/forward, {n/t*1e3:.0f} img/s")
from paper_2006_06443_b200.resnet import fold_dense_batchnorms
for fold in (False, True):
    torch.manual_seed(0)
    dense = torchvision.models.resnet50(weights=None).eval()
    if fold:
        dense = fold_dense_batchnorms(dense)
    dense = dense.cuda().to(torch.bfloat16).to(memory_format=torch.channels_last)
    t2 = tg(dense)
    print(f"dense cuDNN resnet50 (dense BNs folded: {fold}) n={n}: {t2:.3f} ms/forward, {n/t2*1e3:.0f} img/s")
# per compressed layer time
for idx, c in comp.items():
    c.layer.set_timing(True); c.layer.stage_times(reset=True)
with torch.no_grad():
    for _ in range(3): model(x)
torch.cuda.synchronize()
tot = 0
for idx, c in comp.items():
    st = c.layer.stage_times(reset=True)
    us = {k: v[0] / max(v[1], 1) * 1e3 for k, v in st.items()}
    tot += sum(us.values())
    print(idx, c.cfg.in_h, c.cfg.c_in, c.cfg.stride, {k: round(v, 1) for k, v in us.items()})
print(f"sum of compressed-layer kernels {tot:.1f} us")
