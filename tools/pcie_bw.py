"""Host<->device copy bandwidth of pinned buffers the size of C3's per-step X / Y (12.85 MB): H2D, D2H, and both
at once on two streams -- the ceiling of bench.py's e2e number (tools/, not product)."""
import torch, time
n = 12845056
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
h2d = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timeit(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
bb = timeit(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  concurrent both: {n/bb/1e9:.1f} GB/s per direction ({bb*1e6:.0f} us for 12.85 MB each way)")
