"""the B200 replay of the paper's speed-bound study (§4.3
"Speedup bound", :240-296, Tables lr_speedup_x1/x2/x3 at :250-266, :507-541).

For every ResNet-50 conv layer of Table 2 (the 7x7 stem is skipped:
its 3 input channels are below the library's 16-byte TMA rows) at 1x / 2x / 3x input size:
  * dense: cuDNN conv2d (torch, bf16, channels_last) -- the paper's "original layer";
  * low-rank only, at compression 1.5 / 2 / 3 / 5 / 10 / 20x: the paper's CP form
     through the C ABI (LRS_CORE_CP, no sparse term; 1x1 stride-1 layers as
    the SVD pair), rank R = floor(P(W) / (c * P per rank)), P per rank = Cin + Cout + 2k
    (CP) or Cin + Cout (SVD), capped at the library's 256;
  * low rank (5x) + 1 % sparse: the whole compressed layer; its increment over the 5x
    low-rank layer is the sparse term's cost (the paper's "sparse component");
  * sparse only, 1 % ("S"): the paper's sparse-component arm, run as
    the cheapest layer the ABI allows -- L of rank 1 (padded to 16 inside the library)
    plus the 1 % S -- so its time is the sparse term plus a rank-16 chain.
Times are CUDA-event means of 20 back-to-back forwards after warm-up, batch 32 (the
per-GPU batch of C5 at 8 GPUs), synthetic seeded weights (speed does not depend on
trained values).  Writes profiles/r02_f2_speed_bound.json and prints the paper-style
tables: network-level speedup = sum of dense times / sum of compressed times.

usage: python tools/f2_speed_bound.py [batch]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torchvision  # noqa: E402

import workloads  # noqa: E402
from paper_2006_06443_b200 import LrsConv, LrsError  # noqa: E402

COMPRESSIONS = (1.5, 2, 3, 5, 10, 20)
SCALES = (1, 2, 3)


def conv_layers(scale):
    """(index, module, input H, W) of ResNet-50's 53 convs, in Table-2 order."""
    model = torchvision.models.resnet50(weights=None).eval()
    convs = [m for m in model.modules() if isinstance(m, torch.nn.Conv2d)]
    shapes = {}
    hooks = [m.register_forward_hook(lambda m, i, o, k=k: shapes.__setitem__(k, i[0].shape))
             for k, m in enumerate(convs)]
    with torch.no_grad():
        model(torch.zeros(1, 3, 224 * scale, 224 * scale))
    for h in hooks:
        h.remove()
    table = workloads.resnet50_table2()
    out = []
    for k, m in enumerate(convs):
        idx, cin, h, w, cout, kk = table[k]
        assert (m.in_channels, m.out_channels, m.kernel_size[0]) == (cin, cout, kk), (k, m)
        out.append((idx, m, shapes[k][2], shapes[k][3]))
    return out


def time_fn(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def lr_layer(n, h, w, cin, cout, k, s, p, rank, density, seed):
    rng = np.random.default_rng(seed)
    bf = workloads.bf16_round
    nnz = int(round(density * cin * cout * k * k))
    if nnz:
        pos = np.sort(rng.choice(cin * cout * k * k, nnz, replace=False))
        rows, cols = pos // (cin * k * k), pos % (cin * k * k)
        rp = np.zeros(cout + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        rp = np.cumsum(rp)
        vals = bf(rng.standard_normal(nnz).astype(np.float32) * np.sqrt(0.1))
    else:
        rp, cols, vals = np.zeros(cout + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32)
    a = bf((rng.standard_normal((cin, rank)) / np.sqrt(cin)).astype(np.float32))
    d = bf((rng.standard_normal((cout, rank)) / np.sqrt(rank)).astype(np.float32))
    if k == 1 and s == 1 and p == 0:  # SVD pair
        return LrsConv(n, h, w, cin, cout, 1, 1, 0, rank, rank, "bf16", a, None, np.ascontiguousarray(d.T),
                       rp, cols.astype(np.int32), vals)
    b = bf((rng.standard_normal((k, rank)) / np.sqrt(k)).astype(np.float32))
    c = bf((rng.standard_normal((k, rank)) / np.sqrt(k)).astype(np.float32))
    return LrsConv.from_cp(n, h, w, k, s, p, "bf16", a, b, c, d, rp, cols.astype(np.int32), vals)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    dev = torch.device("cuda:0")
    rows = []
    for scale in SCALES:
        for idx, m, h, w in conv_layers(scale):
            cin, cout, k = m.in_channels, m.out_channels, m.kernel_size[0]
            s, p = m.stride[0], m.padding[0]
            if cin % 8:
                continue  # the stem: 3 input channels
            x = torch.randn(n, cin, h, w, device=dev, dtype=torch.bfloat16).contiguous(
                memory_format=torch.channels_last)
            wt = torch.randn(cout, cin, k, k, device=dev, dtype=torch.bfloat16).contiguous(
                memory_format=torch.channels_last)
            t_dense = time_fn(lambda: torch.nn.functional.conv2d(x, wt, stride=s, padding=p))
            p_w = cin * cout * k * k
            per_rank = cin + cout + (0 if (k == 1 and s == 1) else 2 * k)
            row = {"scale": scale, "layer": idx, "cin": cin, "cout": cout, "k": k, "stride": s, "h": h, "w": w,
                   "dense_us": t_dense, "lr": {}}
            for c in COMPRESSIONS + ("5+S", "S"):
                cc = 5 if c == "5+S" else c
                rank = 1 if c == "S" else int(min(256, max(1, p_w // (cc * per_rank))))
                try:
                    layer = lr_layer(n, h, w, cin, cout, k, s, p, rank, 0.01 if c in ("5+S", "S") else 0.0, seed=idx)
                except LrsError as e:  # e.g. output width > 128 at 3x input
                    row["lr"][str(c)] = {"rank": rank, "unsupported": str(e)}
                    continue
                y = torch.empty(n, cout, layer.out_h, layer.out_w, device=dev, dtype=torch.bfloat16).contiguous(
                    memory_format=torch.channels_last)
                t = time_fn(lambda: layer.forward_into(x, y))
                row["lr"][str(c)] = {"rank": rank, "us": t, "speedup": t_dense / t}
                layer.close()
            rows.append(row)
            sp = lambda c: f"{row['lr'][str(c)]['speedup']:.2f}" if "us" in row["lr"][str(c)] else "n/a"  # noqa: E731
            print(f"x{scale} L{idx:2d} {cin:4d}->{cout:4d} k{k} s{s} {h}x{w}: dense {t_dense:8.1f} us | "
                  + " ".join(f"{c}x:{sp(c)}" for c in COMPRESSIONS) + f" | 5x+S {sp('5+S')} | S-only {sp('S')}",
                  flush=True)
            del x, wt
    summary = {}
    for scale in SCALES:
        rs = [r for r in rows if r["scale"] == scale and all("us" in v for v in r["lr"].values())]
        dense = sum(r["dense_us"] for r in rs)
        summary[f"x{scale}"] = {str(c): dense / sum(r["lr"][str(c)]["us"] for r in rs)
                                for c in COMPRESSIONS + ("5+S", "S")}
    out = {"batch": n, "device": torch.cuda.get_device_name(0), "rows": rows, "network_speedup": summary,
           "layers_in_totals": {f"x{s_}": sum(1 for r in rows if r["scale"] == s_ and
                                              all("us" in v for v in r["lr"].values())) for s_ in SCALES},
           "paper_cpu_x1": {"1.5": 1.08, "2": 1.2, "3": 1.39, "5": 1.66, "10": 2.03, "20": 2.33},
           "note": "network speedup = sum of cuDNN dense conv times / sum of compressed-layer times over the "
                   "52 layers (stem excluded); paper_cpu_x1 = PAPER.md:250-266 (i3-8130U CPU), context only"}
    for d in ("profiles", "gpurun_out"):  # gpurun_out/ travels back from the GPU box
        if os.path.isdir(os.path.join(ROOT, d)):
            with open(os.path.join(ROOT, d, "r02_f2_speed_bound.json"), "w") as f:
                json.dump(out, f, indent=1)
    print("\nnetwork-level speedup of the low-rank layers vs cuDNN dense (paper CPU x1 for context):")
    print("compression | " + " | ".join(f"x{s} input" for s in SCALES) + " | paper CPU x1")
    for c in COMPRESSIONS:
        print(f"{c:>5}x      | " + " | ".join(f"{summary[f'x{s}'][str(c)]:.2f}x" for s in SCALES)
              + f" | {out['paper_cpu_x1'][str(c)]}x")
    print("5x + 1% S   | " + " | ".join(f"{summary[f'x{s}']['5+S']:.2f}x" for s in SCALES) + " |")
    print("S only (1%) | " + " | ".join(f"{summary[f'x{s}']['S']:.2f}x" for s in SCALES) + " | paper CPU: up to 13x")


if __name__ == "__main__":
    main()
