#!/usr/bin/env python
"""Benchmark of the B200 compressed convolution W ~ L + S (arXiv 2006.06443).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl lrs|reference]
(N > 1: launched by torchrun, one process per GPU; RANK/WORLD_SIZE from env.)

A step = one forward of the whole hot path (a1 projection, a2 core, a3
expansion + a4 sparse + a5 sum/store) over one batch of the workload.
Default workload: BASELINE.json configs[2] = C3, the largest compressed-conv
layer (ResNet-50 layer4 3x3 512->512 at 7x7, batch 256, Tucker-2 (128,128),
5 % S, bf16).  Strong scaling at N > 1: the config's global batch is split
over the ranks (dist.shard_range; --scaling weak gives every rank a full
batch); weights are replicated, no collective on the data path.

Timing: W untimed warm-up steps, then EXACTLY K steps replayed from a CUDA
graph, bracketed by barrier + cuda.synchronize; CUDA events on the launching
stream; max over ranks.  Inputs rotate over enough X/Y buffer sets of
DISTINCT seeded images to cover 2.1x the L2, so every step reads X from
HBM; >= 10 further replays are timed one by one (median reported).  After
timing (untimed): every rotating Y is checked bitwise against an eager
forward of its X, the shards of set 0 are gathered over NCCL and compared
bitwise with a 1-GPU forward of the whole batch and, on sampled images, with
the fp64 oracle.  Refuses to run with LRS_* experiment variables set.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

CONFIG_TEXT = {
    "c1": "C1: 3x3 conv 64->64 @56x56, stride 1, pad 1, batch 1, Tucker-2 (16,16), S 1% (369 nnz), fp32",
    "c2_f32": "C2: ResNet-50 layer3 3x3 conv 256->256 @14x14, batch 64, Tucker-2 (64,64), S 2%, fp32",
    "c2_bf16": "C2: ResNet-50 layer3 3x3 conv 256->256 @14x14, batch 64, Tucker-2 (64,64), S 2%, bf16",
    "c3": "C3: ResNet-50 layer4 3x3 conv 512->512 @7x7, batch 256, Tucker-2 (128,128), S 5%, bf16",
    "c4": "C4: ResNet-50 1x1 expansion 256->1024 @14x14, batch 128, SVD rank 64, S 1%, bf16",
    "c1_cp": "C1 shape with the paper's CP form of L (SURVEY 8f f1): 3x3 conv 64->64 @56x56, batch 1, "
             "CP rank 16 (1x1, 3x1 + 1x3 depthwise, 1x1), S 1%, fp32",
    "c2_cp": "C2 shape with the paper's CP form of L (SURVEY 8f f1): 3x3 conv 256->256 @14x14, batch 64, "
             "CP rank 64 (1x1, 3x1 + 1x3 depthwise, 1x1), S 2%, bf16",
    "c5": "C5: full ResNet-50 forward, global batch 256 (224x224x3 N(0,1) images), random-init weights, "
          "16 3x3 convs -> Tucker-2 (Cin/4, Cout/4) + 2% S via the C-ABI, other layers dense cuDNN, bf16",
}
METRIC = "compressed-conv images/s and % of roofline at 1/2/4/8 B200 vs CPU oracle"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=sorted(workloads.CONFIGS) + sorted(workloads.CP_CONFIGS) + ["c5"])
    ap.add_argument("--impl", default="lrs", choices=["lrs", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = the config's global batch split over the ranks (default), "
                         "weak = a full batch per rank")
    ap.add_argument("--replays", type=int, default=10, help="separately timed graph replays (median reported)")
    ap.add_argument("--no-dense", action="store_true", help="skip the cuDNN dense context row")
    ap.add_argument("--tucker2", action="store_true",
                    help="with --decompose: L in Tucker-2 form (lrs_tucker2_run, HOOI sweeps) at ranks 128 / 128")
    ap.add_argument("--decompose", action="store_true",
                    help="time the GPU low-rank + sparse decomposition of the layer's weight shape (SURVEY 8f f4)")
    ap.add_argument("--backward", action="store_true",
                    help="time the layer's backward pass (dX + parameter gradients, SURVEY 8f f3) instead")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        return 1


def oracle_rate(cfg, inp, seconds: float, sample_images: int, x_all):
    """Time the fp64 oracle (forward_factored, as it stands) on a bounded
    sample of the workload: repeated calls on `sample_images` images."""
    from oracle import lrs_oracle as O
    x = x_all[:sample_images].astype(np.float64)
    calls, t0 = 0, time.perf_counter()
    while True:
        if isinstance(inp, workloads.CpInputs):
            O.forward_cp(x, inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx, inp.values, cfg.stride, cfg.pad)
        else:
            O.forward_factored(x, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values,
                               cfg.stride, cfg.pad)
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds and calls >= 2:
            break
    return calls * sample_images / el, calls, el


class ClockSampler:
    """NVML SM clock / throttle-reason sampling during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def run_reference(args, cfg):
    """--impl reference: the oracle (fp64 numpy, as it stands) on host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # a bounded sample per step: 8 images (2 for C3, whose fp64 oracle takes ~70 ms/image)
    sample = max(1, min(cfg.batch, 2 if cfg.c_in >= 512 else 8))
    is_cp = args.config in workloads.CP_CONFIGS
    inp = (workloads.generate_cp if is_cp else workloads.generate)(cfg, batch=sample)
    from oracle import lrs_oracle as O
    x = inp.x.astype(np.float64)

    def step():
        if is_cp:
            O.forward_cp(x, inp.a, inp.b, inp.c, inp.d, inp.row_ptr, inp.col_idx, inp.values, cfg.stride, cfg.pad)
        else:
            O.forward_factored(x, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values,
                               cfg.stride, cfg.pad)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps * sample / el
    line = {"metric": METRIC, "value": value, "unit": "images/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads/)",
            "config": {"workload": CONFIG_TEXT[args.config], "config_id": args.config, "images_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
                             "sample": f"{sample} images of {args.config} per step (fp64 numpy oracle, "
                                       f"{'forward_cp' if is_cp else 'forward_factored'})", **host_info()},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference_c5(args):
    """--impl reference for C5: the fp64 CPU reference network (oracle/resnet_oracle.py)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import resnet_oracle as R
    img = workloads.resnet50_images(1)
    for _ in range(min(args.warmup, 1)):
        R.reference_logits(img)
    t0 = time.perf_counter()
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        R.reference_logits(img)
    el = time.perf_counter() - t0
    value = steps / el
    line = {"metric": METRIC, "value": value, "unit": "images/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": el / steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, workloads/)",
            "config": {"workload": CONFIG_TEXT["c5"], "images_per_step": 1},
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
                             "sample": "1 image per step through the fp64 reference network"},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def network_work(model, x1, comp):
    """Algorithmic bytes and FLOPs of ONE image through the compressed ResNet-50, from
    forward hooks: every conv / pool / linear / compressed layer reads its input and
    writes its output once (bf16), every bottleneck reads its identity once for the
    residual add; BN is folded and ReLU / add fused.  FLOPs: 2 per MAC of
    the dense convs and FC, and each compressed layer's chain + in-bounds sparse term."""
    import torch
    from paper_2006_06443_b200 import roofline as RL
    lay = {id(c): c for c in comp.values()}
    acc = {"bytes": 0.0, "flops": 0.0}
    hooks = []

    def hook(m, inp, out):
        i, o = inp[0], out
        acc["bytes"] += 2.0 * (i.numel() + o.numel())
        if isinstance(m, torch.nn.Conv2d):
            acc["flops"] += 2.0 * o.numel() * m.in_channels * m.kernel_size[0] * m.kernel_size[1] / m.groups
        elif isinstance(m, torch.nn.Linear):
            acc["flops"] += 2.0 * m.in_features * m.out_features * o.shape[0]
        elif hasattr(m, "c") and id(m.c) in lay:
            c = m.c
            acc["flops"] += RL.layer_work(c.cfg, 1, workloads.generate_weights(c.cfg).col_idx)["layer"]["flops"]

    def block_hook(m, inp, out):
        acc["bytes"] += 2.0 * out.numel()  # the identity read of the residual add

    for name, m in model.named_modules():
        if isinstance(m, (torch.nn.Conv2d, torch.nn.Linear, torch.nn.MaxPool2d, torch.nn.AdaptiveAvgPool2d)) or (
                hasattr(m, "c") and id(getattr(m, "c")) in lay):
            hooks.append(m.register_forward_hook(hook))
        if type(m).__name__ == "Bottleneck":
            hooks.append(m.register_forward_hook(block_hook))
    with torch.no_grad():
        model(x1)
    torch.cuda.synchronize()
    for h in hooks:
        h.remove()
    return acc


def main_c5(args):
    """C5: the full network.  Global batch 256 split across ranks (strong
    scaling, BASELINE.json configs[4] 'batch-sharded'); one CUDA graph per rank
    holds the whole forward; timed by replaying it K times."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2006_06443_b200 import roofline as RL
    from paper_2006_06443_b200.resnet import build_compressed_resnet50
    from paper_2006_06443_b200.dist import shard_range
    gb = 256
    s0, s1 = shard_range(gb, rank, world)
    per = s1 - s0
    model, comp = build_compressed_resnet50(batch_max=per, device=local)
    img = workloads.resnet50_images(per, seed=rank)
    x = torch.from_numpy(img).to(torch.bfloat16).to(dev).contiguous(memory_format=torch.channels_last)
    stream = torch.cuda.Stream(device=dev)
    with torch.no_grad(), torch.cuda.stream(stream):
        model(x)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            logits = model(x)
    K, W = args.steps, args.warmup
    with torch.cuda.stream(stream):
        for _ in range(W):
            g.replay()
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device() if world == 1 else local)
    barrier()
    with sampler:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(K):
                g.replay()
            ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    t = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = gb * K / (ms_max / 1e3)

    # e2e: pinned host images -> device, graph replay, logits -> host, every step
    xh = torch.from_numpy(img).to(torch.bfloat16).contiguous(memory_format=torch.channels_last).pin_memory()
    lh = torch.empty(logits.shape, dtype=logits.dtype).pin_memory()
    ke = max(3, min(K, 20))
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(ke):
            x.copy_(xh, non_blocking=True)
            g.replay()
            lh.copy_(logits, non_blocking=True)
        e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": gb * ke / (float(te.item()) / 1e3), "unit": "images/s",
           "h2d_bytes_per_step": int(xh.numel() * 2), "d2h_bytes_per_step": int(lh.numel() * 2), "steps": ke,
           "api": "CUDA-graph forward of the compressed network (library layers via lrs_conv_forward)"}

    # per-layer kernel durations (event pairs around every library launch, eager)
    for c in comp.values():
        c.layer.set_timing(True)
        c.layer.stage_times(reset=True)
    with torch.no_grad(), torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e7))
        for _ in range(3):
            model(x)
    torch.cuda.synchronize(dev)
    peaks = RL.measured_peaks()
    tot = {}
    lay_bytes = lay_flops = lay_roof_s = 0.0
    for idx, c in comp.items():
        st = c.layer.stage_times(reset=True)
        for k, v in st.items():
            if v[1]:
                tot[k] = tot.get(k, 0.0) + v[0] / v[1]
        wk = RL.layer_work(c.cfg, per, workloads.generate_weights(c.cfg).col_idx)
        lay_bytes += wk["layer"]["bytes"]
        lay_flops += wk["layer"]["flops"]
        lay_roof_s += RL.layer_roofs(wk, peaks, "bf16")["t_literal_s"]
        c.layer.set_timing(False)
    t_layers = sum(tot.values()) / 1e3
    # network roof: algorithmic activation traffic of every compute op (input
    # read + output written once; residual identity read once; BN folded, ReLU / add fused)
    # and FLOPs (dense convs + FC + the compressed layers' chain + sparse term), per image
    net = network_work(model, x[:1], comp)
    t_net_img = max(net["bytes"] / (peaks["hbm_gbs"] * 1e9), net["flops"] / (peaks["bf16_tflops"] * 1e12))
    ach_gbs = net["bytes"] * value / world / 1e9  # per GPU
    roof = {"bound": "hbm" if net["bytes"] / peaks["hbm_gbs"] >= net["flops"] / peaks["bf16_tflops"] / 1e3 else
            "tensor", "unit": "GB/s", "achieved": ach_gbs, "peak": peaks["hbm_gbs"],
            "frac": ach_gbs / peaks["hbm_gbs"], "traffic": None, "kernel": "whole network (CUDA graph)",
            "peak_kind": "measured (MEASURED_PEAKS.json)",
            "network_roof_images_per_s_per_gpu": 1.0 / t_net_img,
            "frac_of_network_roof": (value / world) * t_net_img,
            "per_image": {"bytes": net["bytes"], "flops": net["flops"]},
            "what": "network roof max(bytes / HBM, FLOPs / bf16 peak) per image vs measured images/s per GPU; "
                    "bytes = every op's input read + output written once + residual reads (BN folded, "
                    "ReLU / add fused), FLOPs = dense convs + FC + compressed layers (chain + sparse)",
            "compressed_layers": {"kernel_us_sum": t_layers * 1e6, "literal_roof_us_sum": lay_roof_s * 1e6,
                                  "frac_literal": lay_roof_s / t_layers if t_layers else None,
                                  "bytes": lay_bytes, "flops": lay_flops,
                                  "stage_us_sum_16_layers": {k: round(v * 1e3, 1) for k, v in tot.items()}}}
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        from oracle import resnet_oracle as R
        one = workloads.resnet50_images(1)
        t0 = time.perf_counter()
        R.reference_logits(one)
        el = time.perf_counter() - t0
        cpu = {"value": 1.0 / el, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"1 image through the fp64 reference network ({el:.1f} s; conv_direct fp64 BLAS convs, "
                         "forward_factored compressed layers)"}
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded N(0,1) images, torchvision random init, seeded factors + S)",
        "config": {"workload": CONFIG_TEXT["c5"], "config_id": "c5", "global_batch": gb, "per_gpu_batch": per,
                   "parallelism": f"dp{world} (batch-sharded, no data-path collective)",
                   "l2": "per-step activation traffic (~14 GB at batch 256) >> L2 126 MiB; no rotation needed",
                   "timing": "CUDA graph of the whole forward replayed K times, CUDA events, max over ranks"},
        "clocks": sampler.summary(),
        "e2e": e2e,
        "gpu_launches": sum(c.layer.launches_per_forward for c in comp.values()) * K,
        "roofline": roof,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class ShardPlan:
    """How bench.py splits a layer workload over `world` ranks.
    strong (default at world > 1): the config's global batch is fixed and rank r takes
    images [start, end) = dist.shard_range(batch, r, world) of every rotating input set;
    set i's global X is workloads.generate_x(cfg, batch, seed=i), so the shards of all
    ranks together are exactly the 1-GPU input.  weak: every rank runs a full batch of
    its own images (seed 1000 (rank + 1) + i).  Used by the gloo test
    (tests/test_dist_cpu.py) to run the bench's own partition on CPU."""

    def __init__(self, cfg, rank: int, world: int, scaling: str = "strong"):
        from paper_2006_06443_b200.dist import shard_range
        self.cfg, self.rank, self.world = cfg, rank, world
        self.strong = scaling == "strong" and world > 1
        self.global_batch = cfg.batch if (self.strong or world == 1) else cfg.batch * world
        self.start, self.end = shard_range(self.global_batch, rank, world) if self.strong else (0, cfg.batch)

    def seed(self, i: int) -> int:
        return i if (self.strong or self.world == 1) else 1000 * (self.rank + 1) + i

    def x(self, i: int) -> np.ndarray:
        """this rank's images of rotating set i (NHWC, storage dtype values as float32)"""
        full = workloads.generate_x(self.cfg, self.cfg.batch, seed=self.seed(i))
        return full[self.start:self.end] if self.strong else full


def refuse_experiment_env():
    """Timing with a plan / engine override or (in experiment builds) a work-skipping
    knob would not measure the product's own path: refuse (include/lrs_conv.h)."""
    bad = sorted(k for k in os.environ if k.startswith("LRS_") and k != "LRS_VERBOSE")
    if bad:
        sys.stderr.write(f"bench.py: refusing to time with experiment variables set: {bad}\n")
        sys.exit(2)


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "affinity_cores": len(os.sched_getaffinity(0)), "os_cpu_count": os.cpu_count()}


def dense_weight(inp, cfg):
    """W = L + S as a dense [Cout, Cin, k, k] tensor (the cuDNN context row's weight;
    measurement-side arithmetic, not the product path)."""
    import torch
    if cfg.svd:
        wl = np.einsum("ca,aj->jc", inp.u_in.astype(np.float64), inp.u_out.astype(np.float64))[:, :, None, None]
    else:
        wl = np.einsum("ca,abyx,bj->jcyx", inp.u_in.astype(np.float64), inp.core.astype(np.float64),
                       inp.u_out.astype(np.float64), optimize=True)
    w = wl.reshape(cfg.c_out, -1).copy()
    rows = np.repeat(np.arange(cfg.c_out), np.diff(inp.row_ptr))
    w[rows, inp.col_idx] += inp.values
    return torch.from_numpy(w.reshape(cfg.c_out, cfg.c_in, cfg.k, cfg.k))


def main():
    args = parse()
    if args.impl != "reference":
        refuse_experiment_env()
    if args.decompose and args.config == "c5":
        main_decomp(args)  # the 16 ResNet-50 3x3 weights, decomposed concurrently
        return
    if args.config == "c5":
        if args.impl == "reference":
            run_reference_c5(args)
        else:
            main_c5(args)
        return
    is_cp = args.config in workloads.CP_CONFIGS
    cfg = workloads.CP_CONFIGS[args.config] if is_cp else workloads.CONFIGS[args.config]
    if args.backward:
        main_bwd(args, cfg)
        return
    if args.decompose:
        main_decomp(args)
        return
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2006_06443_b200 import LrsConv
    from paper_2006_06443_b200 import roofline as RL
    from paper_2006_06443_b200.dist import gather_shards

    # ---- inputs.  Strong scaling (default): the config's global batch is fixed and
    # split over the ranks (shard_range); weak: every rank runs a full batch of its own.
    # Same weights everywhere; X set i = generate_x(cfg, seed=i) (distinct images per set).
    gen = workloads.generate_cp if is_cp else workloads.generate
    inp = gen(cfg, batch=1)
    plan = ShardPlan(cfg, rank, world, args.scaling)
    strong, gb, s0, s1 = plan.strong, plan.global_batch, plan.start, plan.end
    n = s1 - s0
    if is_cp:
        layer = LrsConv.from_cp(n, cfg.in_h, cfg.in_w, cfg.k, cfg.stride, cfg.pad, cfg.dtype, inp.a, inp.b, inp.c,
                                inp.d, inp.row_ptr, inp.col_idx, inp.values, device=local)
    else:
        layer = LrsConv.from_inputs(inp, batch_max=n, device=local)
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    esz = 2 if cfg.dtype == "bf16" else 4
    x_bytes = n * cfg.in_h * cfg.in_w * cfg.c_in * esz
    y_bytes = n * cfg.out_h * cfg.out_w * cfg.c_out * esz
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    n_sets = max(2, math.ceil(2.1 * l2 / (x_bytes + y_bytes)))

    xs_np = [plan.x(i) for i in range(n_sets)]
    xs = [torch.from_numpy(x).to(tdt).to(dev) for x in xs_np]
    ys = [torch.empty((n, cfg.out_h, cfg.out_w, cfg.c_out), dtype=tdt, device=dev) for _ in range(n_sets)]
    stream = torch.cuda.Stream(device=dev)

    def capture(count: int):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for i in range(count):
                    layer.forward_into(xs[i % n_sets], ys[i % n_sets], stream=stream)
        return g

    with torch.cuda.stream(stream):
        for i in range(n_sets):  # eager warm-up (also JIT-loads the module)
            layer.forward_into(xs[i], ys[i], stream=stream)
    torch.cuda.synchronize(dev)
    K, W = args.steps, args.warmup
    g_full = capture(n_sets)
    rem = K % n_sets
    g_rem = capture(rem) if rem else None

    def run_steps(k_full, with_rem):
        for _ in range(k_full):
            g_full.replay()
        if with_rem and g_rem is not None:
            g_rem.replay()

    # ---- warm-up (every graph the timed region replays is replayed once here: a graph's
    # first replay uploads it, which must not land in the timed region)
    for _ in range(max(1, math.ceil(W / n_sets))):
        g_full.replay()
    if g_rem is not None:
        g_rem.replay()
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- timed region: exactly K forwards
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device() if world == 1 else local)
    barrier()
    with sampler:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            run_steps(K // n_sets, True)
            ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / K
    value = gb * K / (ms_max / 1e3)

    # ---- replay statistics: >= 10 separately timed replays of the n_sets-forward graph
    # (SURVEY §8(d) timing protocol: median of >= 10 replays), max over ranks per replay
    reps = []
    for _ in range(max(10, args.replays)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            g_full.replay()
            b.record(stream)
        reps.append((a, b))
    torch.cuda.synchronize(dev)
    rep_ms = torch.tensor([a.elapsed_time(b) for a, b in reps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(rep_ms, op=dist.ReduceOp.MAX)
    rep_us = (rep_ms.cpu().numpy() / n_sets * 1e3)
    replays = {"n": int(len(rep_us)), "forwards_per_replay": n_sets, "median_us_per_step": float(np.median(rep_us)),
               "min_us_per_step": float(rep_us.min()), "max_us_per_step": float(rep_us.max()),
               "median_images_per_s": gb / (float(np.median(rep_us)) * 1e-6)}

    # ---- verification, outside any timed region:
    #  (1) every rotating set's Y (last written by the graph) is bitwise an eager forward of its X;
    #  (2) the ranks' shards of set 0 gathered over NCCL: on rank 0, bitwise the 1-GPU Y of the
    #      whole batch (a second handle) and, on sampled images, the fp64 oracle (bf16 2e-2 /
    #      fp32 1e-5 relL2, per image).
    verify = {}
    ok_rot = True
    for i in range(n_sets):
        ye = torch.empty_like(ys[i])
        layer.forward_into(xs[i], ye)
        torch.cuda.synchronize(dev)
        ok_rot &= bool(torch.equal(ye, ys[i]))
    verify["rotation_bitwise_eager"] = ok_rot
    if strong or world == 1:
        y_full = gather_shards(ys[0], gb) if world > 1 else ys[0]
        if rank == 0:
            if world > 1:
                one = LrsConv.from_inputs(inp, batch_max=gb, device=local) if not is_cp else None
                if one is not None:
                    x_full = torch.from_numpy(workloads.generate_x(cfg, gb, seed=plan.seed(0))).to(tdt).to(dev)
                    y_one = torch.empty_like(y_full)
                    one.forward_into(x_full, y_one)
                    torch.cuda.synchronize(dev)
                    verify["gathered_equals_1gpu_bitwise"] = bool(torch.equal(y_one, y_full))
                    one.close()
            if not args.no_cpu:
                from oracle import lrs_oracle as O
                xg = workloads.generate_x(cfg, gb, seed=plan.seed(0))
                idx = np.unique(np.linspace(0, gb - 1, min(gb, 8)).astype(int))
                if is_cp:
                    ref = O.forward_cp(xg[idx].astype(np.float64), inp.a, inp.b, inp.c, inp.d, inp.row_ptr,
                                       inp.col_idx, inp.values, cfg.stride, cfg.pad)
                else:
                    ref = O.forward_factored(xg[idx].astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                                             inp.col_idx, inp.values, cfg.stride, cfg.pad)
                yv = y_full[torch.from_numpy(idx).to(dev)].float().cpu().numpy().astype(np.float64)
                errs = [float(np.linalg.norm(yv[k] - ref[k]) / np.linalg.norm(ref[k])) for k in range(len(idx))]
                tol = 2e-2 if cfg.dtype == "bf16" else 1e-5
                verify["oracle_images"] = [int(i) for i in idx]
                verify["oracle_max_rel_l2"] = max(errs)
                verify["oracle_ok"] = max(errs) <= tol
    # ---- per-kernel durations: an event pair around every launch.  The
    # launches queue up behind a device-side sleep, so they then run back to
    # back with no host launch gaps inside the event pairs.
    layer.set_timing(True)
    layer.stage_times(reset=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e7))
        for i in range(n_sets):
            layer.forward_into(xs[i], ys[i], stream=stream)
    torch.cuda.synchronize(dev)
    stages = layer.stage_times(reset=True)
    layer.set_timing(False)

    # ---- end to end through the C-ABI with host buffers (H2D + forward + D2H per step)
    e2e = None
    if not args.no_e2e:
        xh = xs[0].cpu().pin_memory()
        yh = torch.empty(ys[0].shape, dtype=tdt).pin_memory()
        with torch.cuda.stream(stream):
            for _ in range(3):
                layer.forward_host(xh, yh, stream=stream)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(3, min(K, 50))
        barrier()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(ke):
                layer.forward_host(xh, yh, stream=stream)
            e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": gb * ke / (float(te.item()) / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": x_bytes, "d2h_bytes_per_step": y_bytes, "steps": ke,
               "api": "lrs_conv_forward_host (pinned host buffers)",
               "note": "bytes are per rank (its shard); value is the whole job"}
        torch.cuda.synchronize(dev)
        ok_e2e = bool(torch.equal(yh, ys[0].cpu()))
        verify["e2e_bitwise_device_forward"] = ok_e2e

    # ---- context: cuDNN dense conv of the reconstructed W = L + S, same images, same
    # rotation (PAPER.md:210-223 -- the paper's "original layer")
    dense = None
    if not is_cp and not args.no_dense:
        wd = dense_weight(inp, cfg).to(tdt).to(dev).contiguous(memory_format=torch.channels_last)
        xd = [x.permute(0, 3, 1, 2) for x in xs]  # channels_last NCHW views of the NHWC buffers
        with torch.backends.cudnn.flags(enabled=True, benchmark=True):
            with torch.cuda.stream(stream):
                for i in range(n_sets):
                    torch.nn.functional.conv2d(xd[i], wd, stride=cfg.stride, padding=cfg.pad)
            torch.cuda.synchronize(dev)
            ke = max(n_sets, (K // n_sets) * n_sets)
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                d0.record(stream)
                for i in range(ke):
                    torch.nn.functional.conv2d(xd[i % n_sets], wd, stride=cfg.stride, padding=cfg.pad)
                d1.record(stream)
            torch.cuda.synchronize(dev)
        us = d0.elapsed_time(d1) / ke * 1e3
        dense = {"us_per_step": us, "images_per_s": n / (us * 1e-6), "steps": ke,
                 "what": "torch.nn.functional.conv2d (cuDNN, benchmark mode) of the dense W = L + S, "
                         f"{cfg.dtype}, channels_last, this rank's {n} images, same X rotation (eager launches)",
                 "compressed_speedup": us / (ms_per_step * 1e3)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel + layer roofs (per GPU: this rank's n images)
    peaks = RL.measured_peaks()
    work = RL.layer_work(cfg, n, inp.col_idx, cp=is_cp)
    roofs = RL.layer_roofs(work, peaks, cfg.dtype)
    avg = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in stages.items()}
    dom = max(avg, key=lambda k: avg[k])
    # With the co-resident schedule (the a1+a2 kernel on the SMs the fused kernel leaves
    # free, overlapping under PDL) the per-launch event intervals overlap and each includes
    # the other kernel's time; the fused expansion + sparse kernel is then the dominant one
    # (serialized ncu launch list, profiles/)
    kernel_overlap = sum(avg.values()) > 1.2 * ms_per_step
    if avg.get("a345_expand_sparse", 0.0) > 0.0 and kernel_overlap:
        dom = "a345_expand_sparse"
    t_dom = avg[dom] / 1e3
    roof = RL.kernel_roofline(dom, work, peaks, cfg.dtype, t_dom, layer.sparse_engine[0])
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (tools/ncu_traffic.py -> profiles/ncu_traffic.json); per launch, cold cache
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config)
        if tr and tr.get("kernel_stage", dom) == dom:
            roof["traffic"] = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            roof["traffic_detail"] = {"kernel": tr["kernel"], "dram_read_bytes": tr["dram_read_bytes"],
                                      "dram_write_bytes": tr["dram_write_bytes"], "source": tr["source"]}
    except (OSError, ValueError, KeyError):
        pass
    roof["stage_us"] = {k: round(v * 1e3, 3) for k, v in avg.items()}
    if kernel_overlap:
        roof["stage_note"] = ("kernels overlap (co-resident under PDL): each stage interval includes waiting for "
                              "the other kernel, so kernel_us is an upper bound on the dominant kernel's own time")
    step_s = ms_per_step / 1e3
    layer_roof = {"literal_roof_us": roofs["t_literal_s"] * 1e6, "three_roof_us": roofs["t_three_roof_s"] * 1e6,
                  "frac_literal": roofs["t_literal_s"] / step_s, "frac_three_roof": roofs["t_three_roof_s"] / step_s,
                  "t_hbm_us": roofs["t_hbm_s"] * 1e6, "t_chain_tc_us": roofs["t_chain_tc_s"] * 1e6,
                  "t_sparse_tc_us": roofs["t_sparse_tc_s"] * 1e6, "t_sparse_fma_us": roofs["t_sparse_fma_s"] * 1e6,
                  "fp32_fma_peak_tflops": roofs["fma_tflops"],
                  "fp32_fma_peak_kind": roofs["fma_kind"],
                  "what": "whole layer (all kernels) per GPU: literal = max(bytes / HBM, all FLOPs incl. the sparse "
                          "term / tensor peak) (BASELINE.json north star); three-roof puts the sparse MACs on the "
                          "FP32 pipe (SURVEY §8d)"}
    eng, mb, rb = layer.sparse_engine
    if eng == 1:
        # the 2:4 engine's own floor: its dense-equivalent MMA work at the 2:4 rate (no
        # more useful work per block than 128 x 64 logical slots, whatever the density)
        layer_roof["engine_floor_us"] = RL.sparse24_floor_s(cfg, n, mb, rb, peaks) * 1e6

    cpu = None
    if world == 1 and not args.no_cpu:
        sample = max(1, min(n, 8))
        rate, calls, el = oracle_rate(cfg, inp, args.cpu_seconds, sample, xs_np[0])
        cpu = {"value": rate, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{calls} oracle forwards x {sample} images of {args.config} ({el:.1f} s, fp64 numpy "
                         "forward_factored; BLAS threads = cores, sparse scatter single-threaded)",
               **host_info()}

    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if (strong or world == 1) else "weak",
        "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded ReLU(N(0,1)) images, N(0,1/fan_in) factors, uniform S)",
        "config": {"workload": CONFIG_TEXT[args.config], "config_id": args.config, "global_batch": gb,
                   "per_gpu_batch": n, "parallelism": f"dp{world} (batch-sharded, no data-path collective)",
                   "l2": f"{n_sets} rotating X/Y buffer sets of distinct images = "
                         f"{n_sets * (x_bytes + y_bytes) / 2**20:.0f} MiB (2.1x L2 {l2 / 2**20:.0f} MiB)",
                   "timing": "CUDA graph replay, CUDA events, max over ranks"},
        "clocks": sampler.summary(),
        "e2e": e2e,
        "gpu_launches": layer.launches_per_forward * K,
        "roofline": roof,
        "roofline_layer": layer_roof,
        "replays": replays,
        "verify": verify,
        "dense_context": dense,
        "cpu_baseline": cpu,
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bwd_work(cfg, n: int, inp) -> dict:
    """Algorithmic work of one backward step on n images (per GPU).  FLOPs: dX as the
    transposed layer's forward (chain 2P(R2 Cout + R1 R2 k^2 + R1 Cin) + 2 x sparse MACs);
    the weight-gradient reductions dU_out 2 P R2 Cout, dG 2 P R1 R2 k^2, dU_in 2 Pin Cin R1,
    dvalues 2 x sparse MACs; the recompute T1, T2, dT2, dT1 (2 Pin Cin R1, 2 P R1 R2 k^2,
    2 P Cout R2, 2 Pin R1 R2 k^2).  Bytes: X, dY read, dX written (bf16) -- each once --
    plus the factors and S (read) and the gradients (fp32, written)."""
    from paper_2006_06443_b200 import roofline as RL
    k2 = cfg.k * cfg.k
    pin = n * cfg.in_h * cfg.in_w
    P = n * cfg.out_h * cfg.out_w
    r1, r2 = cfg.rank_in, (cfg.rank_in if cfg.svd else cfg.rank_out)
    kc = 1 if cfg.svd else k2
    sp = RL.sparse_macs(n, cfg.in_h, cfg.in_w, cfg.k, cfg.stride, cfg.pad, inp.col_idx)
    wg = {"d_u_out": 2 * P * r2 * cfg.c_out, "d_core": 0 if cfg.svd else 2 * P * r1 * r2 * k2,
          "d_u_in": 2 * pin * cfg.c_in * r1, "d_values": 2 * sp}
    # executed by the grouped kernel: dvalues as the dense tap weight gradient
    wg_exec = dict(wg, d_values=2 * P * cfg.c_in * cfg.c_out * k2 if len(inp.col_idx) else 0)
    recompute = 2 * pin * cfg.c_in * r1 + 2 * P * cfg.c_out * r2 + (0 if cfg.svd else 2 * P * r1 * r2 * k2 * 2)
    dx = 2 * P * (r2 * cfg.c_out + (0 if cfg.svd else r1 * r2 * k2)) + 2 * pin * r1 * cfg.c_in + 2 * sp
    nparam = cfg.c_in * r1 + cfg.c_out * r2 + (0 if cfg.svd else r1 * r2 * k2)
    act = 2 * (2 * pin * cfg.c_in + P * cfg.c_out)
    byts = act + 2 * nparam + 8 * len(inp.col_idx) + 4 * (nparam + len(inp.col_idx))
    return {"flops_wgrad": sum(wg.values()), "flops_wgrad_executed": sum(wg_exec.values()),
            "flops_recompute": recompute, "flops_dx": dx, "flops": sum(wg.values()) + recompute + dx,
            "bytes": byts, "wgrad_split": wg}


def main_bwd(args, cfg):
    """--backward: one step = the layer's backward for one batch -- dX and every parameter
    gradient (one lrs_conv_backward call) -- and, at N > 1, the
    data-parallel exchange fine-tuning needs: an NCCL all-reduce of the parameter gradients
    (the one real collective of the path).  Same timing protocol as the forward: CUDA graph of
    the rotating sets (X, dY, dX of distinct seeded images, > 2.1x L2), K timed steps, max over
    ranks, median of >= 10 replays; verification after timing (bitwise vs eager, fp64 oracle)."""
    import torch
    import torch.distributed as dist
    if cfg.dtype != "bf16":
        raise SystemExit("--backward: bf16 layers (c2_bf16, c3, c4)")
    if args.impl == "reference":
        return run_reference_bwd(args, cfg)
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2006_06443_b200 import LrsConvBackward
    from paper_2006_06443_b200 import roofline as RL
    from paper_2006_06443_b200.dist import allreduce_grads
    inp = workloads.generate(cfg, batch=1)
    plan = ShardPlan(cfg, rank, world, args.scaling)
    gb, s0, s1 = plan.global_batch, plan.start, plan.end
    n = s1 - s0
    bw = LrsConvBackward.from_inputs(inp, batch_max=n, device=local)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    set_bytes = 2 * n * (2 * cfg.in_h * cfg.in_w * cfg.c_in + cfg.out_h * cfg.out_w * cfg.c_out)
    n_sets = max(2, math.ceil(2.1 * l2 / set_bytes))
    xs_np = [plan.x(i) for i in range(n_sets)]
    dys_np = [workloads.generate_dy(cfg, cfg.batch, seed=10_000 + plan.seed(i))[s0:s1] if plan.strong or world == 1
              else workloads.generate_dy(cfg, cfg.batch, seed=10_000 + plan.seed(i)) for i in range(n_sets)]
    xs = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in xs_np]
    dys = [torch.from_numpy(d).to(torch.bfloat16).to(dev) for d in dys_np]
    dxs = [torch.empty_like(x) for x in xs]
    grads = bw.alloc_grads()
    gl = [t for t in grads.values() if t is not None and t.numel()]
    stream = torch.cuda.Stream(device=dev)

    def step(i):
        bw.backward_into(xs[i], dys[i], dxs[i], grads, stream=stream)
        allreduce_grads(gl)

    with torch.cuda.stream(stream):
        for i in range(n_sets):
            step(i)
    torch.cuda.synchronize(dev)
    K, W = args.steps, args.warmup

    def capture(count):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for i in range(count):
                    step(i % n_sets)
        return g

    g_full = capture(n_sets)
    rem = K % n_sets
    g_rem = capture(rem) if rem else None
    for _ in range(max(1, math.ceil(W / n_sets))):
        g_full.replay()
    if g_rem is not None:
        g_rem.replay()
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device() if world == 1 else local)
    barrier()
    with sampler:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(K // n_sets):
                g_full.replay()
            if g_rem is not None:
                g_rem.replay()
            ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    t = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / K
    value = gb * K / (ms_max / 1e3)
    reps = []
    for _ in range(max(10, args.replays)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            g_full.replay()
            b.record(stream)
        reps.append((a, b))
    torch.cuda.synchronize(dev)
    rep_ms = torch.tensor([a.elapsed_time(b) for a, b in reps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(rep_ms, op=dist.ReduceOp.MAX)
    rep_us = rep_ms.cpu().numpy() / n_sets * 1e3
    replays = {"n": int(len(rep_us)), "steps_per_replay": n_sets, "median_us_per_step": float(np.median(rep_us)),
               "median_images_per_s": gb / (float(np.median(rep_us)) * 1e-6)}

    # ---- verification (untimed): the graph's last gradients and every dX bitwise = eager
    verify = {}
    last = n_sets - 1  # the replays above ran the full rotation last: grads hold set n_sets - 1
    ge = bw.alloc_grads()
    ok = True
    for i in range(n_sets):
        dxe = torch.empty_like(dxs[i])
        bw.backward_into(xs[i], dys[i], dxe, ge)
        torch.cuda.synchronize(dev)
        ok &= bool(torch.equal(dxe, dxs[i]))
    bw.backward_into(xs[last], dys[last], torch.empty_like(dxs[last]), ge)
    torch.cuda.synchronize(dev)
    allreduce_grads(list(ge.values()))
    verify["dx_rotation_bitwise_eager"] = ok
    verify["grads_bitwise_eager"] = all(torch.equal(ge[k_], grads[k_]) for k_ in ge if ge[k_] is not None)
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import lrs_backward as B
        ref = B.backward_factored(xs_np[last].astype(np.float64), dys_np[last].astype(np.float64), inp.u_in,
                                  inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values, cfg.stride, cfg.pad)
        errs = {}
        for k_ in ("d_u_in", "d_core", "d_u_out", "d_values"):
            if ref[k_] is None or ref[k_].size == 0:
                continue
            gpu = grads[k_].double().cpu().numpy()
            errs[k_] = float(np.linalg.norm(gpu - ref[k_]) / np.linalg.norm(ref[k_]))
        dxl = dxs[last].double().cpu().numpy()
        errs["dx"] = float(np.linalg.norm(dxl - ref["dx"]) / np.linalg.norm(ref["dx"]))
        verify["oracle_rel_l2"] = errs
        verify["oracle_ok"] = max(errs.values()) <= 2e-2

    # ---- per-kernel durations (event pairs around every launch, queued behind a sleep)
    bw.set_timing(True)
    bw.stage_times(reset=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e7))
        for i in range(n_sets):
            bw.backward_into(xs[i], dys[i], dxs[i], grads, stream=stream)
    torch.cuda.synchronize(dev)
    stages = bw.stage_times(reset=True)
    bw.set_timing(False)

    # ---- end to end with host buffers: X, dY in (pinned) -> dX and the gradients out
    e2e = None
    if not args.no_e2e:
        xh = xs[0].cpu().pin_memory()
        dyh = dys[0].cpu().pin_memory()
        dxh = torch.empty(dxs[0].shape, dtype=torch.bfloat16).pin_memory()
        gh = {k_: torch.empty(v.shape, dtype=torch.float32).pin_memory() for k_, v in grads.items()
              if v is not None and v.numel()}
        xd, dyd, dxd = torch.empty_like(xs[0]), torch.empty_like(dys[0]), torch.empty_like(dxs[0])

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            dyd.copy_(dyh, non_blocking=True)
            bw.backward_into(xd, dyd, dxd, grads, stream=stream)
            allreduce_grads(gl)
            dxh.copy_(dxd, non_blocking=True)
            for k_, v in gh.items():
                v.copy_(grads[k_], non_blocking=True)

        with torch.cuda.stream(stream):
            for _ in range(3):
                e2e_step()
        torch.cuda.synchronize(dev)
        ke = max(3, min(K, 50))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(ke):
                e2e_step()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": gb * ke / (float(te.item()) / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": xh.numel() * 2 + dyh.numel() * 2,
               "d2h_bytes_per_step": dxh.numel() * 2 + sum(v.numel() * 4 for v in gh.values()), "steps": ke,
               "api": "LrsConvBackward.backward_into (lrs_conv_backward) with pinned-host copies in and out"}

    # ---- context: cuDNN's backward of the dense layer (dgrad + wgrad of conv2d, W = L + S)
    dense = None
    if not args.no_dense:
        wd = dense_weight(inp, cfg).to(torch.bfloat16).to(dev).contiguous(memory_format=torch.channels_last)
        xd_ = [x.permute(0, 3, 1, 2) for x in xs]
        dyd_ = [d.permute(0, 3, 1, 2) for d in dys]
        gi = torch.nn.grad.conv2d_input
        gw = torch.nn.grad.conv2d_weight
        with torch.backends.cudnn.flags(enabled=True, benchmark=True):
            def dstep(i):
                gi(xd_[i].shape, wd, dyd_[i], stride=cfg.stride, padding=cfg.pad)
                gw(xd_[i], wd.shape, dyd_[i], stride=cfg.stride, padding=cfg.pad)
            with torch.cuda.stream(stream):
                for i in range(n_sets):
                    dstep(i)
            torch.cuda.synchronize(dev)
            ke = max(n_sets, (K // n_sets) * n_sets)
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                d0.record(stream)
                for i in range(ke):
                    dstep(i % n_sets)
                d1.record(stream)
            torch.cuda.synchronize(dev)
        us = d0.elapsed_time(d1) / ke * 1e3
        dense = {"us_per_step": us, "images_per_s": n / (us * 1e-6), "steps": ke,
                 "what": "torch.nn.grad.conv2d_input + conv2d_weight (cuDNN, benchmark mode) of the dense "
                         "W = L + S, bf16, channels_last, this rank's images (eager launches)",
                 "compressed_speedup": us / (ms_per_step * 1e3)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    peaks = RL.measured_peaks()
    work = bwd_work(cfg, n, inp)
    avg = {k_: v[0] / v[1] for k_, v in stages.items() if v[1]}
    t_w = avg["wgrad"] / 1e3
    peak = peaks["bf16_tflops_sustained"]
    roof = {"bound": "tensor", "kernel": "lrs_wgrad_kernel (grouped weight-gradient reductions)",
            "achieved": work["flops_wgrad"] / t_w / 1e12, "peak": peak, "unit": "TFLOP/s",
            "frac": work["flops_wgrad"] / t_w / 1e12 / peak, "traffic": None,
            "peak_kind": "measured sustained bf16 (MEASURED_PEAKS.json bf16_tflops_sustained): the kernel runs "
                         "inside a long step",
            "executed_tflops": work["flops_wgrad_executed"] / t_w / 1e12,
            "executed_frac": work["flops_wgrad_executed"] / t_w / 1e12 / peak,
            "what": "achieved = ALGORITHMIC FLOPs of the four reductions (dU_out, dG, dU_in, and dvalues as the "
                    "sparse MACs only) / the kernel's event-timed launch; executed counts dvalues as the dense "
                    "tap weight gradient the kernel computes before gathering S's support",
            "kernel_us": t_w * 1e6, "work": work,
            "stage_us": {k_: round(v * 1e3, 3) for k_, v in avg.items()}}
    try:  # DRAM bytes per launch of the weight-gradient kernel (committed ncu capture)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config + "_bwd")
        if tr:
            roof["traffic"] = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            roof["traffic_detail"] = tr
    except (OSError, ValueError, KeyError):
        pass
    step_s = ms_per_step / 1e3
    layer_roof = {"t_tensor_us": work["flops"] / (peak * 1e12) * 1e6,
                  "t_hbm_us": work["bytes"] / (peaks["hbm_gbs"] * 1e9) * 1e6}
    layer_roof["frac_literal"] = max(layer_roof["t_tensor_us"], layer_roof["t_hbm_us"]) / (step_s * 1e6)
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = bwd_oracle_rate(cfg, inp, args.cpu_seconds, xs_np[0], dys_np[0])
    _, _, cl = bw.launches
    line = {
        "metric": METRIC + " (backward pass: dX + parameter gradients)", "value": value, "unit": "images/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if (plan.strong or world == 1) else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded ReLU(N(0,1)) images, N(0,1) dY, N(0,1/fan_in) factors, uniform S)",
        "config": {"workload": CONFIG_TEXT[args.config] + " -- BACKWARD (SURVEY 8f f3)", "config_id": args.config + "_bwd",
                   "global_batch": gb, "per_gpu_batch": n,
                   "parallelism": f"dp{world} (batch-sharded; NCCL all-reduce of the parameter gradients)",
                   "l2": f"{n_sets} rotating X/dY/dX sets of distinct images ({n_sets * set_bytes / 2**20:.0f} MiB, "
                         f"2.1x L2)", "timing": "CUDA graph replay, CUDA events, max over ranks"},
        "clocks": sampler.summary(), "e2e": e2e, "gpu_launches": cl * K, "roofline": roof,
        "roofline_layer": layer_roof, "replays": replays, "verify": verify, "dense_context": dense,
        "cpu_baseline": cpu, "host": host_info(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


DECOMP_OF = {"c3": "c3_decomp", "c2_bf16": "c2_decomp", "c2_f32": "c2_decomp"}


def fp64_peak():
    """(TFLOP/s, kind): the measured DFMA peak (tools/dfma_peak.cu) if profiles/ holds it,
    else 148 SMs x 64 DFMA/clk x 2 at the max SM clock (derived)."""
    try:
        with open(os.path.join(ROOT, "profiles", "measured_peaks_extra.json")) as f:
            v = json.load(f).get("fp64_fma_tflops")
        if v:
            return float(v), "measured (tools/dfma_peak.cu, profiles/measured_peaks_extra.json)"
    except (OSError, ValueError):
        pass
    return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SMs x 64 DFMA/clk x 2 x 1965 MHz)"


def main_decomp(args):
    """--decompose: one step = one iteration of the paper's two-step scheme (ALS sweep on
    W - S, then S = P_c(W - L)) on the GPU (lrs_decomp_run), for the weight
    shape of --config (c3 -> 512 x 512 x 3 x 3, CP rank 128, c = 1 %).  A run synchronises
    once per iteration (host stopping rule), so it is timed eagerly (no CUDA graph): CUDA
    events around one run of K iterations after a W-iteration warm-up run.  Replicas only at
    N > 1 (one decomposition per GPU, no collective)."""
    import torch
    if args.tucker2:
        return main_decomp_t2(args)
    if args.impl == "reference":
        return run_reference_decomp(args)
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2006_06443_b200 import LrsDecomp
    if args.config == "c5":
        return main_decomp_network(args, dev, local, rank, world)
    cfg = workloads.DECOMP_CONFIGS[DECOMP_OF.get(args.config, "c3_decomp")]
    w, f0 = workloads.generate_decomp(cfg)
    wd = torch.from_numpy(w).to(dev)
    K, W = args.steps, args.warmup
    never = -float("inf")
    warm = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=max(1, W), tol=never, device=local)
    fs = [torch.from_numpy(f).to(dev) for f in f0]
    warm.run(wd, fs)
    torch.cuda.synchronize(dev)
    dc = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=K, tol=never, device=local)
    fs = [torch.from_numpy(f).to(dev) for f in f0]
    stream = torch.cuda.current_stream(dev)
    sampler = ClockSampler(torch.cuda.current_device())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    with sampler:
        e0.record(stream)
        idx, val, eps = dc.run(wd, fs)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    value = K / (ms / 1e3)
    # verification (untimed): the first iterations against the fp64 oracle, and determinism
    verify = {}
    n_chk = min(3, K)
    chk = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=n_chk, tol=never, device=local)
    fc = [torch.from_numpy(f).to(dev) for f in f0]
    ci, cv, ce = chk.run(wd, fc)
    verify["first_iterations_bitwise_timed_run"] = bool(ce == eps[:n_chk])
    if not args.no_cpu:
        from oracle import lrs_decomp as D
        rf, (ridx, rval), reps = D.decompose_lrs(w, f0, cfg.cardinality, max_iters=n_chk, tol=never)
        verify["oracle_eps"] = reps
        verify["gpu_eps"] = ce
        verify["eps_max_rel_diff"] = float(max(abs(a - b) / b for a, b in zip(ce, reps)))
        verify["s_support_equal"] = bool(np.array_equal(ci.cpu().numpy(), ridx))
        verify["oracle_ok"] = verify["eps_max_rel_diff"] < 1e-7 and verify["s_support_equal"]
    # stage timing over a short run
    st_run = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=min(K, 10), tol=never, device=local)
    fsr = [torch.from_numpy(f).to(dev) for f in f0]
    st_run.set_timing(True)
    st_run.run(wd, fsr)
    torch.cuda.synchronize(dev)
    stages = st_run.stage_times()
    iters_t = min(K, 10)
    avg_iter = {k_: v[0] / iters_t for k_, v in stages.items()}  # ms per iteration per stage
    # e2e: W and the initial factors in from pinned host memory, K iterations, factors + S out
    e2e = None
    if not args.no_e2e:
        wh = torch.from_numpy(w).pin_memory()
        fh = [torch.from_numpy(f).pin_memory() for f in f0]
        oh = [torch.empty(f.shape, dtype=torch.float64).pin_memory() for f in f0]
        e2 = LrsDecomp(cfg.dims, cfg.rank, cfg.cardinality, max_iters=K, tol=never, device=local)
        wd2 = torch.empty_like(wd)
        fd2 = [torch.empty_like(f) for f in fs]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(stream)
        wd2.copy_(wh, non_blocking=True)
        for x, y in zip(fd2, fh):
            x.copy_(y, non_blocking=True)
        i2, v2, _ = e2.run(wd2, fd2)
        for x, y in zip(oh, fd2):
            x.copy_(y, non_blocking=True)
        ih = i2.cpu()
        vh = v2.cpu()
        b.record(stream)
        torch.cuda.synchronize(dev)
        e2e = {"value": K / (a.elapsed_time(b) / 1e3), "unit": "iterations/s",
               "h2d_bytes_per_step": (wh.numel() + sum(f.numel() for f in fh)) * 8 / K,
               "d2h_bytes_per_step": (sum(f.numel() for f in oh) * 8 + ih.numel() * 8 + vh.numel() * 8) / K,
               "api": "LrsDecomp.run (lrs_decomp_run) with pinned-host copies of W, the factors and S",
               "note": "one job = copy in, K iterations, copy out; bytes amortised per iteration"}
    numel = int(np.prod(cfg.dims))
    r = cfg.rank
    flops_mttkrp = 4 * 2 * numel * r  # per iteration: the contraction of T with the rank-r Khatri-Rao, per mode
    flops_res = 2 * numel * r
    peak, kind = fp64_peak()
    t_m = avg_iter["mttkrp"] / 1e3
    t_p = avg_iter["pinv_update"] / 1e3
    # the pseudo-inverse stage: 4 symmetric eigendecompositions (~9 r^3 flops each, the dense
    # tridiagonal-QR count) + P = Q diag Q^T (2 r^3) + the factor update F = M P (2 I_m r^2) + Gram
    flops_pinv = 4 * (11 * r ** 3) + sum(4 * d * r * r for d in cfg.dims)
    mttkrp = {"kernel": "lrs_mttkrp01q_kernel / lrs_mttkrp23_kernel (+ partial sums), 4 per iteration",
              "achieved": flops_mttkrp / t_m / 1e12, "frac": flops_mttkrp / t_m / 1e12 / peak,
              "what": "ALGORITHMIC fp64 FLOPs of the four MTTKRPs (2 numel r each) / their time per iteration"}
    pinv = {"kernel": "lrs_sym_pinv_kernel (one CTA) + lrs_cp_update_kernel + lrs_gram_kernel, 4 per iteration",
            "achieved": flops_pinv / t_p / 1e12, "frac": flops_pinv / t_p / 1e12 / peak,
            "what": "ALGORITHMIC fp64 FLOPs (4 x (9 r^3 eigendecomposition + 2 r^3 pseudo-inverse) + the factor "
                    "updates and Grams) / the stage's time per iteration; a one-CTA kernel can reach at most "
                    "1/148 of the chip's peak"}
    dom = pinv if t_p >= t_m else mttkrp
    roof = {"bound": "alu", "kernel": dom["kernel"], "achieved": dom["achieved"], "peak": peak,
            "unit": "TFLOP/s (fp64)", "frac": dom["frac"], "traffic": None, "peak_kind": kind, "what": dom["what"],
            "stage_ms_per_iteration": {k_: round(v, 4) for k_, v in avg_iter.items()},
            "mttkrp": mttkrp, "pseudo_inverse": pinv,
            "residual_tflops": flops_res / (avg_iter["residual"] / 1e3) / 1e12}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(cfg.name)
        if tr and dom is pinv:
            roof["traffic"] = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            roof["traffic_detail"] = tr
    except (OSError, ValueError, KeyError):
        pass
    cpu = None
    if not args.no_cpu:
        from oracle import lrs_decomp as D
        t0 = time.perf_counter()
        calls = 0
        while True:
            D.decompose_lrs(w, f0, cfg.cardinality, max_iters=1, tol=never)
            calls += 1
            el = time.perf_counter() - t0
            if el >= args.cpu_seconds and calls >= 2:
                break
        cpu = {"value": calls / el, "unit": "iterations/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{calls} oracle iterations (decompose_lrs max_iters=1) of {cfg.name} ({el:.1f} s, fp64 numpy)",
               **host_info()}
    if rank != 0:
        return
    line = {
        "metric": "GPU low-rank + sparse decomposition iterations/s (SURVEY 8f f4)", "value": value,
        "unit": "iterations/s", "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (planted CP rank + N(0, 0.05^2) noise + 1% spikes of magnitude 10; N(0,1) initial factors)",
        "config": {"workload": f"{cfg.name}: W {cfg.dims} (the {args.config} layer's weight shape), CP rank {cfg.rank}, "
                               f"cardinality {cfg.cardinality}, planted rank {cfg.planted_rank}",
                   "config_id": cfg.name, "parallelism": "replicas (one decomposition per GPU)",
                   "timing": "CUDA events around one run of K iterations (host stopping rule: one sync per iteration)",
                   "l2": "W is 2.36M fp64 (18.9 MB): L2-resident by design"},
        "clocks": sampler.summary(), "e2e": e2e, "gpu_launches": dc.launches_per_iteration * K, "roofline": roof,
        "verify": verify,
        "eps_last": eps[-1] if eps else None, "cpu_baseline": cpu, "host": host_info(),
    }
    print(json.dumps(line), flush=True)


def main_decomp_network(args, dev, local, rank, world):
    """--decompose --config c5: the 16 ResNet-50 3x3 weights decomposed CONCURRENTLY (f4
    "batched over layers"): one handle + CUDA stream + host thread per layer (calls on
    distinct handles are independent; ctypes releases the GIL), K iterations each; device time
    from an event before every stream starts to one after every stream ends."""
    import threading
    import torch
    from paper_2006_06443_b200 import LrsDecomp
    cfgs = workloads.resnet50_decomp_configs()
    K, W = args.steps, args.warmup
    never = -float("inf")
    data = []
    for c in cfgs:
        w, f0 = workloads.generate_decomp(c)
        data.append((c, torch.from_numpy(w).to(dev), f0))
    streams = [torch.cuda.Stream(device=dev) for _ in cfgs]

    def run_all(iters, out):
        hs = [LrsDecomp(c.dims, c.rank, c.cardinality, max_iters=iters, tol=never, device=local) for c, _, _ in data]
        fss = [[torch.from_numpy(f).to(dev) for f in f0] for _, _, f0 in data]
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        base = torch.cuda.current_stream(dev)
        e0.record(base)
        for s_ in streams:
            s_.wait_event(e0)

        def one(i):
            torch.cuda.set_device(dev)
            out[i] = hs[i].run(data[i][1], fss[i], stream=streams[i])

        ths = [threading.Thread(target=one, args=(i,)) for i in range(len(data))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        for s_ in streams:
            base.wait_stream(s_)
        e1.record(base)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1), fss, sum(h_.launches_per_iteration for h_ in hs)

    run_all(max(1, W), [None] * len(data))
    sampler = ClockSampler(torch.cuda.current_device())
    res = [None] * len(data)
    with sampler:
        ms, fss, launches = run_all(K, res)
    value = len(data) * K / (ms / 1e3)
    verify = {}
    if not args.no_cpu:  # the first iteration of every layer against the fp64 oracle
        from oracle import lrs_decomp as D
        chk = [None] * len(data)
        run_all(1, chk)
        errs, supp = [], []
        for (c, _, f0), (ci, _, ce) in zip(data, chk):
            w = workloads.generate_decomp(c)[0]
            _, (ridx, _), reps = D.decompose_lrs(w, f0, c.cardinality, max_iters=1, tol=never)
            errs.append(abs(ce[0] - reps[0]) / reps[0])
            supp.append(bool(np.array_equal(ci.cpu().numpy(), ridx)))
        verify = {"eps1_max_rel_diff": float(max(errs)), "s_support_equal_all": all(supp),
                  "oracle_ok": max(errs) < 1e-7 and all(supp)}
    if rank != 0:
        return
    numel = sum(int(np.prod(c.dims)) for c in cfgs)
    line = {
        "metric": "GPU low-rank + sparse decomposition iterations/s (SURVEY 8f f4), 16 layers concurrently",
        "value": value, "unit": "layer-iterations/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (planted CP rank + noise + 1% spikes per layer, N(0,1) initial factors)",
        "config": {"workload": "the 16 ResNet-50 3x3 conv weights (PAPER.md Table 2 shapes), CP rank min(Cin,Cout)/4, "
                               "c = 1 %, one handle + stream + host thread per layer", "config_id": "c5_decomp",
                   "layers": [{"name": c.name, "dims": c.dims, "rank": c.rank} for c in cfgs], "weights_numel": numel,
                   "parallelism": "16 concurrent decompositions on one GPU", "timing": "CUDA events around all streams"},
        "clocks": sampler.summary(), "e2e": None, "gpu_launches": launches * K,
        "roofline": None, "verify": verify, "eps_last": [r_[2][-1] for r_ in res], "cpu_baseline": None,
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)


T2_RANKS = (128, 128)  # the north star's Tucker ranks at the C3 shape (BASELINE.json configs[1])


def main_decomp_t2(args):
    """--decompose --tucker2: one step = one Tucker-2 iteration (a HOOI sweep on W - S, then
    S = P_c(W - L); include/lrs_conv.h "Tucker-2 decomposition") at the c3 weight shape and the
    north star's ranks 128 / 128, timed like main_decomp.  --impl reference: the fp64 oracle."""
    import torch
    cfg = workloads.DECOMP_CONFIGS[DECOMP_OF.get(args.config, "c3_decomp")]
    r1, r2 = T2_RANKS
    w, ui0, uo0 = workloads.generate_decomp_tucker2(cfg, r1, r2)
    K, W = args.steps, args.warmup
    never = -float("inf")
    metric = "GPU low-rank + sparse Tucker-2 decomposition iterations/s (SURVEY 8f f4)"
    workload = f"{cfg.name}_tucker2: W {cfg.dims}, Tucker ranks {r1}/{r2}, cardinality {cfg.cardinality}"

    def oracle_rate(steps):
        from oracle import lrs_decomp as D
        t0 = time.perf_counter()
        D.decompose_lrs_tucker2(w, ui0, uo0, cfg.cardinality, max_iters=steps, tol=never)
        el = time.perf_counter() - t0
        return steps / el, el

    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        oracle_rate(max(1, W))
        v, el = oracle_rate(K)
        print(json.dumps({"impl": "reference", "metric": metric, "value": v, "unit": "iterations/s", "n_gpus": 1,
                          "steps": K, "warmup": W, "ms_per_step": el / K * 1e3, "higher_is_better": True,
                          "dtype": "f64", "config": {"workload": workload, "config_id": cfg.name + "_tucker2"},
                          "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": cpu_threads(), "kind": "oracle",
                                           "sample": f"{K} iterations of {cfg.name}_tucker2"},
                          "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2006_06443_b200 import LrsTucker2Decomp
    wd = torch.from_numpy(w).to(dev)
    fresh = lambda: (torch.from_numpy(ui0).to(dev), torch.from_numpy(uo0).to(dev))

    def handle(iters):
        return LrsTucker2Decomp(cfg.dims, r1, r2, cfg.cardinality, max_iters=iters, tol=never, device=local)
    handle(max(1, W)).run(wd, *fresh())
    torch.cuda.synchronize(dev)
    dc = handle(K)
    ui, uo = fresh()
    stream = torch.cuda.current_stream(dev)
    sampler = ClockSampler(torch.cuda.current_device())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    with sampler:
        e0.record(stream)
        core, idx, val, eps = dc.run(wd, ui, uo)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    value = K / (ms / 1e3)
    verify = {}
    n_chk = min(3, K)
    ci, cv_, ce = None, None, None
    _, ci, _, ce = handle(n_chk).run(wd, *fresh())
    verify["first_iterations_bitwise_timed_run"] = bool(ce == eps[:n_chk])
    if not args.no_cpu:
        from oracle import lrs_decomp as D
        _, (ridx, _), reps = D.decompose_lrs_tucker2(w, ui0, uo0, cfg.cardinality, max_iters=n_chk, tol=never)
        verify["oracle_eps"] = reps
        verify["gpu_eps"] = ce
        verify["eps_max_rel_diff"] = float(max(abs(a - b) / b for a, b in zip(ce, reps)))
        verify["s_support_equal"] = bool(np.array_equal(ci.cpu().numpy(), ridx))
        verify["oracle_ok"] = verify["eps_max_rel_diff"] < 1e-7 and verify["s_support_equal"]
    n_t = min(K, 10)
    st_run = handle(n_t)
    st_run.set_timing(True)
    st_run.run(wd, *fresh())
    torch.cuda.synchronize(dev)
    avg_iter = {k_: v[0] / n_t for k_, v in st_run.stage_times().items()}
    e2e = None
    if not args.no_e2e:
        wh = torch.from_numpy(w).pin_memory()
        uih, uoh = torch.from_numpy(ui0).pin_memory(), torch.from_numpy(uo0).pin_memory()
        e2 = handle(K)
        wd2, ui2, uo2 = torch.empty_like(wd), torch.empty(ui0.shape, dtype=torch.float64, device=dev), \
            torch.empty(uo0.shape, dtype=torch.float64, device=dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(stream)
        wd2.copy_(wh, non_blocking=True)
        ui2.copy_(uih, non_blocking=True)
        uo2.copy_(uoh, non_blocking=True)
        c2, i2, v2, _ = e2.run(wd2, ui2, uo2)
        outs = [t.cpu() for t in (ui2, uo2, c2, i2, v2)]
        b.record(stream)
        torch.cuda.synchronize(dev)
        e2e = {"value": K / (a.elapsed_time(b) / 1e3), "unit": "iterations/s",
               "h2d_bytes_per_step": (w.size + ui0.size + uo0.size) * 8 / K,
               "d2h_bytes_per_step": sum(t.numel() for t in outs) * 8 / K,
               "api": "LrsTucker2Decomp.run (lrs_tucker2_run) with pinned-host copies in, factors + core + S out",
               "note": "one job = copy in, K iterations, copy out; bytes amortised per iteration"}
    cin, cout = cfg.dims[0], cfg.dims[1]
    q = cfg.dims[2] * cfg.dims[3]
    # ALGORITHMIC fp64 FLOPs per sweep of the mode products (Z1, Z2: 2 Cin Cout q R each; G: 2 R1 R2 Cout q;
    # the two subspace steps: 4 rows (R q) R each) -- the stage timed as "mode_products" + "subspace_orth"
    flops_prod = 2 * cin * cout * q * r2 + 2 * cin * cout * q * r1 + 2 * r1 * r2 * cout * q
    flops_sub = 4 * cin * r2 * q * r1 + 4 * cout * r1 * q * r2
    flops_res = 2 * r1 * r2 * cout * q + 2 * cin * cout * q * r1
    peak, kind = fp64_peak()
    t_prod = avg_iter["mode_products"] / 1e3
    roof = {"bound": "alu", "kernel": "lrs_dgemm_kernel (Z1, Z2, G mode products)",
            "achieved": flops_prod / t_prod / 1e12, "peak": peak, "unit": "TFLOP/s (fp64)",
            "frac": flops_prod / t_prod / 1e12 / peak, "traffic": None, "peak_kind": kind,
            "what": "ALGORITHMIC fp64 FLOPs of the three mode products per sweep / their time per iteration",
            "stage_ms_per_iteration": {k_: round(v, 4) for k_, v in avg_iter.items()},
            "subspace_tflops_incl_jacobi": flops_sub / (avg_iter["subspace_orth"] / 1e3) / 1e12,
            "residual_tflops": flops_res / (avg_iter["residual"] / 1e3) / 1e12}
    cpu = None
    if not args.no_cpu:
        v1, el1 = oracle_rate(1)
        calls = max(1, int(args.cpu_seconds / max(el1, 1e-3)))
        v, el = oracle_rate(calls)
        cpu = {"value": v, "unit": "iterations/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{calls} oracle iterations (decompose_lrs_tucker2) of {cfg.name} ({el:.1f} s, fp64 numpy)",
               **host_info()}
    if rank != 0:
        return
    print(json.dumps({
        "metric": metric, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (planted CP rank 96 + N(0, 0.05^2) noise + 1% spikes of magnitude 10; N(0,1) initial bases)",
        "config": {"workload": workload, "config_id": cfg.name + "_tucker2",
                   "parallelism": "replicas (one decomposition per GPU)",
                   "timing": "CUDA events around one run of K iterations (host stopping rule: one sync per iteration)",
                   "l2": "W is 2.36M fp64 (18.9 MB): L2-resident by design"},
        "clocks": sampler.summary(), "e2e": e2e, "roofline": roof, "verify": verify,
        # per sweep: 3 mode products + 2 x (2 GEMMs, Gram, Loewdin, update) + 2 residual GEMMs + the
        # projection (flags, 2 scans, finish, eps; with S: 8 x (histogram, pick) + 2 scans + compaction)
        "gpu_launches": (3 + 10 + 2 + 5 + (19 if dc.nnz > 0 else 0)) * K,
        "eps_last": eps[-1] if eps else None, "cpu_baseline": cpu, "host": host_info()}), flush=True)


def run_reference_decomp(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import lrs_decomp as D
    cfg = workloads.DECOMP_CONFIGS[DECOMP_OF.get(args.config, "c3_decomp")]
    w, f0 = workloads.generate_decomp(cfg)
    never = -float("inf")
    D.decompose_lrs(w, f0, cfg.cardinality, max_iters=max(1, args.warmup), tol=never)
    t0 = time.perf_counter()
    D.decompose_lrs(w, f0, cfg.cardinality, max_iters=args.steps, tol=never)
    el = time.perf_counter() - t0
    v = args.steps / el
    print(json.dumps({"impl": "reference", "metric": "GPU low-rank + sparse decomposition iterations/s (SURVEY 8f f4)",
                      "value": v, "unit": "iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "dtype": "f64",
                      "config": {"workload": cfg.name, "config_id": cfg.name},
                      "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": cpu_threads(), "kind": "oracle",
                                       "sample": f"{args.steps} iterations of {cfg.name}"},
                      "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def bwd_oracle_rate(cfg, inp, seconds, x_all, dy_all, sample=2):
    """The fp64 backward oracle (oracle/lrs_backward.backward_factored, as it stands) on a
    bounded sample: repeated calls on `sample` images."""
    from oracle import lrs_backward as B
    x = x_all[:sample].astype(np.float64)
    dy = dy_all[:sample].astype(np.float64)
    calls, t0 = 0, time.perf_counter()
    while True:
        B.backward_factored(x, dy, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values,
                            cfg.stride, cfg.pad)
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds and calls >= 2:
            break
    return {"value": calls * sample / el, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"{calls} oracle backward calls x {sample} images ({el:.1f} s, fp64 numpy backward_factored)",
            **host_info()}


def run_reference_bwd(args, cfg):
    """--impl reference --backward: the fp64 backward oracle as it stands, on rank 0."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    inp = workloads.generate(cfg, batch=1)
    x = workloads.generate_x(cfg, 2, seed=0)
    dy = workloads.generate_dy(cfg, 2, seed=10_000)
    for _ in range(args.warmup):
        bwd_oracle_rate(cfg, inp, 0.0, x, dy)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        bwd_oracle_rate(cfg, inp, 0.0, x, dy)
    el = time.perf_counter() - t0
    v = 2 * 2 * args.steps / el
    cpu = {"value": v, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
           "sample": f"{args.steps} steps x 2 calls x 2 images of {args.config} backward"}
    print(json.dumps({"impl": "reference", "metric": METRIC + " (backward pass: dX + parameter gradients)",
                      "value": v, "unit": "images/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "dtype": "f64",
                      "config": {"workload": CONFIG_TEXT[args.config] + " -- BACKWARD", "config_id": args.config + "_bwd"},
                      "cpu_baseline": cpu, "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0,
                                                   "d2h_bytes_per_step": 0}}), flush=True)


if __name__ == "__main__":
    main()
