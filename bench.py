#!/usr/bin/env python
"""Benchmark of the B200 compressed convolution W ~ L + S (arXiv 2006.06443).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_bf16] [--impl lrs|reference]
(N > 1: launched by torchrun, one process per GPU; RANK/WORLD_SIZE from env.)

A step = one forward of the whole hot path (a1 projection, a2 core, a3
expansion + a4 sparse + a5 sum/store) over one batch of the workload
(default BASELINE.json configs[1] = C2, ResNet-50 layer3 3x3 256->256 at
14x14, batch 64, bf16).  Weak scaling: every rank runs its own batch (its
own seeded images, same weights); there is no collective on the data path.

Timing: W untimed warm-up steps, then EXACTLY K steps replayed from a CUDA
graph, bracketed by barrier + cuda.synchronize; CUDA events on the launching
stream; max over ranks.  Inputs rotate over enough X/Y buffer sets to cover
2.1x the L2, so every step reads X from HBM.  Rank 0 prints ONE JSON line.
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
    ap.add_argument("--config", default="c2_bf16", choices=sorted(workloads.CONFIGS) + sorted(workloads.CP_CONFIGS) + ["c5"])
    ap.add_argument("--impl", default="lrs", choices=["lrs", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
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


def oracle_rate(cfg, inp, seconds: float, sample_images: int):
    """Time the fp64 oracle (forward_factored, as it stands) on a bounded
    sample of the workload: repeated calls on `sample_images` images."""
    from oracle import lrs_oracle as O
    x = inp.x[:sample_images].astype(np.float64)
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
    sample = max(1, min(cfg.batch, 8))
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
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads/)",
            "config": {"workload": CONFIG_TEXT[args.config], "images_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
                             "sample": f"{sample} images of {args.config} per step (fp64 numpy oracle, "
                                       f"{'forward_cp' if is_cp else 'forward_factored'})"},
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
    fma = RL.fp32_fma_tflops(peaks["sm_max_mhz"])
    tot = {}
    sparse_flops = 0.0
    for idx, c in comp.items():
        st = c.layer.stage_times(reset=True)
        for k, v in st.items():
            if v[1]:
                tot[k] = tot.get(k, 0.0) + v[0] / v[1]
        sparse_flops += RL.layer_work(c.cfg, per, workloads.generate_weights(c.cfg).col_idx)["layer"]["flops_sparse"]
        c.layer.set_timing(False)
    t_a345 = tot["a345_expand_sparse"] / 1e3
    achieved = sparse_flops / t_a345 / 1e12
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
        "roofline": {"bound": "alu", "achieved": achieved, "peak": fma, "unit": "TFLOP/s", "frac": achieved / fma,
                     "traffic": None, "kernel": "a345_expand_sparse (16 compressed layers)",
                     "work": "in-bounds sparse MACs x 2 of the 16 layers / their summed kernel time",
                     "engine": "2:4 sparse tensor cores (tcgen05.mma.sp) fused with the expansion GEMM",
                     "peak_source": "derived: 148 SM x 128 FP32 FMA/clk x 2 x sm_max_mhz (the sparse term's "
                                    "CUDA-core roof, SURVEY §8d three-roof)",
                     "stage_us_sum_16_layers": {k: round(v * 1e3, 1) for k, v in tot.items()}},
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.config == "c5":
        if args.impl == "reference":
            run_reference_c5(args)
        else:
            main_c5(args)
        return
    is_cp = args.config in workloads.CP_CONFIGS
    cfg = workloads.CP_CONFIGS[args.config] if is_cp else workloads.CONFIGS[args.config]
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

    # ---- inputs: same weights everywhere, rank-specific images (weak scaling)
    gen = workloads.generate_cp if is_cp else workloads.generate
    inp = gen(cfg)
    if rank > 0:
        inp.x = gen(cfg, seed=1000 + rank).x
    n = cfg.batch
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
    x0 = torch.from_numpy(inp.x).to(tdt).to(dev)
    xs = [x0] + [x0.clone() for _ in range(n_sets - 1)]
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
    value = world * n * K / (ms_max / 1e3)

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
        xh = x0.cpu().pin_memory()
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
        e2e = {"value": world * n * ke / (float(te.item()) / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": x_bytes, "d2h_bytes_per_step": y_bytes, "steps": ke,
               "api": "lrs_conv_forward_host (pinned host buffers)"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel + layer roofs
    peaks = RL.measured_peaks()
    work = RL.layer_work(cfg, n, inp.col_idx, cp=is_cp)
    roofs = RL.layer_roofs(work, peaks, cfg.dtype)
    avg = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in stages.items()}
    dom = max(avg, key=lambda k: avg[k])
    # With the co-resident schedule (the a1+a2 kernel on the SMs the fused kernel leaves
    # free, overlapping under PDL) the per-launch event intervals overlap and each includes
    # the other kernel's time; the fused expansion + sparse kernel is then the dominant one
    # (serialized ncu launch list, profiles/r01_v16_ncu_launches_c2_bf16.csv: 20.7 vs 16.7 us)
    if avg.get("a345_expand_sparse", 0.0) > 0.0 and sum(avg.values()) > 1.2 * ms_per_step:
        dom = "a345_expand_sparse"
    kernel_overlap = sum(avg.values()) > 1.2 * ms_per_step
    t_dom = avg[dom] / 1e3
    fma_peak = RL.fp32_fma_tflops(peaks["sm_max_mhz"])
    tc_peak = peaks["bf16_tflops"] * (1.0 if cfg.dtype == "bf16" else 0.5 / 3.0)  # fp32: 3xTF32 at TF32 = bf16/2
    eng = layer.sparse_engine[0]
    wk = work[dom]
    # the dominant kernel's algorithmic work per pipe: HBM bytes, FP32-pipe flops (the
    # sparse term -- SURVEY §8d three-roof -- plus whatever the kernel computes on the
    # CUDA cores), tensor-pipe flops; its roofline bound is the pipe with the largest
    # roof time, frac = that roof time / the measured kernel time
    if dom in ("a345_expand_sparse", "a4_sparse_add"):
        if eng == 3:  # the one-kernel fp32 path: the whole layer on the CUDA cores
            lay = work["layer"]
            b_alg, f_fma, f_tc = lay["bytes"], lay["flops_chain"] + lay["flops_sparse"], 0.0
        elif eng == 2:  # expansion + sparse term on the CUDA cores
            b_alg, f_fma, f_tc = wk["bytes"], wk["flops_sparse"] + wk["flops_tc"], 0.0
        else:  # tensor-core expansion (+ 2:4 tensor-core or SIMT sparse term)
            b_alg, f_fma, f_tc = wk["bytes"], wk["flops_sparse"], wk["flops_tc"]
    else:
        b_alg, f_fma, f_tc = wk["bytes"], 0.0, wk["flops"]
    roofs_k = {"hbm": (b_alg / (peaks["hbm_gbs"] * 1e9), b_alg / t_dom / 1e9, peaks["hbm_gbs"], "GB/s"),
               "alu": (f_fma / (fma_peak * 1e12), f_fma / t_dom / 1e12, fma_peak, "TFLOP/s"),
               "tensor": (f_tc / (tc_peak * 1e12), f_tc / t_dom / 1e12, tc_peak, "TFLOP/s")}
    bound = max(roofs_k, key=lambda k: roofs_k[k][0])
    t_roof, achieved, peak, unit = roofs_k[bound]
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": None, "kernel": dom,
            "work": {"bytes": b_alg, "fp32_pipe_flops": f_fma, "tensor_flops": f_tc,
                     "roof_us": {k: v[0] * 1e6 for k, v in roofs_k.items()}, "kernel_us": t_dom * 1e6},
            "engine": {0: "SIMT CSR gather fused into the expansion GEMM epilogue",
                       1: "2:4 sparse tensor cores (tcgen05.mma.sp), fused with the expansion GEMM",
                       2: "SIMT expansion + CSR gather over 4-image shared-memory windows, Y written once",
                       3: "the whole fp32 layer in one SIMT kernel"}.get(eng, "?"),
            "peak_source": {"hbm": "MEASURED_PEAKS.json hbm_gbs",
                            "alu": "derived: 148 SM x 128 FP32 FMA/clk x 2 x sm_max_mhz (SURVEY §8d three-roof)",
                            "tensor": "MEASURED_PEAKS.json bf16_tflops" + (" x 1/6 (3xTF32)" if cfg.dtype != "bf16"
                                                                          else "")}[bound]}
    roof["peak_kind"] = peaks["source"]
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (tools/ncu_traffic.py -> profiles/ncu_traffic.json); per launch, cold cache
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config)
        if tr:
            roof["traffic"] = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            roof["traffic_detail"] = {"kernel": tr["kernel"], "dram_read_bytes": tr["dram_read_bytes"],
                                      "dram_write_bytes": tr["dram_write_bytes"], "source": tr["source"],
                                      "note": "Y's write-back mostly lands in L2 after the kernel ends"}
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
                  "t_sparse_fma_us": roofs["t_sparse_fma_s"] * 1e6}

    cpu = None
    if world == 1 and not args.no_cpu:
        sample = max(1, min(n, 8))
        rate, calls, el = oracle_rate(cfg, inp, args.cpu_seconds, sample)
        cpu = {"value": rate, "unit": "images/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{calls} oracle forwards x {sample} images of {args.config} ({el:.1f} s, fp64 numpy "
                         "forward_factored; BLAS threads = cores, sparse scatter single-threaded)"}

    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded ReLU(N(0,1)) images, N(0,1/fan_in) factors, uniform S)",
        "config": {"workload": CONFIG_TEXT[args.config], "config_id": args.config, "global_batch": n * world,
                   "per_gpu_batch": n, "parallelism": f"dp{world} (batch-sharded, no data-path collective)",
                   "l2": f"{n_sets} rotating X/Y buffer sets = {n_sets * (x_bytes + y_bytes) / 2**20:.0f} MiB "
                         f"(2.1x L2 {l2 / 2**20:.0f} MiB)",
                   "timing": "CUDA graph replay, CUDA events, max over ranks"},
        "clocks": sampler.summary(),
        "e2e": e2e,
        "gpu_launches": layer.launches_per_forward * K,
        "roofline": roof,
        "roofline_layer": layer_roof,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
