"""C5: ResNet-50 with every 3x3 conv replaced by a compressed W ~ L + S layer
(BASELINE.json configs[4]; §5.5, :343-387, the network-integration
experiment, with the thesis' CP term read as Tucker-2 -- DESIGN.md reading #1).

The 16 compressed layers run through the C-ABI library (liblrs_conv.so) via
`CompressedConv2d`; every other layer (stem, 1x1 convs, BN in eval mode,
ReLU, residual adds, pooling, FC) stays dense in torch/cuDNN (DESIGN.md
reading #16 -- those layers are not the hot path).  Activations are bf16
`channels_last`, whose storage is the NHWC layout the ABI takes, so the
library reads and writes torch's tensors in place.  Weights are torchvision's
random init under `torch.manual_seed(seed)`; the compressed factors come from
`workloads.resnet50_compressed_layers` (seeded, synthetic).
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from .lrs_conv import LrsConv


def _torch():
    import torch
    return torch


class CompressedConv2d:
    """A drop-in for a torch 3x3 conv module: y = conv(x, L + S) on the GPU
    library.  Holds one LrsConv handle sized for `batch_max` images."""

    def __init__(self, inp, batch_max: int, device: int = 0, out_scale=None, out_bias=None, out_relu: bool = False):
        torch = _torch()
        self.cfg = inp.cfg
        self.layer = LrsConv.from_inputs(inp, batch_max=batch_max, device=device, out_scale=out_scale,
                                         out_bias=out_bias, out_relu=out_relu)
        self.device = device
        self.stream = None  # None: torch's current stream at call time

    def __call__(self, x):
        torch = self.layer.torch
        if not x.is_contiguous(memory_format=torch.channels_last):
            x = x.contiguous(memory_format=torch.channels_last)
        n = x.shape[0]
        y = torch.empty((n, self.cfg.c_out, self.layer.out_h, self.layer.out_w), dtype=x.dtype, device=x.device,
                        memory_format=torch.channels_last)
        self.layer.forward_into(x, y, stream=self.stream)
        return y

    def close(self):
        self.layer.close()


def _module(conv: CompressedConv2d):
    """nn.Module shim so the library layer can sit inside torchvision's graph."""
    torch = _torch()

    class LrsConvModule(torch.nn.Module):
        def __init__(self, c):
            super().__init__()
            self.c = c

        def forward(self, x):
            return self.c(x)

    return LrsConvModule(conv)


def fold_dense_batchnorms(model):
    """Fold every eval-mode BatchNorm that follows a DENSE conv (stem, bottleneck conv1 /
    conv3, downsample) into that conv's weight and bias -- the standard inference
    transform, y = conv(x, W * g / s) + (b - m * g / s), done in fp32 before the bf16
    cast.  The BatchNorm after each compressed 3x3 conv (bn2) stays a separate op:
    the library layer has no bias (reading #15)."""
    torch = _torch()
    from torch.nn.utils.fusion import fuse_conv_bn_eval
    model.conv1 = fuse_conv_bn_eval(model.conv1, model.bn1)
    model.bn1 = torch.nn.Identity()
    for layer in (model.layer1, model.layer2, model.layer3, model.layer4):
        for blk in layer:
            blk.conv1 = fuse_conv_bn_eval(blk.conv1, blk.bn1)
            blk.bn1 = torch.nn.Identity()
            blk.conv3 = fuse_conv_bn_eval(blk.conv3, blk.bn3)
            blk.bn3 = torch.nn.Identity()
            if blk.downsample is not None:
                blk.downsample = torch.nn.Sequential(fuse_conv_bn_eval(blk.downsample[0], blk.downsample[1]))
    return model


def _bottleneck_forward_fused(self, x):
    """torchvision Bottleneck.forward with bn2 + relu fused into the compressed conv2
    (the library's output epilogue), everything else unchanged."""
    identity = x
    out = self.relu(self.bn1(self.conv1(x)))
    out = self.conv2(out)  # conv + bn2 + relu in one library launch chain
    out = self.bn3(self.conv3(out))
    if self.downsample is not None:
        identity = self.downsample(x)
    out += identity
    return self.relu(out)


def build_compressed_resnet50(batch_max: int, device: int = 0, seed: int = 0, density: float = 0.02,
                              layers: Optional[List] = None, fold_bn: bool = True):
    """torchvision resnet50 (random init under manual_seed(seed), eval mode,
    bf16, channels_last) on cuda:device with its 16 3x3 convs compressed.
    fold_bn: fold the BatchNorms of the dense convs into them (fp32, before the
    bf16 cast), and the BatchNorm + ReLU after each compressed conv into the
    library's fused output epilogue.  Returns (model, {table index:
    CompressedConv2d})."""
    torch = _torch()
    import types
    import torchvision
    import workloads
    torch.manual_seed(seed)
    model = torchvision.models.resnet50(weights=None).eval()
    if fold_bn:
        model = fold_dense_batchnorms(model)
    # bn2's inference affine from its fp32 parameters (before the bf16 cast)
    bn2 = {}
    for idx, name, cfg in (layers or workloads.resnet50_compressed_layers(batch=batch_max, density=density)):
        bn = model.get_submodule(name.rsplit(".", 1)[0] + ".bn2")
        scale = (bn.weight / torch.sqrt(bn.running_var + bn.eps)).detach().float()
        bias = (bn.bias - bn.running_mean * scale).detach().float()
        bn2[idx] = (scale.numpy(), bias.numpy())
    model = model.to(device=f"cuda:{device}", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    comp: Dict[int, CompressedConv2d] = {}
    for idx, name, cfg in (layers or workloads.resnet50_compressed_layers(batch=batch_max, density=density)):
        inp = workloads.generate_weights(cfg)
        parent_name = name.rsplit(".", 1)[0]
        parent = model.get_submodule(parent_name)
        if fold_bn:
            conv = CompressedConv2d(inp, batch_max=batch_max, device=device, out_scale=bn2[idx][0],
                                    out_bias=bn2[idx][1], out_relu=True)
            parent.bn2 = torch.nn.Identity()
            parent.forward = types.MethodType(_bottleneck_forward_fused, parent)
        else:
            conv = CompressedConv2d(inp, batch_max=batch_max, device=device)
        comp[idx] = conv
        setattr(parent, name.rsplit(".", 1)[1], _module(conv))
    return model, comp
