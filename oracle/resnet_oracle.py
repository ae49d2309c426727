"""fp64 CPU oracle of C5: ResNet-50 whose 16 3x3 convs are compressed layers
W ~ L + S (BASELINE.json configs[4]; §5.5, :343-387).

TEST INFRASTRUCTURE ONLY (same rule as lrs_oracle.py): imported by tests/
and bench.py's reference leg only; the product never imports it.

The dense layers are torchvision's resnet50 (a library, independent of the
CUDA path) run on the CPU in fp64 with the SAME parameters the GPU model
holds: torchvision random init under torch.manual_seed(seed), rounded to
bf16 (the GPU model is bf16), widened to fp64.  Each compressed 3x3 conv is
replaced by `lrs_oracle.forward_factored` (PAPER.md:162-168 chain + :189
sparse term) on the seeded factors of `workloads.resnet50_compressed_layers`.
Inputs are the bf16-rounded images.  Pinned (tests/test_oracle_pins.py) by
the same network with each conv2 weight set to the dense reconstruction
W = L + S and run through torch's own fp64 conv2d.
"""
from __future__ import annotations

import numpy as np

from . import lrs_oracle as O


def _bf16_round_tensor(t):
    import torch
    return t.to(torch.bfloat16).to(torch.float64)


class _DirectConv:
    """A dense torch Conv2d evaluated by lrs_oracle.conv_direct (fp64 BLAS, tap
    by tap; PAPER.md:160 written out) -- torch's own fp64 CPU conv2d is too slow
    for 224x224 images; it pins this route in tests/test_oracle_pins.py."""

    def __init__(self, conv):
        self.w = np.transpose(conv.weight.detach().numpy().astype(np.float64), (1, 0, 2, 3))
        self.stride, self.pad = conv.stride[0], conv.padding[0]
        assert conv.bias is None and conv.groups == 1 and conv.stride[0] == conv.stride[1]

    def __call__(self, x):
        import torch
        xn = x.permute(0, 2, 3, 1).contiguous().numpy()
        y = O.conv_direct(xn, self.w, self.stride, self.pad)
        return torch.from_numpy(y).permute(0, 3, 1, 2).contiguous()


class _FactoredConv:
    """Module computing the compressed layer with the fp64 oracle (NCHW in/out)."""

    def __init__(self, inp):
        self.inp = inp

    def __call__(self, x):
        import torch
        c = self.inp.cfg
        xn = x.permute(0, 2, 3, 1).contiguous().numpy()
        y = O.forward_factored(xn, self.inp.u_in, self.inp.core, self.inp.u_out, self.inp.row_ptr,
                               self.inp.col_idx, self.inp.values, c.stride, c.pad)
        return torch.from_numpy(y).permute(0, 3, 1, 2).contiguous()


def _wrap(fn):
    import torch

    class M(torch.nn.Module):
        def __init__(self, f):
            super().__init__()
            self.f = f

        def forward(self, x):
            return self.f(x)

    return M(fn)


def build_reference_resnet50(seed: int = 0, density: float = 0.02, dense_conv2: bool = False,
                             torch_convs: bool = False):
    """The fp64 CPU reference network.  dense_conv2=True instead sets each
    compressed conv's weight to the dense reconstruction of L + S, and
    torch_convs=True keeps torch's own fp64 conv2d for the dense convs (both
    used only to pin this network, at small image sizes)."""
    import torch
    import torchvision
    import workloads
    torch.manual_seed(seed)
    model = torchvision.models.resnet50(weights=None).eval()
    with torch.no_grad():
        for p_ in model.parameters():
            p_.copy_(p_.to(torch.bfloat16).to(torch.float32))
        for b in model.buffers():
            if b.dtype.is_floating_point:
                b.copy_(b.to(torch.bfloat16).to(torch.float32))
    model = model.to(torch.float64)
    for idx, name, cfg in workloads.resnet50_compressed_layers(batch=1, density=density):
        inp = workloads.generate_weights(cfg)
        parent = model.get_submodule(name.rsplit(".", 1)[0])
        leaf = name.rsplit(".", 1)[1]
        if dense_conv2:
            w = O.reconstruct_tucker2(inp.u_in, inp.core, inp.u_out) + O.densify_sparse(
                cfg.c_in, cfg.c_out, 3, inp.row_ptr, inp.col_idx, inp.values)
            conv = getattr(parent, leaf)
            with torch.no_grad():
                conv.weight.copy_(torch.from_numpy(np.transpose(w, (1, 0, 2, 3))))
        else:
            setattr(parent, leaf, _wrap(_FactoredConv(inp)))
    if not torch_convs:
        for name, mod in list(model.named_modules()):
            if isinstance(mod, torch.nn.Conv2d):
                parent = model.get_submodule(name.rsplit(".", 1)[0]) if "." in name else model
                setattr(parent, name.rsplit(".", 1)[-1], _wrap(_DirectConv(mod)))
    return model


def reference_logits(images: np.ndarray, seed: int = 0, density: float = 0.02, dense_conv2: bool = False,
                     torch_convs: bool = False):
    """Logits [n, 1000] in fp64 for NCHW images (bf16-representable float32)."""
    import torch
    model = build_reference_resnet50(seed, density, dense_conv2, torch_convs)
    with torch.no_grad():
        return model(torch.from_numpy(images.astype(np.float64))).numpy()
