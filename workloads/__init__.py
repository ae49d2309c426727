"""Seeded synthetic inputs for the compressed-convolution hot path (W ~ L + S).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NO arithmetic of the method: it only draws random numbers, rounds
them to the storage precision, and builds the CSR index arrays of the sparse
term from sampled positions.  The method itself (how Y is computed from these
arrays) lives in `oracle/` (fp64 CPU reference) and in
`paper_2006_06443_b200/csrc/` (the CUDA path); neither is imported here.

Recipe (SURVEY.md §8(c) readings #7-#11):
  * one numpy Generator(PCG64(seed)); draw order X, U_in, G, U_out,
    S positions, S values;
  * X = ReLU(N(0,1)), NHWC [N, H, W, Cin]                  (BASELINE.json configs)
  * U_in [Cin, R1] ~ N(0, 1/Cin), G [R1, R2, k, k] ~ N(0, 1/(R1 k^2)),
    U_out [R2, Cout] ~ N(0, 1/R2)   -- "N(0, v)" read as variance v;
    SVD pair: U [Cin, R] ~ N(0, 1/Cin), V [R, Cout] ~ N(0, 1/R), core = None;
  * S: nnz = round(d * Cout*Cin*k*k) positions drawn uniformly without
    replacement over the OIHW linear index, sorted; values N(0, 0.1)
    (variance 0.1); CSR by output channel with col = (c*k + y)*k + x;
  * fp64 draws -> fp32 (RNE); bf16 configs additionally round X and the
    factors to bf16 (RNE).  S values stay fp32 for every dtype (SURVEY.md
    §8(c) reading #12: "S values fp32"; the ABI takes fp32 values and a bf16
    layer's engine rounds them itself -- that rounding is part of what the
    parity tests check, reading #12).

The arrays returned are exactly what both sides consume: the GPU gets the
fp32/bf16 bits, the oracle gets the same values widened to fp64.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

__all__ = [
    "LayerConfig", "LayerInputs", "CONFIGS", "generate", "bf16_round",
    "bf16_bits", "resnet50_table2", "RESNET50_COMPRESSED_3X3", "generate_weights",
    "resnet50_compressed_layers", "RESNET50_CONV2_MODULES", "resnet50_images",
    "CpInputs", "generate_cp", "CP_CONFIGS", "generate_x",
]


@dataclasses.dataclass(frozen=True)
class LayerConfig:
    """One compressed conv layer workload (BASELINE.json `configs`)."""
    name: str
    batch: int
    in_h: int
    in_w: int
    c_in: int
    c_out: int
    k: int
    stride: int
    pad: int
    rank_in: int          # R1 (Tucker-2) or R (SVD pair)
    rank_out: int         # R2 (Tucker-2) or R (SVD pair)
    density: float
    dtype: str            # "f32" | "bf16"
    svd: bool = False     # 1x1 layer evaluated as an SVD pair (no core)
    seed: int = 0

    @property
    def out_h(self) -> int:
        return (self.in_h + 2 * self.pad - self.k) // self.stride + 1

    @property
    def out_w(self) -> int:
        return (self.in_w + 2 * self.pad - self.k) // self.stride + 1

    @property
    def numel_w(self) -> int:
        return self.c_out * self.c_in * self.k * self.k

    @property
    def nnz(self) -> int:
        # round half to even never triggers for the shipped configs
        return int(round(self.density * self.numel_w))

    def replace(self, **kw) -> "LayerConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..3] (C1..C4); C2 is listed in both dtypes.
CONFIGS = {
    "c1": LayerConfig("c1", 1, 56, 56, 64, 64, 3, 1, 1, 16, 16, 0.01, "f32"),
    "c2_f32": LayerConfig("c2_f32", 64, 14, 14, 256, 256, 3, 1, 1, 64, 64, 0.02, "f32"),
    "c2_bf16": LayerConfig("c2_bf16", 64, 14, 14, 256, 256, 3, 1, 1, 64, 64, 0.02, "bf16"),
    "c3": LayerConfig("c3", 256, 7, 7, 512, 512, 3, 1, 1, 128, 128, 0.05, "bf16"),
    "c4": LayerConfig("c4", 128, 14, 14, 256, 1024, 1, 1, 0, 64, 64, 0.01, "bf16", svd=True),
}


@dataclasses.dataclass
class LayerInputs:
    cfg: LayerConfig
    x: np.ndarray                 # [N,H,W,Cin] float32 (bf16-representable for bf16)
    u_in: np.ndarray              # [Cin,R1] float32
    core: Optional[np.ndarray]    # [R1,R2,k,k] float32 or None (SVD)
    u_out: np.ndarray             # [R2,Cout] float32
    row_ptr: np.ndarray           # [Cout+1] int64
    col_idx: np.ndarray           # [nnz] int32, col = (c*k + y)*k + x
    values: np.ndarray            # [nnz] float32


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (round-to-nearest-even), returned as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounding_bias = ((u >> 16) & 1) + 0x7FFF
    r = ((u + rounding_bias) >> 16) << 16
    r = r.astype(np.uint32)
    nan = np.isnan(a)
    if nan.any():
        r[nan] = 0x7FC00000
    return r.view(np.float32)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """uint16 bit pattern of bf16-representable float32 values (no rounding)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def _store(a: np.ndarray, dtype: str) -> np.ndarray:
    a = a.astype(np.float32)
    return bf16_round(a) if dtype == "bf16" else a


def generate(cfg: LayerConfig, batch: Optional[int] = None, seed: Optional[int] = None,
             empty_rows_skew: bool = False) -> LayerInputs:
    """Draw the inputs of one layer (draw order fixed, see module doc)."""
    n = cfg.batch if batch is None else batch
    rng = np.random.Generator(np.random.PCG64(cfg.seed if seed is None else seed))
    k = cfg.k
    x = np.maximum(rng.standard_normal((n, cfg.in_h, cfg.in_w, cfg.c_in)), 0.0)
    if cfg.svd:
        u_in = rng.standard_normal((cfg.c_in, cfg.rank_in)) / np.sqrt(cfg.c_in)
        core = None
        u_out = rng.standard_normal((cfg.rank_in, cfg.c_out)) / np.sqrt(cfg.rank_in)
    else:
        u_in = rng.standard_normal((cfg.c_in, cfg.rank_in)) / np.sqrt(cfg.c_in)
        core = rng.standard_normal((cfg.rank_in, cfg.rank_out, k, k)) / np.sqrt(cfg.rank_in * k * k)
        u_out = rng.standard_normal((cfg.rank_out, cfg.c_out)) / np.sqrt(cfg.rank_out)
    numel = cfg.numel_w
    nnz = cfg.nnz
    pos = np.sort(rng.choice(numel, size=nnz, replace=False)) if nnz > 0 else np.zeros(0, np.int64)
    vals = rng.standard_normal(nnz) * np.sqrt(0.1)
    row_len = cfg.c_in * k * k
    rows = pos // row_len
    cols = pos % row_len
    row_ptr = np.zeros(cfg.c_out + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return LayerInputs(
        cfg=cfg,
        x=_store(x, cfg.dtype),
        u_in=_store(u_in, cfg.dtype),
        core=None if core is None else _store(core, cfg.dtype),
        u_out=_store(u_out, cfg.dtype),
        row_ptr=row_ptr,
        col_idx=cols.astype(np.int32),
        values=vals.astype(np.float32),
    )


def generate_x(cfg: LayerConfig, batch: Optional[int] = None, seed: int = 0) -> np.ndarray:
    """Only the input X of `generate(cfg, batch, seed)` (its first draw), so other
    seeds give other images for the same weights: generate_x(cfg, n, s) ==
    generate(cfg, n, seed=s).x."""
    n = cfg.batch if batch is None else batch
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.maximum(rng.standard_normal((n, cfg.in_h, cfg.in_w, cfg.c_in)), 0.0)
    return _store(x, cfg.dtype)


def generate_weights(cfg: LayerConfig, seed: Optional[int] = None) -> LayerInputs:
    """Factors and S of one layer WITHOUT an input X (C5 network layers, whose
    input is the previous layer's output).  Same recipe as `generate`, draw
    order U_in, G, U_out, S positions, S values from PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed if seed is None else seed))
    k = cfg.k
    u_in = rng.standard_normal((cfg.c_in, cfg.rank_in)) / np.sqrt(cfg.c_in)
    if cfg.svd:
        core = None
        u_out = rng.standard_normal((cfg.rank_in, cfg.c_out)) / np.sqrt(cfg.rank_in)
    else:
        core = rng.standard_normal((cfg.rank_in, cfg.rank_out, k, k)) / np.sqrt(cfg.rank_in * k * k)
        u_out = rng.standard_normal((cfg.rank_out, cfg.c_out)) / np.sqrt(cfg.rank_out)
    nnz = cfg.nnz
    pos = np.sort(rng.choice(cfg.numel_w, size=nnz, replace=False)) if nnz > 0 else np.zeros(0, np.int64)
    vals = rng.standard_normal(nnz) * np.sqrt(0.1)
    row_len = cfg.c_in * k * k
    rows, cols = pos // row_len, pos % row_len
    row_ptr = np.zeros(cfg.c_out + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    return LayerInputs(cfg=cfg, x=None, u_in=_store(u_in, cfg.dtype),
                       core=None if core is None else _store(core, cfg.dtype), u_out=_store(u_out, cfg.dtype),
                       row_ptr=np.cumsum(row_ptr), col_idx=cols.astype(np.int32), values=vals.astype(np.float32))


# the paper's own CP form of L at the C1 / C2 shapes,
# rank R = the configs' Tucker ranks (rank_in == rank_out).
CP_CONFIGS = {
    "c1_cp": LayerConfig("c1_cp", 1, 56, 56, 64, 64, 3, 1, 1, 16, 16, 0.01, "f32"),
    "c2_cp": LayerConfig("c2_cp", 64, 14, 14, 256, 256, 3, 1, 1, 64, 64, 0.02, "bf16"),
}


@dataclasses.dataclass
class CpInputs:
    """Inputs of a layer whose L is CP: L_{ijkp} = A_ir B_kr C_pr D_jr."""
    cfg: LayerConfig
    x: np.ndarray                 # [N,H,W,Cin]
    a: np.ndarray                 # [Cin,R]
    b: np.ndarray                 # [k,R]   taps along H
    c: np.ndarray                 # [k,R]   taps along W
    d: np.ndarray                 # [Cout,R]
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray


def generate_cp(cfg: LayerConfig, batch: Optional[int] = None, seed: Optional[int] = None) -> CpInputs:
    """Same recipe as `generate` with the CP factors in place of (U_in, G, U_out):
    draw order X, A ~ N(0, 1/Cin), B ~ N(0, 1/k), C ~ N(0, 1/k), D ~ N(0, 1/R),
    S positions, S values (fan-in variances, reading #8)."""
    n = cfg.batch if batch is None else batch
    rng = np.random.Generator(np.random.PCG64(cfg.seed if seed is None else seed))
    k, r = cfg.k, cfg.rank_in
    x = np.maximum(rng.standard_normal((n, cfg.in_h, cfg.in_w, cfg.c_in)), 0.0)
    a = rng.standard_normal((cfg.c_in, r)) / np.sqrt(cfg.c_in)
    b = rng.standard_normal((k, r)) / np.sqrt(k)
    c = rng.standard_normal((k, r)) / np.sqrt(k)
    d = rng.standard_normal((cfg.c_out, r)) / np.sqrt(r)
    nnz = cfg.nnz
    pos = np.sort(rng.choice(cfg.numel_w, size=nnz, replace=False)) if nnz > 0 else np.zeros(0, np.int64)
    vals = rng.standard_normal(nnz) * np.sqrt(0.1)
    row_len = cfg.c_in * k * k
    rows, cols = pos // row_len, pos % row_len
    row_ptr = np.zeros(cfg.c_out + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    st = lambda t: _store(t, cfg.dtype)  # noqa: E731
    return CpInputs(cfg=cfg, x=st(x), a=st(a), b=st(b), c=st(c), d=st(d), row_ptr=np.cumsum(row_ptr),
                    col_idx=cols.astype(np.int32), values=vals.astype(np.float32))


def resnet50_table2(path: Optional[str] = None):
    """Rows of PAPER.md Table 2 (`table:lshapes`) from the
    committed golden fixture: (index, c_in, in_h, in_w, c_out, k)."""
    import os
    if path is None:
        path = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "resnet50_table2.csv")
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#") or line.startswith("index"):
                continue
            idx, cin, h, w, cout, cin2, kx, ky = (int(t) for t in line.split(","))
            assert cin == cin2 and kx == ky
            rows.append((idx, cin, h, w, cout, kx))
    return rows


# Table-2 indices of the 16 ResNet-50 3x3 convs and their strides (torchvision
# v1.5 puts the stride on conv2 of the first block of layers 2-4; Table 2's
# input/output spatial sizes agree: layer 12 56->28, 25 28->14, 44 14->7).
RESNET50_COMPRESSED_3X3 = {
    2: 1, 6: 1, 9: 1, 12: 2, 16: 1, 19: 1, 22: 1, 25: 2,
    29: 1, 32: 1, 35: 1, 38: 1, 41: 1, 44: 2, 48: 1, 51: 1,
}


# torchvision resnet50 module of each compressed 3x3 conv (Table-2 index -> name)
RESNET50_CONV2_MODULES = {
    2: "layer1.0.conv2", 6: "layer1.1.conv2", 9: "layer1.2.conv2",
    12: "layer2.0.conv2", 16: "layer2.1.conv2", 19: "layer2.2.conv2", 22: "layer2.3.conv2",
    25: "layer3.0.conv2", 29: "layer3.1.conv2", 32: "layer3.2.conv2", 35: "layer3.3.conv2",
    38: "layer3.4.conv2", 41: "layer3.5.conv2",
    44: "layer4.0.conv2", 48: "layer4.1.conv2", 51: "layer4.2.conv2",
}


def resnet50_compressed_layers(batch: int = 256, density: float = 0.02, dtype: str = "bf16"):
    """C5 (BASELINE.json configs[4]): every ResNet-50 3x3 conv replaced by a
    Tucker-2 term with ranks Cin/4, Cout/4 plus a `density` sparse S.  Shapes
    are PAPER.md Table 2 rows (tests/golden/resnet50_table2.csv); strides
    RESNET50_COMPRESSED_3X3; seed 1000 + Table-2 index (reading #11).
    Returns [(table index, torchvision module name, LayerConfig)]."""
    rows = {r[0]: r for r in resnet50_table2()}
    out = []
    for idx, stride in RESNET50_COMPRESSED_3X3.items():
        _, cin, h, w, cout, k = rows[idx]
        assert k == 3
        cfg = LayerConfig(f"c5_l{idx}", batch, h, w, cin, cout, 3, stride, 1, cin // 4, cout // 4, density, dtype,
                          seed=1000 + idx)
        out.append((idx, RESNET50_CONV2_MODULES[idx], cfg))
    return out


def resnet50_images(n: int, seed: int = 0) -> np.ndarray:
    """C5 input: N(0,1) images [n, 3, 224, 224] (NCHW) standing in for
    normalised ImageNet pixels; float32 holding bf16 values."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return bf16_round(rng.standard_normal((n, 3, 224, 224)).astype(np.float32))


def generate_dy(cfg: LayerConfig, batch: Optional[int] = None, seed: int = 1) -> np.ndarray:
    """An upstream gradient dY = dLoss/dY of the layer's output shape for the backward
    pass: N(0, 1) entries from PCG64(seed), rounded like X to the
    layer's dtype.  A loss gradient has no sign structure, so unlike X it is not ReLU'd."""
    n = cfg.batch if batch is None else batch
    rng = np.random.Generator(np.random.PCG64(seed))
    return _store(rng.standard_normal((n, cfg.out_h, cfg.out_w, cfg.c_out)), cfg.dtype)


# ---------------------------------------------------------------- decomposition inputs (f4)
@dataclasses.dataclass(frozen=True)
class DecompConfig:
    """A weight tensor to decompose: dims (in, out, kh, kw), a planted CP
    rank, the decomposition's rank and cardinality, and the seed."""
    name: str
    dims: tuple
    planted_rank: int
    rank: int
    cardinality: float
    noise: float = 0.05
    spike: float = 10.0
    seed: int = 0


DECOMP_CONFIGS = {
    # the C3 layer's weight shape (ResNet-50 layer4 3x3 512 -> 512), CP rank 128, c = 1 %
    "c3_decomp": DecompConfig("c3_decomp", (512, 512, 3, 3), 96, 128, 0.01),
    # the C2 layer's weight shape (layer3 3x3 256 -> 256), CP rank 64
    "c2_decomp": DecompConfig("c2_decomp", (256, 256, 3, 3), 48, 64, 0.01),
}


def generate_decomp(cfg: DecompConfig):
    """(W, initial factors) for a decomposition run, from PCG64(seed), draw order: the planted
    factors (N(0,1) each, [dims[m], planted_rank]), the noise (N(0, noise^2)), the spike
    positions (uniform without replacement, round(cardinality * numel) of them), the spike signs,
    then the initial factors (N(0,1) [dims[m], rank]).  W = (planted CP tensor) / sqrt(planted_rank)
    + noise + spike * sign at the spike positions: a weight with a low-rank body and a few large
    entries -- the structure the paper's W ~ L + S targets (pretrained weights are unavailable)."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    pf = [rng.standard_normal((d, cfg.planted_rank)) for d in cfg.dims]
    w = np.ascontiguousarray(np.einsum("ar,br,cr,dr->abcd", *pf, optimize=True)) / np.sqrt(cfg.planted_rank)
    w += cfg.noise * rng.standard_normal(cfg.dims)
    numel = int(np.prod(cfg.dims))
    n = int(round(cfg.cardinality * numel))
    pos = rng.choice(numel, size=n, replace=False)
    w.flat[pos] += cfg.spike * np.sign(rng.standard_normal(n))
    f0 = [rng.standard_normal((d, cfg.rank)) for d in cfg.dims]
    return w, f0


def resnet50_decomp_configs(cardinality: float = 0.01):
    """The 16 ResNet-50 3x3 weights of C5 as decomposition inputs (f4 "batched over layers"):
    dims (Cin, Cout, 3, 3), CP rank min(Cin, Cout) / 4, a planted rank of 3/4 of it,
    cardinality 1 %, seed 1000 + the Table-2 index."""
    out = []
    for idx, _, cfg in resnet50_compressed_layers():
        r = min(cfg.c_in, cfg.c_out) // 4
        out.append(DecompConfig(f"l{idx}", (cfg.c_in, cfg.c_out, 3, 3), (3 * r) // 4, r, cardinality, seed=1000 + idx))
    return out


def generate_decomp_tucker2(cfg: DecompConfig, r1: int, r2: int):
    """(W, U_in0, U_out0) for a Tucker-2 decomposition run: W of generate_decomp(cfg) (a planted
    CP tensor is a Tucker-2 tensor of channel ranks <= planted_rank, plus noise and spikes); the
    initial channel bases N(0,1) [dims[0], r1] and [dims[1], r2] from PCG64(seed + 1000)."""
    w, _ = generate_decomp(cfg)
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 1000))
    return w, rng.standard_normal((cfg.dims[0], r1)), rng.standard_normal((cfg.dims[1], r2))
