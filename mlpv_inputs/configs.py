"""Config registry and seeded generators for BASELINE.json:configs.

All randomness comes from ``numpy.random.default_rng([12933, cfg, purpose])`` with purpose
0 = weights, 1 = base inputs, 2 = pixel subset, 3 = Philox key.  cfg5's two variants share
cfg5's draws.  The quantisers below (fp32 -> bf16 / Q4.12 / int8) *define* the synthetic net's
exact operands: the oracle and the CUDA path both receive the quantised integers / bf16 bits.
No forward pass, predicate, covering method or property lives here.
"""
from __future__ import annotations

import copy
import math
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

# enum values mirror include/mlpv.h (plain integers; the oracle has its own copy)
NUM_FP32, NUM_BF16, NUM_Q4_12, NUM_INT8 = 0, 1, 2, 3
ACT_SIGMOID, ACT_PL_SIGMOID, ACT_RELU = 0, 1, 2
PERT_TUPLE_REPLACE, PERT_SUBSET_OFFSET, PERT_SUBSET_REPLACE, PERT_PHILOX_LATTICE, PERT_PHILOX_BOX = 0, 1, 2, 3, 4
PERT_PHILOX_CLAMP = 5
PROP_ARGMAX_UNCHANGED, PROP_TARGET_NEVER, PROP_THRESHOLD_LITERAL, PROP_THRESHOLD_LITERAL_ALL = 0, 1, 2, 3

CONFIG_IDS = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5_bf16", "cfg5_int8"]

# Requantisation shifts of the int8 nets (C18).  Written by tools/calibrate_int8.py, which calls
# only oracle/: sh_l is the smallest shift with max over base inputs of ReLU(acc_l) >> sh_l <= 255.
INT8_SHIFTS = {
    "cfg3": [10, 7],
    "cfg5_int8": [12, 9],
}

INPUT_DTYPE = {NUM_FP32: np.float32, NUM_BF16: np.uint16, NUM_Q4_12: np.int16, NUM_INT8: np.uint8}
WEIGHT_DTYPE = {NUM_FP32: np.float32, NUM_BF16: np.uint16, NUM_Q4_12: np.int16, NUM_INT8: np.int8}
LEVEL_DTYPE = {NUM_FP32: np.float32, NUM_BF16: np.uint16, NUM_Q4_12: np.int16, NUM_INT8: np.int16}


# ----------------------------------------------------------------------------- bit helpers
def f32_to_bf16_bits(x) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round to nearest even (finite inputs only)."""
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(b) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _bf16_scalar(v: float) -> float:
    return float(bf16_bits_to_f32(f32_to_bf16_bits(np.array([v], np.float32)))[0])


# ----------------------------------------------------------------------------- data classes
@dataclass
class Net:
    sizes: List[int]                  # n_0 .. n_L
    act: int                          # hidden activation (output layer has none)
    numeric: int
    W: List[np.ndarray]               # [L] (n_l, n_{l-1}) storage dtype
    b: List[np.ndarray]               # [L] float32 (float numerics) | int32 accumulator units (fixed)
    requant_shift: Optional[List[int]] = None    # INT8: [L-1]
    sigmoid_knots: Optional[np.ndarray] = None   # PL_SIGMOID: int16[129]
    acc_scale: Optional[List[float]] = None      # [L] real value of one accumulator unit

    @property
    def L(self) -> int:
        return len(self.sizes) - 1


@dataclass
class Pert:
    kind: int
    tuple: int = 0
    pixels: Optional[np.ndarray] = None          # int32, strictly ascending
    levels: Optional[np.ndarray] = None          # LEVEL_DTYPE[numeric]
    seed: int = 0
    n_samples: int = 0
    lattice_step: float = 0.0
    lattice_origin: float = 0.0
    index_begin: int = 0
    index_end: int = 0
    restrict_l2: float = 0.0                     # restriction R (reading C27): 0 = none

    def space_size(self, n0: int) -> int:
        if self.kind == PERT_TUPLE_REPLACE:
            return math.comb(n0, self.tuple) * len(self.levels) ** self.tuple
        if self.kind in (PERT_SUBSET_OFFSET, PERT_SUBSET_REPLACE):
            return len(self.levels) ** len(self.pixels)
        return int(self.n_samples)

    def with_range(self, begin: int, end: int) -> "Pert":
        return replace(self, index_begin=int(begin), index_end=int(end))


@dataclass
class Prop:
    kind: int = PROP_ARGMAX_UNCHANGED
    target: int = -1
    V: float = 0.0


@dataclass
class CovSpec:
    pairs: List[int] = field(default_factory=list)   # lower layer k of pair (k, k+1), 1 <= k < L
    d_value: float = 0.1
    d_distance: float = 0.1
    near_tie: float = 1e-5


@dataclass
class Config:
    name: str
    description: str
    net: Net
    bases: np.ndarray                 # (n_base, n_0) INPUT_DTYPE[numeric]
    pert: Pert
    prop: Prop
    cov: CovSpec

    @property
    def n_base(self) -> int:
        return int(self.bases.shape[0])

    @property
    def space(self) -> int:
        return self.pert.space_size(self.net.sizes[0])

    def subset(self, n_base: Optional[int] = None, begin: int = 0, end: Optional[int] = None,
               base_start: int = 0) -> "Config":
        """Copy restricted to bases[base_start:base_start+n_base] and index range [begin, end)."""
        c = copy.copy(self)
        nb = self.n_base - base_start if n_base is None else n_base
        c.bases = np.ascontiguousarray(self.bases[base_start:base_start + nb])
        e = self.space if end is None else min(int(end), self.space)
        c.pert = self.pert.with_range(begin, e)
        return c


# ----------------------------------------------------------------------------- generators
def _rng(cfg: int, purpose: int) -> np.random.Generator:
    return np.random.default_rng([12933, cfg, purpose])


def _master_net(cfg: int, sizes: List[int], w_var_num: float):
    """fp32 masters: W ~ N(0, w_var_num/fan_in), b ~ N(0, 1/fan_in)."""
    rng = _rng(cfg, 0)
    W, b = [], []
    for l in range(1, len(sizes)):
        fan_in = sizes[l - 1]
        W.append(rng.normal(0.0, math.sqrt(w_var_num / fan_in), (sizes[l], fan_in)).astype(np.float32))
        b.append(rng.normal(0.0, math.sqrt(1.0 / fan_in), sizes[l]).astype(np.float32))
    return W, b


def smooth_blobs(rng: np.random.Generator, n: int, side: int = 28) -> np.ndarray:
    """MNIST-shaped stand-in: 2-4 Gaussian blobs, centres U[6,22)^2, sigma U[1.5,4),
    amplitude U[0.6,1), summed and clipped to [0,1]."""
    yy, xx = np.mgrid[0:side, 0:side].astype(np.float64)
    out = np.zeros((n, side * side), dtype=np.float32)
    for i in range(n):
        img = np.zeros((side, side))
        for _ in range(int(rng.integers(2, 5))):
            cy, cx = rng.uniform(6.0, 22.0, 2)
            sig = rng.uniform(1.5, 4.0)
            amp = rng.uniform(0.6, 1.0)
            img += amp * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2.0 * sig * sig))
        out[i] = np.clip(img, 0.0, 1.0).reshape(-1)
    return out


def pl_sigmoid_knots() -> np.ndarray:
    """C17: 129 knots T[m] = RNE(4096 * sigma(-8 + m/8)), shipped to both sides as data.
    (The table realises the paper's sigmoid lookup table, §IV.D.)"""
    m = np.arange(129, dtype=np.float64)
    return np.rint(4096.0 / (1.0 + np.exp(-(-8.0 + m / 8.0)))).astype(np.int16)


def _quant_q412(W: List[np.ndarray], b: List[np.ndarray]):
    """C16: raw = sat16(RNE(v * 4096)); bias in Q8.24 accumulator units = b_raw << 12."""
    Wq = [np.clip(np.rint(w.astype(np.float64) * 4096.0), -32768, 32767).astype(np.int16) for w in W]
    bq = [(np.clip(np.rint(v.astype(np.float64) * 4096.0), -32768, 32767).astype(np.int32) << 12) for v in b]
    return Wq, bq


def _quant_int8(W: List[np.ndarray], b: List[np.ndarray], shifts: List[int]):
    """C18: per-layer symmetric int8 weights, int32 biases in accumulator units."""
    s_in = 1.0 / 255.0
    Wq, bq, acc_scale = [], [], []
    for l, (w, v) in enumerate(zip(W, b)):
        s = float(np.max(np.abs(w.astype(np.float64)))) / 127.0
        Wq.append(np.clip(np.rint(w.astype(np.float64) / s), -127, 127).astype(np.int8))
        a = s * s_in
        bq.append(np.rint(v.astype(np.float64) / a).astype(np.int32))
        acc_scale.append(a)
        if l < len(W) - 1:
            s_in = a * (2.0 ** shifts[l])
    return Wq, bq, acc_scale


def _cfg1() -> Config:
    sizes = [25, 10, 5]
    W, b = _master_net(1, sizes, 1.0)
    bases = _rng(1, 1).random((1, 25), dtype=np.float32)
    levels = np.array([l / 15.0 for l in range(16)], dtype=np.float32)
    net = Net(sizes, ACT_SIGMOID, NUM_FP32, W, b, acc_scale=[1.0, 1.0])
    pert = Pert(PERT_TUPLE_REPLACE, tuple=2, levels=levels)
    pert.index_end = pert.space_size(25)
    return Config("cfg1", "25-10-5 sigmoid fp32, 1 base, all pixel pairs x 16 levels (76,800)",
                  net, bases, pert, Prop(), CovSpec([1]))


def _cfg2() -> Config:
    sizes = [25, 10, 5]
    W, b = _master_net(1, sizes, 1.0)                      # cfg1's master net (BASELINE cfg2)
    Wq, bq = _quant_q412(W, b)
    x = _rng(2, 1).random((10, 25), dtype=np.float32)
    bases = np.rint(x.astype(np.float64) * 4096.0).astype(np.int16)
    pixels = np.sort(_rng(2, 2).choice(25, 8, replace=False)).astype(np.int32)
    eps_raw = int(np.rint(0.1 * 4096.0))                   # 410
    levels = np.array([np.rint(eps_raw * (2 * d - 4) / 4.0) for d in range(5)], dtype=np.int16)
    net = Net(sizes, ACT_PL_SIGMOID, NUM_Q4_12, Wq, bq, sigmoid_knots=pl_sigmoid_knots(),
              acc_scale=[2.0 ** -24, 2.0 ** -24])
    pert = Pert(PERT_SUBSET_OFFSET, pixels=pixels, levels=levels)
    pert.index_end = pert.space_size(25)
    return Config("cfg2", "25-10-5 PL-sigmoid Q4.12, 10 bases, 8 pixels x 5 offsets (390,625/base)",
                  net, bases, pert, Prop(), CovSpec([1]))


def _cfg3() -> Config:
    sizes = [784, 64, 32, 10]
    W, b = _master_net(3, sizes, 2.0)
    sh = INT8_SHIFTS["cfg3"]
    Wq, bq, acc_scale = _quant_int8(W, b, sh)
    img = smooth_blobs(_rng(3, 1), 100)
    bases = np.rint(img.astype(np.float64) * 255.0).astype(np.uint8)
    cand = np.array([r * 28 + c for r in range(4, 24) for c in range(4, 24)])
    pixels = np.sort(_rng(3, 2).choice(cand, 6, replace=False)).astype(np.int32)
    levels = np.array([17 * l for l in range(16)], dtype=np.int16)
    net = Net(sizes, ACT_RELU, NUM_INT8, Wq, bq, requant_shift=list(sh), acc_scale=acc_scale)
    pert = Pert(PERT_SUBSET_REPLACE, pixels=pixels, levels=levels)
    pert.index_end = pert.space_size(784)
    return Config("cfg3", "784-64-32-10 ReLU int8, 100 bases, 6 pixels x 16 values (16.7M/base)",
                  net, bases, pert, Prop(), CovSpec([1, 2]))


def cfg4_lattice(eps: float = 0.05):
    """(step, origin) of cfg4's 16-level lattice: step = bf16(2 eps / 15) (a dyadic value; for
    eps = 0.05 it is 109 * 2^-14), origin = -7.5 step, so the offsets origin + l step, l = 0..15,
    are the odd multiples of step / 2 in [-7.5 step, 7.5 step] (radius 7.5 step = 0.0499 for
    eps = 0.05)."""
    step = _bf16_scalar(2.0 * eps / 15.0)
    return step, -7.5 * step


def eight_bit_bf16(img: np.ndarray) -> np.ndarray:
    """An image in [0, 1] as an 8-bit image (u8 / 255, as MNIST's pixels) stored as bf16 bits:
    every pixel is 0 or >= 1/255."""
    q = np.rint(np.clip(img.astype(np.float64), 0.0, 1.0) * 255.0) / 255.0
    return f32_to_bf16_bits(q.astype(np.float32))


def _cfg4() -> Config:
    sizes = [784, 256, 256, 10]
    W, b = _master_net(4, sizes, 2.0)
    Wb = [f32_to_bf16_bits(w) for w in W]
    img = smooth_blobs(_rng(4, 1), 1000)
    bases = eight_bit_bf16(img)
    seed = int(_rng(4, 3).integers(2 ** 64, dtype=np.uint64))
    net = Net(sizes, ACT_RELU, NUM_BF16, Wb, b, acc_scale=[1.0, 1.0, 1.0])
    # the L-inf box lattice of radius ~0.05 clamped to the image domain [0, 1] (reading C14)
    step, origin = cfg4_lattice(0.05)
    pert = Pert(PERT_PHILOX_CLAMP, seed=seed, n_samples=2 ** 32, lattice_step=step, lattice_origin=origin)
    pert.index_end = pert.n_samples
    return Config("cfg4", "784-256-256-10 ReLU bf16, 1000 bases, 2^32 Philox L-inf eps=0.05 samples/base, "
                  "clamped to [0,1]", net, bases, pert, Prop(), CovSpec([1, 2]))


def _cfg4_box() -> Config:
    """cfg4's net and bases on the unclamped box (PHILOX_BOX, reading C14b): an extra space."""
    c = copy.copy(_cfg4())
    c.name = "cfg4_box"
    c.pert = replace(c.pert, kind=PERT_PHILOX_BOX)
    return c


def _cfg5(variant: str) -> Config:
    sizes = [3072, 1024, 512, 10]
    W, b = _master_net(5, sizes, 2.0)
    # 8-bit images (CIFAR's pixels are u8): the bf16 variant holds u8 / 255 as bf16, the int8 one u8
    x = np.rint(_rng(5, 1).random((256, 3072), dtype=np.float32).astype(np.float64) * 255.0) / 255.0
    seed = int(_rng(5, 3).integers(2 ** 64, dtype=np.uint64))
    if variant == "bf16":
        net = Net(sizes, ACT_RELU, NUM_BF16, [f32_to_bf16_bits(w) for w in W], b, acc_scale=[1.0] * 3)
        bases = eight_bit_bf16(x)
        # offsets (l - 8) step, step = bf16(1/255) = 129 * 2^-15, clamped to [0, 1] (reading C14);
        # the int8 variant takes the same draws as u8 offsets l - 8
        step = _bf16_scalar(1.0 / 255.0)
        pert = Pert(PERT_PHILOX_CLAMP, seed=seed, n_samples=2 ** 30,
                    lattice_step=step, lattice_origin=-8.0 * step)
        name = "cfg5_bf16"
    else:
        sh = INT8_SHIFTS["cfg5_int8"]
        Wq, bq, acc_scale = _quant_int8(W, b, sh)
        net = Net(sizes, ACT_RELU, NUM_INT8, Wq, bq, requant_shift=list(sh), acc_scale=acc_scale)
        bases = np.rint(x.astype(np.float64) * 255.0).astype(np.uint8)
        pert = Pert(PERT_PHILOX_LATTICE, seed=seed, n_samples=2 ** 30,
                    lattice_step=1.0, lattice_origin=-8.0)
        name = "cfg5_int8"
    pert.index_end = pert.n_samples
    return Config(name, f"3072-1024-512-10 ReLU {variant}, 256 bases, 2^30 Philox samples/base (eps=8/255)",
                  net, bases, pert, Prop(), CovSpec([1, 2]))


_CACHE = {}


def make_config(name: str) -> Config:
    """Full-size config by name (cached; callers get a shallow copy)."""
    if name not in _CACHE:
        builders = {"cfg1": _cfg1, "cfg2": _cfg2, "cfg3": _cfg3, "cfg4": _cfg4, "cfg4_box": _cfg4_box,
                    "cfg5_bf16": lambda: _cfg5("bf16"), "cfg5_int8": lambda: _cfg5("int8")}
        _CACHE[name] = builders[name]()
    return copy.copy(_CACHE[name])


# ------------------------------------------------------------ dataset-pair workload (NEXT-3)
def vowel_net(numeric: int = NUM_Q4_12, seed: int = 0) -> Net:
    """A random-init 25-5-4-5 sigmoid net, the architecture of the paper's vocalic classifier
    (Table II's 14 neurons).  Q4.12: PL-sigmoid table (readings
    C16/C17), W in Q4.12, b in Q8.24; FP32: the exact logistic sigmoid on W / 4096, b * 2^-24."""
    return _vowel_net(np.random.default_rng([12933, 77, seed]), numeric)


def _vowel_net(rng: np.random.Generator, numeric: int) -> Net:
    sizes = [25, 5, 4, 5]
    W, b = [], []
    for l in range(1, 4):
        w = rng.normal(0.0, np.sqrt(4.0 / sizes[l - 1]), (sizes[l], sizes[l - 1]))
        W.append(np.clip(np.rint(w * 4096), -32768, 32767).astype(np.int16))
        b.append((np.rint(rng.normal(0.0, 0.5, sizes[l]) * 4096).astype(np.int64) << 12).astype(np.int32))
    if numeric == NUM_Q4_12:
        return Net(sizes, ACT_PL_SIGMOID, NUM_Q4_12, W, b, sigmoid_knots=pl_sigmoid_knots(),
                   acc_scale=[2.0 ** -24] * 3)
    assert numeric == NUM_FP32
    return Net(sizes, ACT_SIGMOID, NUM_FP32, [(w.astype(np.float64) / 4096).astype(np.float32) for w in W],
               [(v.astype(np.float64) * 2.0 ** -24).astype(np.float32) for v in b], acc_scale=[1.0] * 3)


def pair_images(net: Net, n: int, seed: int = 0) -> np.ndarray:
    """n seeded images for the dataset-pair workload, in the net's input element type.
    n_0 = 25: 5x5 glyph-like stand-ins for the vocalic images and their noisy variants
    (Fig. 4): pixels on with p = 0.4 at U[0.7, 1) plus N(0, 0.05) noise, clipped
    to [0, 1].  n_0 = 784: smooth_blobs (28x28).  Otherwise U[0, 1) pixels."""
    rng = np.random.default_rng([12933, 303, seed])
    n0 = net.sizes[0]
    if n0 == 25:
        x = (rng.random((n, 25)) < 0.4) * rng.uniform(0.7, 1.0, (n, 25)) + rng.normal(0.0, 0.05, (n, 25))
        x = np.clip(x, 0.0, 1.0)
    elif n0 == 784:
        x = smooth_blobs(rng, n).astype(np.float64)
    else:
        x = rng.random((n, n0))
    if net.numeric == NUM_FP32:
        return x.astype(np.float32)
    if net.numeric == NUM_BF16:
        return f32_to_bf16_bits(x.astype(np.float32))
    if net.numeric == NUM_Q4_12:
        return np.rint(x * 4096.0).astype(np.int16)
    return np.rint(x * 255.0).astype(np.uint8)


def gamma_config(n_base: int = 50) -> Config:
    """Table III-style workload (NEXT-1 / NEXT-2): vowel_net(Q4.12), n_base 5x5
    binary images (pixels on with p = 0.4), a SUBSET_REPLACE space over 8 pixels x levels
    {0, 0.5, 1} (6,561 candidates per base), property "class unchanged"."""
    rng = np.random.default_rng([12933, 77, 0])
    net = _vowel_net(rng, NUM_Q4_12)
    bases = (rng.random((n_base, 25)) < 0.4).astype(np.int16) * 4096
    pixels = np.sort(rng.choice(25, 8, replace=False)).astype(np.int32)
    pert = Pert(PERT_SUBSET_REPLACE, pixels=pixels, levels=np.array([0, 2048, 4096], np.int16),
                index_begin=0, index_end=3 ** 8)
    return Config("gamma", "25-5-4-5 PL-sigmoid Q4.12", net, bases, pert, Prop(), CovSpec([1, 2]))
