"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds random-number recipes only -- none of the method's arithmetic
(no packing, no convolution, no thresholding).  Every array is drawn from
``numpy.random.Generator(PCG64(seed))`` so the oracle and the CUDA path are fed
the very same buffers.  The recipes are stated in DESIGN.md ("Input recipe").

The paper's data (NIH pancreas CT) is not available; the
CT-like volumes below stand in for it (Gaussian-blurred noise scaled to a
HU-like range, BASELINE.json configs[2..4]).
"""
from __future__ import annotations

import math

import numpy as np

# BASELINE.json configs, 0-based (SURVEY.md §0 "Config indexing").
CONFIGS = {
    "C0": dict(kind="conv", x_shape=(1, 16, 32, 32, 32), k=16, p0_x=0.5, p0_w=0.5,
               seed_x=0, seed_w=1, requant=False),
    "C1": dict(kind="conv", x_shape=(1, 64, 64, 128, 128), k=64, p0_x=0.5, p0_w=0.6,
               seed_x=10, seed_w=11, seed_t=12, requant=True),
    "C2": dict(kind="fcn", vol_shape=(1, 1, 96, 144, 144), seeds=(20,), seed_params=21),
    "C3": dict(kind="fcn", vol_shape=(1, 1, 128, 256, 256), seeds=tuple(100 + i for i in range(8)),
               seed_params=21),
    "C4": dict(kind="fcn", vol_shape=(1, 1, 256, 512, 512), seeds=(200,), seed_params=21),
}

# Weight shapes (cin, cout) of the 14 ternary layers the FCN configs draw
# parameters for (input recipe only; the topology itself is stated separately
# by the oracle and by the CUDA path's layer table).
FCN_WEIGHT_SHAPES = [(1, 16), (16, 16), (16, 16), (16, 32), (32, 32), (32, 64), (64, 64),
                     (64, 64), (128, 64), (64, 32), (64, 32), (32, 16), (32, 16), (16, 16)]

# HU-like scale of the CT stand-in and the matching Eq. 6 input thresholds
# (zero mean, sigma = 400 HU -> t = mu +- 0.5 sigma).
CT_SIGMA_HU = 400.0
CT_T_LO = -200.0
CT_T_HI = 200.0


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def ternary_codes(shape, p0: float, seed: int) -> np.ndarray:
    """int8 codes in {-1,0,+1}: P(0) = p0, P(+1) = P(-1) = (1 - p0)/2."""
    u = rng(seed).random(size=shape)
    out = np.zeros(shape, dtype=np.int8)
    half = (1.0 - p0) / 2.0
    out[u < half] = -1
    out[u >= 1.0 - half] = 1
    return out


def jittered_thresholds(k: int, base: int, seed: int):
    """Per-channel integer thresholds hi = base + j, lo = -base - j', j,j' in {-1,0,1}."""
    g = rng(seed)
    jh = g.integers(-1, 2, size=k)
    jl = g.integers(-1, 2, size=k)
    hi = (base + jh).astype(np.int32)
    lo = (-base - jl).astype(np.int32)
    return lo, hi


def threshold_base(cin: int, p_a: float, p_w: float = 0.4, taps: int = 27) -> int:
    """Quartile of an acc ~ N(0, taps*cin*p_a*p_w): about half the outputs become 0."""
    return int(round(0.6745 * math.sqrt(taps * cin * p_a * p_w)))


def ct_volume(shape, seed: int) -> np.ndarray:
    """CT-like float32 volume: N(0,1) -> separable Gaussian blur (sigma 2 voxels,
    radius 8, reflect, float64) -> / std -> * 400 -> clip [-1000, 1000]."""
    from scipy.ndimage import gaussian_filter1d

    v = rng(seed).standard_normal(size=shape)
    for ax in range(len(shape) - 3, len(shape)):
        v = gaussian_filter1d(v, sigma=2.0, axis=ax, mode="reflect", truncate=4.0)
    v /= v.std()
    v *= CT_SIGMA_HU
    np.clip(v, -1000.0, 1000.0, out=v)
    return v.astype(np.float32)


def conv_config(name: str):
    """(x codes int8 NCDHW, w codes int8 [k,c,3,3,3], lo, hi or None) for C0/C1."""
    cfg = CONFIGS[name]
    x = ternary_codes(cfg["x_shape"], cfg["p0_x"], cfg["seed_x"])
    c = cfg["x_shape"][1]
    w = ternary_codes((cfg["k"], c, 3, 3, 3), cfg["p0_w"], cfg["seed_w"])
    lo = hi = None
    if cfg["requant"]:
        base = threshold_base(c, 1.0 - cfg["p0_x"], 1.0 - cfg["p0_w"])
        lo, hi = jittered_thresholds(cfg["k"], base, cfg["seed_t"])
    return x, w, lo, hi


def binary_config():
    """NEXT-4 binary workload on C1's shape: {-1,+1} activations (seed 13) and weights (seed 14),
    sign thresholds hi in {-2, 0, 2} (seed 15) with lo = hi - 1 (acc is always even)."""
    x = ternary_codes((1, 64, 64, 128, 128), 0.0, seed=13)
    w = ternary_codes((64, 64, 3, 3, 3), 0.0, seed=14)
    hi = (2 * rng(15).integers(-1, 2, size=64)).astype(np.int32)
    return x, w, hi - 1, hi


def sample_positions(shape, k, m, seed):
    """m random output coordinates (n, k, z, y, x) of a stride-1 conv over shape (for sampled parity)."""
    g = rng(seed)
    n, _, d, h, w = shape
    return np.stack([g.integers(0, n, m), g.integers(0, k, m), g.integers(0, d, m),
                     g.integers(0, h, m), g.integers(0, w, m)], 1).astype(np.int32)


def fcn_params(seed: int = 21):
    """Ternary weights, integer thresholds and prediction weights for the FCN.

    Layer i (0-based) weights: P(0)=0.6, seed = seed + i.  Thresholds: base
    from :func:`threshold_base` (p_a = 0.38 for the first layer, whose input
    is the ternarised CT volume, else 0.5), jitter seed 40 + i.  Prediction:
    w ~ N(0, 0.25^2) [2,16], b ~ N(0, 0.1^2) [2], seed 60.
    """
    weights, lo, hi = [], [], []
    for i, (cin, cout) in enumerate(FCN_WEIGHT_SHAPES):
        weights.append(ternary_codes((cout, cin, 3, 3, 3), 0.6, seed + i))
        base = threshold_base(cin, 0.38 if i == 0 else 0.5)
        l, h = jittered_thresholds(cout, base, 40 + i)
        lo.append(l)
        hi.append(h)
    g = rng(60)
    pred_w = (0.25 * g.standard_normal(size=(2, 16))).astype(np.float32)
    pred_b = (0.1 * g.standard_normal(size=(2,))).astype(np.float32)
    return dict(weights=weights, lo=lo, hi=hi, pred_w=pred_w, pred_b=pred_b,
                t_lo=CT_T_LO, t_hi=CT_T_HI)


# NEXT-4: Table 1's 2.5D U-Net (reading R18).  (cin, cout, kernel) of its 14 ternary layers --
# input recipe only; the topology is stated separately by the oracle and the binding.
FCN25_WEIGHT_SHAPES = [(15, 32, 3), (32, 64, 3), (64, 64, 3), (64, 128, 3), (128, 128, 3), (128, 256, 3),
                       (256, 256, 1), (256, 256, 1), (512, 256, 3), (256, 128, 3), (256, 128, 3), (128, 64, 3),
                       (128, 64, 3), (64, 64, 3)]
# stack geometry: 15 neighbouring slices of 240 x 176 voxels (Table 1's 236 x 172
# input rounded up to a multiple of 8 for its three /2 levels); one volume = 138 stacks (the
# 138-slice ROI of PAPER.md:180)
STACK_SLICES, STACK_H, STACK_W, ROI_STACKS = 15, 240, 176, 138


def fcn25_params(seed: int = 81):
    """Weights of the 2D layers as [cout][cin][3][3][3] codes with P(0) = 0.6 on the active taps
    (the middle plane dz = 1 for 3x3 layers, the centre tap for 1x1 layers) and 0 elsewhere
    (those taps only ever meet the zero padding of one-plane inputs); thresholds from
    threshold_base with taps = 9 or 1 (p_a = 0.38 for layer 1, else 0.5), jitter seed 100 + i;
    prediction w ~ N(0, 0.25^2) [2][64], b ~ N(0, 0.1^2) (seed 61)."""
    weights, lo, hi = [], [], []
    for i, (cin, cout, k) in enumerate(FCN25_WEIGHT_SHAPES):
        w = np.zeros((cout, cin, 3, 3, 3), np.int8)
        act = ternary_codes((cout, cin, k, k), 0.6, seed + i)
        if k == 3:
            w[:, :, 1] = act
        else:
            w[:, :, 1, 1, 1] = act[:, :, 0, 0]
        weights.append(w)
        base = threshold_base(cin, 0.38 if i == 0 else 0.5, taps=k * k)
        l, h = jittered_thresholds(cout, base, 100 + i)
        lo.append(l)
        hi.append(h)
    g = rng(61)
    pred_w = (0.25 * g.standard_normal(size=(2, 64))).astype(np.float32)
    pred_b = (0.1 * g.standard_normal(size=(2,))).astype(np.float32)
    return dict(weights=weights, lo=lo, hi=hi, pred_w=pred_w, pred_b=pred_b, t_lo=CT_T_LO, t_hi=CT_T_HI)


def ct_stacks(n_stacks: int, h: int, w: int, seed: int) -> np.ndarray:
    """float32 [n_stacks][15][1][h][w]: stack s holds slices s-7 .. s+7 of a CT-like volume of
    n_stacks slices (ct_volume recipe), zero outside the volume ('a stack of several
    neighbouring slices (15 in our experiments)' per central slice)."""
    vol = ct_volume((1, 1, n_stacks, h, w), seed)[0, 0]
    half = STACK_SLICES // 2
    out = np.zeros((n_stacks, STACK_SLICES, 1, h, w), np.float32)
    for s in range(n_stacks):
        for j in range(STACK_SLICES):
            z = s + j - half
            if 0 <= z < n_stacks:
                out[s, j, 0] = vol[z]
    return out
