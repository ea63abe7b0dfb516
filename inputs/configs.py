"""Seeded synthetic inputs for BASELINE.json's configs.

No public dataset is involved: the configs are synthetic by definition.  Configs 0 and 1 are
drawn with the reference's own RNG stack (std::mt19937_64 + libstdc++ normal_distribution,
seed 0; sampler = sample_uniform, observations.hpp:90-121).  Configs 2-4 draw the small factor
matrices the same way and the bulk noise / indices with numpy's PCG64 (config 2) or on the
device with a counter-based generator (configs 3-4: inputs/synth_math.h, the same bits on the host and on the device).

Noise "N(0, 1e-2)" is read as VARIANCE 1e-2 (std 0.1); SURVEY §8d records the choice.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class AlignedConfig:
    name: str
    shape: list
    r: int
    lam: float
    points: np.ndarray
    kernel: str            # "gaussian" | "matern32"
    ell: float
    factors: list          # truth; factors[0] = K W_true
    w_true: np.ndarray
    tensor: np.ndarray = field(repr=False, default=None)   # flat column-major


@dataclass
class UnalignedConfig:
    name: str
    shape: list
    r: int
    lam: float
    rho: float
    tol: float
    max_iter: int
    points: np.ndarray
    kernel: str
    ell: float
    factors: list
    w_true: np.ndarray
    idx: np.ndarray = field(repr=False, default=None)      # (d, q) int32
    vals: np.ndarray = field(repr=False, default=None)     # (q,)
    multiset: bool = False


def _rng(seed):
    from . import Mt19937_64
    return Mt19937_64(seed)


def sample_uniform(shape, tensor_flat, q, seed):
    """sample_uniform (observations.hpp:90-121) on a column-major tensor: (d, q) int32 indices of q
    distinct entries (partial Fisher-Yates, mt19937_64(seed)) and their values."""
    from . import sample_uniform_linear
    picked = sample_uniform_linear(int(np.prod(shape)), q, seed)
    idx = np.zeros((len(shape), q), dtype=np.int32)
    lin = picked.copy()
    for k, s in enumerate(shape):
        idx[k] = lin % s
        lin //= s
    return idx, np.asarray(tensor_flat)[picked]


def _normal_matrix(rng, rows, cols):
    return np.asfortranarray(rng.normal(0.0, 1.0, rows * cols).reshape((rows, cols), order="F"))


def kernel_matrix(points, kind, ell):
    x = np.asarray(points, dtype=np.float64)
    d = np.abs(x[:, None] - x[None, :])
    if kind == "gaussian":
        return np.exp(-d * d * (1.0 / (2.0 * ell * ell)))
    a = np.sqrt(3.0) / ell * d
    return (1.0 + a) * np.exp(-a)


def _full_3way(a1, a2, a3):
    """[[A1, A2, A3]] flattened column-major (i1 fastest)."""
    n1, n2, n3 = a1.shape[0], a2.shape[0], a3.shape[0]
    t = np.empty((n1, n2, n3), order="F")
    for i3 in range(n3):
        t[:, :, i3] = a1 @ (a2 * a3[i3][None, :]).T
    return t.reshape(-1, order="F")


def config0() -> AlignedConfig:
    """Aligned 200x100x100, mode-1 RBF(0.1) on a uniform grid, rank 10, lambda 1e-3."""
    n, r = 200, 10
    pts = np.arange(n, dtype=np.float64) / (n - 1)
    rng = _rng(0)
    w = _normal_matrix(rng, n, r)
    a2 = _normal_matrix(rng, 100, r)
    a3 = _normal_matrix(rng, 100, r)
    kmat = kernel_matrix(pts, "gaussian", 0.1)
    a1 = np.asfortranarray(kmat @ w)
    t = _full_3way(a1, a2, a3)
    t = t + rng.normal(0.0, 0.1, t.size)
    return AlignedConfig("config0", [n, 100, 100], r, 1e-3, pts, "gaussian", 0.1, [a1, a2, a3], w, t)


def config1() -> UnalignedConfig:
    """Unaligned version of config 0: q = 200k distinct entries (10 %), PCG tol 1e-8."""
    c0 = config0()
    idx, vals = sample_uniform(c0.shape, c0.tensor, 200_000, 1)
    return UnalignedConfig("config1", c0.shape, c0.r, 1e-3, 1e-6, 1e-8, 500, c0.points, "gaussian", 0.1,
                           c0.factors, c0.w_true, idx, vals)


def config2() -> AlignedConfig:
    """Aligned 1024x256x256, RBF(0.05) on sorted uniform points, rank 32, lambda 1e-4."""
    n, r = 1024, 32
    rng = _rng(0)
    pts = np.sort(rng.uniform_real(0.0, 1.0, n))
    w = _normal_matrix(rng, n, r)
    a2 = _normal_matrix(rng, 256, r)
    a3 = _normal_matrix(rng, 256, r)
    kmat = kernel_matrix(pts, "gaussian", 0.05)
    a1 = np.asfortranarray(kmat @ w)
    t = _full_3way(a1, a2, a3)
    t += np.random.default_rng(2).normal(0.0, 0.1, t.size)
    return AlignedConfig("config2", [n, 256, 256], r, 1e-4, pts, "gaussian", 0.05, [a1, a2, a3], w, t)


def small_unaligned(shape=(40, 12, 10), r=4, q=1500, seed=5) -> UnalignedConfig:
    """A scaled-down config-1 analogue for quick parity checks."""
    rng = _rng(seed)
    n = shape[0]
    pts = np.arange(n, dtype=np.float64) / (n - 1)
    w = _normal_matrix(rng, n, r)
    others = [_normal_matrix(rng, s, r) for s in shape[1:]]
    kmat = kernel_matrix(pts, "gaussian", 0.1)
    a1 = np.asfortranarray(kmat @ w)
    factors = [a1] + others
    t = _full_3way(*factors) if len(shape) == 3 else None
    t = t + rng.normal(0.0, 0.1, t.size)
    idx, vals = sample_uniform(list(shape), t, q, seed + 1)
    return UnalignedConfig("small", list(shape), r, 1e-3, 1e-6, 1e-8, 500, pts, "gaussian", 0.1, factors, w,
                           idx, vals)


# ---- configs 3 and 4: observations generated on the device --------------------------------
@dataclass
class DeviceUnalignedConfig:
    """Factors are host arrays; the q observations are drawn on the GPU by
    cphifi_synth_observations (counter-based, seed-reproducible)."""
    name: str
    shape: list
    r: int
    lam: float
    rho: float
    tol: float
    max_iter: int
    points: np.ndarray
    kernel: str
    ell: float
    factors: list
    w_true: np.ndarray
    q: int
    seed: int
    zipf_mode: int
    zipf_s: float
    noise_std: float = 0.1
    coalesce: bool = False  # merge repeated draws in the plan (CPHIFI_OBS_COALESCE_DUPLICATES)


def config3() -> DeviceUnalignedConfig:
    """Unaligned 4-way 2048x256x256x256, Matern-3/2 (0.05) on 2048 sorted uniform points,
    q = 2e8 uniform draws (multiset), rank 32, lambda 1e-4, PCG tol 1e-8."""
    n, r = 2048, 32
    rng = _rng(3)
    pts = np.sort(rng.uniform_real(0.0, 1.0, n))
    w = _normal_matrix(rng, n, r)
    others = [_normal_matrix(rng, 256, r) for _ in range(3)]
    a1 = np.asfortranarray(kernel_matrix(pts, "matern32", 0.05) @ w)
    return DeviceUnalignedConfig("config3", [n, 256, 256, 256], r, 1e-4, 1e-6, 1e-8, 500, pts, "matern32", 0.05,
                                 [a1] + others, w, 200_000_000, 3, -1, 0.0)


def config4() -> DeviceUnalignedConfig:
    """Unaligned skewed 3-way 4096x512x512, RBF (0.02) on 4096 clustered points (8 Gaussian
    clusters, sigma 0.03, clipped to [0,1]), q = 1e9 draws with i_1 ~ Zipf(1.1), rank 64,
    lambda 1e-5, PCG tol 1e-8."""
    n, r = 4096, 64
    rng = _rng(4)
    centres = rng.uniform_real(0.0, 1.0, 8)
    which = rng.uniform_int(0, 7, n)
    pts = np.sort(np.clip(centres[which] + 0.03 * rng.normal(0.0, 1.0, n), 0.0, 1.0))
    w = _normal_matrix(rng, n, r)
    others = [_normal_matrix(rng, 512, r) for _ in range(2)]
    a1 = np.asfortranarray(kernel_matrix(pts, "gaussian", 0.02) @ w)
    return DeviceUnalignedConfig("config4", [n, 512, 512], r, 1e-5, 1e-6, 1e-8, 500, pts, "gaussian", 0.02,
                                 [a1] + others, w, 1_000_000_000, 4, 0, 1.1, coalesce=True)


def generate_host(cfg: DeviceUnalignedConfig, l0: int = 0, l1: int | None = None, values: bool = True,
                  threads: int | None = None):
    """Draws [l0, l1) of cfg's observations on the host (bit-identical to the device generator,
    paper_2603_25691_b200.synth_observations_device): idx (d, l1 - l0) int32, vals fp64 or None."""
    from . import synth_observations
    l1 = cfg.q if l1 is None else l1
    return synth_observations(cfg.shape, l0, l1, cfg.seed, cfg.zipf_mode, cfg.zipf_s, cfg.factors, cfg.noise_std,
                              values=values, threads=threads)
