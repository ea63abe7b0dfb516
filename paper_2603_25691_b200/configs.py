"""Seeded synthetic inputs for BASELINE.json's configs.

No public dataset is involved: the configs are synthetic by definition.  Configs 0 and 1 are
drawn with the reference's own RNG stack (std::mt19937_64 + libstdc++ normal_distribution,
seed 0; sampler = sample_uniform, observations.hpp:90-121).  Configs 2-4 draw the small factor
matrices the same way and the bulk noise / indices with numpy's PCG64 (config 2) or on the
device with a counter-based generator (configs 3-4, see synth_observations).

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
    import paper_2603_25691_b200 as cp
    return cp.Mt19937_64(seed)


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
    from . import sample_uniform, DenseTensor
    obs = sample_uniform(DenseTensor(c0.shape, c0.tensor), 200_000, 1)
    return UnalignedConfig("config1", c0.shape, c0.r, 1e-3, 1e-6, 1e-8, 500, c0.points, "gaussian", 0.1,
                           c0.factors, c0.w_true, obs.index_array(), obs.values())


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
    from . import sample_uniform, DenseTensor
    obs = sample_uniform(DenseTensor(list(shape), t), q, seed + 1)
    return UnalignedConfig("small", list(shape), r, 1e-3, 1e-6, 1e-8, 500, pts, "gaussian", 0.1, factors, w,
                           obs.index_array(), obs.values())
