"""Rebuilds the reference tests' seeded instances bit-for-bit (test infrastructure).

The reference generates every test input with std::mt19937_64 and libstdc++ distributions
(proj/tests/test_util.hpp:10-44); Mt19937_64 in the product library uses the same engine and
distributions (pinned by tests/golden/rng_golden.json), so e.g. the 50-seed dense sweep of
tests/test_unaligned_solvers.cpp:171-186 is reproduced instance for instance.
"""
from __future__ import annotations

import numpy as np

from inputs import Mt19937_64
from oracle import oracle as orc


def random_matrix(rng, rows, cols, lo=-1.0, hi=1.0):
    return rng.random_matrix(rows, cols, lo, hi)


def random_spd(rng, n, shift=0.5):
    a = random_matrix(rng, n, n)
    return np.asfortranarray(a @ a.T + shift * np.eye(n))


def random_tensor(shape, rng):
    """test_util.hpp:24-30: uniform(-1,1) in storage order."""
    n = int(np.prod(shape))
    return rng.uniform_real(-1.0, 1.0, n)  # flat, column-major storage order


def random_model(shape, r, rng):
    return [random_matrix(rng, n, r) for n in shape]


def sample(shape, flat, q, seed):
    """sample_uniform (observations.hpp:90-121): (d, q) int32 indices and values."""
    from inputs import sample_uniform_linear
    picked = sample_uniform_linear(int(flat.size), q, seed)
    idx = np.zeros((len(shape), q), dtype=np.int32)
    lin = picked.copy()
    for k, s in enumerate(shape):
        idx[k] = lin % s
        lin //= s
    return idx, flat[picked].copy()


def full_obs(shape, flat):
    n = flat.size
    lin = np.arange(n, dtype=np.int64)
    idx = np.zeros((len(shape), n), dtype=np.int32)
    for k, s in enumerate(shape):
        idx[k] = lin % s
        lin //= s
    return idx, flat.copy()


def grid_points(n):
    return np.arange(1, n + 1, dtype=np.float64)


def identity_points(n):
    return 1e6 * np.arange(n, dtype=np.float64)


class Inst:
    """random_instance (test_unaligned_solvers.cpp:36-47)."""

    def __init__(self, shape, r, q, k, sigma, lam, rho, seed, acceptance_rng=None):
        if acceptance_rng is None:
            rng = Mt19937_64(seed)
            self.flat = random_tensor(shape, rng)
            self.idx, self.vals = sample(shape, self.flat, q, seed + 1)
            self.factors = random_model(shape, r, rng)
            self.rng = rng
        else:  # acceptance_test.cpp:93-104 order: tensor, model, then rng() as the seed
            rng = acceptance_rng
            self.flat = random_tensor(shape, rng)
            self.factors = random_model(shape, r, rng)
            self.idx, self.vals = sample(shape, self.flat, q, rng())
            self.rng = rng
        self.shape = list(shape)
        self.k, self.r, self.sigma, self.lam, self.rho = k, r, sigma, lam, rho
        self.points = grid_points(shape[k])
        self.kernel = orc.gaussian_kernel(self.points, sigma)
        self.sub = orc.make_unaligned_subproblem(self.shape, self.idx, self.vals, self.factors, k,
                                                 self.kernel, lam, rho)


def build_f(sub):
    """build_F (unaligned.hpp:52-62): row l = zhat(l,:) kron khat(l,:) — test-only dense oracle."""
    n, r, q = sub.n, sub.r, sub.q
    khat = sub.kernel[sub.idx[sub.k], :]
    f = np.zeros((q, r * n))
    for j in range(r):
        f[:, j * n:(j + 1) * n] = sub.zhat[:, j:j + 1] * khat
    return f


def dense_sym_operator(sub):
    """test_unaligned_solvers.cpp:50-56: F'F + lambda (I kron K) + rho I."""
    f = build_f(sub)
    sysm = f.T @ f + sub.lam * np.kron(np.eye(sub.r), sub.kernel)
    sysm[np.diag_indices_from(sysm)] += sub.rho
    return sysm


def dense_preconditioner(sub):
    k2 = sub.kernel @ sub.kernel
    m = sub.density * np.kron(sub.v, k2) + sub.lam * np.kron(np.eye(sub.r), sub.kernel)
    m[np.diag_indices_from(m)] += sub.rho
    return m


def rel(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)
