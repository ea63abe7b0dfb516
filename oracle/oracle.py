"""CPU ORACLE wrapper (test infrastructure only — never imported by the product package).

ctypes front-end over ``oracle/_build/libcphifi_oracle.so`` (the plain-C restatement in
``cphifi_oracle.c``) plus two small pure-numpy restatements:

* :func:`pcg` — ``pcg`` (proj/include/cphifi/solvers.hpp:38-88), line for line: zero
  initial guess unless given, recurrence residual, break before the preconditioner, the
  same two ``runtime_error`` checks and the ``bnorm == 0`` early exit.
* :func:`sym_eig` — ``sym_eig`` (kernel.hpp:40-49): symmetry check at
  ``1e-12 * max(scale, 1)``, LAPACK ``dsyevd`` (numpy) instead of Eigen's
  ``SelfAdjointEigenSolver`` (parity unpinned at the Eigen boundary), clamp
  at 0.  The device path is fed the SAME eigendecomposition in parity tests.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs use this
module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libcphifi_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_lp = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64


class InvalidArgument(ValueError):
    """Mirrors std::invalid_argument."""


class RuntimeFailure(RuntimeError):
    """Mirrors std::runtime_error."""


def build() -> str:
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise InvalidArgument(msg)
    raise RuntimeFailure(msg)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _factor_ptrs(factors, k):
    arrs = [None if (i == k or f is None) else _f64(f) for i, f in enumerate(factors)]
    ptrs = (_dp * len(arrs))(*[(_d(a) if a is not None else _dp()) for a in arrs])
    return arrs, ptrs


def max_threads() -> int:
    return lib().orc_max_threads()


# ---- dense algebra ---------------------------------------------------------------------
def gemm(a, b, ta=False, tb=False, threads=1) -> np.ndarray:
    a = _f64(a); b = _f64(b)
    m = a.shape[1] if ta else a.shape[0]
    kk = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    c = np.zeros((m, n), order="F")
    lib().orc_gemm(int(ta), int(tb), _i64(m), _i64(n), _i64(kk), ctypes.c_double(1.0), _d(a),
                   _i64(a.shape[0]), _d(b), _i64(b.shape[0]), ctypes.c_double(0.0), _d(c),
                   _i64(m), threads)
    return c


# ---- kernel.hpp ------------------------------------------------------------------------
def gaussian_kernel(points, sigma) -> np.ndarray:
    p = np.ascontiguousarray(points, dtype=np.float64)
    k = np.zeros((p.size, p.size), order="F")
    _check(lib().orc_gaussian_kernel(_d(p), _i64(p.size), ctypes.c_double(sigma), _d(k)))
    return k


def matern32_kernel(points, ell) -> np.ndarray:
    p = np.ascontiguousarray(points, dtype=np.float64)
    k = np.zeros((p.size, p.size), order="F")
    _check(lib().orc_matern32_kernel(_d(p), _i64(p.size), ctypes.c_double(ell), _d(k)))
    return k


@dataclass
class SymEig:
    u: np.ndarray
    d: np.ndarray


def sym_eig(k) -> SymEig:
    """kernel.hpp:40-49 (LAPACK dsyevd in place of Eigen; see module doc)."""
    k = np.asarray(k, dtype=np.float64)
    scale = np.abs(k).max() if k.size else 0.0
    if k.size and np.abs(k - k.T).max() > 1e-12 * max(scale, 1.0):
        raise InvalidArgument("sym_eig: matrix is not symmetric")
    w, u = np.linalg.eigh(k)
    if not (np.all(np.isfinite(w)) and np.all(np.isfinite(u))):
        raise RuntimeFailure("sym_eig: eigendecomposition failed")
    return SymEig(np.asfortranarray(u), np.maximum(w, 0.0))


# ---- observations.hpp ------------------------------------------------------------------
def build_zhat(shape, k, idx, factors) -> np.ndarray:
    """observations.hpp:142-158; idx is a (d, q) int array."""
    shape = np.ascontiguousarray(shape, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    d, q = idx.shape
    r = next(np.asarray(f).shape[1] for i, f in enumerate(factors) if i != k)
    for i in range(d):
        if i != k and np.asarray(factors[i]).shape[0] != shape[i]:
            raise InvalidArgument("build_zhat: shape mismatch")
    arrs, ptrs = _factor_ptrs(factors, k)
    z = np.zeros((q, r), order="F")
    lib().orc_build_zhat(d, shape.ctypes.data_as(_lp), k, _i64(q), idx.ctypes.data_as(_ip),
                         _i64(r), ptrs, _d(z))
    return z


def gather_rows(xhat, zhat, idx_k) -> np.ndarray:
    """observations.hpp:191-198."""
    xhat = _f64(xhat); zhat = _f64(zhat)
    idx_k = np.ascontiguousarray(idx_k, dtype=np.int32)
    if zhat.shape[0] != idx_k.size:
        raise InvalidArgument("gather_rows: row count mismatch")
    out = np.zeros(idx_k.size)
    lib().orc_gather_rows(_i64(xhat.shape[0]), _i64(xhat.shape[1]), _d(xhat), _i64(idx_k.size),
                          _d(zhat), idx_k.ctypes.data_as(_ip), _d(out))
    return out


def sampled_mttkrp(n, zhat, idx_k, weights) -> np.ndarray:
    """observations.hpp:174-184."""
    zhat = _f64(zhat)
    idx_k = np.ascontiguousarray(idx_k, dtype=np.int32)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if zhat.shape[0] != idx_k.size or w.size != idx_k.size:
        raise InvalidArgument("sampled_mttkrp: row count mismatch")
    out = np.zeros((n, zhat.shape[1]), order="F")
    lib().orc_sampled_mttkrp(_i64(n), _i64(zhat.shape[1]), _i64(idx_k.size), _d(zhat),
                             idx_k.ctypes.data_as(_ip), _d(w), _d(out))
    return out


# ---- tensor.hpp ------------------------------------------------------------------------
def khatri_rao_excluding(shape, factors, k) -> np.ndarray:
    shape = np.ascontiguousarray(shape, dtype=np.int64)
    d = shape.size
    r = next(np.asarray(f).shape[1] for i, f in enumerate(factors) if i != k)
    rows = int(np.prod([shape[i] for i in range(d) if i != k]))
    arrs, ptrs = _factor_ptrs(factors, k)
    z = np.zeros((rows, r), order="F")
    lib().orc_khatri_rao_excluding(d, shape.ctypes.data_as(_lp), k, _i64(r), ptrs, _d(z))
    return z


def mttkrp(tensor, factors, k, threads=1) -> np.ndarray:
    """tensor.hpp:174-182 (unfold copy + materialised Khatri-Rao + GEMM)."""
    t = np.asfortranarray(tensor, dtype=np.float64)
    shape = np.ascontiguousarray(t.shape, dtype=np.int64)
    d = shape.size
    for i in range(d):
        if i != k and np.asarray(factors[i]).shape[0] != shape[i]:
            raise InvalidArgument("mttkrp: shape mismatch")
    r = next(np.asarray(f).shape[1] for i, f in enumerate(factors) if i != k)
    arrs, ptrs = _factor_ptrs(factors, k)
    b = np.zeros((shape[k], r), order="F")
    _check(lib().orc_mttkrp(d, shape.ctypes.data_as(_lp), _d(t), k, _i64(r), ptrs, _d(b), threads))
    return b


def gram_khatri_rao(factors, k) -> np.ndarray:
    """tensor.hpp:186-194."""
    shape = np.ascontiguousarray([np.asarray(f).shape[0] for f in factors], dtype=np.int64)
    r = np.asarray(factors[0 if k != 0 else 1]).shape[1]
    arrs, ptrs = _factor_ptrs(factors, -1)
    v = np.zeros((r, r), order="F")
    lib().orc_gram_khatri_rao(shape.size, shape.ctypes.data_as(_lp), _i64(r), ptrs, k, _d(v))
    return v


# ---- unaligned.hpp ---------------------------------------------------------------------
@dataclass
class UnalignedSubproblem:
    """unaligned.hpp:18-33 (+ the flat index arrays of the ObservationSet it points at)."""
    shape: np.ndarray
    k: int
    idx: np.ndarray       # (d, q) int32
    values: np.ndarray    # (q,)
    factors: list
    kernel: np.ndarray    # n x n
    lam: float
    rho: float
    zhat: np.ndarray
    b: np.ndarray
    v: np.ndarray

    @property
    def n(self):
        return self.kernel.shape[0]

    @property
    def r(self):
        return self.zhat.shape[1]

    @property
    def q(self):
        return self.idx.shape[1]

    @property
    def density(self):
        # observations.hpp:58-60: q / prod(shape) over ALL modes including k
        return float(self.q) / float(np.prod(self.shape.astype(np.float64)))


def make_unaligned_subproblem(shape, idx, values, factors, k, kernel, lam, rho):
    """unaligned.hpp:35-48."""
    shape = np.ascontiguousarray(shape, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    zhat = build_zhat(shape, k, idx, factors)
    b = sampled_mttkrp(shape[k], zhat, idx[k], values)
    v = gram_khatri_rao(factors, k)
    return UnalignedSubproblem(shape, k, idx, np.ascontiguousarray(values, dtype=np.float64),
                               list(factors), _f64(kernel), float(lam), float(rho), zhat, b, v)


def unaligned_matvec(p: UnalignedSubproblem, x, threads=1) -> np.ndarray:
    """unaligned.hpp:101-115 (reference-faithful)."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    if x.size != p.n * p.r:
        raise InvalidArgument("unaligned_matvec: size mismatch")
    y = np.zeros(p.n * p.r)
    idx_k = np.ascontiguousarray(p.idx[p.k])
    _check(lib().orc_unaligned_matvec(_i64(p.n), _i64(p.r), _d(p.kernel), ctypes.c_double(p.lam),
                                      ctypes.c_double(p.rho), _i64(p.q), _d(p.zhat),
                                      idx_k.ctypes.data_as(_ip), _d(x), _d(y), threads))
    return y


def scatter_gather_stream(shape, k, idx, factors, xhat, threads=None) -> np.ndarray:
    """Fused streaming Yhat = sampled_mttkrp(gather_rows(Xhat)) (multiset semantics)."""
    shape = np.ascontiguousarray(shape, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    d, q = idx.shape
    xhat = _f64(xhat)
    n, r = xhat.shape
    arrs, ptrs = _factor_ptrs(factors, k)
    y = np.zeros((n, r), order="F")
    _check(lib().orc_scatter_gather_stream(d, shape.ctypes.data_as(_lp), k, _i64(q),
                                           idx.ctypes.data_as(_ip), _i64(r), ptrs, _i64(n),
                                           _d(xhat), _d(y), threads or max_threads()))
    return y


def sampled_mttkrp_stream(shape, k, idx, values, factors, n, threads=None) -> np.ndarray:
    shape = np.ascontiguousarray(shape, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    vals = np.ascontiguousarray(values, dtype=np.float64)
    d, q = idx.shape
    r = next(np.asarray(f).shape[1] for i, f in enumerate(factors) if i != k)
    arrs, ptrs = _factor_ptrs(factors, k)
    b = np.zeros((n, r), order="F")
    _check(lib().orc_sampled_mttkrp_stream(d, shape.ctypes.data_as(_lp), k, _i64(q),
                                           idx.ctypes.data_as(_ip), _d(vals), _i64(r), ptrs,
                                           _i64(n), _d(b), threads or max_threads()))
    return b


def unaligned_matvec_stream(shape, k, idx, factors, kernel, lam, rho, x, threads=None):
    shape = np.ascontiguousarray(shape, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    d, q = idx.shape
    kern = _f64(kernel)
    n = kern.shape[0]
    r = next(np.asarray(f).shape[1] for i, f in enumerate(factors) if i != k)
    arrs, ptrs = _factor_ptrs(factors, k)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.zeros(n * r)
    _check(lib().orc_unaligned_matvec_stream(d, shape.ctypes.data_as(_lp), k, _i64(q),
                                             idx.ctypes.data_as(_ip), _i64(r), ptrs, _i64(n),
                                             _d(kern), ctypes.c_double(lam), ctypes.c_double(rho),
                                             _d(x), _d(y), threads or max_threads()))
    return y


def build_F(p: UnalignedSubproblem, dense_cap=6000) -> np.ndarray:
    """unaligned.hpp:52-62: F = S'(Z kron K), row l = zhat(l,:) kron khat(l,:) (khat: observations.hpp:161-169)."""
    if p.n * p.r > dense_cap:
        raise InvalidArgument("build_F: rn exceeds memory cap")
    khat = p.kernel[p.idx[p.k], :]
    f = np.zeros((p.q, p.r * p.n))
    for j in range(p.r):
        f[:, j * p.n:(j + 1) * p.n] = p.zhat[:, j:j + 1] * khat
    return f


def build_G(p: UnalignedSubproblem, dense_cap=6000) -> np.ndarray:
    """unaligned.hpp:65-75: G = S'(Z kron I), row l = zhat(l,:) kron e_{i_k(l)}'."""
    if p.n * p.r > dense_cap:
        raise InvalidArgument("build_G: rn exceeds memory cap")
    g = np.zeros((p.q, p.r * p.n))
    rows = np.arange(p.q)
    for j in range(p.r):
        g[rows, j * p.n + p.idx[p.k]] = p.zhat[:, j]
    return g


def lu_solve(a, b) -> np.ndarray:
    """solvers.hpp:99-106: partial-pivot LU (LAPACK getrf / getrs via numpy), then the residual check."""
    try:
        x = np.linalg.solve(a, b)
    except np.linalg.LinAlgError:
        raise RuntimeFailure("lu_solve: matrix is singular or severely ill-conditioned")
    res = float(np.linalg.norm(a @ x - b))
    if not np.isfinite(res) or res > 1e-6 * max(float(np.linalg.norm(b)), 1.0):
        raise RuntimeFailure("lu_solve: matrix is singular or severely ill-conditioned")
    return x


def solve_unaligned_direct_nonsym(p: UnalignedSubproblem, report: SolveReport | None = None, dense_cap=6000):
    """unaligned.hpp:77-96: LU solve of (G'F + lambda I) vec(W) = vec(B)."""
    import time
    t0 = time.perf_counter()
    sys_ = build_G(p, dense_cap).T @ build_F(p, dense_cap)
    sys_[np.diag_indices_from(sys_)] += p.lam
    rhs = p.b.reshape(-1, order="F")
    w = lu_solve(sys_, rhs)
    if report is not None:
        bn = float(np.linalg.norm(rhs))
        report.iterations = 1
        report.relative_residual = 0.0 if bn == 0.0 else float(np.linalg.norm(sys_ @ w - rhs)) / bn
        report.converged = True
        report.wall_time_s = time.perf_counter() - t0
    return w.reshape((p.n, p.r), order="F")


def assemble_unaligned_sym_dense(p: UnalignedSubproblem, dense_cap=6000):
    """unaligned.hpp:164-174: (F'F + lambda (I kron K) + rho I, vec(K B))."""
    if p.n * p.r > dense_cap:
        raise InvalidArgument("assemble_unaligned_sym_dense: rn exceeds memory cap")
    f = build_F(p, dense_cap)
    sys_ = f.T @ f + p.lam * np.kron(np.eye(p.r), p.kernel)
    sys_[np.diag_indices_from(sys_)] += p.rho
    return sys_, (p.kernel @ p.b).reshape(-1, order="F")


@dataclass
class Preconditioner:
    """build_preconditioner (unaligned.hpp:120-140) given eig(K) and eig(V)."""
    uk: np.ndarray
    uv: np.ndarray
    dmat: np.ndarray

    def apply(self, x, threads=1) -> np.ndarray:
        n, r = self.dmat.shape
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        y = np.zeros(n * r)
        _check(lib().orc_precond_apply(_i64(n), _i64(r), _d(self.uk), _d(self.uv), _d(self.dmat),
                                       _d(x), _d(y), threads))
        return y


def build_preconditioner(p: UnalignedSubproblem, ek: SymEig, ev: SymEig | None = None):
    ev = ev if ev is not None else sym_eig(p.v)
    dmat = np.zeros((p.n, p.r), order="F")
    muk = np.ascontiguousarray(ek.d); sv = np.ascontiguousarray(ev.d)
    _check(lib().orc_precond_diag(_i64(p.n), _i64(p.r), _d(muk), _d(sv),
                                  ctypes.c_double(p.density), ctypes.c_double(p.lam),
                                  ctypes.c_double(p.rho), _d(dmat)))
    return Preconditioner(_f64(ek.u), _f64(ev.u), dmat)


# ---- solvers.hpp -----------------------------------------------------------------------
@dataclass
class PcgConfig:
    tol: float = 1e-6
    max_iter: int = 75
    record_history: bool = False


@dataclass
class SolveReport:
    iterations: int = 0
    relative_residual: float = 0.0
    wall_time_s: float = 0.0
    converged: bool = False
    residual_history: list = field(default_factory=list)


def pcg(apply_a, apply_m, b, cfg: PcgConfig, report: SolveReport | None = None, x0=None):
    """solvers.hpp:38-88, restated line for line."""
    import time
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    if cfg.tol <= 0.0 or cfg.max_iter < 1:
        raise InvalidArgument("pcg: invalid config")
    t0 = time.perf_counter()
    bnorm = float(np.linalg.norm(b))
    rep = SolveReport()
    x = np.array(x0, dtype=np.float64).reshape(-1) if x0 is not None else np.zeros_like(b)
    if bnorm == 0.0:
        x[:] = 0.0
        rep.converged = True
        if report is not None:
            report.__dict__.update(rep.__dict__)
        return x
    r = (b - apply_a(x)) if x0 is not None else b.copy()
    z = apply_m(r)
    p = z.copy()
    rz = float(r @ z)
    rel = float(np.linalg.norm(r)) / bnorm
    if cfg.record_history:
        rep.residual_history.append(rel)
    it = 0
    while rel > cfg.tol and it < cfg.max_iter:
        ap = apply_a(p)
        pap = float(p @ ap)
        if not np.isfinite(pap):
            raise RuntimeFailure("pcg: non-finite value encountered")
        if pap <= 0.0:
            raise RuntimeFailure("pcg: operator not positive definite (p'Ap <= 0)")
        alpha = rz / pap
        x += alpha * p
        r -= alpha * ap
        it += 1
        rel = float(np.linalg.norm(r)) / bnorm
        if cfg.record_history:
            rep.residual_history.append(rel)
        if rel <= cfg.tol:
            break
        z = apply_m(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    rep.iterations = it
    rep.relative_residual = rel
    rep.converged = rel <= cfg.tol
    rep.wall_time_s = time.perf_counter() - t0
    if report is not None:
        report.__dict__.update(rep.__dict__)
    return x


def solve_unaligned_pcg(p: UnalignedSubproblem, cfg: PcgConfig, ek: SymEig, ev: SymEig | None = None,
                        report: SolveReport | None = None, warm_start=None, threads=1):
    """unaligned.hpp:143-161."""
    if p.rho <= 0.0:
        raise InvalidArgument("solve_unaligned_pcg: rho must be positive")
    kb = gemm(p.kernel, p.b, threads=threads)
    rhs = kb.reshape(-1, order="F")
    m_inv = build_preconditioner(p, ek, ev)
    x0 = None if warm_start is None else np.asarray(warm_start, dtype=np.float64).reshape(-1, order="F")
    w = pcg(lambda v: unaligned_matvec(p, v, threads), lambda v: m_inv.apply(v, threads), rhs, cfg,
            report, x0)
    return w.reshape((p.n, p.r), order="F")


# ---- aligned.hpp -----------------------------------------------------------------------
def solve_aligned_decoupled(b, ek: SymEig, ev: SymEig, lam, threads=1) -> np.ndarray:
    """aligned.hpp:41-54 with a given eig(K), eig(V)."""
    b = _f64(b)
    n, r = b.shape
    w = np.zeros((n, r), order="F")
    _check(lib().orc_solve_aligned_decoupled(_i64(n), _i64(r), _d(_f64(ek.u)), _d(np.ascontiguousarray(ek.d)),
                                             _d(_f64(ev.u)), _d(np.ascontiguousarray(ev.d)),
                                             ctypes.c_double(lam), _d(b), _d(w), threads))
    return w


def aligned_matvec(x, dk, v, lam) -> np.ndarray:
    """aligned.hpp:58-67: vec(diag(d_K) (X V) + lambda X) with X = reshape(x, n, r) (column-major)."""
    dk = np.asarray(dk, dtype=np.float64).reshape(-1)
    v = np.asarray(v, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    n, r = dk.size, v.shape[0]
    if x.size != n * r:
        raise InvalidArgument("aligned_matvec: size mismatch")
    xm = x.reshape((n, r), order="F")
    return (dk[:, None] * (xm @ v) + lam * xm).reshape(-1, order="F")


def solve_aligned_pcg(b, ek: SymEig, v, lam, cfg: PcgConfig, report: SolveReport | None = None,
                      warm_start=None) -> np.ndarray:
    """aligned.hpp:72-100: PCG on (V kron D_K + lambda I) vec(Wbar) = vec(U_K' B), diagonal
    preconditioner 1 / (V(j,j) d_K(i) + lambda) (:83-89), warm start rotated (:92-96), W = U_K Wbar."""
    b = np.asarray(b, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n, r = b.shape
    bbar = (ek.u.T @ b).reshape(-1, order="F")
    dinv = (1.0 / (np.diag(v)[None, :] * ek.d[:, None] + lam)).reshape(-1, order="F")
    x0 = None
    if warm_start is not None:
        x0 = (ek.u.T @ np.asarray(warm_start, dtype=np.float64)).reshape(-1, order="F")
    wbar = pcg(lambda x: aligned_matvec(x, ek.d, v, lam), lambda x: dinv * x, bbar, cfg, report, x0)
    return ek.u @ wbar.reshape((n, r), order="F")


def solve_aligned_direct(b, kernel, v, lam, direct_cap=6000) -> np.ndarray:
    """aligned.hpp:28-37: (V kron K + lambda I) vec(W) = vec(B) by Cholesky (solvers.hpp:91-96)."""
    b = np.asarray(b, dtype=np.float64)
    n, r = b.shape
    if n * r > direct_cap:
        raise InvalidArgument("solve_aligned_direct: rn exceeds memory cap")
    sys_ = np.kron(np.asarray(v, dtype=np.float64), np.asarray(kernel, dtype=np.float64))
    sys_[np.diag_indices_from(sys_)] += lam
    try:
        c = np.linalg.cholesky(sys_)
    except np.linalg.LinAlgError:
        raise RuntimeFailure("cholesky_solve: matrix is not positive definite")
    w = np.linalg.solve(c.T, np.linalg.solve(c, b.reshape(-1, order="F")))
    return w.reshape((n, r), order="F")


def aligned_residual_dense(b, kernel, v, lam, w) -> float:
    """aligned.hpp:104-108: ||K W V + lambda W - B|| / ||B||."""
    b = np.asarray(b, dtype=np.float64)
    res = kernel @ w @ v + lam * w - b
    bn = float(np.linalg.norm(b))
    return float(np.linalg.norm(res)) / bn if bn != 0.0 else float(np.linalg.norm(res))
