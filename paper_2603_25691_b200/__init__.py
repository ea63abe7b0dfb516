"""paper_2603_25691_b200 — B200-native CP-HIFI infinite-mode subproblem solver.

Python mirror of the reference's C++ interface for the hot path (names, argument meaning and
exception classes follow proj/include/cphifi/*.hpp).  Every compute call
goes through the C-ABI of ``libcphifi_b200.so`` (include/cphifi_b200.h) to hand-written
sm_100a kernels; there is no CPU fallback.

Reference object                        -> here
  RkhsMode (kernel.hpp:53-101)          -> RkhsMode (device kernel + cached device eig)
  ObservationSet (observations.hpp:18)  -> ObservationSet (host arrays; device plans per k)
  KruskalModel / DenseTensor            -> KruskalModel / DenseTensor (numpy, column-major)
  make_unaligned_subproblem (unaligned.hpp:35-48), unaligned_matvec (:101-115),
  build_preconditioner (:120-140), solve_unaligned_pcg (:143-161)
  mttkrp / gram_khatri_rao (tensor.hpp:174-194), solve_aligned_decoupled (aligned.hpp:41-54)
  PcgConfig / SolveReport (solvers.hpp:23-35)
std::invalid_argument -> CphifiInvalidArgument (a ValueError); std::runtime_error ->
CphifiRuntimeError (a RuntimeError).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import (CphifiDeviceError, CphifiInvalidArgument, CphifiRuntimeError, c_double_p, c_int64_p,
                    call)

__all__ = [
    "Context", "VirtualComm", "default_context", "RkhsMode", "SymEig", "ObservationSet", "DenseTensor", "KruskalModel",
    "sample_uniform", "full_observations", "make_unaligned_subproblem", "UnalignedSubproblem",
    "unaligned_matvec", "build_preconditioner", "LinearOperator", "solve_unaligned_pcg", "PcgConfig",
    "AlsUpdate", "update_infinite_mode_unaligned", "update_infinite_mode_aligned",
    "read_observations", "write_observations", "update_finite_mode_unaligned", "unaligned_relative_error",
    "UnalignedAlsState", "FitIteration", "AlignedAlsState", "update_finite_mode_aligned",
    "SolveReport", "mttkrp", "gram_khatri_rao", "AlignedSubproblem", "solve_aligned_decoupled",
    "aligned_matvec", "solve_aligned_pcg", "solve_aligned_direct", "solve_unaligned_direct_nonsym",
    "assemble_unaligned_sym_dense",
    "aligned_solve", "Mt19937_64", "synth_observations_device", "CphifiInvalidArgument", "CphifiRuntimeError", "CphifiDeviceError",
]


def _dp(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ---- context ---------------------------------------------------------------------------
class Context:
    """One GPU (and optionally an NCCL communicator) — owns the CUDA stream."""

    def __init__(self, device: int | None = None):
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", os.environ.get("CPHIFI_DEVICE", "0")))
        h = ctypes.c_void_p()
        call("cphifi_ctx_create", device, ctypes.byref(h))
        self.handle = h
        self.device = device

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        call("cphifi_comm_unique_id", buf)
        return buf.raw

    def init_comm(self, nranks: int, rank: int, uid: bytes) -> None:
        call("cphifi_ctx_init_comm", self.handle, nranks, rank, uid)

    def init_vcomm(self, vc: "VirtualComm", rank: int) -> None:
        """Join a one-GPU virtual communicator as `rank` (test hook for the multi-rank paths)."""
        call("cphifi_ctx_init_vcomm", self.handle, vc.handle, rank)
        self._vc = vc  # the communicator outlives its contexts

    def world(self):
        n, r = ctypes.c_int(), ctypes.c_int()
        call("cphifi_ctx_world", self.handle, ctypes.byref(n), ctypes.byref(r))
        return n.value, r.value

    def stream(self) -> int:
        s = ctypes.c_void_p()
        call("cphifi_ctx_stream", self.handle, ctypes.byref(s))
        return s.value or 0

    def synchronize(self) -> None:
        call("cphifi_ctx_synchronize", self.handle)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _capi.load().cphifi_ctx_destroy(self.handle)
            self.handle = None


class VirtualComm:
    """cphifi_vcomm: `nranks` contexts on ONE GPU, each driven by its own host thread, standing in
    for NCCL ranks (collectives = rank-order sums); every multi-rank code path runs without a
    second GPU.  Test hook, see include/cphifi_b200.h."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        call("cphifi_vcomm_create", nranks, ctypes.byref(h))
        self.handle = h
        self.nranks = nranks

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                _capi.load().cphifi_vcomm_destroy(self.handle)
            except AttributeError:  # interpreter shutdown: module globals already cleared
                pass
            self.handle = None


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


# ---- RNG (std::mt19937_64 + libstdc++ distributions; test/bench inputs) -------------------
# The seeded input generators live in the separate `inputs` library (inputs/synth_host.cpp), so
# that bench.py's reference arm and the oracle never load this package's library.
from inputs import Mt19937_64  # noqa: E402  (re-exported: the reference tests' RNG)
from inputs import sample_uniform_linear as _sample_uniform_linear  # noqa: E402


# ---- kernel.hpp ------------------------------------------------------------------------
@dataclass
class SymEig:
    u: np.ndarray
    d: np.ndarray


class RkhsMode:
    """RkhsMode(points, sigma, lambda) (kernel.hpp:53-101) with the kernel and its one-time
    eigendecomposition resident on the GPU."""

    def __init__(self, design_points, sigma: float, lambda_: float, ctx: Context | None = None,
                 kernel: str = "gaussian", kernel_matrix=None):
        self.ctx = ctx or default_context()
        pts = np.ascontiguousarray(design_points, dtype=np.float64).reshape(-1)
        self._points = pts
        self._sigma = float(sigma)
        self._lambda = float(lambda_)
        h = ctypes.c_void_p()
        if kernel_matrix is not None:
            km = _f64(kernel_matrix)
            call("cphifi_mode_create", self.ctx.handle, km.shape[0], _dp(km), self._lambda, ctypes.byref(h))
        elif kernel == "gaussian":
            call("cphifi_mode_create_gaussian", self.ctx.handle, pts.size, _dp(pts), self._sigma, self._lambda,
                 ctypes.byref(h))
        elif kernel == "matern32":
            call("cphifi_mode_create_matern32", self.ctx.handle, pts.size, _dp(pts), self._sigma, self._lambda,
                 ctypes.byref(h))
        else:
            raise CphifiInvalidArgument(f"RkhsMode: unknown kernel {kernel!r}")
        self.handle = h

    @staticmethod
    def regular_grid(n: int, sigma: float, lambda_: float, ctx: Context | None = None) -> "RkhsMode":
        return RkhsMode(np.arange(1, n + 1, dtype=np.float64), sigma, lambda_, ctx)

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                _capi.load().cphifi_mode_destroy(self.handle)
            except AttributeError:  # interpreter shutdown: module globals already cleared
                pass

    def size(self) -> int:
        n = ctypes.c_int64()
        call("cphifi_mode_size", self.handle, ctypes.byref(n))
        return n.value

    def sigma(self) -> float:
        return self._sigma

    def lambda_(self) -> float:
        return self._lambda

    def points(self) -> np.ndarray:
        return self._points

    def kernel(self) -> np.ndarray:
        n = self.size()
        k = np.zeros((n, n), order="F")
        call("cphifi_mode_get_kernel", self.handle, _dp(k))
        return k

    def eig(self) -> SymEig:
        n = self.size()
        u = np.zeros((n, n), order="F")
        d = np.zeros(n)
        call("cphifi_mode_get_eig", self.handle, _dp(u), _dp(d))
        return SymEig(u, d)

    def set_eig(self, u, d) -> None:
        """Install a shared eigendecomposition."""
        u = _f64(u)
        d = np.ascontiguousarray(d, dtype=np.float64)
        call("cphifi_mode_set_eig", self.handle, _dp(u), _dp(d))

    def eig_factorization_count(self) -> int:
        c = ctypes.c_int()
        call("cphifi_mode_eig_count", self.handle, ctypes.byref(c))
        return c.value


# ---- tensor.hpp ------------------------------------------------------------------------
class DenseTensor:
    """Dense d-way tensor, column-major (tensor.hpp:14-68), host resident."""

    def __init__(self, shape, data=None):
        shape = [int(s) for s in shape]
        if not shape:
            raise CphifiInvalidArgument("DenseTensor: empty shape")
        if any(s <= 0 for s in shape):
            raise CphifiInvalidArgument("DenseTensor: nonpositive mode size")
        n = int(np.prod(shape))
        if data is None:
            flat = np.zeros(n)
        else:
            flat = np.asarray(data, dtype=np.float64).reshape(-1, order="F")
            if flat.size != n:
                raise CphifiInvalidArgument("DenseTensor: data length does not match shape")
        self._shape = shape
        self._data = np.ascontiguousarray(flat)

    @staticmethod
    def from_array(a: np.ndarray) -> "DenseTensor":
        return DenseTensor(a.shape, np.asarray(a).reshape(-1, order="F"))

    def order(self) -> int:
        return len(self._shape)

    def shape(self):
        return list(self._shape)

    def size(self) -> int:
        return self._data.size

    def data(self) -> np.ndarray:
        return self._data

    def array(self) -> np.ndarray:
        return self._data.reshape(self._shape, order="F")


class KruskalModel:
    def __init__(self, factors):
        if not factors:
            raise CphifiInvalidArgument("KruskalModel: no factors")
        self.factors = [_f64(f) for f in factors]
        r = self.rank()
        for a in self.factors:
            if a.shape[1] != r:
                raise CphifiInvalidArgument("KruskalModel: rank mismatch")

    def order(self) -> int:
        return len(self.factors)

    def rank(self) -> int:
        return self.factors[0].shape[1]

    def shape(self):
        return [a.shape[0] for a in self.factors]


def _factor_array(factors, skip: int):
    arrs = [None if (i == skip or f is None) else _f64(f) for i, f in enumerate(factors)]
    ptrs = (c_double_p * len(arrs))(*[(_dp(a) if a is not None else c_double_p()) for a in arrs])
    return arrs, ptrs


# ---- observations.hpp ------------------------------------------------------------------
class ObservationSet:
    """The set Omega (observations.hpp:18-79).  Indices are held host-side as (d, q) int32;
    device plans (lexicographic order, CSR over i_k, sharded) are built per mode on first use.
    With ``multiset=True`` repeated multi-indices are summed instead of rejected;
    ``coalesce=True`` additionally merges them in the plan into one weighted entry (same
    operator, fewer entries streamed per application)."""

    def __init__(self, shape, indices, values, multiset: bool = False, coalesce: bool = False):
        self._shape = [int(s) for s in shape]
        d = len(self._shape)
        vals = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        idx = np.asarray(indices, dtype=np.int64)
        if idx.size == 0:
            idx = np.zeros((d, 0), dtype=np.int64)
        elif idx.ndim == 2 and idx.shape[1] == d and idx.shape[0] == vals.size and not (
                idx.shape[0] == d and idx.shape[1] == vals.size):
            idx = idx.T
        if idx.ndim != 2 or idx.shape[1] != vals.size:
            raise CphifiInvalidArgument("ObservationSet: index/value count mismatch")
        if idx.shape[0] != d:
            raise CphifiInvalidArgument("ObservationSet: index arity mismatch")
        for k in range(d):
            if idx.shape[1] and (idx[k].min() < 0 or idx[k].max() >= self._shape[k]):
                raise CphifiInvalidArgument("ObservationSet: index out of range")
        self._idx = np.ascontiguousarray(idx.astype(np.int32))
        self._values = vals
        self.multiset = multiset
        self.coalesce = bool(coalesce and multiset)
        self.equal_count_shards = False  # shards > 1: equal counts of observations instead of balanced cost
        self.shard_by_entries = False    # shards > 1: balance plan entries (row-Gram build) instead of q-pass time
        self._plans = {}
        if not multiset and vals.size > 1:
            strides = np.cumprod([1] + self._shape[:-1]).astype(np.int64)
            lin = (self._idx.astype(np.int64) * strides[:, None]).sum(axis=0)
            if np.unique(lin).size != lin.size:
                raise CphifiInvalidArgument("ObservationSet: duplicate index")

    def shape(self):
        return list(self._shape)

    def num_obs(self) -> int:
        return self._values.size

    def num_entries(self) -> int:
        return int(np.prod(self._shape))

    def density(self) -> float:
        return float(self.num_obs()) / float(self.num_entries())

    def aligned(self) -> bool:
        return self.num_obs() == self.num_entries()

    def values(self) -> np.ndarray:
        return self._values

    def index_array(self) -> np.ndarray:
        return self._idx

    def index(self, l: int, k: int) -> int:
        return int(self._idx[k, l])

    def plan(self, k: int, ctx: Context, shard: int = 0, shards: int = 1):
        key = (k, id(ctx), shard, shards, self.equal_count_shards, self.shard_by_entries)
        if key not in self._plans:
            h = ctypes.c_void_p()
            shape = np.ascontiguousarray(self._shape, dtype=np.int64)
            flags = (_capi.OBS_COALESCE_DUPLICATES if self.coalesce else 0) if self.multiset \
                else _capi.OBS_REJECT_DUPLICATES
            if self.equal_count_shards:
                flags |= _capi.OBS_SHARD_EQUAL_COUNT
            if self.shard_by_entries:
                flags |= _capi.OBS_SHARD_BY_ENTRIES
            call("cphifi_obs_create", ctx.handle, len(self._shape), shape.ctypes.data_as(c_int64_p),
                 self.num_obs(), self._idx.ctypes.data, self._values.ctypes.data, k, flags, shard, shards,
                 ctypes.byref(h))
            self._plans[key] = _Handle(h, "cphifi_obs_destroy", deps=(ctx,))
        return self._plans[key]


class DeviceObservations:
    """Observations already resident on the GPU (d x q int32 indices, q fp64 values, e.g. torch
    tensors or raw device pointers): multiset semantics, no host copy.  Plans are built per
    (k, shard) exactly like ObservationSet.plan."""

    def __init__(self, shape, idx_ptr: int, vals_ptr: int, q: int, keepalive=(), coalesce: bool = False):
        self._shape = [int(s) for s in shape]
        self.coalesce = bool(coalesce)
        self._idx_ptr = int(idx_ptr)
        self._vals_ptr = int(vals_ptr)
        self._q = int(q)
        self._keep = tuple(keepalive)
        self._plans = {}
        self.multiset = True
        self.equal_count_shards = False
        self.shard_by_entries = False

    def shape(self):
        return list(self._shape)

    def num_obs(self) -> int:
        return self._q

    def num_entries(self) -> int:
        return int(np.prod(self._shape))

    def density(self) -> float:
        return float(self._q) / float(np.prod(np.asarray(self._shape, dtype=np.float64)))

    def plan(self, k: int, ctx: "Context", shard: int = 0, shards: int = 1):
        key = (k, id(ctx), shard, shards, self.equal_count_shards, self.shard_by_entries)
        if key not in self._plans:
            h = ctypes.c_void_p()
            shape = np.ascontiguousarray(self._shape, dtype=np.int64)
            call("cphifi_obs_create", ctx.handle, len(self._shape), shape.ctypes.data_as(c_int64_p), self._q,
                 ctypes.c_void_p(self._idx_ptr), ctypes.c_void_p(self._vals_ptr), k,
                 _capi.OBS_DEVICE_INPUT | (_capi.OBS_COALESCE_DUPLICATES if self.coalesce else 0)
                 | (_capi.OBS_SHARD_EQUAL_COUNT if self.equal_count_shards else 0)
                 | (_capi.OBS_SHARD_BY_ENTRIES if self.shard_by_entries else 0),
                 shard, shards, ctypes.byref(h))
            self._plans[key] = _Handle(h, "cphifi_obs_destroy", deps=(ctx,))
        return self._plans[key]

    def release_inputs(self):
        """Drop the references to the raw input buffers (plans own sorted copies)."""
        self._keep = ()


class _Handle:
    """Owns one C-ABI handle.  `deps` keeps the handles it points into (observation plan,
    mode, context) alive until after this one is destroyed."""

    def __init__(self, h, destroy, deps=()):
        self.h = h
        self.destroy = destroy
        self.deps = tuple(deps)

    def __del__(self):
        if self.h:
            try:
                getattr(_capi.load(), self.destroy)(self.h)
            except AttributeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None


def sample_uniform(source: DenseTensor, q: int, seed: int, multiset: bool = False) -> ObservationSet:
    """observations.hpp:90-121: q distinct entries drawn by partial Fisher-Yates."""
    n_total = source.size()
    if q > n_total:
        raise CphifiInvalidArgument("sample_uniform: q exceeds tensor size")
    picked = _sample_uniform_linear(n_total, q, seed)
    shape = source.shape()
    idx = np.zeros((len(shape), q), dtype=np.int64)
    lin = picked.copy()
    for k, s in enumerate(shape):
        idx[k] = lin % s
        lin //= s
    return ObservationSet(shape, idx, source.data()[picked], multiset=multiset)


def full_observations(t: DenseTensor) -> ObservationSet:
    """observations.hpp:124-138: every entry in storage order."""
    shape = t.shape()
    lin = np.arange(t.size(), dtype=np.int64)
    idx = np.zeros((len(shape), t.size()), dtype=np.int64)
    for k, s in enumerate(shape):
        idx[k] = lin % s
        lin //= s
    return ObservationSet(shape, idx, t.data().copy())


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
    setup_s: float = 0.0
    matvecs: int = 0


@dataclass
class LinearOperator:
    dim: int
    apply: object


# ---- unaligned.hpp ---------------------------------------------------------------------
class UnalignedSubproblem:
    """unaligned.hpp:18-33 — a device plan: sorted observations, packed factors, B, V."""

    def __init__(self, obs: ObservationSet, model: KruskalModel, k: int, mode: RkhsMode, rho: float,
                 shard: int = 0, shards: int = 1, ctx: Context | None = None):
        self.obs = obs
        self.mode = mode
        self.mode_index = k
        self.rho = float(rho)
        for i in range(model.order()):
            if i != k and model.factors[i].shape[0] != obs.shape()[i]:
                raise CphifiInvalidArgument("build_zhat: shape mismatch")
        self._r = model.rank()
        # mode None: a finite-mode subproblem (B, V, row Grams; no operator) for the row updates
        self._n = mode.size() if mode is not None else obs.shape()[k]
        ctx = mode.ctx if mode is not None else (ctx or default_context())
        arrs, ptrs = _factor_array(model.factors, k)
        plan = obs.plan(k, ctx, shard, shards)
        h = ctypes.c_void_p()
        call("cphifi_unaligned_create", plan.h, mode.handle if mode is not None else None, self._r, ptrs, self.rho,
             ctypes.byref(h))
        self._h = _Handle(h, "cphifi_unaligned_destroy", deps=(plan, mode) if mode is not None else (plan,))
        self.handle = h

    def n(self) -> int:
        return self._n

    def r(self) -> int:
        return self._r

    def q(self) -> int:
        return self.obs.num_obs()

    def lambda_(self) -> float:
        return self.mode.lambda_()

    def density(self) -> float:
        return self.obs.density()

    @property
    def b(self) -> np.ndarray:
        out = np.zeros((self._n, self._r), order="F")
        call("cphifi_unaligned_get_b", self.handle, _dp(out))
        return out

    @property
    def v(self) -> np.ndarray:
        out = np.zeros((self._r, self._r), order="F")
        call("cphifi_unaligned_get_v", self.handle, _dp(out))
        return out

    _OPS = {"stream": 0, "gram": 1, "auto": 2}

    def set_operator(self, op: str) -> str:
        """'stream' (reference structure, default), 'gram' (row-Gram form, G built once) or
        'auto'; returns the resolved form."""
        call("cphifi_unaligned_set_operator", self.handle, self._OPS[op])
        return self.operator()

    def operator(self) -> str:
        v = ctypes.c_int()
        call("cphifi_unaligned_get_operator", self.handle, ctypes.byref(v))
        return "gram" if v.value == 1 else "stream"

    def set_v_eig(self, u, d) -> None:
        u = _f64(u)
        d = np.ascontiguousarray(d, dtype=np.float64)
        call("cphifi_unaligned_set_v_eig", self.handle, _dp(u), _dp(d))

    def v_eig(self) -> SymEig:
        u = np.zeros((self._r, self._r), order="F")
        d = np.zeros(self._r)
        call("cphifi_unaligned_get_v_eig", self.handle, _dp(u), _dp(d))
        return SymEig(u, d)

    def qpass_plan(self) -> dict:
        """The stream operator's q-pass plan: run-kernel parts, dense rows (GEMM form), entries
        left to the run kernel, parts run by the cross-run kernel k_xruns.cu (their runs padded to even
        lengths: sparse_entries counts the padding) (cphifi_unaligned_qpass_plan)."""
        v = (ctypes.c_int64 * 8)()
        call("cphifi_unaligned_qpass_plan", self.handle, v, 8)
        return {"parts": v[0], "dense_rows": v[1], "sparse_entries": v[2], "sparse_draws": v[3],
                "dense_n1p": v[4], "dense_n2p": v[5], "xruns_parts": v[6], "sparse_entries_unpadded": v[7]}

    def scatter_gather(self, xhat) -> np.ndarray:
        """Yhat = sampled_mttkrp(gather_rows(Xhat)) (observations.hpp:174-198), fused."""
        xhat = _f64(xhat)
        out = np.zeros((self._n, self._r), order="F")
        call("cphifi_unaligned_scatter_gather", self.handle, _dp(xhat), _dp(out))
        return out


def make_unaligned_subproblem(obs: ObservationSet, model: KruskalModel, k: int, mode: RkhsMode,
                              rho: float, shard: int = 0, shards: int = 1) -> UnalignedSubproblem:
    """unaligned.hpp:35-48."""
    return UnalignedSubproblem(obs, model, k, mode, rho, shard, shards)


def unaligned_matvec(p: UnalignedSubproblem, x) -> np.ndarray:
    """unaligned.hpp:101-115: y = (F'F + lambda (I kron K) + rho I) x."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    if x.size != p.n() * p.r():
        raise CphifiInvalidArgument("unaligned_matvec: size mismatch")
    y = np.zeros_like(x)
    call("cphifi_unaligned_matvec", p.handle, _dp(x), _dp(y))
    return y


def build_preconditioner(p: UnalignedSubproblem) -> LinearOperator:
    """unaligned.hpp:120-140: M^-1 = U_K((U_K' X U_V) .* D)U_V' on device."""
    p.v_eig()  # builds eig(V) and D now, like the reference (throws here on bad D)

    def apply(x):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        y = np.zeros_like(x)
        call("cphifi_unaligned_precond_apply", p.handle, _dp(x), _dp(y))
        return y

    return LinearOperator(p.n() * p.r(), apply)


def solve_unaligned_pcg(p: UnalignedSubproblem, cfg: PcgConfig | None = None, report: SolveReport | None = None,
                        warm_start=None) -> np.ndarray:
    """unaligned.hpp:143-161 / solvers.hpp:38-88, entirely on device."""
    cfg = cfg or PcgConfig()
    n, r = p.n(), p.r()
    ccfg = _capi.PcgConfigC(cfg.tol, int(cfg.max_iter), int(bool(cfg.record_history)))
    cap = int(cfg.max_iter) + 2
    hist = np.zeros(cap)
    rep = _capi.SolveReportC()
    rep.residual_history = _dp(hist)
    rep.history_capacity = cap
    w = np.zeros((n, r), order="F")
    ws = None if warm_start is None else _f64(warm_start)
    call("cphifi_solve_unaligned_pcg", p.handle, ctypes.byref(ccfg), ctypes.byref(rep),
         _dp(ws) if ws is not None else c_double_p(), _dp(w))
    if report is not None:
        report.iterations = rep.iterations
        report.relative_residual = rep.relative_residual
        report.wall_time_s = rep.wall_time_s
        report.converged = bool(rep.converged)
        report.residual_history = list(hist[: rep.history_len]) if cfg.record_history else []
        report.setup_s = rep.setup_s
        report.matvecs = rep.matvecs
    return w


def solve_unaligned_direct_nonsym(p: UnalignedSubproblem, report: SolveReport | None = None,
                                  dense_cap: int = 6000) -> np.ndarray:
    """unaligned.hpp:77-96: LU solve of (G'F + lambda I) vec(W) = vec(B) — the nonsymmetric direct
    baseline, its system assembled on device from the row Grams."""
    n, r = p.n(), p.r()
    w = np.zeros((n, r), order="F")
    rep = _capi.SolveReportC()
    call("cphifi_solve_unaligned_direct_nonsym", p.handle, int(dense_cap), ctypes.byref(rep), _dp(w))
    if report is not None:
        report.iterations = rep.iterations
        report.relative_residual = rep.relative_residual
        report.wall_time_s = rep.wall_time_s
        report.converged = bool(rep.converged)
        report.residual_history = []
    return w


def assemble_unaligned_sym_dense(p: UnalignedSubproblem, dense_cap: int = 6000):
    """unaligned.hpp:164-174 (test oracle): (F'F + lambda (I kron K) + rho I, vec(K B)), assembled on
    device."""
    rn = p.n() * p.r()
    if rn > dense_cap:  # checked before allocating the rn x rn host buffer
        raise CphifiInvalidArgument("assemble_unaligned_sym_dense: rn exceeds memory cap")
    sys_ = np.zeros((rn, rn), order="F")
    rhs = np.zeros(rn)
    call("cphifi_unaligned_assemble_sym_dense", p.handle, int(dense_cap), _dp(sys_), _dp(rhs))
    return sys_, rhs


# ---- aligned path ----------------------------------------------------------------------
class _DeviceTensor:
    def __init__(self, t: DenseTensor, ctx: Context, shard=0, shards=1):
        shape = np.ascontiguousarray(t.shape(), dtype=np.int64)
        h = ctypes.c_void_p()
        call("cphifi_tensor_create", ctx.handle, len(t.shape()), shape.ctypes.data_as(c_int64_p),
             t.data().ctypes.data, 0, shard, shards, ctypes.byref(h))
        self._h = _Handle(h, "cphifi_tensor_destroy", deps=(ctx,))
        self.handle = h


def _device_tensor(t: DenseTensor, ctx: Context, shard=0, shards=1):
    cache = t.__dict__.setdefault("_dev", {})
    key = (id(ctx), shard, shards)
    if key not in cache:
        cache[key] = _DeviceTensor(t, ctx, shard, shards)
    return cache[key]


def mttkrp(t: DenseTensor, model: KruskalModel, k: int, ctx: Context | None = None, shard: int = 0,
           shards: int = 1) -> np.ndarray:
    """tensor.hpp:174-182 on device: k = 0 (the infinite mode) for any order; k = 1, 2 for 3-way
    tensors with even n0 (the finite-mode updates).  shards > 1: this rank holds mode-1 slab
    `shard` and B is all-reduced over the communicator."""
    ctx = ctx or default_context()
    if t.order() != model.order():
        raise CphifiInvalidArgument("mttkrp: order mismatch")
    for i in range(t.order()):
        if i != k and t.shape()[i] != model.factors[i].shape[0]:
            raise CphifiInvalidArgument("mttkrp: shape mismatch")
    dt = _device_tensor(t, ctx, shard, shards)
    arrs, ptrs = _factor_array(model.factors, k)
    b = np.zeros((t.shape()[k], model.rank()), order="F")
    call("cphifi_mttkrp", dt.handle, k, model.rank(), ptrs, _dp(b))
    return b


def gram_khatri_rao(model: KruskalModel, k: int, ctx: Context | None = None) -> np.ndarray:
    """tensor.hpp:186-194."""
    ctx = ctx or default_context()
    shape = np.ascontiguousarray(model.shape(), dtype=np.int64)
    arrs, ptrs = _factor_array(model.factors, k)
    r = model.rank()
    v = np.zeros((r, r), order="F")
    call("cphifi_gram_khatri_rao", ctx.handle, model.order(), shape.ctypes.data_as(c_int64_p), r, ptrs, k, _dp(v))
    return v


@dataclass
class AlignedSubproblem:
    """aligned.hpp:16-25."""
    b: np.ndarray
    v: np.ndarray
    mode: RkhsMode
    direct_cap: int = 6000  # guard on rn for the materialised path (aligned.hpp:20)

    def n(self):
        return self.b.shape[0]

    def r(self):
        return self.b.shape[1]


def solve_aligned_decoupled(p: AlignedSubproblem, v_eig: SymEig | None = None) -> np.ndarray:
    """aligned.hpp:41-54 on device; eig(V) on device unless a shared one is given."""
    b = _f64(p.b)
    v = _f64(p.v)
    n, r = b.shape
    w = np.zeros((n, r), order="F")
    if v_eig is not None:
        uv = _f64(v_eig.u)
        sv = np.ascontiguousarray(v_eig.d, dtype=np.float64)
        call("cphifi_solve_aligned_decoupled", p.mode.handle, r, _dp(b), _dp(v), _dp(uv), _dp(sv), _dp(w))
    else:
        call("cphifi_solve_aligned_decoupled", p.mode.handle, r, _dp(b), _dp(v), c_double_p(), c_double_p(),
             _dp(w))
    return w


def aligned_matvec(x, d_k, v, lam, ctx: Context | None = None) -> np.ndarray:
    """aligned.hpp:58-67 on device: vec(diag(d_k) X V + lambda X), X = reshape(x, n, r)."""
    ctx = ctx or default_context()
    d_k = np.ascontiguousarray(d_k, dtype=np.float64).reshape(-1)
    v = _f64(v)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    n, r = d_k.size, v.shape[0]
    if x.size != n * r:
        raise CphifiInvalidArgument("aligned_matvec: size mismatch")
    y = np.zeros(n * r)
    call("cphifi_aligned_matvec", ctx.handle, n, r, _dp(x), _dp(d_k), _dp(v), float(lam), _dp(y))
    return y


def solve_aligned_pcg(p: AlignedSubproblem, cfg: PcgConfig | None = None, report: SolveReport | None = None,
                      warm_start=None) -> np.ndarray:
    """aligned.hpp:72-100 on device (PCG on the eigen-rotated system, diagonal preconditioner)."""
    cfg = cfg or PcgConfig()
    b = _f64(p.b)
    n, r = b.shape
    ccfg = _capi.PcgConfigC(cfg.tol, int(cfg.max_iter), int(bool(cfg.record_history)))
    cap = int(cfg.max_iter) + 2
    hist = np.zeros(cap)
    rep = _capi.SolveReportC()
    rep.residual_history = _dp(hist)
    rep.history_capacity = cap
    w = np.zeros((n, r), order="F")
    ws = None if warm_start is None else _f64(warm_start)
    call("cphifi_solve_aligned_pcg", p.mode.handle, r, _dp(b), _dp(_f64(p.v)), ctypes.byref(ccfg), ctypes.byref(rep),
         _dp(ws) if ws is not None else c_double_p(), _dp(w))
    if report is not None:
        report.iterations = rep.iterations
        report.relative_residual = rep.relative_residual
        report.wall_time_s = rep.wall_time_s
        report.converged = bool(rep.converged)
        report.residual_history = list(hist[: rep.history_len]) if cfg.record_history else []
        report.matvecs = rep.matvecs
    return w


def solve_aligned_direct(p: AlignedSubproblem) -> np.ndarray:
    """aligned.hpp:28-37 on device: V kron K + lambda I materialised, Cholesky (cuSOLVER)."""
    b = _f64(p.b)
    n, r = b.shape
    w = np.zeros((n, r), order="F")
    call("cphifi_solve_aligned_direct", p.mode.handle, r, _dp(b), _dp(_f64(p.v)), int(p.direct_cap), _dp(w))
    return w


# ---- io.hpp: observation files ----------------------------------------
def read_observations(path: str, multiset: bool = False, coalesce: bool = False) -> ObservationSet:
    """read_observations (io.hpp:110-131): the reference text format (1-based lines, parsed on all
    host threads) or the binary format written by write_observations(..., binary=True)."""
    d = ctypes.c_int()
    shape = (ctypes.c_int64 * 8)()
    q = ctypes.c_int64()
    binary = ctypes.c_int()
    bp = os.fsencode(path)
    call("cphifi_obs_file_info", bp, ctypes.byref(d), shape, ctypes.byref(q), ctypes.byref(binary))
    idx = np.zeros((d.value, q.value), dtype=np.int32)
    vals = np.zeros(q.value, dtype=np.float64)
    call("cphifi_obs_file_read", bp, d.value, q.value, idx.ctypes.data_as(ctypes.c_void_p), _dp(vals))
    return ObservationSet([shape[m] for m in range(d.value)], idx, vals, multiset=multiset, coalesce=coalesce)


def write_observations(path: str, obs: ObservationSet, binary: bool = False) -> None:
    """write_observations (io.hpp:97-107): text, 1-based, 17 significant digits; or the binary
    format (int32 SoA indices + fp64 values after the `shape:` header)."""
    shape = np.ascontiguousarray(obs.shape(), dtype=np.int64)
    idx = np.ascontiguousarray(obs.index_array(), dtype=np.int32)
    vals = np.ascontiguousarray(obs.values(), dtype=np.float64)
    call("cphifi_obs_file_write", os.fsencode(path), int(bool(binary)), len(shape),
         shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), vals.size, idx.ctypes.data_as(ctypes.c_void_p), _dp(vals))


# ---- als.hpp: the infinite-mode update of one ALS sweep -----------------
@dataclass
class AlsUpdate:
    """AlsState::update_infinite_mode (als.hpp:170-218) + relative_error (:221-237) + this mode's
    objective term lambda trace(W'KW) (:243-255), computed in one device pass."""
    w: np.ndarray
    a: np.ndarray                # the updated factor A_k = K W (als.hpp:214)
    relative_error: float
    data_norm: float
    reg: float
    residual: float              # aligned_residual (aligned) / PCG relative residual (unaligned)
    solve_s: float = 0.0
    update_s: float = 0.0
    report: SolveReport | None = None

    def objective_term(self) -> float:
        """(relative_error * data_norm)^2 + lambda trace(W'KW): objective_from_error with only this
        infinite mode (als.hpp:243-255)."""
        fit = self.relative_error * self.data_norm
        return fit * fit + self.reg


def _als_from(c, w, a, report=None) -> AlsUpdate:
    return AlsUpdate(w, a, c.relative_error, c.data_norm, c.reg, c.residual, c.solve_s, c.update_s, report)


def update_infinite_mode_unaligned(p: UnalignedSubproblem, cfg: PcgConfig | None = None,
                                   warm_start=None) -> AlsUpdate:
    """The unaligned branch of update_infinite_mode (PCG, als.hpp:198-210) on device."""
    cfg = cfg or PcgConfig()
    n, r = p.n(), p.r()
    ccfg = _capi.PcgConfigC(cfg.tol, int(cfg.max_iter), int(bool(cfg.record_history)))
    cap = int(cfg.max_iter) + 2
    hist = np.zeros(cap)
    rep = _capi.SolveReportC()
    rep.residual_history = _dp(hist)
    rep.history_capacity = cap
    w = np.zeros((n, r), order="F")
    a = np.zeros((n, r), order="F")
    ws = None if warm_start is None else _f64(warm_start)
    c = _capi.AlsReportC()
    call("cphifi_als_update_infinite_unaligned", p.handle, ctypes.byref(ccfg),
         _dp(ws) if ws is not None else c_double_p(), _dp(w), _dp(a), ctypes.byref(rep), ctypes.byref(c))
    sr = SolveReport(rep.iterations, rep.relative_residual, rep.wall_time_s, bool(rep.converged),
                     list(hist[: rep.history_len]) if cfg.record_history else [], rep.setup_s, rep.matvecs)
    return _als_from(c, w, a, sr)


def update_finite_mode_unaligned(obs: ObservationSet, model: KruskalModel, k: int, ctx: Context | None = None,
                                 shard: int = 0, shards: int = 1) -> np.ndarray:
    """update_finite_mode, unaligned branch (als.hpp:144-162) on device: the minimum-norm least-
    squares row fits of mode k (rows without observations stay zero).  Returns A_k (n_k x r).
    shards > 1: this rank's observation shard; the row Grams and B are summed over the ranks."""
    p = UnalignedSubproblem(obs, model, k, None, 1e-6, shard, shards, ctx=ctx)
    a = np.zeros((p.n(), p.r()), order="F")
    call("cphifi_als_update_finite_unaligned", p.handle, _dp(a))
    return a


def unaligned_relative_error(p: UnalignedSubproblem, a_k) -> tuple[float, float]:
    """relative_error (als.hpp:221-237) with factor k = a_k and the plan's other factors.
    Returns (relative error, ||v||)."""
    rel, nrm = ctypes.c_double(), ctypes.c_double()
    call("cphifi_unaligned_relative_error", p.handle, _dp(_f64(a_k)), ctypes.byref(rel), ctypes.byref(nrm))
    return rel.value, nrm.value


@dataclass
class FitIteration:
    """als.hpp FitIteration: the relative error / objective after a sweep and its wall time."""
    rel_error: float
    objective: float
    wall_time_s: float = 0.0
    pcg_iterations: int = 0


class UnalignedAlsState:
    """AlsState (als.hpp:66-275) for unaligned data with mode 0 the infinite (RKHS) mode and the
    other modes finite, every update on device: update_infinite_mode (PCG warm-started from the
    previous W, A_0 = K W), update_finite_mode (row least squares), relative_error and the
    objective.  Factors stay host-side between calls (the reference's KruskalModel)."""

    def __init__(self, obs: ObservationSet, mode: RkhsMode, model: KruskalModel, rho: float = 1e-6,
                 inner: PcgConfig | None = None, warm_start: bool = True):
        self.obs, self.mode, self.rho = obs, mode, float(rho)
        self.model = KruskalModel([np.array(f, order="F", dtype=np.float64) for f in model.factors])
        self.inner = inner or PcgConfig()
        self.warm_start = warm_start
        self.weights = None  # W of mode 0 (als.hpp weights_[0])

    def update_infinite_mode(self) -> AlsUpdate:
        p = make_unaligned_subproblem(self.obs, self.model, 0, self.mode, self.rho)
        u = update_infinite_mode_unaligned(p, self.inner, self.weights if self.warm_start else None)
        self.weights = u.w
        self.model.factors[0] = u.a
        return u

    def update_finite_mode(self, k: int) -> None:
        self.model.factors[k] = update_finite_mode_unaligned(self.obs, self.model, k)

    def relative_error(self) -> float:
        p = UnalignedSubproblem(self.obs, self.model, 0, None, self.rho)
        return unaligned_relative_error(p, self.model.factors[0])[0]

    def objective_from_error(self, rel: float) -> float:
        """als.hpp:243-255: fit^2 + lambda trace(W'KW) for the infinite mode."""
        nrm = float(np.linalg.norm(self.obs.values()))
        obj = (rel * nrm) ** 2
        if self.weights is not None:
            obj += self.mode.lambda_() * float(np.sum(self.weights * self.model.factors[0]))
        return obj

    def sweep(self) -> FitIteration:
        """One outer iteration of run_cp_hifi (als.hpp:303-314): every mode in order, then the error."""
        import time as _time
        t0 = _time.perf_counter()
        u = self.update_infinite_mode()
        for k in range(1, self.model.order()):
            self.update_finite_mode(k)
        rel = self.relative_error()
        return FitIteration(rel, self.objective_from_error(rel), _time.perf_counter() - t0,
                            u.report.iterations if u.report else 0)


def update_finite_mode_aligned(t: DenseTensor, model: KruskalModel, k: int, ctx: Context | None = None):
    """update_finite_mode, aligned branch (als.hpp:139-143) on device: A_k = B_k V_k^+.  Returns
    (A_k, relative error of the model after the update)."""
    ctx = ctx or default_context()
    dt = _device_tensor(t, ctx)
    arrs, ptrs = _factor_array(model.factors, k)
    a = np.zeros((t.shape()[k], model.rank()), order="F")
    rel = ctypes.c_double()
    call("cphifi_als_update_finite_aligned", dt.handle, k, model.rank(), ptrs, _dp(a), ctypes.byref(rel))
    return a, rel.value


class AlignedAlsState:
    """AlsState (als.hpp:66-275) for aligned (dense) data with mode 0 the infinite (RKHS) mode and the
    other modes finite, every update on device: update_infinite_mode (decoupled solve, A_0 = K W),
    update_finite_mode (A_k = B_k V_k^+), and relative_error from the last update's MTTKRP and Gram
    (no N-sized reconstruction)."""

    def __init__(self, t: DenseTensor, mode: RkhsMode, model: KruskalModel):
        self.t, self.mode = t, mode
        self.model = KruskalModel([np.array(f, order="F", dtype=np.float64) for f in model.factors])
        self.weights = None

    def sweep(self) -> FitIteration:
        import time as _time
        t0 = _time.perf_counter()
        u = update_infinite_mode_aligned(self.t, self.model, 0, self.mode)
        self.weights = u.w
        self.model.factors[0] = u.a
        rel = u.relative_error
        for k in range(1, self.model.order()):
            self.model.factors[k], rel = update_finite_mode_aligned(self.t, self.model, k, self.mode.ctx)
        nrm = u.data_norm
        obj = (rel * nrm) ** 2 + self.mode.lambda_() * float(np.sum(self.weights * self.model.factors[0]))
        return FitIteration(rel, obj, _time.perf_counter() - t0, 0)


def update_infinite_mode_aligned(t: DenseTensor, model: KruskalModel, k: int, mode: RkhsMode) -> AlsUpdate:
    """The aligned decoupled branch of update_infinite_mode (als.hpp:181-197) on device."""
    dt = _device_tensor(t, mode.ctx)
    arrs, ptrs = _factor_array(model.factors, k)
    n, r = mode.size(), model.rank()
    w = np.zeros((n, r), order="F")
    a = np.zeros((n, r), order="F")
    c = _capi.AlsReportC()
    call("cphifi_als_update_infinite_aligned", dt.handle, mode.handle, k, r, ptrs, _dp(w), _dp(a), ctypes.byref(c))
    return _als_from(c, w, a)


def aligned_solve(t: DenseTensor, model: KruskalModel, k: int, mode: RkhsMode):
    """Fused aligned update (MTTKRP + Gram + decoupled solve on device). Returns (W, B, V)."""
    dt = _device_tensor(t, mode.ctx)
    arrs, ptrs = _factor_array(model.factors, k)
    n, r = mode.size(), model.rank()
    w = np.zeros((n, r), order="F")
    b = np.zeros((n, r), order="F")
    v = np.zeros((r, r), order="F")
    call("cphifi_aligned_solve", dt.handle, mode.handle, k, r, ptrs, _dp(w), _dp(b), _dp(v))
    return w, b, v


def synth_observations_device(cfg, ctx: Context, q: int | None = None):
    """Draw cfg's observations (inputs.configs.DeviceUnalignedConfig) on cfg's GPU with the
    counter-based generator (cphifi_synth_observations; bit-identical to inputs.configs.generate_host):
    returns torch tensors idx (d, q) int32 and vals (q,) fp64."""
    import torch
    q = cfg.q if q is None else q
    d = len(cfg.shape)
    dev = torch.device("cuda", ctx.device)
    idx = torch.empty((d, q), dtype=torch.int32, device=dev)
    vals = torch.empty(q, dtype=torch.float64, device=dev)
    shape = np.ascontiguousarray(cfg.shape, dtype=np.int64)
    facs = [np.asfortranarray(f) for f in cfg.factors]
    ptrs = (c_double_p * d)(*[f.ctypes.data_as(c_double_p) for f in facs])
    call("cphifi_synth_observations", ctx.handle, d, shape.ctypes.data_as(c_int64_p), q, ctypes.c_uint64(cfg.seed),
         cfg.zipf_mode, cfg.zipf_s, cfg.r, ptrs, cfg.noise_std, idx.data_ptr(), vals.data_ptr())
    return idx, vals
