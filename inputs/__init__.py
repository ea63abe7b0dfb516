"""Seeded test / benchmark inputs (not the solver, not the oracle).

ctypes front-end over ``inputs/_build/libcphifi_inputs.so`` (``synth_host.cpp``): the
reference's RNG stack (std::mt19937_64 + libstdc++ distributions), sample_uniform's index draw
(observations.hpp:90-121) and the counter-based observation generator of configs 3/4
(``synth_math.h``, bit-identical to the device generator in the product's k_synth.cu).

It is shared by the product tests, the oracle tests, both arms of bench.py and the fixture
scripts; it never loads the product library, so bench.py's reference arm stays product-free.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libcphifi_inputs.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)
_up = ctypes.POINTER(ctypes.c_uint64)
_ip = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("synth_host.cpp", "synth_math.h")]
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(s) for s in srcs):
            build()
        L = ctypes.CDLL(_SO)
        L.inp_rng_create.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        L.inp_rng_destroy.argtypes = [ctypes.c_void_p]
        L.inp_rng_destroy.restype = None
        L.inp_rng_next_u64.argtypes = [ctypes.c_void_p, _up, ctypes.c_int64]
        L.inp_rng_uniform_real.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _dp, ctypes.c_int64]
        L.inp_rng_uniform_int.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, _lp, ctypes.c_int64]
        L.inp_rng_normal.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _dp, ctypes.c_int64]
        L.inp_rng_normal_reset.argtypes = [ctypes.c_void_p]
        L.inp_sample_uniform_linear.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, _lp]
        L.inp_zipf_cdf.argtypes = [ctypes.c_int64, ctypes.c_double, _dp]
        L.inp_zipf_cdf.restype = None
        L.inp_synth_observations.argtypes = [ctypes.c_int, _lp, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                             ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                             ctypes.POINTER(_dp), ctypes.c_double, _ip, _dp, ctypes.c_int]
        L.inp_syn_log.argtypes = [ctypes.c_double]
        L.inp_syn_log.restype = ctypes.c_double
        L.inp_syn_cos2pi.argtypes = [ctypes.c_double]
        L.inp_syn_cos2pi.restype = ctypes.c_double
        _lib = L
    return _lib


def _ok(rc):
    if rc != 0:
        raise ValueError("inputs: invalid argument")


class Mt19937_64:
    """std::mt19937_64 with libstdc++'s distributions (one normal_distribution per engine)."""

    def __init__(self, seed: int):
        h = ctypes.c_void_p()
        _ok(lib().inp_rng_create(ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.inp_rng_destroy(self.h)
            self.h = None

    def __call__(self) -> int:
        return int(self.next_u64(1)[0])

    def next_u64(self, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint64)
        _ok(lib().inp_rng_next_u64(self.h, out.ctypes.data_as(_up), count))
        return out

    def uniform_real(self, lo: float, hi: float, count: int) -> np.ndarray:
        out = np.zeros(count)
        _ok(lib().inp_rng_uniform_real(self.h, lo, hi, out.ctypes.data_as(_dp), count))
        return out

    def uniform_int(self, lo: int, hi: int, count: int = 1) -> np.ndarray:
        out = np.zeros(count, dtype=np.int64)
        _ok(lib().inp_rng_uniform_int(self.h, lo, hi, out.ctypes.data_as(_lp), count))
        return out

    def normal(self, mean: float, std: float, count: int) -> np.ndarray:
        out = np.zeros(count)
        _ok(lib().inp_rng_normal(self.h, mean, std, out.ctypes.data_as(_dp), count))
        return out

    def normal_reset(self) -> None:
        _ok(lib().inp_rng_normal_reset(self.h))

    def random_matrix(self, rows: int, cols: int, lo=-1.0, hi=1.0) -> np.ndarray:
        """test_util.hpp:10-17: column-major fill."""
        return np.asfortranarray(self.uniform_real(lo, hi, rows * cols).reshape((rows, cols), order="F"))


def sample_uniform_linear(n_total: int, q: int, seed: int) -> np.ndarray:
    """observations.hpp:90-107: q distinct linear indices of [0, n_total)."""
    if q > n_total:
        raise ValueError("sample_uniform: q exceeds tensor size")
    picked = np.zeros(max(q, 0), dtype=np.int64)
    _ok(lib().inp_sample_uniform_linear(n_total, q, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
                                        picked.ctypes.data_as(_lp)))
    return picked


def zipf_cdf(n: int, s: float) -> np.ndarray:
    out = np.zeros(n)
    lib().inp_zipf_cdf(n, s, out.ctypes.data_as(_dp))
    return out


def synth_observations(shape, l0: int, l1: int, seed: int, zipf_mode: int, zipf_s: float, factors,
                       noise_std: float, values: bool = True, threads: int | None = None):
    """Draws [l0, l1) of the counter-based generator (synth_math.h): idx (d, l1 - l0) int32 and
    values (l1 - l0,) fp64 (None with values=False)."""
    d = len(shape)
    cnt = int(l1 - l0)
    sh = np.ascontiguousarray(shape, dtype=np.int64)
    idx = np.empty((d, cnt), dtype=np.int32)
    vals = np.empty(cnt) if values else None
    facs = [np.asfortranarray(f, dtype=np.float64) for f in factors]
    r = facs[0].shape[1]
    ptrs = (_dp * d)(*[f.ctypes.data_as(_dp) for f in facs])
    threads = threads or os.cpu_count() or 1
    _ok(lib().inp_synth_observations(d, sh.ctypes.data_as(_lp), int(l0), int(l1),
                                     ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), zipf_mode, zipf_s, r, ptrs,
                                     noise_std, idx.ctypes.data_as(_ip),
                                     vals.ctypes.data_as(_dp) if values else _dp(), threads))
    return idx, vals
