"""ctypes binding of libcphifi_b200.so (the C-ABI in include/cphifi_b200.h).

The library is built in-tree (``python -m paper_2603_25691_b200.build``).  There is no
fallback: if the shared library is missing or no GPU is present, compute entry points raise.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcphifi_b200.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_uint64_p = ctypes.POINTER(ctypes.c_uint64)
c_void_pp = ctypes.POINTER(ctypes.c_void_p)

OK, INVALID_ARGUMENT, RUNTIME_ERROR, CUDA_ERROR, NCCL_ERROR = 0, 1, 2, 3, 4
OBS_DEVICE_INPUT = 1
OBS_REJECT_DUPLICATES = 2
OBS_COALESCE_DUPLICATES = 4
OBS_SHARD_EQUAL_COUNT = 8
OBS_SHARD_BY_ENTRIES = 16
TENSOR_DEVICE_INPUT = 1


class PcgConfigC(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int32), ("record_history", ctypes.c_int32)]


class AlsReportC(ctypes.Structure):
    _fields_ = [
        ("relative_error", ctypes.c_double),
        ("data_norm", ctypes.c_double),
        ("reg", ctypes.c_double),
        ("residual", ctypes.c_double),
        ("solve_s", ctypes.c_double),
        ("update_s", ctypes.c_double),
    ]


class SolveReportC(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("relative_residual", ctypes.c_double),
        ("wall_time_s", ctypes.c_double),
        ("residual_history", c_double_p),
        ("history_capacity", ctypes.c_int32),
        ("history_len", ctypes.c_int32),
        ("setup_s", ctypes.c_double),
        ("matvec_s", ctypes.c_double),
        ("precond_s", ctypes.c_double),
        ("matvecs", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
    ]


class CphifiInvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class CphifiRuntimeError(RuntimeError):
    """std::runtime_error in the reference."""


class CphifiDeviceError(RuntimeError):
    """CUDA or NCCL failure."""


# (name, restype, argtypes)
_H = ctypes.c_void_p
_SIGS = [
    ("cphifi_last_error", ctypes.c_char_p, []),
    ("cphifi_abi_version", ctypes.c_int, []),
    ("cphifi_ctx_create", ctypes.c_int, [ctypes.c_int, c_void_pp]),
    ("cphifi_ctx_destroy", ctypes.c_int, [_H]),
    ("cphifi_ctx_synchronize", ctypes.c_int, [_H]),
    ("cphifi_ctx_stream", ctypes.c_int, [_H, c_void_pp]),
    ("cphifi_fp64_peak", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_comm_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("cphifi_ctx_init_comm", ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]),
    ("cphifi_vcomm_create", ctypes.c_int, [ctypes.c_int, c_void_pp]),
    ("cphifi_vcomm_destroy", ctypes.c_int, [_H]),
    ("cphifi_ctx_init_vcomm", ctypes.c_int, [_H, _H, ctypes.c_int]),
    ("cphifi_ctx_world", ctypes.c_int, [_H, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("cphifi_mode_create_gaussian", ctypes.c_int,
     [_H, ctypes.c_int64, c_double_p, ctypes.c_double, ctypes.c_double, c_void_pp]),
    ("cphifi_mode_create_matern32", ctypes.c_int,
     [_H, ctypes.c_int64, c_double_p, ctypes.c_double, ctypes.c_double, c_void_pp]),
    ("cphifi_mode_create", ctypes.c_int, [_H, ctypes.c_int64, c_double_p, ctypes.c_double, c_void_pp]),
    ("cphifi_mode_destroy", ctypes.c_int, [_H]),
    ("cphifi_mode_size", ctypes.c_int, [_H, c_int64_p]),
    ("cphifi_mode_lambda", ctypes.c_int, [_H, c_double_p]),
    ("cphifi_mode_get_kernel", ctypes.c_int, [_H, c_double_p]),
    ("cphifi_mode_eig", ctypes.c_int, [_H]),
    ("cphifi_mode_set_eig", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_mode_get_eig", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_mode_eig_count", ctypes.c_int, [_H, ctypes.POINTER(ctypes.c_int)]),
    ("cphifi_obs_create", ctypes.c_int,
     [_H, ctypes.c_int, c_int64_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
      ctypes.c_uint32, ctypes.c_int, ctypes.c_int, c_void_pp]),
    ("cphifi_obs_destroy", ctypes.c_int, [_H]),
    ("cphifi_obs_info", ctypes.c_int, [_H, c_int64_p, c_int64_p, c_double_p]),
    ("cphifi_obs_shard_rows", ctypes.c_int, [_H, c_int64_p, c_int64_p, c_int64_p]),
    ("cphifi_unaligned_create", ctypes.c_int,
     [_H, _H, ctypes.c_int64, ctypes.POINTER(c_double_p), ctypes.c_double, c_void_pp]),
    ("cphifi_unaligned_destroy", ctypes.c_int, [_H]),
    ("cphifi_unaligned_get_b", ctypes.c_int, [_H, c_double_p]),
    ("cphifi_unaligned_get_v", ctypes.c_int, [_H, c_double_p]),
    ("cphifi_unaligned_set_operator", ctypes.c_int, [_H, ctypes.c_int]),
    ("cphifi_unaligned_get_operator", ctypes.c_int, [_H, ctypes.POINTER(ctypes.c_int)]),
    ("cphifi_unaligned_matvec", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_unaligned_matvec_device", ctypes.c_int, [_H, ctypes.c_void_p, ctypes.c_void_p]),
    ("cphifi_unaligned_set_v_eig", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_unaligned_get_v_eig", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_unaligned_precond_apply", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_unaligned_precond_apply_device", ctypes.c_int, [_H, ctypes.c_void_p, ctypes.c_void_p]),
    ("cphifi_solve_unaligned_pcg", ctypes.c_int,
     [_H, ctypes.POINTER(PcgConfigC), ctypes.POINTER(SolveReportC), c_double_p, c_double_p]),
    ("cphifi_unaligned_qpass_plan", ctypes.c_int, [_H, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    ("cphifi_unaligned_matvec_launches", ctypes.c_int, [_H, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    ("cphifi_unaligned_matvec_timed", ctypes.c_int, [_H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, c_double_p]),
    ("cphifi_unaligned_matvec_cycle_timed", ctypes.c_int,
     [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
      ctypes.c_int, ctypes.POINTER(ctypes.c_float)]),
    ("cphifi_unaligned_matvec_graph_timed", ctypes.c_int,
     [_H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
      ctypes.POINTER(ctypes.c_float)]),
    ("cphifi_unaligned_matvec_trace", ctypes.c_int,
     [_H, ctypes.c_void_p, ctypes.c_void_p, c_uint64_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("cphifi_unaligned_scatter_gather", ctypes.c_int, [_H, c_double_p, c_double_p]),
    ("cphifi_tensor_create", ctypes.c_int,
     [_H, ctypes.c_int, c_int64_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, c_void_pp]),
    ("cphifi_tensor_destroy", ctypes.c_int, [_H]),
    ("cphifi_mttkrp", ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(c_double_p), c_double_p]),
    ("cphifi_gram_khatri_rao", ctypes.c_int,
     [_H, ctypes.c_int, c_int64_p, ctypes.c_int64, ctypes.POINTER(c_double_p), ctypes.c_int, c_double_p]),
    ("cphifi_solve_aligned_decoupled", ctypes.c_int,
     [_H, ctypes.c_int64, c_double_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    ("cphifi_aligned_matvec", ctypes.c_int,
     [_H, ctypes.c_int64, ctypes.c_int64, c_double_p, c_double_p, c_double_p, ctypes.c_double, c_double_p]),
    ("cphifi_solve_aligned_pcg", ctypes.c_int,
     [_H, ctypes.c_int64, c_double_p, c_double_p, ctypes.POINTER(PcgConfigC), ctypes.POINTER(SolveReportC),
      c_double_p, c_double_p]),
    ("cphifi_solve_unaligned_direct_nonsym", ctypes.c_int, [_H, ctypes.c_int64, ctypes.c_void_p, c_double_p]),
    ("cphifi_unaligned_assemble_sym_dense", ctypes.c_int, [_H, ctypes.c_int64, c_double_p, c_double_p]),
    ("cphifi_solve_aligned_direct", ctypes.c_int,
     [_H, ctypes.c_int64, c_double_p, c_double_p, ctypes.c_int64, c_double_p]),
    ("cphifi_aligned_solve", ctypes.c_int,
     [_H, _H, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(c_double_p), c_double_p, c_double_p, c_double_p]),
    ("cphifi_obs_file_info", ctypes.c_int,
     [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
      ctypes.POINTER(ctypes.c_int)]),
    ("cphifi_obs_file_read", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, c_double_p]),
    ("cphifi_obs_file_write", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_void_p,
      c_double_p]),
    ("cphifi_als_update_finite_unaligned", ctypes.c_int, [_H, c_double_p]),
    ("cphifi_als_update_finite_aligned", ctypes.c_int,
     [_H, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(c_double_p), c_double_p, ctypes.POINTER(ctypes.c_double)]),
    ("cphifi_unaligned_relative_error", ctypes.c_int, [_H, c_double_p, c_double_p, c_double_p]),
    ("cphifi_als_update_infinite_unaligned", ctypes.c_int,
     [_H, ctypes.c_void_p, c_double_p, c_double_p, c_double_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("cphifi_als_update_infinite_aligned", ctypes.c_int,
     [_H, _H, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(c_double_p), c_double_p, c_double_p, ctypes.c_void_p]),
    ("cphifi_aligned_solve_timed", ctypes.c_int,
     [_H, _H, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(c_double_p), ctypes.c_int, c_double_p, c_double_p]),
    ("cphifi_synth_observations", ctypes.c_int,
     [_H, ctypes.c_int, c_int64_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
      ctypes.POINTER(c_double_p), ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
]

EXPORTED = [s[0] for s in _SIGS]
_lib = None


def load():
    """Load the in-tree shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2603_25691_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = load().cphifi_last_error().decode()
    if rc == INVALID_ARGUMENT:
        raise CphifiInvalidArgument(msg)
    if rc == RUNTIME_ERROR:
        raise CphifiRuntimeError(msg)
    raise CphifiDeviceError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
