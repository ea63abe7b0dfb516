"""The C-ABI library loads on a CPU-only host and exports every symbol include/*.h declares
(no compute calls: those need a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cphifi_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cphifi_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(built_lib):
    lib = ctypes.CDLL(built_lib)
    names = declared_functions()
    assert len(names) >= 45
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header(built_lib):
    from paper_2603_25691_b200 import _capi
    assert set(declared_functions()) == set(_capi.EXPORTED)
    assert _capi.load().cphifi_abi_version() == 1


def test_no_gpu_fails_loudly(built_lib):
    """Without a GPU the context cannot be created: a CUDA error, never a CPU fallback."""
    import torch
    if torch.cuda.is_available():
        return
    from paper_2603_25691_b200 import _capi
    h = ctypes.c_void_p()
    rc = _capi.load().cphifi_ctx_create(0, ctypes.byref(h))
    assert rc == _capi.CUDA_ERROR
    assert _capi.load().cphifi_last_error()


def test_sm100a_code_present(built_lib):
    """The fat binary carries sm_100a SASS with FP64 tensor-core (DMMA) instructions."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", built_lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", built_lib], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    gemm = [f for f in funcs if "gemm_dmma_kernel" in f.split("\n", 1)[0]]
    assert gemm and all("DMMA" in f for f in gemm)
    mtt = [f for f in funcs if "mttkrp_dmma_kernel" in f.split("\n", 1)[0]]
    assert mtt and all("DMMA" in f for f in mtt)
