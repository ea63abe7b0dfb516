"""In-tree build of libcphifi_b200.so (sm_100a) — `python -m paper_2603_25691_b200.build`.

Every .cu/.cpp under csrc/ is compiled with nvcc for `-gencode arch=compute_100a,code=sm_100a`
(lineinfo on, so ncu's source page maps to our code) and linked into one shared library next
to this file, together with cuSOLVER (setup eigendecompositions) and NCCL (multi-GPU).
Object files are cached under build/ keyed by source mtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libcphifi_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ccbin", "/usr/bin/g++",
          f"-I{os.path.join(ROOT, 'include')}"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "cphifi_b200.h"))
    hs.append(os.path.join(ROOT, "inputs", "synth_math.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, verbose_ptxas: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _headers_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", path, "-o", obj]
    if src.endswith(".cu") and verbose_ptxas:
        cmd[1:1] = ["-Xptxas", "-v"]
    if src.endswith(".cpp"):
        cmd += ["-x", "c++"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    if verbose_ptxas and res.stderr:
        with open(os.path.join(OBJ, src + ".ptxas.txt"), "w") as f:
            f.write(res.stderr)
    return obj


def _torch_nccl_dir():
    """The NCCL that torch.distributed loads (pip nvidia-nccl).  Linking the same file keeps
    one libnccl.so.2 in the process whichever of torch / this library loads first."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return d
    return None


def build(verbose_ptxas: bool = True, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    if force:
        for s in srcs:
            o = os.path.join(OBJ, s + ".o")
            if os.path.exists(o):
                os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose_ptxas), srcs))
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    nccl_dir = _torch_nccl_dir()
    nccl = ([f"-L{nccl_dir}", "-Xlinker", "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_dir}"]
            if nccl_dir else ["-lnccl"])
    link = [NVCC, *ARCH, "-shared", "-ccbin", "/usr/bin/g++", "-o", LIB, *objs,
            f"-L{CUDA}/lib64", "-lcusolver", *nccl, "-lcudart",
            "-Xlinker", f"-rpath={CUDA}/lib64"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
