"""Build libinferix_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

    python -m paper_2511_20714_b200._build      # or __graft_entry__.build()
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libinferix_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["attn_fwd_sm100.cu", "gemm_sm100.cu", "attn_few_keys.cu", "kv_ops.cu", "kv_latent.cu", "peer.cu", "comm.cpp", "gemm_lt.cpp", "abi.cpp", "pagetable.cpp", "noise_host.cpp"]


def _npyrandom() -> str:
    """numpy's static distributions library (ziggurat normal), linked for bit-exact noise."""
    import numpy.random
    path = os.path.join(os.path.dirname(numpy.random.__file__), "lib", "libnpyrandom.a")
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing (numpy 2.3 wheel layout expected)")
    return path
FLAGS = ["-O3", "-std=c++17", "-lineinfo", *os.environ.get("IFX_NVCC_EXTRA", "").split(), "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-I", os.path.join(ROOT, "include")]


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, src + ".o")
    path = os.path.join(CSRC, src)
    deps = [path] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "ifx_abi.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-x", "cu" if src.endswith(".cu") else "c++", "-c", path, "-o", obj]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"] if os.environ.get("IFX_PTXAS_V") else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and os.environ.get("IFX_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return obj


def _cublaslt_dir() -> str:
    """The cuBLASLt torch itself loads (the pip `nvidia-cublas` wheel): one copy per process
    whichever of torch and this library is loaded first. Linking the toolkit's newer copy
    instead made torch's libcublas run against a mismatched libcublasLt when this library
    was loaded before torch (CUBLAS_STATUS_INVALID_VALUE in torch GEMMs)."""
    try:
        import nvidia.cublas as nc
        d = os.path.join(list(nc.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libcublasLt.so.12")):
            return d
    except ImportError:
        pass
    return "/usr/local/cuda/lib64"


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(o) for o in objs):
        return OUT
    lt = _cublaslt_dir()
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT + ".tmp", *objs, _npyrandom(), "-lcudart_static",
           f"-L{lt}", "-l:libcublasLt.so.12", "-Xlinker", f"-rpath={lt}",
           "-Xlinker", "--disable-new-dtags",  # DT_RPATH: wins over LD_LIBRARY_PATH
           "-Xlinker", "--exclude-libs,ALL", "-lm", "-ldl", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print("built", OUT)
    return OUT


if __name__ == "__main__":
    build(verbose=True)
