"""Build libsv.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a -lineinfo).

Usage: python paper_2106_13995_b200/build.py [--force] [--verbose]
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsv.so")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("NCCL (nvidia-nccl wheel) not found; needed for the sharded layer")


SOURCES = ["kernels.cu", "ir.cpp", "planner.cpp", "capi.cpp", "sharded.cpp", "comm.cpp", "jit.cpp"]
HEADERS = ["sv_internal.hpp", "sv_kernels.hpp", "engine.hpp", "state.hpp", "comm.hpp", "jit.hpp"]
CUDA_LIB = "/usr/local/cuda/lib64"


def _newest_header():
    hs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "sv.h")]
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, inc_nccl, verbose, force):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    path = os.path.join(CSRC, src)
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _newest_header()):
        return obj
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + CSRC, "-I" + os.path.join(ROOT, "include"),
              "-I" + inc_nccl]
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
               *common, "-c", path, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *common, "-x", "c++", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = nccl_dirs()
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, inc, verbose, force), SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        # NVRTC is linked statically (CUDA 12.9, sm_100a-aware) with its symbols kept local: a
        # process that imported torch first already has torch's own libnvrtc.so.12 (12.8)
        # loaded, and binding to it produced 1.8x more instructions in the generated kernels.
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L" + libdir, "-l:libnccl.so.2",
               "-L" + CUDA_LIB, "-l:libnvrtc_static.a", "-l:libnvrtc-builtins_static.a",
               "-l:libnvptxcompiler_static.a", "-Xlinker", "--exclude-libs,ALL",
               "-Xlinker", "-rpath=" + libdir]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
