"""CPU emulation of the generated tile-pass kernels (test and debugging tool, not a product path).

The CUDA source of every TILE pass of a plan (``Plan.source(i)``) is rewritten into host C++:
the packed-complex64 PTX helpers become bit-exact scalar float code (f32x2 add/mul/fma are
two independent IEEE RNE operations), CUDA built-ins become per-thread variables, and each CTA
runs as a group of std::threads meeting at a std::barrier for ``__syncthreads()``.  A plan's
passes then run in order on a host buffer.  Small states only (one thread per CUDA thread).

    from tools.emulate import run_plan_on_host
    out = run_plan_on_host(plan, psi)          # psi: complex64/complex128 numpy array (copied)

Used by tests/test_generator_cpu.py (the generated code checked against the oracle without a
GPU) and for debugging generator changes here.  Only TILE passes are supported.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import re
import subprocess
import tempfile

import numpy as np

_CACHE = os.path.join(tempfile.gettempdir(), "svb_emulate_cache")

_PRELUDE_C64 = r"""
#include <cstdint>
#include <cstring>
#include <cmath>
typedef unsigned long long C;
static inline float lo(C a){uint32_t u=(uint32_t)a; float f; std::memcpy(&f,&u,4); return f;}
static inline float hi(C a){uint32_t u=(uint32_t)(a>>32); float f; std::memcpy(&f,&u,4); return f;}
static inline C pk(float x,float y){uint32_t a,b; std::memcpy(&a,&x,4); std::memcpy(&b,&y,4); return (C)a|((C)b<<32);}
static inline C A(C a,C b){return pk(lo(a)+lo(b),hi(a)+hi(b));}
static inline C M(C a,C b){return pk(lo(a)*lo(b),hi(a)*hi(b));}
static inline C F2(C a,C b,C c){return pk(std::fmaf(lo(a),lo(b),lo(c)),std::fmaf(hi(a),hi(b),hi(c)));}
static inline C F1(C a,C b,C c){return pk(std::fmaf(lo(a),lo(b),lo(c)),std::fmaf(hi(a),hi(b),hi(c)));}
static inline C N(C a){return pk(-lo(a),-hi(a));}
static inline C I(C a){return pk(-hi(a),lo(a));}
static inline C NI(C a){return pk(hi(a),-lo(a));}
static inline C SX(C a,C s){return a^(s&0x8000000080000000ull);}
static inline C CM(C a,C b){return pk(lo(a)*lo(b)-hi(a)*hi(b),lo(a)*hi(b)+hi(a)*lo(b));}
static inline void SS(C* p,C v){*p=v;}
static inline unsigned long long W64(unsigned x){return x;}
static inline void SS2(C* p,C a,C b){p[0]=a;p[1]=b;}
struct ulonglong2 { unsigned long long x, y; };
static inline void SG(C* p,C v){*p=v;}
"""

_PRELUDE_C128 = r"""
#include <cstdint>
#include <cmath>
typedef double R;
struct alignas(16) C { R x, y; };
static inline C mk(R x, R y){C c; c.x=x; c.y=y; return c;}
static inline C CM(C a, C b){return mk(a.x*b.x-a.y*b.y, a.x*b.y+a.y*b.x);}
static inline unsigned long long W64(unsigned x){return x;}
"""

_RUNNER = r"""
#include <barrier>
#include <thread>
#include <vector>
struct Dim { unsigned x; };
static thread_local Dim threadIdx, blockIdx, gridDim;
static thread_local C* g_sm;
static std::barrier<>* g_bar;
static inline void __syncthreads() { g_bar->arrive_and_wait(); }
KERNEL_BODY
extern "C" int emu_run(void* psi, unsigned long long grid, int threads, unsigned long long smem_bytes
                       EXTRA_PARAM) {
    std::vector<C> smem(smem_bytes / sizeof(C) + 1);
    for (unsigned long long b = 0; b < grid; ++b) {
        std::barrier<> bar(threads);
        g_bar = &bar;
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t)
            th.emplace_back([&, t, b]() {
                threadIdx.x = (unsigned)t;
                blockIdx.x = (unsigned)b;
                gridDim.x = (unsigned)grid;
                g_sm = smem.data();
                svpass((C*)psi EXTRA_ARG);
            });
        for (auto& x : th) x.join();
    }
    return 0;
}
"""


def _translate(src: str, basis: bool) -> str:
    dbl = "typedef double R;" in src
    lines = src.splitlines()
    # drop the CUDA prelude (everything before the kernel signature)
    k = next(i for i, l in enumerate(lines) if l.startswith('extern "C" __global__'))
    body = "\n".join(lines[k:])
    body = re.sub(r'extern "C" __global__ void __launch_bounds__\([^)]*\) svpass\(', "static void svpass(", body)
    body = body.replace("extern __shared__ C sm_[];", "C* sm_ = g_sm;")
    body = body.replace("extern __shared__ C sm[];", "C* sm = g_sm;")
    if "#define F F1" in src:
        body = "#define F F1\n" + body
    elif "#define F F2" in src:
        body = "#define F F2\n" + body
    pre = _PRELUDE_C128 if dbl else _PRELUDE_C64
    runner = _RUNNER.replace("KERNEL_BODY", body)
    if basis:
        runner = runner.replace("EXTRA_PARAM", ", unsigned long long kb").replace("EXTRA_ARG", ", kb")
    else:
        runner = runner.replace("EXTRA_PARAM", "").replace("EXTRA_ARG", "")
    return pre + runner


def _compile(cpp: str) -> ctypes.CDLL:
    os.makedirs(_CACHE, exist_ok=True)
    h = hashlib.sha1(cpp.encode()).hexdigest()[:20]
    so = os.path.join(_CACHE, f"emu_{h}.so")
    if not os.path.exists(so):
        src = os.path.join(_CACHE, f"emu_{h}.cpp")
        open(src, "w").write(cpp)
        tmp = so + f".{os.getpid()}.tmp"
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-ffp-contract=off", "-shared", "-fPIC", "-pthread",
                            src, "-o", tmp], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("emulation build failed:\n" + r.stderr[-4000:])
        os.replace(tmp, so)
    return ctypes.CDLL(so)


def geometry(src: str, n: int):
    hdr = src.splitlines()[0]
    m = int(re.search(r"m=(\d+)", hdr).group(1))
    rb = int(re.search(r"rb=(\d+)", hdr).group(1))
    threads = 1 << (m - rb)
    tpc = 1
    mt = re.search(r"__launch_bounds__\((\d+),", src)
    if mt:
        tpc = int(mt.group(1)) // threads
    ntiles = 1 << (n - m)
    dbl = "typedef double R;" in src
    smem = (1 << m) * (16 if dbl else 8) * tpc
    return ntiles // tpc, threads * tpc, smem


def run_pass_on_host(src: str, psi: np.ndarray, n: int, basis: int | None = None) -> None:
    lib = _compile(_translate(src, basis is not None))
    grid, threads, smem = geometry(src, n)
    ptr = psi.ctypes.data_as(ctypes.c_void_p)
    if basis is None:
        lib.emu_run(ptr, ctypes.c_ulonglong(grid), ctypes.c_int(threads), ctypes.c_ulonglong(smem))
    else:
        lib.emu_run(ptr, ctypes.c_ulonglong(grid), ctypes.c_int(threads), ctypes.c_ulonglong(smem),
                    ctypes.c_ulonglong(basis))


def to_logical(phys_psi: np.ndarray, qmap, n: int) -> np.ndarray:
    """Reorder a state held in a relabelled physical layout (qmap: logical -> physical bit)."""
    idx = np.arange(1 << n, dtype=np.int64)
    src = np.zeros_like(idx)
    for q in range(n):
        src |= ((idx >> q) & 1) << qmap[q]
    return phys_psi[src]


def run_plan_on_host(plan, psi: np.ndarray) -> np.ndarray:
    """Apply every (TILE) pass of `plan` to a copy of psi (logical order in, logical order out:
    the plan's final qubit map is undone on the host)."""
    out = np.array(psi, copy=True)
    info = plan.info()
    n = info["n"]
    for i in range(info["passes"]):
        src = plan.source(i)
        if not src or "svpass(C* __restrict__ psi" not in src:
            raise NotImplementedError(f"pass {i} is not a tile pass")
        run_pass_on_host(src, out, n)
    return to_logical(out, plan.qubit_map(), n)
