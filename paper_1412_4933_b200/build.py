"""In-tree build of the CUDA library (sm_100a) and the checkers.

    python -m paper_1412_4933_b200.build

nvcc cross-compiles without a GPU. The product library is
paper_1412_4933_b200/libpedflow_b200.so (static cudart, --fmad=false so that
no floating-point contraction can change a bit). The C++
drop-in demo (tools/pedflow_gpu_demo.cpp, via include/pedflow_gpu.hpp) is built
beside it.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpedflow_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = GENCODE + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
                     "-I", os.path.join(ROOT, "include")]
SOURCES = ["pf_kernels.cu", "pf_bitstep.cu", "pf_bitstep_ns8.cu", "pf_bitstep_ns10.cu", "pf_bitstep_small.cu", "pf_cluster.cu",
           "pf_context.cu", "pf_setup.cpp"]


def _run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, **kw)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose_ptxas: bool = False) -> str:
    """Compile every source to an object in parallel (the kernel template is
    instantiated in three translation units), then link the shared library."""
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "pf_gpu.h")]
    if force or _stale(LIB, deps):
        from concurrent.futures import ThreadPoolExecutor

        objdir = os.path.join(PKG, "build_obj")
        os.makedirs(objdir, exist_ok=True)
        extra = ["-Xptxas", "-v"] if verbose_ptxas else []
        jobs = [(os.path.join(CSRC, src), os.path.join(objdir, src + ".o")) for src in SOURCES]
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as pool:
            for f in [pool.submit(_run, [NVCC] + NVFLAGS + extra + ["-c", "-o", obj, src]) for src, obj in jobs]:
                f.result()
        _run([NVCC] + GENCODE + ["-shared", "-o", LIB] + [obj for _, obj in jobs])
    return LIB


def build_demo(force: bool = False) -> str:
    src = os.path.join(ROOT, "tools", "pedflow_gpu_demo.cpp")
    out = os.path.join(ROOT, "tools", "pedflow_gpu_demo")
    hdr = os.path.join(ROOT, "include", "pedflow_gpu.hpp")
    if not os.path.exists(src):
        return ""
    if force or _stale(out, [src, hdr, LIB]):
        _run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-o", out, src,
              f"-L{PKG}", "-lpedflow_b200", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../paper_1412_4933_b200"])
    return out


def build_oracle() -> None:
    """The checkers (test infrastructure): oracle/liboracle.so always, and
    oracle/_ref from the reference sources when /root/reference is present."""
    _run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"])
    if os.path.isdir("/root/reference/proj/src"):
        ref = os.path.join(ROOT, "oracle", "_ref", "libpedflow_ref.so")
        srcs = [os.path.join("/root/reference/proj/src", f) for f in os.listdir("/root/reference/proj/src")]
        if _stale(ref, srcs + [os.path.join(ROOT, "oracle", "ref_shim.cpp")]):
            _run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])


def build_all(force: bool = False) -> None:
    build_lib(force)
    build_demo(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
