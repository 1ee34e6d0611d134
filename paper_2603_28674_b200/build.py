"""Build the native libraries in-tree (they travel to the GPU box with the repo).

    python -m paper_2603_28674_b200.build

* ``lib/librgg_gpu.so``   — the CUDA engine (csrc/rgg_kernels.cu + csrc/rgg_capi.cu),
  nvcc for sm_100a only, -lineinfo for ncu source mapping, static cudart.
* ``lib/librgg_build.so`` — the CPU roadmap producer (csrc/producer.cpp).
* ``lib/_rggfast*.so``    — CPython binding of the per-update call (csrc/pyfast.c), linked to
  librgg_gpu.so; engine.GpuEngine uses it for batch_update.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
ROOT = os.path.dirname(PKG)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
GPU_SOURCES = ["rgg_kernels.cu", "rgg_resolve.cu", "rgg_store.cu", "rgg_capi.cu"]
GPU_DEPS = GPU_SOURCES + ["rgg_device.cuh", "rgg_kernels.cuh"]
PRODUCER_SOURCES = ["producer.cpp", "swept_gpu.cu", "rgg_prm.cu"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_gpu(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "librgg_gpu.so")
    deps = [os.path.join(CSRC, f) for f in GPU_DEPS] + [os.path.join(ROOT, "include", "rgg_gpu.h")]
    if force or _stale(out, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-Xptxas", "-v" if verbose else "-O3", "-o", out] + [os.path.join(CSRC, f) for f in GPU_SOURCES]
        subprocess.check_call(cmd)
    return out


def build_producer(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "librgg_build.so")
    srcs = [os.path.join(CSRC, f) for f in PRODUCER_SOURCES]
    deps = srcs + [os.path.join(ROOT, "include", h) for h in ("rgg_build.h", "rgg_prm.h")] + [
        os.path.join(CSRC, "swept_gpu.h")]
    if not all(os.path.exists(s) for s in srcs):
        return ""
    if force or _stale(out, deps):
        # host part with g++ (the reference's flags); the GPU fit and PRM with nvcc -fmad=false
        objs = [os.path.join(LIB, os.path.splitext(f)[0] + ".o") for f in PRODUCER_SOURCES]
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-pthread", "-c",
                               "-I", os.path.join(ROOT, "include"), "-o", objs[0], srcs[0]])
        for src, obj in zip(srcs[1:], objs[1:]):
            subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler",
                                   "-fPIC,-ffp-contract=off", "-c", "-o", obj, src])
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs, "-Xcompiler", "-pthread"])
        for o in objs:
            os.remove(o)
    return out


def build_pyfast(force: bool = False) -> str:
    import sysconfig

    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "_rggfast" + sysconfig.get_config_var("EXT_SUFFIX"))
    src = os.path.join(CSRC, "pyfast.c")
    deps = [src, os.path.join(ROOT, "include", "rgg_gpu.h"), os.path.join(LIB, "librgg_gpu.so")]
    if force or _stale(out, deps):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-I", sysconfig.get_paths()["include"], "-o", out, src,
               "-L", LIB, "-lrgg_gpu", "-Wl,-rpath,$ORIGIN"]
        subprocess.check_call(cmd)
    return out


def build_all(force: bool = False) -> None:
    build_gpu(force)
    build_producer(force)
    build_pyfast(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
