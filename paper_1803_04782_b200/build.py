"""In-tree build of the socfield B200 engine.

    python -m paper_1803_04782_b200.build [--force]

Produces, under paper_1803_04782_b200/lib/ (git-ignored, shipped to the GPU box as built):

  libsocfield_cuda.so        the sm_100a kernels + C ABI (include/socfield_cuda.h); nvcc
  libsocfield_b200.so        the C++ host mirror of the socfield API (include/socfield/*.hpp); g++
  socfield/_core*.so         pybind11 module with the reference's Python surface

and, under oracle/build/ (test infrastructure, not product): libsocfield_b200_shim.so, oracle/socfield_shim.cpp
compiled against the mirror — the same flat-C driver the tests run the unmodified reference through.

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU-only build container.
"""
from __future__ import annotations

import os
import shlex
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")

CUDA_SOURCES = ["sfc_api.cu", "sfc_ped_kernels.cu", "sfc_k5_writeback.cu", "sfc_k5_window.cu", "sfc_k5_listwalk.cu", "sfc_k5_pairs.cu", "sfc_k5_field.cu", "sfc_rasterize.cu", "sfc_slab.cu", "sfc_digest.cu"]
HOST_SOURCES = ["model.cpp", "engine.cpp", "raster.cpp", "scenario.cpp", "bench.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "--fmad=false",  # decisions and field sums must not contract a*b+c
]
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-ffp-contract=off", "-Wl,-Bsymbolic"]
# One shared C++ runtime for every library in the process: this image's g++ wrapper finds only
# the static libstdc++.a, and several private copies of it (one per .so) corrupt iostream state.
STDCXX = ["-L/usr/lib/x86_64-linux-gnu", "-l:libstdc++.so.6"]


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print("+", " ".join(shlex.quote(c) for c in cmd), flush=True)
    subprocess.check_call(cmd)


def _headers() -> list[str]:
    out = [os.path.join(INCLUDE, "socfield_cuda.h")]
    for d in (os.path.join(INCLUDE, "socfield"), CSRC, HOST):
        out += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".hpp", ".cuh", ".h"))]
    return out


def build_cuda(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(LIB, exist_ok=True)
    target = os.path.join(LIB, "libsocfield_cuda.so")
    sources = [os.path.join(CSRC, s) for s in CUDA_SOURCES]
    # one object per translation unit (only the changed ones are recompiled, in parallel), then link
    objdir = os.path.join(LIB, "obj")
    os.makedirs(objdir, exist_ok=True)
    objects, stale = [], []
    for src in sources:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objects.append(obj)
        if force or _newer(obj, [src] + _headers()):
            stale.append([NVCC, *NVCC_FLAGS, "-I" + INCLUDE, "-I" + CSRC, "-c", "-o", obj, src])
    if stale:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=min(len(stale), os.cpu_count() or 1)) as pool:
            list(pool.map(lambda cmd: _run(cmd, verbose), stale))
    if stale or _newer(target, objects):
        _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target, *objects], verbose)
    return target


def build_host(force: bool = False, verbose: bool = True) -> str:
    cuda = build_cuda(force, verbose)
    target = os.path.join(LIB, "libsocfield_b200.so")
    sources = [os.path.join(HOST, s) for s in HOST_SOURCES]
    if force or _newer(target, sources + _headers() + [cuda]):
        _run([CXX, *CXX_FLAGS, "-I" + INCLUDE, "-I" + HOST, "-shared", "-o", target, *sources,
              "-L" + LIB, "-lsocfield_cuda", *STDCXX, "-Wl,-rpath,$ORIGIN"], verbose)
    return target


def build_shim(force: bool = False, verbose: bool = True) -> str:
    host = build_host(force, verbose)
    outdir = os.path.join(ROOT, "oracle", "build")  # a test driver: kept out of the product's lib/
    os.makedirs(outdir, exist_ok=True)
    target = os.path.join(outdir, "libsocfield_b200_shim.so")
    src = os.path.join(ROOT, "oracle", "socfield_shim.cpp")
    hdr = os.path.join(ROOT, "oracle", "socfield_shim.h")
    if force or _newer(target, [src, hdr, host] + _headers()):
        _run([CXX, *CXX_FLAGS, "-Wno-comment", "-I" + INCLUDE, "-I" + os.path.join(ROOT, "oracle"),
              '-DSHIM_IMPL_NAME="b200-cuda"', "-shared", "-o", target, src,
              "-L" + LIB, "-lsocfield_b200", "-lsocfield_cuda", *STDCXX,
              "-Wl,-rpath,$ORIGIN/../../paper_1803_04782_b200/lib"], verbose)
    return target


def build_pybind(force: bool = False, verbose: bool = True) -> str:
    import pybind11

    host = build_host(force, verbose)
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    outdir = os.path.join(PKG, "socfield")
    os.makedirs(outdir, exist_ok=True)
    target = os.path.join(outdir, "_core" + suffix)
    src = os.path.join(PKG, "bindings", "module.cpp")
    if force or _newer(target, [src, host] + _headers()):
        _run([CXX, *CXX_FLAGS, "-I" + INCLUDE, "-I" + HOST, "-I" + pybind11.get_include(),
              "-I" + sysconfig.get_paths()["include"], "-shared", "-o", target, src,
              "-L" + LIB, "-lsocfield_b200", "-lsocfield_cuda", *STDCXX, "-Wl,-rpath,$ORIGIN/../lib"], verbose)
    return target


def build_all(force: bool = False, verbose: bool = True) -> dict[str, str]:
    return {
        "cuda": build_cuda(force, verbose),
        "host": build_host(False, verbose),
        "shim": build_shim(False, verbose),
        "pybind": build_pybind(False, verbose),
    }


if __name__ == "__main__":
    built = build_all(force="--force" in sys.argv)
    for k, v in built.items():
        print(f"{k}: {v}")
