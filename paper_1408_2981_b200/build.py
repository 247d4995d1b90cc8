"""In-tree build of the CUDA extension (sm_100a) and of the CPU oracle.

    python -m paper_1408_2981_b200.build [--force]

Produces, next to this file:
  libtpmg_b200.so       the product: the reference's exact operation order (--fmad=false,
                        true IEEE divisions), bitwise comparable to the oracle
  libtpmg_b200_fma.so   experimental: DFMA contraction + one reciprocal per Thomas level
and oracle/liboracle.so (test infrastructure).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = [os.path.join(CSRC, "tpmg_kernels.cu"), os.path.join(CSRC, "tpmg_host.cpp"),
           os.path.join(CSRC, "tpmg_io.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "tpmg_kernels.cuh"), os.path.join(ROOT, "include", "tpmg_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-shared",
          f"-I{os.path.join(ROOT, 'include')}", "-ldl"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build_lib(variant: str, force: bool = False, verbose: bool = False) -> str:
    name = "libtpmg_b200.so" if variant == "exact" else "libtpmg_b200_fma.so"
    out = os.path.join(PKG, name)
    if not force and not _stale(out):
        return out
    flags = list(COMMON)
    if variant == "exact":
        flags += ["--fmad=false", "-DTPMG_STRICT=1"]
    cmd = [_nvcc(), *ARCH, *flags, *SOURCES, "-o", out + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build_oracle(force: bool = False) -> str:
    odir = os.path.join(ROOT, "oracle")
    args = ["make", "-s", "-C", odir, "liboracle.so"]
    if force:
        args.insert(1, "-B")
    subprocess.run(args, check=True)
    return os.path.join(odir, "liboracle.so")


def build_all(force: bool = False, verbose: bool = False):
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(3) as ex:  # nvcc runs are independent processes
        jobs = [ex.submit(build_lib, "exact", force, verbose), ex.submit(build_lib, "fma", force, verbose),
                ex.submit(build_oracle, force)]
        return [j.result() for j in jobs]


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv, verbose=True):
        print("built", p)
