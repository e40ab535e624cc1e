"""Build the in-tree CUDA library libsl7.so for sm_100a (nvcc; no GPU needed to compile).

usage: python -m paper_2302_05170_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsl7.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["sl7_host.cpp", "sl7_kernels.cu", "sl7_tc.cu", "sl7_cdc.cu", "sl7_em.cu", "sl7_cir.cu"]
HEADERS = ["sl7_internal.h", "sl7_device.cuh", "sl7_tc.cuh"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "sl7.h"),
                                                                  os.path.abspath(__file__)]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, extra=()):
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v", *extra,
           "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return cmd, r


def build(force: bool = False, verbose: bool = True, ab: bool = False) -> str:
    """ab=True: the experiment build libsl7_ab.so (-DSL7_AB_HOOKS: SL7_TC_VARIANT selects the epilogue
    variants of DESIGN.md §6; load it with SL7_LIB=...); never used by the tests, smoke() or bench.py."""
    lib = LIB if not ab else os.path.join(PKG, "libsl7_ab.so")
    extra = ("-DSL7_AB_HOOKS",) if ab else ()
    if not ab and not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    srcs = [os.path.join(CSRC, f) for f in SOURCES if os.path.exists(os.path.join(CSRC, f))]
    objdir = os.path.join(PKG, "build" if not ab else "build_ab")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]
    with ThreadPoolExecutor(len(srcs)) as ex:
        results = list(ex.map(lambda so: _compile(*so, extra), zip(srcs, objs)))
    log = os.path.join(PKG, "build_ptxas.log")
    with open(log, "w") as f:
        for cmd, r in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    for cmd, r in results:
        if verbose:
            print(" ".join(cmd), flush=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed (see %s)" % log)
    link = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", lib + ".tmp", *objs]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, ab="--ab" in sys.argv))
