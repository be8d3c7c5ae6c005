"""Build libut.so (the C-ABI gather library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libut.so")
SOURCES = [os.path.join(CSRC, "ut.cu"), os.path.join(CSRC, "ut_sample.cu"), os.path.join(CSRC, "ut_coop.cu"),
           os.path.join(CSRC, "ut_pool.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "ut_kernels.cuh"), os.path.join(CSRC, "ut_internal.h"),
                  os.path.join(CSRC, "ut_scan.cuh"),
                  os.path.join(INCLUDE, "ut.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def command(out: str = LIB, extra: list[str] | None = None) -> list[str]:
    return [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
            "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v", "-I", INCLUDE,
            "-cudart", "static", *(extra or []), "-o", out, *SOURCES]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    p = subprocess.run(command(tmp), capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + p.stdout + p.stderr)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write(p.stderr)
    if verbose:
        print(p.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True)
