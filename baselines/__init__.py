"""Comparison baselines reported beside the gather (not on the product path).

``cpu_staged``: the paper's CPU-centric "Py" path (Fig. 2a): multithreaded CPU
gather into a pinned staging buffer, then one host-to-device DMA."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cpu_staged.c")
_SO = os.path.join(_HERE, "libcpu_staged.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC],
                       check=True)
        os.replace(tmp, _SO)
    return _SO


def lib():
    """The compiled baselines (loaded once; call it before concurrent use)."""
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.cpu_staged_gather.restype = None
        L.cpu_staged_gather.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int]
        _lib = L
    return _lib


def cpu_staged_gather(table_addr: int, rb: int, idx_addr: int, n: int, staging_addr: int,
                      threads: int = 0) -> None:
    lib().cpu_staged_gather(table_addr, rb, idx_addr, n, staging_addr, threads)


def host_read_gbs(addr: int, nbytes: int, threads: int = 0, reps: int = 3) -> float:
    """Best-of-`reps` multithreaded host read bandwidth over [addr, addr+nbytes) (GB/s)."""
    import time
    L = ctypes.CDLL(build())
    L.host_read_sum.restype = ctypes.c_uint64
    L.host_read_sum.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int]
    best = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        L.host_read_sum(addr, nbytes, threads)
        best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
    return best
