"""oracle — TEST INFRASTRUCTURE ONLY: the plain CPU definition of the unified-tensor gather.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. The product path
(``paper_2101_07956_b200``) never imports, links or executes anything here, and this package
shares no code with it; both take their inputs from ``workloads`` only.

* ``gather`` wraps ``ut_oracle.c``: ``out[i] = table[idx[i]]`` row by row (PAPER.md:377,
  Table 1; Listing 2), out-of-range rows zero-filled and the first
  offending position returned (reading R4). Pinned by tests/test_oracle.py.
* ``access_model`` is the paper's thread-per-element indexing kernel and its circular-shift
  variant written out as access traces, with the (warp, cacheline) request count the paper
  quotes (§4.5; Figs. 5/6). Pinned by the paper's 7 -> 5 example.
* ``pool_model`` replays the unified allocator's block recycling (P:530-531 under SPEC's reading,
  DESIGN.md R19). Pinned by tests/test_pool_model.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ut_oracle.c")
_SRC_SAMPLE = os.path.join(_HERE, "ut_oracle_sample.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile ut_oracle.c (plain C, -O2, single-threaded) into oracle/liboracle.so."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_SRC_SAMPLE))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, _SRC_SAMPLE],
                       check=True)
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_gather.restype = ctypes.c_int64
        L.oracle_gather.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.oracle_sample.restype = ctypes.c_int64
        L.oracle_sample.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                                    ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_sample_hash.restype = ctypes.c_uint64
        L.oracle_sample_hash.argtypes = [ctypes.c_uint64] * 4
        _lib = L
    return _lib


def gather_into(table_addr: int, rows: int, rb: int, idx: np.ndarray, out: np.ndarray) -> int:
    """Oracle gather from a table at a raw host address into ``out`` (uint8, >= n*rb bytes).

    Returns the first out-of-range position, or -1."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    n = idx.size
    assert out.dtype == np.uint8 and out.flags.c_contiguous and out.nbytes >= n * rb
    return int(_load().oracle_gather(table_addr, rows, rb, idx.ctypes.data, n, out.ctypes.data))


def gather(table, rows: int, rb: int, idx) -> tuple[np.ndarray, int]:
    """``(out, first_bad)`` with out[i*rb:(i+1)*rb] = table row idx[i] (bytes).

    ``table`` is a uint8 numpy array of >= rows*rb bytes or a raw host address (int)."""
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    out = np.empty(idx.size * rb, dtype=np.uint8)
    if isinstance(table, np.ndarray):
        t = np.ascontiguousarray(table).view(np.uint8).reshape(-1)
        assert t.nbytes >= rows * rb
        addr = t.ctypes.data
    else:
        addr = int(table)
    bad = gather_into(addr, rows, rb, idx, out)
    return out, bad


def sample(indptr_addr: int, indices_addr: int, n_nodes: int, seeds, fanouts, seed: int) -> np.ndarray:
    """Oracle multi-hop neighbour sampling (ut_oracle_sample.c): the minibatch node list."""
    seeds = np.ascontiguousarray(seeds, dtype=np.int64)
    fan = np.ascontiguousarray(fanouts, dtype=np.int32)
    need = ctypes.c_uint64(0)
    cap = max(16, seeds.size * 4)
    while True:
        out = np.empty(cap, dtype=np.int64)
        rc = _load().oracle_sample(indptr_addr, indices_addr, n_nodes, seeds.ctypes.data,
                                   seeds.size, fan.ctypes.data, fan.size,
                                   seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data, cap,
                                   ctypes.byref(need))
        if rc >= 0:
            return out[:rc]
        if rc == -1:
            cap = int(need.value)
            continue
        raise ValueError("seed out of range" if rc == -2 else "allocation failure")


def sample_hash(seed: int, hop: int, v: int, t: int) -> int:
    return int(_load().oracle_sample_hash(seed & 0xFFFFFFFFFFFFFFFF, hop, v, t))
